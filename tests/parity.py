"""Helpers of the GPU parity tests: move a Dem's state/history into the
oracle's representation and compare with the SURVEY §8(c) thresholds.
Test infrastructure (imports both sides; neither side imports it)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def oracle_inputs(d, K: int):
    """(State, History) of a Dem's current state in its internal order."""
    s = d.get_state()
    st = orc.State.from_arrays(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"], s["id"],
                               s.get("material"))
    if d.params.model == 0:
        id_i, id_j, dt3 = d.get_contacts()
        h = orc.History.from_pairs(st.id, K, id_i, id_j, dt3.astype(np.float64))
    else:
        h = orc.History.empty(st.n, K)
    return st, h


def contacts_dict(d) -> dict:
    id_i, id_j, dt3 = d.get_contacts()
    return {(int(a), int(b)): v.astype(np.float64) for a, b, v in zip(id_i, id_j, dt3)}


def assert_T2_forces(F_gpu, T_gpu, res, rel=1e-4, floor=1e-5, mask=None, what=""):
    """|F_gpu - F_orc| <= rel |F_orc| + floor * Fabs, where
    the absolute floor's scale Fabs is the oracle's cancellation scale: the sum
    over the particle's contacts of the magnitudes of the terms Eq. 4 adds
    (|k_n δ| + |η v_n| + |k_t δ_t| + |η v_t|; Eq. 1's for the simple model).
    The same for T with Σ r_i (|k_t δ_t| + |η v_t| + μ(|k_n δ| + |η v_n|)) —
    Eq. 5 makes a capped F_t inherit the cancellation of |F_n|. DESIGN.md §3."""
    F_gpu = np.asarray(F_gpu, np.float64)
    T_gpu = np.asarray(T_gpu, np.float64)
    sel = slice(None) if mask is None else mask
    dF = np.linalg.norm(F_gpu[sel] - res.F[sel], axis=1)
    tolF = rel * np.linalg.norm(res.F[sel], axis=1) + floor * res.Fabs[sel]
    bad = np.nonzero(dF > tolF)[0]
    assert bad.size == 0, (f"{what} F: {bad.size} particles over T2; worst excess "
                           f"{np.max(dF - tolF):.3e} N at {bad[:5]}")
    dT = np.linalg.norm(T_gpu[sel] - res.T[sel], axis=1)
    tolT = rel * np.linalg.norm(res.T[sel], axis=1) + floor * res.Tabs[sel] + 1e-30
    bad = np.nonzero(dT > tolT)[0]
    assert bad.size == 0, (f"{what} T: {bad.size} particles over T2; worst excess "
                           f"{np.max(dT - tolT):.3e} N m at {bad[:5]}")


def assert_T2_history(gpu: dict, orc_hist: dict, d_len=1e-3, rel=1e-4, abs_frac=1e-6):
    """Same contact keys bit-exactly; |Δδ_t| <= rel |δ_t| + abs_frac d."""
    assert gpu.keys() == orc_hist.keys(), (
        f"contact sets differ: gpu-only {sorted(set(gpu) - set(orc_hist))[:5]}, "
        f"oracle-only {sorted(set(orc_hist) - set(gpu))[:5]}")
    worst = 0.0
    for k, v in orc_hist.items():
        err = np.linalg.norm(gpu[k] - v)
        tol = rel * np.linalg.norm(v) + abs_frac * d_len
        worst = max(worst, err - tol)
    assert worst <= 0.0, f"δ_t over tolerance by {worst:.3e} m"
