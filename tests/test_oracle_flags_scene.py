"""The scene of the GPU flag parity tests (tests/test_gpu_parity.py::
test_flags_one_step_T2) exercises what it is meant to: on the oracle, the
clamp flag (reading R3), the truncation flag (R4) and C_t (Eq. 9) each change
the step's forces or tangential histories on it well beyond the T2 tolerance,
so a GPU branch that ignored one of them would fail that test."""
import numpy as np

from paper_1301_1714_b200 import scenes as S


def step_after(orc, sc, warm=3):
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, sc.params.max_contacts)
    for _ in range(warm):
        assert orc.step(p, st, h).rc == 0
    return p, st, h


def test_flags_change_the_step(orc):
    base = S.flag_gas()
    p, st, h = step_after(orc, base)
    ref = orc.step(p, st.copy(), h.copy())
    tol = 1e-4 * np.linalg.norm(ref.F, axis=1) + 1e-5 * ref.Fabs
    variants = {
        "clamp": S.flag_gas(clamp_fn=True).params,
        "truncate": S.flag_gas(truncate_dt=True).params,
        "Ct=Cn": base.params.replace(stiffness_t=base.params.stiffness_n),
    }
    for name, sp in variants.items():
        q = orc.make_params(sp, base.radius)
        st2, h2 = st.copy(), h.copy()
        r = orc.step(q, st2, h2)
        assert r.rc == 0
        if name == "truncate":  # F is the same this step; δ_t of the capped contacts is not
            da, db = h.copy(), h2
            orc.step(p, st.copy(), da)
            diff = np.abs(da.dt - db.dt).max(axis=(1, 2))
            assert (diff > 1e-6 * 1e-3).sum() > 100, name
        else:
            changed = np.linalg.norm(r.F - ref.F, axis=1) > 10 * tol
            assert changed.sum() > 50, (name, changed.sum())
