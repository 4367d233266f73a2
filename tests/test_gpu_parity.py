"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs. Run on a B200 via gpurun:
    python -m pytest tests -m gpu -x -q
"""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1301_1714_b200 import scenes as S
from paper_1301_1714_b200.dem import (DEM_ECOINCIDENT, DEM_EESCAPED, DEM_ENONFINITE, DEM_EOVERFLOW, DEM_F_DIAG, DEM_F_FORCE_DENSE,
                                      DEM_F_FORCE_WS,
                                      DEM_F_FORCE_LANES, DEM_F_FORCE_LIGHT, DEM_F_FULL_SORT, DEM_F_GENERAL_DETECT,
                                      DEM_F_HALF_LISTS,
                                      DEM_F_NO_GRAPH, DEM_F_SPLIT_SWEEP, DEM_F_THREAD_PER_PARTICLE,
                                      DEM_ORDER_ID,
                                      Dem, DemError)

from .parity import assert_T2_forces, assert_T2_history, contacts_dict, oracle_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


def make(sc, flags=DEM_F_DIAG, **kw) -> Dem:
    d = Dem(sc.params, flags=flags, **kw)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    return d


def scenes_small():
    return [S.C1(), S.random_gas(3000, 14.0, 5, r_range=(0.25e-3, 0.5e-3), v_sigma=0.05,
                                 params=S.SimParams(max_contacts=32))]


# --------------------------------------------------------- T1 bit-exact ----

@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_hash_sort_offsets_bit_exact(name):
    sc = S.CONFIGS[name]()
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc, flags=0)
    key0, _, _ = d.get_grid()
    s0 = d.get_state()
    CM = orc.hash_cells(p, s0["pos"].astype(np.float64))
    assert np.array_equal(key0, CM)
    d.step(1)
    key1, perm, off = d.get_grid()
    SCM, SCCM = orc.sort_map(CM)
    assert np.array_equal(perm, SCCM)  # Eq. 11, stable
    assert np.array_equal(off, orc.cell_offsets(SCM, off.shape[0] - 1))
    s1 = d.get_state()
    assert np.array_equal(s1["id"], s0["id"][SCCM])  # the reorder of step 4
    assert np.array_equal(key1, orc.hash_cells(p, s1["pos"].astype(np.float64)))


# ------------------------------------------ merge re-sort -----

def _check_sorts(d, nsteps, per_call=1):
    """Eq. 11 (stable, R16) and the lower-bound offsets of every step, taken
    from the key array before it, against the oracle's definitions."""
    for _ in range(nsteps // per_call):
        key0, _, _ = d.get_grid()
        d.step(per_call)
        if per_call == 1:
            _, perm, off = d.get_grid()
            SCM, SCCM = orc.sort_map(key0)
            assert np.array_equal(perm, SCCM)
            assert np.array_equal(off, orc.cell_offsets(SCM, off.shape[0] - 1))


@pytest.mark.parametrize("name", ["C1", "C3", "gas"])
@pytest.mark.parametrize("graph", [True, False])
def test_merge_resort_bit_exact(name, graph):
    """After the first step the state is in the last sorted order and only the
    particles that changed cell are merged in (k_merge): SCCM and the offsets stay bit-exact every step."""
    sc = scenes_small()[1] if name == "gas" else S.CONFIGS[name]()
    d = make(sc, flags=0 if graph else DEM_F_NO_GRAPH)
    _check_sorts(d, 25)
    assert d.stats()["full_sorts"] == 1


def cell_crossers_scene(n_side=24, gap=3e-8):
    """n_side³ separated spheres (no contacts, g = 0), each 3e-8 m below a
    cell face in x and moving +x at 0.01 m/s (2e-8 m per step): none changes
    cell in step 1, all of them (> 4,096) in step 2, so step 3 has more movers
    than the merge re-sort takes and must be redone by counting."""
    p = S.SimParams(gravity=(0.0, 0.0, 0.0))
    h = 2.0 * S.R * (1.0 + 2.0 ** -10)
    L = (3 * n_side + 4) * h
    p = p.replace(box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    g = np.stack(np.meshgrid(*[np.arange(n_side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    c = (3 * g + 2).astype(np.float64)
    pos = (c + 0.5) * h
    pos[:, 0] = (c[:, 0] + 1.0) * h - gap  # just below the face x = (c + 1) h
    vel = np.zeros_like(pos)
    vel[:, 0] = 0.01
    return S.make_scene("crossers", p, pos.astype(np.float32), vel.astype(np.float32))


@pytest.mark.parametrize("graph", [True, False])
def test_merge_resort_overflow_fallback(graph):
    """More movers than the list holds (4,096 at this size): that step is
    rolled back and redone by the counting sort, and the rest of the
    20-step call merges again; the run equals the counting-sort-only run
    bitwise and the grid stays bit-exact."""
    sc = cell_crossers_scene()
    assert sc.n > 4096
    base = 0 if graph else DEM_F_NO_GRAPH
    a = make(sc, flags=DEM_F_DIAG | base)
    b = make(sc, flags=DEM_F_DIAG | base | DEM_F_FULL_SORT)
    a.step(20)
    b.step(20)
    assert a.stats()["full_sorts"] == 2  # step 1 and the redone step 3; steps 4-20 merged
    sa, sb = a.get_state(forces=True), b.get_state(forces=True)
    for k in ("pos", "vel", "omega", "id", "force"):
        assert np.array_equal(sa[k], sb[k]), k
    c = make(sc, flags=base)
    _check_sorts(c, 6)  # one step per call: step 3 overflows, later calls merge again
    assert c.stats()["full_sorts"] == 2


@pytest.mark.parametrize("n_side", [7, 10, 15])
def test_merge_resort_mover_counts(n_side):
    """All n_side³ spheres change cell in step 2, so step 3 merges 343, 1,000
    or 3,375 movers, more events per k_merge block than its shared-memory
    list holds (the exact per-slot path): the grid is bit-exact every step,
    with no fallback to counting, and the run equals the counting-sort run
    bitwise."""
    sc = cell_crossers_scene(n_side=n_side)
    d = make(sc, flags=0)
    _check_sorts(d, 2)
    assert d.analyze()["movers"] == n_side ** 3  # step 2 moved every sphere: step 3 merges them
    _check_sorts(d, 3)
    assert d.stats()["full_sorts"] == 1
    a = make(sc, flags=DEM_F_DIAG)
    b = make(sc, flags=DEM_F_DIAG | DEM_F_FULL_SORT)
    a.step(5)
    b.step(5)
    sa, sb = a.get_state(forces=True), b.get_state(forces=True)
    for k in ("pos", "vel", "omega", "id", "force"):
        assert np.array_equal(sa[k], sb[k]), k


def test_merge_resort_equals_counting_sort_bitwise():
    """Whole runs with the merge re-sort and with the counting sort every
    step (DEM_F_FULL_SORT) agree bitwise (C3: settled contacts, migrations
    between cells every step)."""
    sc = S.C3()
    runs = []
    for f in (0, DEM_F_FULL_SORT):
        d = make(sc, flags=DEM_F_DIAG | f)
        d.step(30)
        runs.append((d.get_state(forces=True), contacts_dict(d), d.get_grid()))
    for k in ("pos", "vel", "omega", "id", "force", "torque"):
        assert np.array_equal(runs[0][0][k], runs[1][0][k]), k
    assert runs[0][1].keys() == runs[1][1].keys()
    for x, y in zip(runs[0][2], runs[1][2]):
        assert np.array_equal(x, y)


# ------------------------------------------------------ T2 one step -------

@pytest.mark.parametrize("variant", [0, DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES,
                                     DEM_F_FORCE_WS, DEM_F_GENERAL_DETECT, DEM_F_HALF_LISTS,
                                     DEM_F_THREAD_PER_PARTICLE, DEM_F_SPLIT_SWEEP,
                                     DEM_F_SPLIT_SWEEP | DEM_F_FORCE_DENSE,
                                     DEM_F_SPLIT_SWEEP | DEM_F_FORCE_LIGHT])
@pytest.mark.parametrize("idx", [0, 1])
def test_one_step_T2(idx, variant):
    sc = scenes_small()[idx]
    K = sc.params.max_contacts
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc, flags=DEM_F_DIAG | variant)
    for k in range(4):  # steps 1..4 each from the GPU's own state + history
        st, h = oracle_inputs(d, K)
        d.step(1)
        g = d.get_state(forces=True)
        res = orc.step(p, st, h)
        assert res.rc == 0
        assert np.array_equal(g["id"], st.id)  # same sorted order
        assert_T2_forces(g["force"], g["torque"], res, what=f"{sc.name} step {k + 1}")
        assert_T2_history(contacts_dict(d), h.as_dict(st.id))
        # integrated state: within the force tolerance carried through Δt, plus fp32 rounding
        dt = p.dt
        tolF = 1e-4 * np.linalg.norm(res.F, axis=1) + 1e-5 * res.Fabs
        dv = np.linalg.norm(g["vel"] - st.vel, axis=1)
        assert np.all(dv <= tolF / st.mass * dt + 3e-7 * np.linalg.norm(st.vel, axis=1) + 1e-12)
        dx = np.abs(g["pos"] - st.pos).max(axis=1)
        assert np.all(dx <= dv * dt + 2 * np.spacing(np.abs(st.pos).astype(np.float32)).max(axis=1))


@pytest.mark.parametrize("variant", [0, DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES,
                                     DEM_F_THREAD_PER_PARTICLE, DEM_F_SPLIT_SWEEP])
@pytest.mark.parametrize("flags", ["clamp", "truncate", "clamp+truncate", "none"])
def test_flags_one_step_T2(flags, variant):
    """Readings R3 (DEM_F_CLAMP_FN) and R4 (DEM_F_TRUNCATE_DT) and a scalar
    C_t != C_n, T2 against the oracle for four consecutive steps."""
    sc = S.flag_gas(clamp_fn="clamp" in flags, truncate_dt="trunc" in flags)
    K = sc.params.max_contacts
    p = orc.make_params(sc.params, sc.radius)
    assert p.Ct == pytest.approx(2.5 * p.Cn, rel=1e-7)
    d = make(sc, flags=DEM_F_DIAG | variant)
    for k in range(4):
        st, h = oracle_inputs(d, K)
        d.step(1)
        g = d.get_state(forces=True)
        res = orc.step(p, st, h)
        assert res.rc == 0
        assert np.array_equal(g["id"], st.id)
        assert_T2_forces(g["force"], g["torque"], res, what=f"{flags} step {k + 1}")
        assert_T2_history(contacts_dict(d), h.as_dict(st.id))


@pytest.mark.parametrize("name", ["C3", "C4/4", "C5/4"])
def test_bench_instantiation_bitwise(name):
    """The bench runs k_force without DEM_F_DIAG (no F/T output) while every
    T2 test sets it: the two instantiations must produce the same run bitwise
    (state and δ_t), in the same force configuration."""
    sc = S.C3() if name == "C3" else S.C4(scale=4) if name == "C4/4" else S.C5(scale=4)
    runs = []
    # the bench's kernel (no DIAG; one radius: detection fused into it), its DIAG twin, and the
    # split path (k_detect writing lists to HBM, then k_force)
    for flags in (DEM_F_DIAG, 0, DEM_F_SPLIT_SWEEP):
        d = make(sc, flags=flags)
        d.step(12)
        runs.append((d.get_state(), contacts_dict(d), d.stats()["force_cfg"],
                     d.stats()["fused_sweep"]))
    assert {r[2] for r in runs} == {"dense" if name == "C3" else "light"}
    assert [r[3] for r in runs] == ([True, True, False] if name != "C5/4" else [False] * 3)
    for r in runs[1:]:
        for k in ("pos", "vel", "omega", "id"):
            assert np.array_equal(runs[0][0][k], r[0][k]), k
        assert runs[0][1].keys() == r[1].keys()
        assert all(np.array_equal(runs[0][1][x], r[1][x]) for x in runs[0][1])


def test_one_step_T2_C2_both_models():
    for model in ("practical", "simple"):
        sc = S.C2(S.SimParams(model=model))
        p = orc.make_params(sc.params, sc.radius)
        d = make(sc)
        d.step(3)
        st, h = oracle_inputs(d, 16)
        d.step(1)
        g = d.get_state(forces=True)
        res = orc.step(p, st, h)
        assert np.array_equal(g["id"], st.id)
        assert_T2_forces(g["force"], g["torque"], res, what=f"C2 {model}")
        if model == "practical":
            assert_T2_history(contacts_dict(d), h.as_dict(st.id))


def test_one_step_T2_C3_full():
    sc = S.C3()
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc)
    d.step(2)
    st, h = oracle_inputs(d, 16)
    d.step(1)
    g = d.get_state(forces=True)
    res = orc.step(p, st, h)
    assert np.array_equal(g["id"], st.id)
    assert_T2_forces(g["force"], g["torque"], res, what="C3")
    assert_T2_history(contacts_dict(d), h.as_dict(st.id))


def band_pairs_scene(seed=11, m=8, mono=False):
    """m³ isolated pairs at separations S(1 + k 2⁻²³), |k| <= 40 (before the
    fp32 rounding of the positions): ~60 pairs fall inside the ±16u fp32 band
    of R14, where k_detect must rescan with the exact fp64 predicate. mono:
    every radius r (k_detect's constant-S² test)."""
    rng = np.random.default_rng(seed)
    g = np.stack(np.meshgrid(*[np.arange(m)] * 3, indexing="ij"), -1).reshape(-1, 3)
    a = (g * 4.0 + 2.0) * S.D
    u = rng.normal(size=a.shape)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    r = rng.choice([S.R] if mono else [0.5 * S.R, 0.75 * S.R, S.R], size=(a.shape[0], 2))
    sep = (r[:, 0] + r[:, 1]) * (1.0 + rng.integers(-40, 41, a.shape[0]) * 2.0 ** -23)
    b = a + u * sep[:, None]
    pos = np.concatenate([a, b]).astype(np.float32)
    rad = np.concatenate([r[:, 0], r[:, 1]]).astype(np.float32)
    L = (4.0 * m + 1.0) * S.D
    p = S.SimParams(gravity=(0.0, 0.0, 0.0)).replace(box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    return S.make_scene("band_pairs", p, pos, radius=rad)


@pytest.mark.parametrize("mono", [False, True])
def test_touching_pairs_in_fp32_band(mono):
    sc = band_pairs_scene(mono=mono)
    p = orc.make_params(sc.params, sc.radius)
    # the decisions the band has to settle: fp32 d², S² vs the exact fp64 predicate
    n = sc.n // 2
    A, B = sc.pos[:n].astype(np.float64), sc.pos[n:].astype(np.float64)
    S2 = (sc.radius[:n].astype(np.float64) + sc.radius[n:]) ** 2
    exact = ((B - A) ** 2).sum(1) < S2
    d2f = ((sc.pos[n:] - sc.pos[:n]) ** 2).sum(1, dtype=np.float32)
    in_band = np.abs(d2f.astype(np.float64) - S2) <= 16 * 2.0 ** -24 * S2
    assert in_band.sum() >= 40 and exact[in_band].any() and not exact[in_band].all()
    for flags in (DEM_F_DIAG | DEM_F_FORCE_DENSE, DEM_F_DIAG | DEM_F_FORCE_LIGHT,
                  DEM_F_DIAG | DEM_F_SPLIT_SWEEP | DEM_F_FORCE_DENSE,
                  DEM_F_DIAG | DEM_F_SPLIT_SWEEP | DEM_F_FORCE_LIGHT,
                  DEM_F_DIAG | DEM_F_FORCE_LANES, DEM_F_DIAG | DEM_F_GENERAL_DETECT,
                  DEM_F_DIAG | DEM_F_THREAD_PER_PARTICLE, DEM_F_DIAG | DEM_F_HALF_LISTS):
        d = make(sc, flags=flags)
        st, h = oracle_inputs(d, 16)
        d.step(1)
        res = orc.step(p, st, h)
        assert res.rc == 0
        got = contacts_dict(d)
        assert got.keys() == h.as_dict(st.id).keys()
        assert len(got) == 2 * int(exact.sum())  # each contact seen from both sides


def test_full_size_C4_sampled():
    """4M-particle settling bed in the bench's launch configuration (graph
    replay): grid bit-exact for every particle; forces, torques and histories
    of ~300 sampled particles against the oracle evaluated one by one."""
    sc = S.C4()
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc)
    d.step(20)
    K = int(d.stats()["max_contacts_seen"]) + 2
    st, h = oracle_inputs(d, K)
    key0, _, _ = d.get_grid()
    CM = orc.hash_cells(p, st.pos)
    assert np.array_equal(key0, CM)
    d.step(1)
    key1, perm, off = d.get_grid()
    SCM, SCCM = orc.sort_map(CM)
    assert np.array_equal(perm, SCCM)
    assert np.array_equal(off, orc.cell_offsets(SCM, off.shape[0] - 1))
    g = d.get_state(forces=True)
    rng = np.random.default_rng(44)
    mask = np.zeros(sc.n, bool)
    mask[rng.choice(sc.n, 256, replace=False)] = True
    near = np.nonzero(g["pos"][:, 1] < 0.6e-3)[0]  # floor contacts too
    mask[near[:32]] = True
    res = orc.step(p, st, h, only=mask)
    assert np.array_equal(g["id"], st.id)
    assert_T2_forces(g["force"], g["torque"], res, mask=mask, what="C4 sampled")
    sample_ids = st.id[mask]
    id_i, id_j, dt3 = d.get_contacts()
    keep = np.isin(id_i, sample_ids)
    gc = {(int(a), int(b)): v.astype(np.float64)
          for a, b, v in zip(id_i[keep], id_j[keep], dt3[keep])}
    oc = {}
    for s in np.nonzero(mask)[0]:
        for k in range(int(h.cnt[s])):
            oc[(int(st.id[s]), int(h.pid[s, k]))] = h.dt[s, k].copy()
    assert_T2_history(gc, oc)


def test_full_size_C5_sampled():
    """2M-particle polydisperse bed (K = 32: per-pair S = r_i + r_j, lists of
    sorted slots through SCCM — the bench's C5 launch configuration), after
    200 steps of settling: grid bit-exact for every particle; forces,
    torques and histories of ~300 sampled particles against the oracle."""
    sc = S.C5()
    assert sc.params.max_contacts == 32 and sc.radius.min() < sc.radius.max()
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc)
    d.step(200)
    assert d.stats()["fused_sweep"] is False
    K = int(d.stats()["max_contacts_seen"]) + 2
    st, h = oracle_inputs(d, K)
    key0, _, _ = d.get_grid()
    CM = orc.hash_cells(p, st.pos)
    assert np.array_equal(key0, CM)
    d.step(1)
    key1, perm, off = d.get_grid()
    SCM, SCCM = orc.sort_map(CM)
    assert np.array_equal(perm, SCCM)
    assert np.array_equal(off, orc.cell_offsets(SCM, off.shape[0] - 1))
    g = d.get_state(forces=True)
    rng = np.random.default_rng(45)
    mask = np.zeros(sc.n, bool)
    mask[rng.choice(sc.n, 256, replace=False)] = True
    busy = np.nonzero(h.cnt >= 3)[0]  # particles with several contacts
    mask[busy[:48]] = True
    res = orc.step(p, st, h, only=mask)
    assert np.array_equal(g["id"], st.id)
    assert_T2_forces(g["force"], g["torque"], res, mask=mask, what="C5 sampled")
    sample_ids = st.id[mask]
    id_i, id_j, dt3 = d.get_contacts()
    keep = np.isin(id_i, sample_ids)
    gc = {(int(a), int(b)): v.astype(np.float64)
          for a, b, v in zip(id_i[keep], id_j[keep], dt3[keep])}
    oc = {}
    for s in np.nonzero(mask)[0]:
        for k in range(int(h.cnt[s])):
            oc[(int(st.id[s]), int(h.pid[s, k]))] = h.dt[s, k].copy()
    assert_T2_history(gc, oc)


# ------------------------------------------- T3 shadow bound, 100 steps ----

def test_shadow_bound_100_steps():
    sc = S.C1()
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc, flags=0)
    st = orc.State.from_scene(sc)
    hx = orc.History.empty(sc.n, 16)
    st_r = st.copy()
    hr = orc.History.empty(sc.n, 16)
    for _ in range(100):
        assert orc.step(p, st, hx).rc == 0
        assert orc.step(p, st_r, hr).rc == 0
        r = st_r.rounded_fp32()
        st_r.pos, st_r.vel, st_r.omega = r.pos, r.vel, r.omega
        hr.dt = hr.dt.astype(np.float32).astype(np.float64)
    d.step(100)
    g = d.get_state(order=DEM_ORDER_ID)
    o = np.argsort(st.id)
    o_r = np.argsort(st_r.id)
    shadow = np.abs(st.pos[o] - st_r.pos[o_r]).max()
    err = np.abs(g["pos"] - st.pos[o]).max()
    L = max(abs(x) for x in sc.params.box_hi)
    bound = max(10 * shadow, 8 * 100 * np.spacing(np.float32(L)))
    assert err <= bound, (err, shadow, bound)
    vshadow = np.abs(st.vel[o] - st_r.vel[o_r]).max()
    verr = np.abs(g["vel"] - st.vel[o]).max()
    assert verr <= max(10 * vshadow, 8 * 100 * np.spacing(np.float32(np.abs(st.vel).max()))), (
        verr, vshadow)


# ------------------------------------------------- invariants ------------

def test_third_law_bitwise_history():
    """P11 on the GPU: δ_t,ij = -δ_t,ji bitwise for every pair contact."""
    sc = S.C2()
    d = make(sc, flags=0)
    d.step(30)
    c = contacts_dict(d)
    pairs = [(a, b) for (a, b) in c if b < S_WALL]
    assert len(pairs) > 10000
    for a, b in pairs:
        assert np.array_equal(c[(a, b)].astype(np.float32), -c[(b, a)].astype(np.float32))


S_WALL = 0xFFFFFFF0


def test_kissing_bound_and_contact_symmetry():
    sc = S.C3()
    d = make(sc, flags=0)
    for _ in range(3):
        d.step(10)
        id_i, id_j, _ = d.get_contacts()
        pair = id_j < S_WALL
        per = np.bincount(id_i[pair], minlength=sc.n)
        assert per.max() <= 12
        st = d.stats()
        assert st["contacts"] == len(id_i)
        assert st["max_contacts_seen"] <= 16


def test_momentum_conservation_gpu():
    """T4/P12: g = 0, no walls touched: |ΔΣmv| within fp32 accumulation."""
    c1 = S.C1()
    sp = S.SimParams(gravity=(0.0, 0.0, 0.0), box_hi=(0.016, 0.02, 0.016))
    sc = S.make_scene("free", sp, c1.pos + np.float32(2e-3), c1.vel, c1.omega)
    d = make(sc, flags=0)
    s0 = d.get_state()
    P0 = (s0["mass"][:, None].astype(np.float64) * s0["vel"]).sum(0)
    A = (s0["mass"][:, None].astype(np.float64) * np.abs(s0["vel"])).sum()
    d.step(2000)
    s1 = d.get_state()
    P1 = (s1["mass"][:, None].astype(np.float64) * s1["vel"]).sum(0)
    assert np.abs(P1 - P0).max() <= 1e-4 * A


def test_energy_conservation_gpu():
    """α = 0, μ = 0, g = 0, elastic walls: the GPU run's total energy (kinetic,
    rotational and Hertz elastic, evaluated in fp64 from the fp32 state) stays
    within the oracle's bound of the same experiment, with no secular drift."""
    from .test_oracle_dynamics import total_energy
    c1 = S.C1()
    sp = S.SimParams(gravity=(0.0, 0.0, 0.0), damping=0.0, friction=0.0)
    sc = S.make_scene("c1", sp.replace(box_hi=c1.params.box_hi), c1.pos, c1.vel * np.float32(4),
                      c1.omega)
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc, flags=0)

    def energy():
        s = d.get_state()
        st = orc.State.from_arrays(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"],
                                   s["id"])
        return total_energy(orc, st, p)
    E0 = energy()
    dev = []
    for _ in range(20):
        d.step(100)
        dev.append(energy() / E0 - 1)
    assert np.mean(np.abs(dev)) < 3e-3
    assert abs(np.mean(dev[-5:]) - np.mean(dev[:5])) < 2e-3  # no drift


def test_determinism_and_graph_equivalence():
    sc = S.C2()
    outs = []
    for flags in (0, 0, DEM_F_NO_GRAPH):
        d = make(sc, flags=flags)
        d.step(41)
        s = d.get_state()
        outs.append((s, d.get_contacts()))
    def as_dict(c):  # history lists are looked up by partner id: compare as maps
        return {(int(a), int(b)): v.tobytes() for a, b, v in zip(*c)}
    for s, c in outs[1:]:
        for k in ("pos", "vel", "omega", "id"):
            assert np.array_equal(s[k], outs[0][0][k])
        assert as_dict(c) == as_dict(outs[0][1])  # bitwise δ_t per contact


@pytest.mark.parametrize("other", [DEM_F_HALF_LISTS, DEM_F_THREAD_PER_PARTICLE])
def test_sweep_variants_agree(other):
    """The force-kernel mappings (contact lists, warp-flattened rounds, the
    paper's fused thread per particle) evaluate the same contacts with the
    same arithmetic and summation order; only the compiler's FMA contraction
    may differ between kernels, so one step agrees to fp32 rounding and the
    contact sets bit-exactly."""
    sc = S.C2()
    a = make(sc, flags=DEM_F_DIAG)
    b = make(sc, flags=DEM_F_DIAG | other)
    a.step(5)
    b.step(5)
    sa, sb = a.get_state(forces=True), b.get_state(forces=True)
    assert np.array_equal(sa["id"], sb["id"])
    scale = np.abs(sa["force"]).max()
    assert np.abs(sa["force"] - sb["force"]).max() <= 1e-5 * scale
    assert contacts_dict(a).keys() == contacts_dict(b).keys()


@pytest.mark.parametrize("name", ["C2", "gas"])
def test_force_configs_bitwise(name):
    """The dense, light and lanes force configurations differ only in how a
    warp's contacts are dealt to lanes and where owner state and partner slots
    are staged: same contacts, same arithmetic, same per-owner summation
    order, so whole runs agree bitwise."""
    sc = S.C2() if name == "C2" else scenes_small()[1]
    runs = []
    for f in (DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES, DEM_F_FORCE_WS,
              DEM_F_FORCE_DENSE | DEM_F_SPLIT_SWEEP, DEM_F_FORCE_LIGHT | DEM_F_SPLIT_SWEEP):
        d = make(sc, flags=DEM_F_DIAG | f)
        d.step(12)
        runs.append((d.get_state(forces=True), contacts_dict(d), d.stats()["force_cfg"]))
    assert [r[2] for r in runs] == ["dense", "light", "lanes", "ws", "dense", "light"]
    for r in runs[1:]:
        for k in ("pos", "vel", "omega", "id", "force", "torque"):
            assert np.array_equal(runs[0][0][k], r[0][k]), k
        assert runs[0][1].keys() == r[1].keys()
        assert all(np.array_equal(runs[0][1][x], r[1][x]) for x in runs[0][1])


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_mono_detect_bitwise(name):
    """One radius: k_detect's constant-S² candidate test makes the decisions of
    the per-pair S = r_i + r_j test (DEM_F_GENERAL_DETECT), so whole runs agree
    bitwise."""
    sc = S.CONFIGS[name]()
    assert np.all(sc.radius == sc.radius[0])
    runs = []
    for f in (0, DEM_F_GENERAL_DETECT):
        d = make(sc, flags=DEM_F_DIAG | f)
        d.step(8)
        runs.append((d.get_state(forces=True), contacts_dict(d)))
    for k in ("pos", "vel", "omega", "id", "force", "torque"):
        assert np.array_equal(runs[0][0][k], runs[1][0][k]), k
    assert runs[0][1].keys() == runs[1][1].keys()


def test_force_config_choice():
    """Automatic choice after the first step: dense for the jittered FCC
    packing (c̄ ≈ 11), light for the simple-cubic settling bed (c̄ ≈ 5)."""
    fcc = make(S.C3(), flags=0)
    assert fcc.stats()["force_cfg"] is None
    fcc.step(2)
    assert fcc.stats()["force_cfg"] == "dense"
    bed = make(S.C4(scale=4), flags=0)
    bed.step(2)
    assert bed.stats()["force_cfg"] == "light"


def analysis_from_oracle(p, s, K):
    """The §6 quantities of dem_analyze, recomputed from the oracle's grid
    (hash, stable sort, offsets, 27-cell neighbour sets) and its contact set
    for the same input state."""
    pos = s["pos"].astype(np.float64)
    n = pos.shape[0]
    nx, ny, nz = orc.grid_dims(p)
    CM = orc.hash_cells(p, pos)
    SCM, SCCM = orc.sort_map(CM)
    off = orc.cell_offsets(SCM, nx * ny * nz).astype(np.int64)
    pop = np.diff(off)
    cand_cell = {}
    cand = np.empty(n, np.int64)
    for j in range(n):
        c = int(SCM[j])
        if c not in cand_cell:
            cand_cell[c] = sum(int(pop[x]) for x in orc.neighbor_cells(p, c)) - 1
        cand[j] = cand_cell[c]
    pairs = orc.contacts_grid(p, pos, s["radius"])
    cont = np.bincount(pairs.ravel().astype(np.int64), minlength=n)[SCCM]  # sorted order
    w = lambda a: int(sum(32 * a[i:i + 32].max() for i in range(0, n, 32)))
    return dict(n=n, candidates=int(cand.sum()), max_candidates=int(cand.max()),
                contacts=int(cont.sum()), max_contacts=int(cont.max()),
                warp_candidate_slots=w(cand), warp_contact_slots=w(cont),
                max_per_cell=int(pop.max()), occupied_cells=int((pop > 0).sum()),
                contact_hist=list(np.bincount(np.minimum(cont, 32), minlength=33)))


@pytest.mark.parametrize("variant", [0, DEM_F_HALF_LISTS, DEM_F_THREAD_PER_PARTICLE])
@pytest.mark.parametrize("idx", [0, 1])
def test_analysis_matches_oracle(idx, variant):
    """dem_analyze (the paper's §6 counts: candidates, contacts, SIMT lane
    slots of the thread-per-particle mapping, cell populations) equals the
    same counts taken from the oracle's grid and contact set, exactly."""
    sc = [S.C2(), scenes_small()[1]][idx]
    p = orc.make_params(sc.params, sc.radius)
    d = make(sc, flags=variant)
    d.step(3)
    s = d.get_state()
    d.step(1)
    got = d.analyze()
    want = analysis_from_oracle(p, s, sc.params.max_contacts)
    for k, v in want.items():
        assert got[k] == v, (k, got[k], v)
    if idx == 0:  # equal spheres: the kissing bound of PAPER.md:155
        assert got["max_contacts"] <= 12


def test_set_particles_accepts_what_a_step_produces():
    """dem_set_particles takes centres up to r beyond a wall (a particle in
    contact with it, R18), like the step's escape check, and rejects more."""
    sc = S.C1()
    pos = sc.pos.copy()
    for frac, ok in ((0.5, True), (2.0, False)):
        pos[0, 0] = sc.params.box_lo[0] - frac * sc.radius[0]
        d = Dem(sc.params)
        if ok:
            d.set_particles(pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
        else:
            with pytest.raises(DemError) as e:
                d.set_particles(pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
            assert "outside" in str(e.value)


# ------------------------------------------- material pairs (Eqs. 5, 8-10) --

def mixed(M=3, n=3000, seed=7):
    return S.mixed_gas(n, 14.0, seed, M=M, r_range=(0.25e-3, 0.5e-3), v_sigma=0.05,
                       params=S.SimParams(max_contacts=32))


@pytest.mark.parametrize("variant", [DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES,
                                     DEM_F_HALF_LISTS, DEM_F_THREAD_PER_PARTICLE])
def test_materials_one_step_T2(variant):
    """Each particle pair takes C_n, C_t, α, μ from its two materials and each
    wall contact from the particle's material: T2 against the oracle."""
    sc = mixed()
    p = orc.make_params(sc.params, sc.radius)
    d = Dem(sc.params, flags=DEM_F_DIAG | variant)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id, material=sc.material)
    for k in range(3):
        st, h = oracle_inputs(d, 32)
        assert st.mat is not None and st.mat.max() > 0
        d.step(1)
        g = d.get_state(forces=True)
        res = orc.step(p, st, h)
        assert res.rc == 0
        assert np.array_equal(g["id"], st.id) and np.array_equal(g["material"], st.mat)
        assert_T2_forces(g["force"], g["torque"], res, what=f"mixed step {k + 1}")
        assert_T2_history(contacts_dict(d), h.as_dict(st.id))


def test_materials_uniform_table_bitwise():
    """A table whose every entry is the scalar parameters reproduces the
    scalar run bitwise on the GPU."""
    sc = scenes_small()[1]
    sp = sc.params
    c = (sp.stiffness_n, sp.stiffness_t, sp.damping, sp.friction)
    spm = sp.replace(materials=((c, c), (c, c)), wall_materials=(c, c))
    runs = []
    for params, mat in ((sp, None), (spm, (np.arange(sc.n) % 2).astype(np.uint32))):
        d = Dem(params, flags=DEM_F_DIAG)
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id, material=mat)
        d.step(10)
        runs.append(d.get_state(forces=True))
    for k in ("pos", "vel", "omega", "id", "force", "torque"):
        assert np.array_equal(runs[0][k], runs[1][k]), k


def test_materials_checkpoint_and_validation():
    sc = mixed(n=1500, seed=3)
    d = Dem(sc.params, flags=0)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id, material=sc.material)
    d.step(8)
    s = d.get_state()
    ci, cj, cd = d.get_contacts()
    assert set(np.unique(s["material"])) == {0, 1, 2}
    assert s["id"].max() < sc.n  # the material bits are not part of the id
    e = Dem(sc.params, flags=0)
    e.set_particles(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"], s["id"],
                    material=s["material"])
    e.set_contacts(ci, cj, cd)
    d.step(7)
    e.step(7)
    a, b = d.get_state(), e.get_state()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    bad = sc.material.copy()
    bad[0] = 3  # only 3 materials
    with pytest.raises(DemError):
        Dem(sc.params).set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id,
                                     material=bad)


# ------------------------------------------------- plates (R23, slit box) --

def plate_gas(seed=5, n=2500, materials=False):
    """A gas crossing three plates (a large horizontal one, a vertical one, a
    small tilted one): face, edge and corner contacts, both sides."""
    L = 14.0 * S.D
    c = 0.5 * L
    t = np.array([1.0, 0.0, 1.0]) / math.sqrt(2.0)
    plates = (S.plate((c, c, c), (0, 1, 0), (1, 0, 0), 4 * S.D, 3 * S.D),
              S.plate((c - 3 * S.D, c, c), (1, 0, 0), (0, 0, 1), 2 * S.D, 2.5 * S.D),
              S.plate((c + 3 * S.D, c - 3 * S.D, c + 2 * S.D), tuple(t), (0, 1, 0), 1.5 * S.D,
                      1.0 * S.D))
    kw = dict(r_range=(0.3e-3, 0.5e-3), v_sigma=0.2,
              params=S.SimParams(max_contacts=32, plates=plates))
    if materials:
        return S.mixed_gas(n, 14.0, seed, M=2, **kw)
    return S.random_gas(n, 14.0, seed, **kw)


@pytest.mark.parametrize("variant", [DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES,
                                     DEM_F_HALF_LISTS, DEM_F_THREAD_PER_PARTICLE,
                                     DEM_F_SPLIT_SWEEP])
@pytest.mark.parametrize("kind", ["plates", "plates+materials", "slit"])
def test_plates_one_step_T2(kind, variant):
    """Plate contacts (faces, edges, corners, both sides) bit-exactly the
    oracle's (their history entries are part of the contact set), forces and
    torques within T2, for every force-kernel variant."""
    sc = S.slit_box((16, 6, 16)) if kind == "slit" else plate_gas(materials="mat" in kind)
    K = sc.params.max_contacts
    p = orc.make_params(sc.params, sc.radius)
    d = Dem(sc.params, flags=DEM_F_DIAG | variant)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id,
                    material=getattr(sc, "material", None))
    plate_contacts = 0
    for k in range(3):
        st, h = oracle_inputs(d, K)
        d.step(1)
        g = d.get_state(forces=True)
        res = orc.step(p, st, h)
        assert res.rc == 0
        assert np.array_equal(g["id"], st.id)
        assert_T2_forces(g["force"], g["torque"], res, what=f"{kind} step {k + 1}")
        got = contacts_dict(d)
        assert_T2_history(got, h.as_dict(st.id))
        plate_contacts += sum(1 for (_, b) in got if b >= 0xFFFFFFF6)
    assert plate_contacts > 0


def test_slit_box_flows_through_the_slit():
    """The §5 experiment at small scale: particles above the slit fall
    through it onto the floor, those beside it stay on the box bottom, none
    leaves the domain, no error."""
    sc = S.slit_box((16, 6, 16))
    d = Dem(sc.params)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    d.step(30000)  # 60 ms: the column above the slit has reached the floor
    s = d.get_state()
    y = s["pos"][:, 1]
    below = y < sc.meta["y_bottom"]
    assert 0 < below.sum() < sc.n
    assert (y > 0).all() and (y < sc.params.box_hi[1]).all()
    assert (s["pos"][below, 1] < sc.meta["y_bottom"] - 5 * S.D).mean() > 0.5
    assert d.stats()["max_speed"] > 0


def test_checkpoint_roundtrip_bitwise():
    sc = S.C1()
    d1 = make(sc, flags=0)
    d1.step(25)
    s = d1.get_state()
    id_i, id_j, dt3 = d1.get_contacts()
    d2 = Dem(sc.params)
    d2.set_particles(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"], s["id"])
    d2.set_contacts(id_i, id_j, dt3)
    d1.step(15)
    d2.step(15)
    a, b = d1.get_state(), d2.get_state()
    for k in ("pos", "vel", "omega", "id"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("K", [6, 9])
@pytest.mark.parametrize("split", [False, True])
def test_overflow_rejects_step_and_keeps_last_good_state(K, split):
    # (C1 has one radius: by default the dense configuration detects inside k_force)
    fl = DEM_F_SPLIT_SWEEP if split else 0
    sc = S.C1(S.SimParams(max_contacts=K))
    d = make(sc, flags=fl)
    with pytest.raises(DemError) as e:
        for _ in range(200):
            d.step(1)
    assert e.value.code == DEM_EOVERFLOW
    done = d.stats()["steps"]
    ref = make(sc, flags=fl)
    if done:
        ref.step(done)
    a, b = d.get_state(), ref.get_state()
    for k in ("pos", "vel", "omega", "id"):
        assert np.array_equal(a[k], b[k])
    # the same failure happens inside a multi-step graph replay
    d3 = make(sc, flags=fl)
    with pytest.raises(DemError):
        d3.step(200)
    assert d3.stats()["steps"] == done
    assert np.array_equal(d3.get_state()["pos"], a["pos"])


def test_escape_is_reported():
    sc = S.C1()
    vel = sc.vel.copy()
    vel[0] = (0.0, -4000.0, 0.0)  # crosses the floor within a step
    sc2 = S.make_scene("esc", sc.params, sc.pos, vel, sc.omega)
    d = make(sc2, flags=0)
    with pytest.raises(DemError) as e:
        d.step(5)
    assert e.value.code == DEM_EESCAPED
    assert "particle id 0" in str(e.value)


def test_coincident_centres_are_reported():
    """R18: two centres at the same point while in contact leave n undefined:
    DEM_ECOINCIDENT from the step (the oracle says the same for this input),
    the state stays that of the last good step."""
    sc = S.C1()
    pos = sc.pos.copy()
    pos[1] = pos[0]
    sc2 = S.make_scene("coinc", sc.params, pos, sc.vel, sc.omega)
    p = orc.make_params(sc2.params, sc2.radius)
    d = make(sc2, flags=0)
    s0 = d.get_state()
    with pytest.raises(DemError) as e:
        d.step(3)
    assert e.value.code == DEM_ECOINCIDENT
    assert "particle id 0" in str(e.value) or "particle id 1" in str(e.value)
    assert d.stats()["steps"] == 0
    assert np.array_equal(d.get_state()["pos"], s0["pos"])
    st = orc.State.from_scene(sc2)
    assert orc.step(p, st, orc.History.empty(sc2.n, 16)).rc == orc.ECOINCIDENT


@pytest.mark.parametrize("graph", [True, False])
def test_nonfinite_is_reported(graph):
    """NaN injection through the public API: a checkpointed tangential history
    (dem_set_contacts does not validate δ_t values) with one NaN entry makes
    that particle's force, velocity and position NaN in the next step, which
    the integrator reports as DEM_ENONFINITE with the particle's id; the state
    stays the last good one."""
    sc = S.C1()
    base = 0 if graph else DEM_F_NO_GRAPH
    d = make(sc, flags=base)
    d.step(5)
    s = d.get_state()
    ci, cj, cd = d.get_contacts()
    slot = {int(i): x for x, i in enumerate(s["id"])}
    pair = np.nonzero(cj < S_WALL)[0]
    a = np.array([slot[int(i)] for i in ci[pair]])
    b = np.array([slot[int(j)] for j in cj[pair]])
    ov = s["radius"][a] + s["radius"][b] - np.linalg.norm(s["pos"][a] - s["pos"][b], axis=1)
    k = int(pair[np.argmax(ov)])  # the deepest contact: still touching next step
    cd = cd.copy()
    cd[k, 1] = np.nan
    e = Dem(sc.params, flags=base)
    e.set_particles(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"], s["id"])
    e.set_contacts(ci, cj, cd)
    with pytest.raises(DemError) as err:
        e.step(4)
    assert err.value.code == DEM_ENONFINITE
    assert f"particle id {int(ci[k])} " in str(err.value)
    assert e.stats()["steps"] == 0
    assert np.array_equal(e.get_state()["pos"], s["pos"])


def test_device_tensors_and_order_id(cuda):
    torch = cuda
    sc = S.C1()
    d = Dem(sc.params)
    t = lambda a: torch.as_tensor(a).cuda()  # noqa: E731
    d.set_particles(t(sc.pos), t(sc.vel), t(sc.omega), t(sc.radius), t(sc.mass),
                    t(sc.id.astype(np.int32)))
    d.step(3)
    out = {k: torch.empty(v, dtype=torch.float32, device="cuda")
           for k, v in (("pos", (sc.n, 3)), ("vel", (sc.n, 3)), ("omega", (sc.n, 3)))}
    out["id"] = torch.empty(sc.n, dtype=torch.int32, device="cuda")
    d.get_state(order=DEM_ORDER_ID, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out["id"].cpu(), torch.arange(sc.n, dtype=torch.int32))
    h = make(sc, flags=0)
    h.step(3)
    ref = h.get_state(order=DEM_ORDER_ID)
    assert np.array_equal(out["pos"].cpu().numpy(), ref["pos"])


def test_profile_mode_times_every_kernel():
    sc = S.C2()
    d = make(sc, flags=0)
    d.profile(True)
    d.step(10)
    st = d.stats()
    for k in ("rank", "sweep"):
        assert st["kernel_count"][k] == 10
        assert st["kernel_ms"][k] > 0
    # C2 (one radius, dense): detection inside the force kernel; split: k_detect
    assert st["fused_sweep"] and st["kernel_count"]["detect"] == 0
    sp = make(sc, flags=DEM_F_SPLIT_SWEEP)
    sp.profile(True)
    sp.step(10)
    assert not sp.stats()["fused_sweep"] and sp.stats()["kernel_count"]["detect"] == 10
    # the counting sort (cell counts, scan, scatter) runs only in the first
    # step; the merge re-sort's one kernel is timed as rank afterwards
    assert st["kernel_count"]["hash"] == 1 and st["kernel_count"]["scan"] == 1
    assert st["kernel_count"]["scatter"] == 1
    assert st["full_sorts"] == 1
    assert st["steps"] == 10
    f = make(sc, flags=DEM_F_FULL_SORT)
    f.profile(True)
    f.step(10)
    assert all(f.stats()["kernel_count"][k] == 10 for k in ("scan", "scatter", "rank", "sweep"))
