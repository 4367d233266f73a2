"""GPU tests of the slab decomposition on one B200:
P slab ranks as separate handles — in one process (neighbours connected by
device pointer) and in two processes (connected by CUDA IPC handles, the
multi-GPU transport) — against the fp64 oracle on the gathered state, and
against the single-GPU path. Run via gpurun: python -m pytest tests -m gpu."""
import multiprocessing as mp

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1301_1714_b200 import scenes as S
from paper_1301_1714_b200.dem import DEM_F_DIAG, Dem, DemError

from .parity import assert_T2_forces, assert_T2_history

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


def fast_gas(seed=3, n=6000):
    """Dense polydisperse gas with fast particles: migrations every step."""
    return S.random_gas(n, 18.0, seed, r_range=(0.3e-3, 0.5e-3), v_sigma=3.0, w_sigma=50.0,
                        params=S.SimParams(max_contacts=32, gravity=(0.0, -9.81, 0.0)))


def make_slabs(sc, P, flags=DEM_F_DIAG):
    ds = [Dem(sc.params, flags=flags, rank=r, world=P) for r in range(P)]
    for d in ds:
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    for r, d in enumerate(ds):
        d.connect_local(ds[r - 1] if r > 0 else None, ds[r + 1] if r < P - 1 else None)
    return ds


def step_all(ds, n=1):
    for _ in range(n):
        for d in ds:
            d.step(1)


def union_state(ds, forces=False):
    parts = [d.get_state(forces=forces) for d in ds]
    cat = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    o = np.argsort(cat["id"], kind="stable")
    return {k: v[o] for k, v in cat.items()}


def union_contacts(ds):
    out = {}
    for d in ds:
        a, b, v = d.get_contacts()
        for x, y, z in zip(a, b, v):
            key = (int(x), int(y))
            assert key not in out  # each particle is reported by exactly one rank
            out[key] = z.astype(np.float64)
    return out


@pytest.mark.parametrize("P", [2, 3])
def test_partition_is_exact(P):
    sc = S.C2()
    ds = make_slabs(sc, P)
    ns = [d.n for d in ds]
    assert sum(ns) == sc.n and min(ns) > 0
    u = union_state(ds)
    assert np.array_equal(u["id"], np.sort(sc.id))


@pytest.mark.parametrize("P", [2, 3])
def test_slab_steps_match_oracle(P):
    """Every step, the union of the ranks' outputs equals one oracle step of the
    union of their inputs: same contact pairs bit-exactly, T2 forces/torques,
    with particles migrating between slabs."""
    sc = fast_gas()
    p = orc.make_params(sc.params, sc.radius)
    ds = make_slabs(sc, P)
    migrated = 0
    owner = {int(i): r for r, d in enumerate(ds) for i in d.get_state()["id"]}
    for k in range(6):
        u = union_state(ds)
        st = orc.State.from_arrays(u["pos"], u["vel"], u["omega"], u["radius"], u["mass"], u["id"])
        c = union_contacts(ds) if k else {}
        if c:
            keys = sorted(c)
            h = orc.History.from_pairs(st.id, 32, [a for a, _ in keys], [b for _, b in keys],
                                       np.array([c[x] for x in keys]))
        else:
            h = orc.History.empty(st.n, 32)
        step_all(ds)
        res = orc.step(p, st, h)
        assert res.rc == 0
        g = union_state(ds, forces=True)
        o = np.argsort(st.id)  # oracle output (its sorted order) -> id order
        assert np.array_equal(g["id"], st.id[o])

        class R:  # the oracle result in id order
            F, T, Fabs, Tabs = res.F[o], res.T[o], res.Fabs[o], res.Tabs[o]
        assert_T2_forces(g["force"], g["torque"], R, what=f"P={P} step {k + 1}")
        assert_T2_history(union_contacts(ds), h.as_dict(st.id))
        now = {int(i): r for r, d in enumerate(ds) for i in d.get_state()["id"]}
        migrated += sum(1 for i in now if now[i] != owner[i])
        owner = now
    assert migrated > 0  # the test exercised migration


def test_slabs_agree_with_single_gpu():
    sc = S.C2()
    one = Dem(sc.params, flags=DEM_F_DIAG)
    one.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    ds = make_slabs(sc, 3)
    one.step(1)
    step_all(ds)
    a = one.get_state(forces=True)
    o = np.argsort(a["id"])
    a = {k: v[o] for k, v in a.items()}
    b = union_state(ds, forces=True)
    assert np.array_equal(a["id"], b["id"])
    scale = np.abs(a["force"]).max()
    assert np.abs(a["force"] - b["force"]).max() <= 1e-5 * scale
    ca = {}
    for x, y, z in zip(*one.get_contacts()):
        ca[(int(x), int(y))] = z
    assert ca.keys() == union_contacts(ds).keys()


def test_slab_run_is_deterministic():
    sc = fast_gas(seed=9, n=4000)
    runs = []
    for _ in range(2):
        ds = make_slabs(sc, 2, flags=0)
        step_all(ds, 15)
        runs.append(union_state(ds))
    for k in ("pos", "vel", "omega", "id"):
        assert np.array_equal(runs[0][k], runs[1][k])


def _ipc_rank(rank, world, q_out, q_in, steps, result):
    import torch  # noqa: F401  (CUDA context in the child)
    sc = fast_gas(seed=9, n=4000)
    d = Dem(sc.params, flags=0, rank=rank, world=world, torch_allocator=False)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    q_out.put((rank, d.exchange_handle()))
    handles = dict([q_in.get() for _ in range(world - 1)])
    d.connect(handles.get(rank - 1), handles.get(rank + 1))
    d.step(steps)
    s = d.get_state()
    result.put((rank, {k: v.copy() for k, v in s.items()}))


def test_two_process_ipc_matches_single_process():
    """The CUDA IPC transport (two processes sharing the GPU, as two GPUs
    would over NVLink) reproduces the in-process slab run bitwise."""
    ctx = mp.get_context("spawn")
    q0, q1, res = ctx.Queue(), ctx.Queue(), ctx.Queue()
    steps = 15
    # rank r publishes on q_r and reads the other's
    procs = [ctx.Process(target=_ipc_rank, args=(0, 2, q0, q1, steps, res)),
             ctx.Process(target=_ipc_rank, args=(1, 2, q1, q0, steps, res))]
    for p in procs:
        p.start()
    parts = dict(res.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cat = {k: np.concatenate([parts[0][k], parts[1][k]]) for k in parts[0]}
    o = np.argsort(cat["id"], kind="stable")
    ipc = {k: v[o] for k, v in cat.items()}
    ds = make_slabs(fast_gas(seed=9, n=4000), 2, flags=0)
    step_all(ds, steps)
    ref = union_state(ds)
    for k in ("pos", "vel", "omega", "id"):
        assert np.array_equal(ipc[k], ref[k])


def test_reset_particles_between_runs():
    """Setting the particles again restarts every rank; stale publications of
    the previous run are never taken for the new one (exchange tag epochs)."""
    sc = fast_gas(seed=4, n=3000)
    ds = make_slabs(sc, 2, flags=0)
    step_all(ds, 3)
    for d in ds:
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    step_all(ds, 5)
    a = union_state(ds)
    fresh = make_slabs(sc, 2, flags=0)
    step_all(fresh, 5)
    b = union_state(fresh)
    for k in ("pos", "vel", "omega", "id"):
        assert np.array_equal(a[k], b[k])


def test_slab_checkpoint_roundtrip():
    """Restart from a checkpoint: every rank is given the gathered state and
    the gathered contact list (dem_set_contacts keeps each rank's own) and
    the run continues as the uninterrupted one: same contact pairs, state
    equal to fp32 summation-order rounding (in-cell ties follow the new input
    order)."""
    sc = fast_gas(seed=6, n=5000)
    ds = make_slabs(sc, 2, flags=0)
    step_all(ds, 4)
    u = union_state(ds)
    c = union_contacts(ds)
    step_all(ds, 6)
    ref = union_state(ds)
    keys = sorted(c)
    ii = np.array([a for a, _ in keys], np.uint32)
    jj = np.array([b for _, b in keys], np.uint32)
    vv = np.array([c[k] for k in keys], np.float32)
    fresh = [Dem(sc.params, flags=0, rank=r, world=2) for r in range(2)]
    for d in fresh:
        d.set_particles(u["pos"], u["vel"], u["omega"], u["radius"], u["mass"], u["id"])
        d.set_contacts(ii, jj, vv)
    for r, d in enumerate(fresh):
        d.connect_local(fresh[r - 1] if r > 0 else None, fresh[r + 1] if r < 1 else None)
    step_all(fresh, 6)
    got = union_state(fresh)
    assert np.array_equal(got["id"], ref["id"])
    assert np.abs(got["pos"] - ref["pos"]).max() <= 1e-6 * np.abs(ref["pos"]).max()
    assert np.abs(got["vel"] - ref["vel"]).max() <= 1e-4 * np.abs(ref["vel"]).max()
    assert union_contacts(fresh).keys() == union_contacts(ds).keys()


def test_slab_set_contacts_global_list():
    """Every rank given the same global contact list keeps exactly its own."""
    sc = fast_gas(seed=8, n=4000)
    ds = make_slabs(sc, 3, flags=0)
    step_all(ds, 3)
    before = union_contacts(ds)
    keys = sorted(before)
    ii = np.array([a for a, _ in keys], np.uint32)
    jj = np.array([b for _, b in keys], np.uint32)
    vv = np.array([before[k] for k in keys], np.float32)
    for d in ds:
        d.set_contacts(ii, jj, vv)
    after = union_contacts(ds)
    assert after.keys() == before.keys()
    assert all(np.array_equal(after[k], before[k].astype(np.float32)) for k in keys)


@pytest.mark.parametrize("P", [2, 3])
def test_slabs_settling_bed_match_single_gpu(P):
    """The bench's workload (a settling bed, dense boundary planes, slabs of
    unequal plane counts): slab ranks agree with the single-GPU run."""
    sc = S.C4(scale=8)
    one = Dem(sc.params, flags=DEM_F_DIAG)
    one.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    ds = make_slabs(sc, P)
    one.step(4)
    step_all(ds, 4)
    a = one.get_state(forces=True)
    o = np.argsort(a["id"])
    a = {k: v[o] for k, v in a.items()}
    b = union_state(ds, forces=True)
    assert np.array_equal(a["id"], b["id"])
    assert np.abs(a["pos"] - b["pos"]).max() <= 1e-6 * np.abs(a["pos"]).max()
    ca = {(int(x), int(y)) for x, y, _ in zip(*one.get_contacts())}
    assert ca == set(union_contacts(ds))


@pytest.mark.parametrize("name", ["bed", "gas"])
def test_slab_long_run_matches_single_gpu(name):
    """300 steps as 3 slab ranks (merge re-sort, ghost planes sorted by their
    senders; the gas sends particles across slabs every step) against the
    single-GPU run: the same particles, the same contact pairs, and the same
    trajectories — both paths evaluate every contact with the same
    arithmetic in the same candidate order, so the runs stay bitwise equal."""
    sc = S.C4(scale=8) if name == "bed" else fast_gas(seed=13, n=5000)
    one = Dem(sc.params, flags=0)
    one.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    ds = make_slabs(sc, 3, flags=0)
    owner0 = {int(i): r for r, d in enumerate(ds) for i in d.get_state()["id"]}
    for _ in range(3):
        one.step(100)
        step_all(ds, 100)
    owner1 = {int(i): r for r, d in enumerate(ds) for i in d.get_state()["id"]}
    if name == "gas":
        assert sum(owner0[i] != owner1[i] for i in owner1) > 100  # particles changed slab
    a = one.get_state()
    o = np.argsort(a["id"])
    a = {k: v[o] for k, v in a.items()}
    b = union_state(ds)
    assert np.array_equal(a["id"], b["id"])
    for k in ("pos", "vel", "omega"):
        assert np.array_equal(a[k], b[k]), (k, np.abs(a[k] - b[k]).max())
    ca = {(int(x), int(y)) for x, y, _ in zip(*one.get_contacts())}
    assert ca == set(union_contacts(ds))


def test_slab_ranks_with_different_sets_refuse_to_connect():
    """Every rank must be given the same particle set (the exchange layout is
    derived from it); otherwise connecting fails instead of mis-reading."""
    sc = S.C4(scale=8)
    ds = [Dem(sc.params, flags=0, rank=r, world=2) for r in range(2)]
    ds[0].set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    m = np.arange(sc.n) % 2 == 0  # half the particles on rank 1: sparser planes
    ds[1].set_particles(sc.pos[m], sc.vel[m], sc.omega[m], sc.radius[m], sc.mass[m], sc.id[m])
    with pytest.raises(DemError) as e:
        ds[0].connect_local(None, ds[1])
    assert "layout" in str(e.value)


def test_slab_overflow_fails_fast():
    """A whole z-plane of spheres (49 x 49) crosses the slab boundary in one
    step: more migrants than the exchange blocks hold (capacity from the most
    populated plane: max(1024, (2 x 2,402 + 1,024) / 4) = 1,457). The sending
    rank's step fails with DEM_EOVERFLOW; its publication carries the failure,
    so the neighbour's next step fails with DEM_EPEER at once — not after the
    ~30 s tag timeout, and without reading past the exchange block."""
    import time

    from paper_1301_1714_b200.dem import DEM_EOVERFLOW, DEM_EPEER

    L = 60e-3
    params = S.SimParams(gravity=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    h = 2 * S.R * (1 + 2.0**-10)
    nz = int(np.floor(L / h))
    zb = (nz // 2) * h  # rank 1's first plane (planes split evenly)
    g = 0.6e-3 + 1.2e-3 * np.arange(49)
    x, y = np.meshgrid(g, g, indexing="ij")
    pos = np.stack([x.ravel(), y.ravel(), np.full(x.size, zb - 0.2e-3)], 1)
    vel = np.zeros_like(pos)
    vel[:, 2] = 0.4e-3 / params.dt  # 0.4 mm in one step: into rank 1's first plane
    sc = S.make_scene("plane_crossing", params, pos, vel)
    ds = make_slabs(sc, 2, flags=0)
    assert len(ds[0].get_state()["id"]) == sc.n
    with pytest.raises(DemError) as e:
        ds[0].step(1)
    assert e.value.code == DEM_EOVERFLOW
    ds[1].step(1)  # reads rank 0's publication from dem_set_particles: fine
    t0 = time.perf_counter()
    with pytest.raises(DemError) as e:
        ds[1].step(1)  # reads rank 0's failed step
    assert e.value.code == DEM_EPEER and "neighbour's step failed" in str(e.value)
    assert time.perf_counter() - t0 < 10.0
