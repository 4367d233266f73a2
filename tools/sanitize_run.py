"""Small workloads for compute-sanitizer (tools/sanitize.sh): every step
kernel of every force-kernel variant, slabs, materials, plates, on C1/C2-sized
scenes, eager launches, the library's own allocator."""
import sys

sys.path.insert(0, ".")
from paper_1301_1714_b200 import scenes as S  # noqa: E402
import numpy as np  # noqa: E402
from paper_1301_1714_b200.dem import (DEM_F_DIAG, DEM_F_FORCE_DENSE, DEM_F_FORCE_LANES, DEM_F_FORCE_WS,  # noqa: E402
                                      DEM_F_FORCE_LIGHT, DEM_F_HALF_LISTS, DEM_F_NO_GRAPH,
                                      DEM_F_SPLIT_SWEEP, DEM_F_THREAD_PER_PARTICLE, Dem)


def run(sc, flags, steps=3, material=None):
    d = Dem(sc.params, flags=flags | DEM_F_NO_GRAPH | DEM_F_DIAG, torch_allocator=False)
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id, material=material)
    d.step(steps)
    d.get_state(forces=True)
    ci, cj, cd = d.get_contacts()
    d.set_contacts(ci, cj, cd)
    d.step(1)
    d.analyze()
    d.stats()
    d.close()


for f in (DEM_F_FORCE_DENSE, DEM_F_FORCE_LIGHT, DEM_F_FORCE_LANES, DEM_F_FORCE_WS, DEM_F_HALF_LISTS,
          DEM_F_THREAD_PER_PARTICLE, DEM_F_SPLIT_SWEEP | DEM_F_FORCE_DENSE):
    run(S.C1(), f)  # (C1 has one radius: dense = detection fused into k_force)


def crossers(n_side, gap=3e-8):
    """n_side³ separated spheres just below a cell face, moving +x: all change
    cell in step 2, so step 3's merge re-sort takes n_side³ movers (512, 729:
    more events per k_merge block than its shared list; 13,824: more movers
    than the list holds, so that step is rolled back and redone by counting)."""
    p = S.SimParams(gravity=(0.0, 0.0, 0.0))
    h = 2.0 * S.R * (1.0 + 2.0 ** -10)
    L = (3 * n_side + 4) * h
    p = p.replace(box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    g = np.stack(np.meshgrid(*[np.arange(n_side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    c = (3 * g + 2).astype(np.float64)
    pos = (c + 0.5) * h
    pos[:, 0] = (c[:, 0] + 1.0) * h - gap
    vel = np.zeros_like(pos)
    vel[:, 0] = 0.01
    return S.make_scene("crossers", p, pos.astype(np.float32), vel.astype(np.float32))


for ns in (8, 9, 24):
    run(crossers(ns), 0, steps=4)
run(S.C2(S.SimParams(model="simple")), 0)
mg = S.mixed_gas(800, 10.0, 2, M=3, params=S.SimParams(max_contacts=32))
run(mg, DEM_F_FORCE_LIGHT, material=mg.material)
run(S.slit_box((8, 4, 8)), DEM_F_FORCE_DENSE)
# two slab ranks in one process
sc = S.random_gas(3000, 16.0, 3, r_range=(0.3e-3, 0.5e-3), v_sigma=2.0,
                  params=S.SimParams(max_contacts=32))
ds = [Dem(sc.params, flags=DEM_F_NO_GRAPH, rank=r, world=2, torch_allocator=False) for r in range(2)]
for d in ds:
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
ds[0].connect_local(None, ds[1])
ds[1].connect_local(ds[0], None)
for _ in range(3):
    for d in ds:
        d.step(1)
print("sanitize workload done", flush=True)
