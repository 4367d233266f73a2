"""P in-process slab ranks (C4 narrowed by --scale) stepped in turn on one
B200, for an ncu launch list of the slab step's kernels:
    ncu --metrics gpu__time_duration.sum -s S -c C --csv --log-file X.csv \\
        python tools/slab_launches.py --scale 2 --P 2
Single-GPU reference at one rank's size: --P 1 --z 2 (the bed narrowed in z)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=2)
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--z", type=int, default=1, help="single GPU: narrow the bed in z by this")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
sc = S.C4(scale=a.scale)
if a.z > 1:
    m = sc.meta["nxyz"]
    sc = S.settling_bed(f"{sc.name}/z{a.z}", (m[0], m[1], m[2] // a.z), (m[0] + 2, 72, m[2] // a.z + 2),
                        seed=4)
ds = [Dem(sc.params, rank=r, world=a.P) if a.P > 1 else Dem(sc.params) for r in range(a.P)]
for x in ds:
    x.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
if a.P > 1:
    for r, x in enumerate(ds):
        x.connect_local(ds[r - 1] if r > 0 else None, ds[r + 1] if r < a.P - 1 else None)
for _ in range(a.steps):
    for x in ds:
        x.step(1)
print("ok", [x.stats()["n"] for x in ds])
