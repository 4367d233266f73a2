"""In-process slab ranks (device-pointer connection) on the settling bed."""
import sys
sys.path.insert(0, ".")
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sc = S.C4(scale=scale)
ds = [Dem(sc.params, flags=0, rank=r, world=P) for r in range(P)]
for d in ds:
    d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    print("rank", d.rank, "n", d.n, flush=True)
for r, d in enumerate(ds):
    d.connect_local(ds[r - 1] if r > 0 else None, ds[r + 1] if r < P - 1 else None)
for k in range(3):
    for d in ds:
        try:
            d.step(1)
            print("rank", d.rank, "step", k, "ok n", d.n, flush=True)
        except Exception as e:  # noqa: BLE001
            print("rank", d.rank, "step", k, "FAILED", e, flush=True)
            sys.exit(1)
