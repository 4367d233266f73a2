"""Per-rank kernel breakdown of the slab path against the single-GPU path on
one B200: C4 narrowed by --scale as one handle, and as P slab
ranks in one process (neighbours by device pointer), each rank stepped in
turn with per-kernel CUDA events (dem_profile). Prints µs per step and ns per
owned particle per kernel class."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=2)
ap.add_argument("--P", type=int, nargs="+", default=[2, 3])
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--warmup", type=int, default=10)
a = ap.parse_args()
sc = S.C4(scale=a.scale)
out = {"scene": sc.name, "n": sc.n}


def breakdown(ds, steps):
    for d in ds:
        d.profile(True)
    for _ in range(steps):
        for d in ds:
            d.step(1)
    res = []
    for d in ds:
        st = d.stats()
        n = st["n"]
        k = {c: st["kernel_ms"][c] / steps * 1e3 for c in st["kernel_ms"] if st["kernel_count"][c]}
        res.append({"n_owned": n, "us_per_step": k, "total_us": sum(k.values()),
                    "ns_per_particle": sum(k.values()) * 1e3 / n,
                    "full_sorts": st["full_sorts"]})
        d.profile(False)
    return res


d = Dem(sc.params)
d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
d.step(a.warmup)
out["single"] = breakdown([d], a.steps)[0]
d.close()
for P in a.P:  # the same bed narrowed in z to one rank's share: a single GPU at rank size
    m = sc.meta["nxyz"]
    sub_sc = S.settling_bed(f"{sc.name}/z{P}", (m[0], m[1], m[2] // P),
                            (m[0] + 2, 72, m[2] // P + 2), seed=4)
    d = Dem(sub_sc.params)
    d.set_particles(sub_sc.pos, sub_sc.vel, sub_sc.omega, sub_sc.radius, sub_sc.mass, sub_sc.id)
    d.step(a.warmup)
    out[f"single_z{P}"] = breakdown([d], a.steps)[0]
    d.close()
for P in a.P:
    ds = [Dem(sc.params, rank=r, world=P) for r in range(P)]
    for x in ds:
        x.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    for r, x in enumerate(ds):
        x.connect_local(ds[r - 1] if r > 0 else None, ds[r + 1] if r < P - 1 else None)
    for _ in range(a.warmup):
        for x in ds:
            x.step(1)
    out[f"P{P}"] = breakdown(ds, a.steps)
    for x in ds:
        x.close()
print(json.dumps(out))
print("single ns/particle", round(out["single"]["ns_per_particle"], 3))
for P in a.P:
    s = out[f"single_z{P}"]["ns_per_particle"]
    print(f"single at rank size (n {out[f'single_z{P}']['n_owned']}) ns/particle {s:.3f}",
          {k: round(v, 1) for k, v in out[f"single_z{P}"]["us_per_step"].items()})
    for r, x in enumerate(out[f"P{P}"]):
        print(f"P{P} rank{r}: n {x['n_owned']} ns/particle {x['ns_per_particle']:.2f} "
              f"({x['ns_per_particle'] / s - 1:+.1%}) ",
              {k: round(v, 1) for k, v in x["us_per_step"].items()})
print("single", {k: round(v, 1) for k, v in out["single"]["us_per_step"].items()})
