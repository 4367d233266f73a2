"""How fast does the C5 polydisperse bed compact? Stages g-multiplier:alpha:steps[:mu]
(each a new handle fed with the previous one's state and tangential history
through the public API); prints c̄ (history entries per particle) and
the largest speed. GPU only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
stages = [tuple(int(x) if i == 2 else float(x) for i, x in enumerate(a.split(":")))
          for a in (sys.argv[2:] or ["1:1:60000", "1:0.2522:3000"])]
sc = S.C5(scale=scale)
state, contacts = None, None
t0 = time.time()
for stage in stages:
    gmul, alpha, steps = stage[:3]
    sp = sc.params.replace(gravity=(0.0, -9.81 * gmul, 0.0), damping=alpha)
    if len(stage) > 3:
        sp = sp.replace(friction=stage[3])
    d = Dem(sp)
    if state is None:
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
    else:
        s = state
        d.set_particles(s["pos"], s["vel"], s["omega"], s["radius"], s["mass"], s["id"])
        d.set_contacts(*contacts)
    for k in range(0, steps, 1000 if steps <= 10000 else 5000):
        d.step(1000 if steps <= 10000 else 5000)
        st = d.stats()
        print(f"g x{gmul:g} alpha {sp.damping} mu {sp.friction}: +{k:5d}+ cbar {st['contacts'] / st['n']:.3f} "
              f"vmax {st['max_speed']:.3f} t {time.time() - t0:.1f}s", flush=True)
    state, contacts = d.get_state(), d.get_contacts()
    d.close()
