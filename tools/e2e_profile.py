"""Wall-clock breakdown of one end-to-end step through the public API (C4)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402

sc = S.C4()
d = Dem(sc.params)
d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
d.step(3)
s = d.get_state()
ci, cj, cd = d.get_contacts()


def pinned(a):
    t = torch.empty(a.shape, dtype={np.float32: torch.float32, np.uint32: torch.int32}[a.dtype.type],
                    pin_memory=True)
    o = t.numpy().view(a.dtype)
    o[...] = a
    return o


H = {k: pinned(v) for k, v in s.items()}
out = {k: pinned(v) for k, v in s.items()}
hci, hcj, hcd = pinned(np.concatenate([ci, ci])), pinned(np.concatenate([cj, cj])), pinned(np.concatenate([cd, cd]))
for rep in range(3):
    t = [time.perf_counter()]
    d.set_particles(H["pos"], H["vel"], H["omega"], H["radius"], H["mass"], H["id"])
    t.append(time.perf_counter())
    d.set_contacts(hci[:len(ci)], hcj[:len(ci)], hcd[:len(ci)])
    t.append(time.perf_counter())
    d.step(1)
    t.append(time.perf_counter())
    d.get_state(out=out)
    t.append(time.perf_counter())
    a, b, c = d.get_contacts(out=(hci, hcj, hcd))
    t.append(time.perf_counter())
    names = ["set_particles", "set_contacts", "step", "get_state", "get_contacts"]
    print({nm: round((t[i + 1] - t[i]) * 1e3, 2) for i, nm in enumerate(names)},
          "total ms", round((t[-1] - t[0]) * 1e3, 1), "contacts", len(a), flush=True)
