"""The paper's §5 experiment on one B200: 2^17 equal spheres
fall from a box through a slit onto the floor; the run continues until the
largest displacement of a step is below eps (checked every `chunk` steps).
Prints one JSON line: particles/s over the whole run (the paper's Table 3
"computing speed", N x steps / time), steps, simulated time, how many
particles went through the slit.

    python tools/slit_run.py [--nxyz 64 32 64] [--eps 1e-9] [--max-steps 2000000]
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1301_1714_b200 import scenes as S  # noqa: E402
from paper_1301_1714_b200.dem import Dem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nxyz", type=int, nargs=3, default=[64, 32, 64])
    ap.add_argument("--eps", type=float, default=1e-9, help="termination: max step displacement [m]")
    ap.add_argument("--chunk", type=int, default=2000)
    ap.add_argument("--max-steps", type=int, default=2_000_000)
    ap.add_argument("--model", default="practical")
    a = ap.parse_args()
    sc = S.slit_box(tuple(a.nxyz), params=S.SimParams(model=a.model))
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        d = Dem(sc.params, stream=stream)
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        steps, vmax, trace = 0, float("inf"), []
        while steps < a.max_steps:
            d.step(a.chunk)
            steps += a.chunk
            st = d.stats()
            vmax = st["max_speed"]
            if steps % (50 * a.chunk) == 0:
                trace.append((steps, vmax))
            if vmax * sc.params.dt < a.eps:
                break
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = e0.elapsed_time(e1)
        s = d.get_state()
        an = d.analyze()
    below = int((s["pos"][:, 1] < sc.meta["y_bottom"]).sum())
    print(json.dumps({
        "experiment": "PAPER.md §5 box with a slit (geometry: scenes.slit_box, DESIGN.md R23)",
        "n_particles": sc.n, "model": a.model, "steps": steps,
        "terminated": bool(vmax * sc.params.dt < a.eps), "eps_m": a.eps,
        "final_max_step_displacement_m": vmax * sc.params.dt,
        "simulated_s": steps * sc.params.dt, "device_s": ms / 1e3, "wall_s": wall,
        "particles_per_s": sc.n * steps / (ms / 1e3),
        "paper_particles_per_s": {"practical OpenCL GPU (C2050)": 2.960e6,
                                  "practical C++ CPU (X5670, 1 core)": 0.474e6,
                                  "simple CUDA GPU": 22.359e6},
        "through_slit": below, "contacts_mean_last_step": an["contacts_mean"],
        "max_contacts_last_step": an["max_contacts"], "trace_steps_vmax": trace[-20:],
    }), flush=True)


if __name__ == "__main__":
    main()
