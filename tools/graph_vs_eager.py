"""Compare dem_step timing: CUDA-graph replay vs eager launches (no events)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1301_1714_b200 import scenes as S
from paper_1301_1714_b200.dem import DEM_F_NO_GRAPH, Dem

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
sc = S.CONFIGS[cfg]()
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for name, flags in (("graph", 0), ("eager", DEM_F_NO_GRAPH), ("graph", 0), ("eager", DEM_F_NO_GRAPH)):
        d = Dem(sc.params, flags=flags, stream=stream)
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
        d.step(6)
        res = []
        for K in (2, 20, 100):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            d.step(K)
            b.record(stream)
            torch.cuda.synchronize()
            res.append((K, round(a.elapsed_time(b) / K, 4)))
        print(cfg, name, res, flush=True)
        del d
