"""Two slab ranks in two processes on one GPU (gloo): the bench's multi-rank
flow on a small bed, for debugging the exchange. Usage: python tools/mg_debug.py [flags]"""
import os
import sys

import torch.multiprocessing as mp


def rank_main(rank, world, flags, scale, steps, talloc, use_stream, scene):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ".")
    from paper_1301_1714_b200 import scenes as S
    from paper_1301_1714_b200.dem import Dem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29541"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = S.C4(scale=scale) if scene == "bed" else S.random_gas(6000, 18.0, 3, r_range=(0.3e-3, 0.5e-3), v_sigma=3.0, w_sigma=50.0, params=S.SimParams(max_contacts=32, gravity=(0.0, -9.81, 0.0)))
    stream = torch.cuda.Stream() if use_stream else None
    with torch.cuda.stream(stream or torch.cuda.current_stream()):
        d = Dem(sc.params, flags=flags, stream=stream, rank=rank, world=world, torch_allocator=bool(talloc))
        d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
        d.connect_group()
        for k in range(steps):
            try:
                d.step(1)
            except Exception as e:  # noqa: BLE001
                print(f"rank {rank} step {k}: {e}", flush=True)
                break
        print(f"rank {rank} done n={d.n} stats={d.stats()['steps']} cfg={d.stats()['force_cfg']}",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    talloc = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    use_stream = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    scene = sys.argv[6] if len(sys.argv) > 6 else "bed"
    mp.spawn(rank_main, args=(2, flags, scale, steps, talloc, use_stream, scene), nprocs=2)
