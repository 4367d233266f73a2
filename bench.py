#!/usr/bin/env python
"""Benchmark of the B200 DEM timestep (arXiv 1301.1714 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Default workload (N=1): C4, the 4,194,304-sphere settling bed on which
BASELINE.json's metric (particle-steps/s at 1/2/4/8 B200, % of HBM roofline)
is quoted. Prints ONE JSON line on rank 0.

Timed regions (our arm), each bracketed by barrier + synchronize, max over
ranks: (1) K profiled steps with CUDA events around every kernel on the
handle's stream (dem_profile: eager launches) -> per-kernel durations for the
roofline and ms_per_step_profiled; (2) K steps replaying the captured CUDA
graph (the library's default path) -> the headline value and ms_per_step.
The per-step working set (>1 GB at C4) is far larger than the 126 MB L2, so
no L2 flush is needed.

--impl reference: the fp64 CPU oracle (oracle/, test infrastructure) timed on
the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (ms/step) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "particle-steps/s"
KERNELS = ("hash", "scan", "scatter", "rank", "sweep", "other", "detect", "finish")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------ clocks -------
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)  # the timed region can be ~20 ms

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------- scenes ------
def make_scene(name: str, model: str, rank: int):
    from paper_1301_1714_b200 import scenes as S
    sp = S.SimParams(model=model)
    if name == "C5":
        return S.C5(sp.replace(max_contacts=32), rank=rank)
    return S.CONFIGS[name](sp)


def describe(sc) -> str:
    m = sc.meta
    if sc.name.startswith("C4"):
        return (f"{sc.name}: {sc.n:,}-sphere pre-compressed settling bed (SC {m['nxyz']}, "
                f"spacing 0.998 d, r = 0.5 mm) under gravity, {sc.params.model} model")
    if m.get("kind") == "poly_bed":
        return (f"{sc.name}: {sc.n:,}-sphere polydisperse bed (r ~ U[0.25, 0.5] mm capped to "
                f"touch, SC {m['nxyz']} sites at {m['spacing'] * 1e3:.2f} mm) compacted under "
                f"gravity before timing, {sc.params.model} model, K = {sc.params.max_contacts}")
    if m.get("kind") == "fcc":
        return (f"{sc.name}: {sc.n:,}-sphere jittered FCC dense packing {m['ncells']} cells, "
                f"{sc.params.model} model")
    return f"{sc.name}: {sc.n:,} spheres, {sc.params.model} model"


# ------------------------------------------------- algorithmic bytes -------
def alg_bytes(model: str, rho_c: float, c_bar: float):
    """Algorithmic bytes per particle-step.

    The sweep (steps 5-8 and 1: detection, contact forces, walls, integration
    — k_detect + k_force, the dominant part of the step): state
    read + write 96, SCCM read 4, next CM write 4, cell offsets read 4 rho_c,
    history counts r+w 8, history entries r+w 32 c_bar -> 112 + 4 rho_c +
    32 c_bar (practical); simple model (no history, no spin update):
    position + velocity r+w 64, radius/mass/id carried 16, SCCM 4, CM 4,
    offsets 4 rho_c -> 88 + 4 rho_c.
    Whole step: 120 + 8 rho_c + 32 c_bar (practical),
    88 + 8 rho_c (simple)."""
    if model == "practical":
        return 112 + 4 * rho_c + 32 * c_bar, 120 + 8 * rho_c + 32 * c_bar
    return 88 + 4 * rho_c, 88 + 8 * rho_c


def l2_note(step_bytes: float) -> str:
    """How the per-step working set compares with the L2 (queried on the box)."""
    try:
        import torch
        l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    except Exception:
        l2 = 126 * 2**20
    mb = step_bytes / 2**20
    if step_bytes > 4 * l2:
        return f"working set ~{mb:.0f} MB per step >> {l2 / 2**20:.0f} MB L2; no flush needed"
    return (f"working set ~{mb:.0f} MB per step vs {l2 / 2**20:.0f} MB L2: partly L2-resident "
            f"across steps (no flush; not a bandwidth measurement)")


# ------------------------------------------------------- reference arm -----
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    steps_total = args.warmup + args.steps
    sc, sample = reference_sample(args.config, args.model, steps_total)
    p = orc.make_params(sc.params, sc.radius)
    st = orc.State.from_scene(sc)
    h = orc.History.empty(sc.n, sc.params.max_contacts)
    for _ in range(args.warmup):
        orc.step(p, st, h)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rc = orc.step(p, st, h).rc
        assert rc == 0, rc
    t = time.perf_counter() - t0
    value = sc.n * args.steps / t
    cores = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": describe(sc), "n_particles": sc.n,
                                        "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def reference_sample(config: str, model: str, steps_total: int, budget_s: float = 150.0):
    """A bounded sample of the workload: the same scene generator, narrowed so
    that steps_total oracle steps take about budget_s (oracle ~0.35 M
    particle-steps/s on one core)."""
    from paper_1301_1714_b200 import scenes as S
    sp = S.SimParams(model=model)
    if config == "C4":
        target = budget_s * 3.5e5 / max(1, steps_total)
        scale = 1
        while 4194304 // (scale * scale) > target and scale < 64:
            scale *= 2
        sc = S.C4(sp, scale=scale)
        return sc, (f"C4 generator narrowed {scale}x in x and z: {sc.n:,} spheres "
                    f"(same bed height, spacing, jitter), from t=0")
    sc = make_scene(config, model, 0)
    return sc, f"{config} full ({sc.n:,} spheres) from t=0"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_on_state(d, sc, budget_s: float = 12.0):
    """Time the fp64 oracle (as it stands, single thread) on the GPU's own
    warmed-up state of the same workload; whole steps until ~budget_s."""
    from oracle import oracle as orc
    from tests.parity import oracle_inputs
    K = int(d.stats()["max_contacts_seen"]) + 2
    st, h = oracle_inputs(d, max(K, 4))
    p = orc.make_params(sc.params, sc.radius)
    n_steps, t = 0, 0.0
    while t < budget_s and n_steps < 50:
        t0 = time.perf_counter()
        rc = orc.step(p, st, h).rc
        t += time.perf_counter() - t0
        n_steps += 1
        if rc != 0:
            break
    return {"value": sc.n * n_steps / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": (f"{n_steps} whole step(s) of the full {sc.name} state ({sc.n:,} spheres) "
                       f"after the GPU warm-up, fp64, one thread"), "cpu": cpu_model(),
            "seconds": t}


# ------------------------------------------------------------- our arm -----
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1301_1714_b200.dem import DEM_F_NO_GRAPH, Dem

    rank, world, local = dist_env()
    # DEM_BENCH_SHARE_GPU=1: all ranks on cuda:0 with a gloo group — a functional
    # check of the multi-rank path on a one-GPU box (timings are not meaningful)
    share = os.environ.get("DEM_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl", init_method="env://")
    torch.cuda.set_device(local)
    peak_gbs, peak_src = load_peaks()
    stream = torch.cuda.Stream()
    sc = make_scene(args.config, args.model, 0 if args.config != "C5" else rank)

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        from paper_1301_1714_b200.dem import (DEM_F_FORCE_LANES, DEM_F_FORCE_WS, DEM_F_HALF_LISTS,
                                              DEM_F_SPLIT_SWEEP, DEM_F_THREAD_PER_PARTICLE)
        d = Dem(sc.params, device=local, stream=stream, rank=rank, world=world,
                flags={"full": 0, "half": DEM_F_HALF_LISTS,
                       "tpp": DEM_F_THREAD_PER_PARTICLE, "lanes": DEM_F_FORCE_LANES,
                       "ws": DEM_F_FORCE_WS, "split": DEM_F_SPLIT_SWEEP}[args.sweep]
                | args.extra_flags)
        # every rank passes the whole set; a slab rank keeps its own planes
        if args.config == "C5" and args.c5_prep > 0:
            # C5: the loose polydisperse lattice is compacted under gravity
            # first (untimed; strong damping so it comes to rest within the
            # preparation), then handed over with its tangential history
            prep = Dem(sc.params.replace(damping=1.0), device=local, stream=stream)
            prep.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
            prep.step(args.c5_prep)
            s0, c0 = prep.get_state(), prep.get_contacts()
            prep.close()
            d.set_particles(s0["pos"], s0["vel"], s0["omega"], s0["radius"], s0["mass"], s0["id"])
            d.set_contacts(*c0)
        else:
            d.set_particles(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id)
        if world > 1:
            d.connect_group()
        d.step(max(args.warmup, 3))
        # build the step graphs of both parities (one- and two-step) before
        # any timed region: dem_step captures them lazily on first use
        for k in (1, 1, 2, 2):
            d.step(k)
        stats0 = d.stats()
        # timed region: K steps, CUDA events around every kernel on the handle's stream
        launches0 = d.stats()["launches"]
        d.profile(True)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            e0.record(stream)
            d.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        st = d.stats()
        launches_timed = st["launches"] - launches0
        d.profile(False)
        c_bar = st["contacts"] / max(1, st["n"]) if sc.params.model == "practical" else 0.0
        # graph-replay regions (the library's default path): --reps repetitions
        # of exactly K steps, each bracketed by barrier + synchronize; the
        # headline is their median
        ms_reps = []
        with ClockSampler(torch.cuda.current_device()) as clk_graph:
            for _ in range(args.reps):
                torch.cuda.synchronize()
                barrier()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                d.step(args.steps)
                g1.record(stream)
                torch.cuda.synchronize()
                barrier()
                ms_reps.append(g0.elapsed_time(g1))
        st_graph = d.stats()

    ms_max = ms
    ms_reps_max = list(ms_reps)
    if world > 1:
        t = torch.tensor([ms] + ms_reps, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max, ms_reps_max = float(t[0]), [float(x) for x in t[1:]]
    ms_graph_max = statistics.median(ms_reps_max)

    # headline: the graph-replay region; the profiled region (events around every
    # kernel) gives the per-kernel durations of the roofline
    ms_step = ms_graph_max / args.steps
    ms_step_profiled = ms_max / args.steps
    slab = world > 1 and args.config != "C5"
    # C4 (strong scaling): the whole set is split into slabs; C5 (weak): each
    # rank holds its own 2M-particle bed
    total = sc.n if slab else world * sc.n
    value = total * args.steps / (ms_graph_max * 1e-3)
    n_local = int(d.stats()["n"]) if world > 1 else sc.n
    rho_c = stats0["ncells"] / max(1, n_local)
    b_sweep, b_step = alg_bytes(sc.params.model, rho_c, c_bar)
    kernel_avg = {k: (st["kernel_ms"][k] / st["kernel_count"][k]) if st["kernel_count"][k] else 0.0
                  for k in KERNELS}
    sweep_ms = kernel_avg["detect"] + kernel_avg["sweep"] + kernel_avg["finish"]
    achieved = b_sweep * n_local / (sweep_ms * 1e-3) / 1e9
    step_kernel_ms = sum(kernel_avg.values())
    # DRAM bytes of one k_detect + k_force launch from a committed ncu --set
    # full capture of this bench command (tools/ncu_traffic.sh), with the c̄ and
    # step of that capture beside it (ncu cannot run inside the timed region)
    traffic, traffic_src, issue = None, None, None
    tr_path = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.model}.json")
    if os.path.exists(tr_path) and args.sweep == "full":
        try:
            tj = json.load(open(tr_path))
            traffic = tj.get("sweep_dram_bytes_per_step")
            traffic_src = {k: tj.get(k) for k in ("file", "step", "c_bar", "commit",
                                                  "bytes_per_particle", "alg_bytes_per_particle")}
            # the binding resource of the sweep: instruction issue. Warp
            # instructions per step from the same capture, over this run's
            # sweep time, against 4 issue slots per SM per cycle at the clock
            # sampled during the profiled region (informational: the roofline
            # above stays the north star's HBM one)
            wi = tj.get("sweep_warp_inst_per_step")
            mhz = clk.summary().get("sm_mhz")
            if wi and mhz and sweep_ms > 0:
                sms = torch.cuda.get_device_properties(local).multi_processor_count
                ach = wi / (sweep_ms * 1e-3)
                peak = sms * 4 * mhz * 1e6
                issue = {"warp_inst_per_step": wi, "achieved_warp_inst_per_s": ach,
                         "peak_warp_inst_per_s": peak, "frac": ach / peak,
                         "peak_basis": f"{sms} SMs x 4 schedulers x 1 warp instruction per "
                                       f"cycle at {mhz} MHz (profiled-region clock)",
                         "source": {k: tj.get(k) for k in ("file", "step", "c_bar", "commit")}}
        except Exception:
            traffic, issue = None, None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if (world == 1 or slab) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {
            "workload": describe(sc), "n_particles": sc.n, "ncells": stats0["ncells"],
            "grid": list(stats0["dims"]), "rho_c": rho_c, "c_bar": c_bar,
            "parallelism": (f"slabs{world} (z planes, migrant + ghost exchange over CUDA IPC "
                            f"peer memory)" if slab else
                            (f"replicas{world}" if world > 1 else "single-gpu")),
            "n_particles_rank0": n_local,
            "l2": l2_note(b_step * n_local),
            "dt": sc.params.dt, "sweep": args.sweep,
            **({"extra_flags": args.extra_flags} if args.extra_flags else {}),
            "untimed_graph_build_steps": 6,  # after the W warm-up steps (both parities, 1 and 2 steps)
            "c_bar_after_graph_reps": (st_graph["contacts"] / max(1, st_graph["n"])
                                       if sc.params.model == "practical" else 0.0),
            **({"prep_steps": args.c5_prep} if args.config == "C5" else {}),
        },
        "roofline": {
            "bound": "hbm",
            "kernel": {"half": "sweep = k_detect_half + k_pair + k_finish",
                       "full": ("sweep = k_force with fused detection" if kernel_avg["detect"] == 0
                                else "sweep = k_detect + k_force"),
                       "split": "sweep = k_detect + k_force",
                       "tpp": "sweep = k_sweep_tpp",
                       "lanes": "sweep = k_detect + k_force_lane",
                       "ws": "sweep = k_detect + k_force_ws"}[args.sweep],
            "achieved": achieved, "peak": peak_gbs,
            "unit": "GB/s", "frac": achieved / peak_gbs, "traffic": traffic,
            "traffic_source": traffic_src,
            "issue": issue,
            "alg_bytes_per_particle": b_sweep, "peak_source": peak_src,
            "kernel_ms_avg": sweep_ms, "kernel_share_of_step": sweep_ms / step_kernel_ms
            if step_kernel_ms else None,
            "step_alg_bytes_per_particle": b_step,
            "step_frac": b_step * n_local / (ms_step * 1e-3) / 1e9 / peak_gbs,
            "step_frac_of_8TBps": b_step * n_local / (ms_step * 1e-3) / 8e12,
        },
        "kernel_ms_avg": kernel_avg,
        "kernel_classes": {"hash": "k_count (counting-sort steps after a merge run)",
                           "scan": "k_tile_sum + k_scan_apply (counting sort)",
                           "scatter": "k_scatter (counting sort)",
                           "rank": "k_merge (merge re-sort) or k_rank (counting sort)",
                           "detect": "k_detect / k_detect_half",
                           "sweep": "k_force / k_force_lane / k_pair / k_sweep_tpp",
                           "finish": "k_finish (half lists)", "other": "slab exchange"},
        "ms_per_step_profiled": ms_step_profiled,
        "ms_per_step_reps": [x / args.steps for x in ms_reps_max],
        "timing": (f"value/ms_per_step: median of {args.reps} K-step CUDA-graph replay regions "
                   "(CUDA events on the handle's stream, max over ranks); roofline kernel "
                   "durations: CUDA events around every kernel over a separate K-step region of "
                   "eager launches timed just before them (ms_per_step_profiled)"),
        "gpu_launches": int(launches_timed),
        "clocks": clk_graph.summary(),
        "clocks_profiled": clk.summary(),
    }
    # the paper's §6 quantities for the last timed step (outside the timed regions)
    an = d.analyze()
    line["analysis"] = {
        "scope": "last timed step" + (" (rank 0 slab)" if world > 1 else ""),
        **{k: an[k] for k in ("candidates_mean", "max_candidates", "contacts_mean",
                              "max_contacts", "contact_fraction",
                              "tpp_candidate_lane_efficiency", "tpp_contact_lane_efficiency",
                              "max_per_cell", "movers")},
        "force_cfg": d.stats()["force_cfg"],
        "full_sorts": d.stats()["full_sorts"],
    }
    # end to end through the public API with pinned host buffers
    if not args.no_e2e and world == 1:
        line["e2e"] = run_e2e(d, sc, stream, min(args.steps, args.e2e_steps), world, barrier)
    elif not args.no_e2e:
        line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None,
                       "d2h_bytes_per_step": None,
                       "unavailable": ("a per-step host round trip at N > 1 needs every rank's "
                                       "results gathered on the host each step (dem_get_state "
                                       "returns a rank's own particles only); not built")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_on_state(d, sc)
    elif rank == 0:
        line["cpu_baseline"] = None
    d.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(d, sc, stream, steps, world, barrier):
    """Each step: dem_set_particles + dem_set_contacts from pinned host memory,
    dem_step(1), dem_get_state + dem_get_contacts into pinned host memory. Two
    pinned buffer sets alternate (a step's outputs are the next step's inputs),
    as a host-driven user loop would run it."""
    import torch

    s = d.get_state()
    ci, cj, cd = d.get_contacts()
    n = sc.n

    def pinned(shape, dtype):
        t = torch.empty(shape, dtype={np.float32: torch.float32, np.uint32: torch.int32}[dtype],
                        pin_memory=True)
        return t.numpy().view(dtype)

    cap = max(2 * len(ci), 1024)
    sets = []
    for _ in range(2):
        st = {k: pinned(v.shape, v.dtype.type) for k, v in s.items()}
        ct = (pinned((cap,), np.uint32), pinned((cap,), np.uint32), pinned((cap, 3), np.float32))
        sets.append((st, ct))
    for k, v in s.items():
        sets[0][0][k][...] = v
    m = len(ci)
    sets[0][1][0][:m], sets[0][1][1][:m], sets[0][1][2][:m] = ci, cj, cd
    h2d = d2h = 0
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    parts = np.zeros(5)
    for k in range(steps):
        (H, (hi, hj, hd)), (O, oc) = sets[k % 2], sets[(k + 1) % 2]
        tt = [time.perf_counter()]
        d.set_particles(H["pos"], H["vel"], H["omega"], H["radius"], H["mass"], H["id"])
        tt.append(time.perf_counter())
        d.set_contacts(hi[:m], hj[:m], hd[:m])
        tt.append(time.perf_counter())
        d.step(1)
        tt.append(time.perf_counter())
        d.get_state(out=O)
        tt.append(time.perf_counter())
        h2d += n * 48 + m * 20
        m = len(d.get_contacts(out=oc)[0])
        tt.append(time.perf_counter())
        d2h += n * 48 + m * 20
        parts += np.diff(tt)
    barrier()
    t = time.perf_counter() - t0
    return {"value": world * n * steps / t, "unit": UNIT,
            "h2d_bytes_per_step": h2d // max(1, steps), "d2h_bytes_per_step": d2h // max(1, steps),
            "steps": steps, "api": "dem_set_particles+dem_set_contacts+dem_step(1)+"
                                   "dem_get_state+dem_get_contacts per step, pinned host buffers",
            "ms_per_call": dict(zip(("set_particles", "set_contacts", "step", "get_state",
                                     "get_contacts"), (parts * 1e3 / max(1, steps)).round(2).tolist()))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--model", default="practical", choices=["practical", "simple"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweep", default="full", choices=["full", "half", "tpp", "lanes", "ws", "split"],
                    help="full: the default path (one radius: detection inside k_force; "
                         "else k_detect + k_force, warp-flattened force rounds); split: "
                         "k_detect + k_force always; ablations: half lists (each pair once, "
                         "Newton's third law), tpp (the paper's fused thread per particle), "
                         "lanes, ws (warp-specialised)")
    ap.add_argument("--extra-flags", type=int, default=0,
                    help="dem_flags OR-ed into the handle's (A/B runs, e.g. a force configuration)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5, help="timed K-step graph regions (median)")
    ap.add_argument("--c5-prep", type=int, default=100000,
                    help="C5: untimed compaction steps under gravity before the warm-up")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
