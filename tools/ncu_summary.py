"""Summarise an .ncu-rep: key metrics + top stall SASS lines (needs ncu locally)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_average_branch_targets_threads_uniform.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(hdr, units, r)})
    return res


def stalls(rep, top=25, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", kernel]
    out = subprocess.check_output(cmd, text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    # multi-kernel reports: keep the first kernel's table
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    if len(starts) > 1:
        rows = rows[starts[0]:starts[1]]
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_th = hdr.index("Avg. Threads Executed")
    tot = sum(int(r[i_s] or 0) for r in data)
    idx = sorted(range(len(data)), key=lambda k: -int(data[k][i_s] or 0))[:top]
    lines = [f"total stall samples {tot}"]
    for k in sorted(idx):
        r = data[k]
        lines.append(f"{k:5d} {int(r[i_s]) / tot * 100:5.1f}% thr={r[i_th]:>4} {r[i_src][:80]}")
    return "\n".join(lines)


if __name__ == "__main__":
    rep = sys.argv[1]
    for i, k in enumerate(raw(rep)):
        name = k.get("Kernel Name", ("?",))[0]
        print(f"== launch {i}: {name[:100]}")
        for key in KEYS:
            if key in k:
                print(f"   {key:70s} {k[key][0]:>16} {k[key][1]}")
    if "--stalls" in sys.argv:
        kern = sys.argv[sys.argv.index("--stalls") + 1] if len(sys.argv) > sys.argv.index("--stalls") + 1 else None
        print(stalls(rep, kernel=kern))
