"""Stall breakdown (warps stalled per issue-active cycle, by reason) of every
kernel in an .ncu-rep: python tools/ncu_stalls.py rep [rep...]."""
import csv
import io
import subprocess
import sys

for rep in sys.argv[1:]:
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        items = []
        for h, v in d.items():
            if h.startswith(pre) and h.endswith(suf):
                try:
                    items.append((float(v), h[len(pre):-len(suf)]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items)
        print(d.get("Kernel Name", "?")[:60], f"total {tot:.2f} warps/issue")
        print("   " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(items, reverse=True)[:9]))
