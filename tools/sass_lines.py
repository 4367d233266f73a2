"""Per-source-line totals of an ncu SASS source page (instructions executed,
thread instructions, stall samples), mapped to CUDA lines through the line
table of `nvdisasm -g` (the ncu CSV itself carries no line numbers).

  ncu -i rep --page source --csv --print-source sass -k regex:NAME > sass.csv
  cuobjdump -xelf all libdem.so; nvdisasm -g -c dem_kernels.sm_100a.cubin > all.sass
  python tools/sass_lines.py sass.csv all.sass MANGLED_NAME [top]
"""
import csv
import re
import sys
from collections import defaultdict


def line_table(sass_path, func):
    tab, cur, inside = {}, None, False
    for ln in open(sass_path):
        if ln.startswith("//---------------------"):
            inside = (".text." + func + " ") in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File ".*", line (\d+)', ln)
        if m:
            cur = int(m.group(1))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m:
            tab[int(m.group(1), 16)] = cur
    return tab


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Address":  # a second kernel's table: keep the first
            break
        if len(r) >= len(hdr) - 1:
            data.append(r)
    ia, ii, it, iss = (hdr.index(k) for k in ("Address", "Instructions Executed",
                                             "Thread Instructions Executed",
                                             "Warp Stall Sampling (All Samples)"))
    tab = line_table(sys.argv[2], sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    a0 = int(data[0][ia], 16)
    agg = defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in data:
        line = tab.get(int(r[ia], 16) - a0)
        v = [int(r[ii] or 0), int(r[it] or 0), int(r[iss] or 0)]
        for k in range(3):
            agg[line][k] += v[k]
            tot[k] += v[k]
    print(f"total warp inst {tot[0]:,}  thread inst {tot[1]:,}  stall samples {tot[2]:,}")
    src = open(sys.argv[5]).read().split("\n") if len(sys.argv) > 5 else None
    for line, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        txt = src[line - 1].strip()[:70] if src and line else ""
        print(f"line {line!s:>5}: inst {v[0] / tot[0] * 100:5.1f}%  thr/inst {v[1] / max(v[0], 1):5.1f}"
              f"  stalls {v[2] / max(tot[2], 1) * 100:5.1f}%  {txt}")


if __name__ == "__main__":
    main()
