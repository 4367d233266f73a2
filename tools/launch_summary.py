"""Per-kernel averages and step shares from an ncu launch list
(--metrics gpu__time_duration.sum --csv --log-file X.csv)."""
import collections
import csv
import io
import sys


def main(path, title):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]  # skip the profiled program's own output
    rows = list(csv.DictReader(io.StringIO(txt)))
    t = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("dem::", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        t[name].append(v * scale.get(r["Metric Unit"], 1.0))
    tot = sum(sum(v) for v in t.values())
    print(title)
    print(f"{'kernel':30s} launches  avg_us   share")
    for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
        print(f"{k:30s} {len(v):6d} {sum(v) / len(v):8.1f} {sum(v) / tot * 100:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
