"""Write profiles/traffic_<config>_<model>.json from an ncu --set full capture
of the sweep's launches (k_detect + k_force, or the fused k_force alone; one
or more steps: per-kernel figures are averaged over that kernel's launches)
and the bench line that run printed: DRAM bytes of the sweep per step, with
the capture's first step index and c̄ beside it (bench.py copies them into
roofline.traffic).

    python tools/traffic_json.py gpurun_out/full_C4_TAG.ncu-rep gpurun_out/ncu_TAG.log \
        --skip 8 --warmup 5 [--config C4 --model practical]
"""
import argparse
import csv
import io
import json
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("log")
ap.add_argument("--skip", type=int, default=8, help="matching launches ncu skipped (-s)")
ap.add_argument("--config", default="C4")
ap.add_argument("--model", default="practical")
a = ap.parse_args()
out = subprocess.check_output(["ncu", "-i", a.rep, "--page", "raw", "--csv"], text=True,
                              stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
per, inst, cnt = {}, {}, {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("<")[0].split("(")[0].replace("void ", "").strip()
    b = sum(float(d[k].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            for k, u in ((k, rows[1][hdr.index(k)]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))
    cnt[name] = cnt.get(name, 0) + 1
    per[name] = per.get(name, 0.0) + b
    if "smsp__inst_executed.sum" in d:  # warp instructions issued by the launch
        inst[name] = inst.get(name, 0.0) + float(d["smsp__inst_executed.sum"].replace(",", ""))
per = {k: v / cnt[k] for k, v in per.items()}
inst = {k: v / cnt[k] for k, v in inst.items()}
kps = len(per)  # sweep kernels per step
line = None
for ln in open(a.log):
    ln = ln.strip()
    if ln.startswith("{"):
        line = json.loads(ln)
n = line["config"]["n_particles_rank0"]
tot = sum(per.values())
commit = subprocess.check_output(["git", "rev-parse", "--short", "HEAD"], text=True).strip()
res = {
    "sweep_dram_bytes_per_step": tot,
    "per_kernel": per,
    "sweep_warp_inst_per_step": sum(inst.values()) if inst else None,
    "warp_inst_per_kernel": inst,
    "bytes_per_particle": tot / n,
    "alg_bytes_per_particle": line["roofline"]["alg_bytes_per_particle"],
    "step": a.skip // kps + 1,
    "launches_averaged": cnt,
    "c_bar": line["config"]["c_bar"],
    "n_particles": n,
    "commit": commit,
    "file": os.path.basename(a.rep),
    "source": (f"ncu --set full --clock-control none of bench.py --config {a.config}: launch "
               f"step {a.skip // kps + 1} on of {' + '.join(sorted(per))} (dram__bytes_read.sum + "
               f"dram__bytes_write.sum); c_bar = the bench line of the same run (its "
               f"profiled region, steps warmup+1..warmup+K)"),
}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    f"traffic_{a.config}_{a.model}.json")
json.dump(res, open(path, "w"), indent=1)
print(path, json.dumps(res))
