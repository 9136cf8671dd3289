"""Copy the judged evidence from gpurun_out/ (scratch) into profiles/<round>/ (tracked).
python tools/save_profiles.py r01"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
# optional second argument: an export root used instead of profiles/ (on the GPU box, so the
# summaries travel back inside gpurun_out/ without the large .ncu-rep files)
proot = os.path.abspath(sys.argv[2]) if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(proot, rnd)
os.makedirs(dst, exist_ok=True)


def last_json(p):
    for ln in reversed(open(p).read().strip().splitlines()):
        if ln.startswith("{"):
            return ln
    return None


for name, out in [("bench_default.log", "bench_cfg2.jsonl"), ("bench_reference.log", "bench_reference_cfg2.jsonl")] + \
        [(f"bench_cfg{c}.log", f"bench_cfg{c}.jsonl") for c in (1, 3, 4, 5)]:
    p = os.path.join(src, name)
    if os.path.exists(p) and last_json(p):
        open(os.path.join(dst, out), "w").write(last_json(p) + "\n")

# launch list: per-kernel share of device time
lp = os.path.join(src, "launches_cfg2.csv")
if os.path.exists(lp):
    shutil.copy(lp, os.path.join(dst, "launches_cfg2.csv"))
    rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, per = 0.0, {}
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0].split("<")[0].replace("void ", "")
        per[k] = per.get(k, 0.0) + v
        tot += v
    with open(os.path.join(dst, "launches_cfg2_shares.txt"), "w") as f:
        for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
            f.write(f"{100 * v / tot:6.2f}%  {v / 1e3:10.1f} us  {k}\n")

traffic = {}
tp = os.path.join(proot, "traffic.json")
for cand in (tp, os.path.join(ROOT, "profiles", "traffic.json")):
    if os.path.exists(cand):
        traffic = json.load(open(cand))
        break
for rep, tag in [("prof_cfg2.ncu-rep", "ncu_full_cfg2"), ("prof_fused_cfg2.ncu-rep", "ncu_full_fused_cfg2"),
                 ("prof_cfg3.ncu-rep", "ncu_full_cfg3"), ("prof_cfg4.ncu-rep", "ncu_full_cfg4"),
                 ("prof_cfg5r.ncu-rep", "ncu_full_cfg5_eval"), ("prof_cfg5.ncu-rep", "ncu_full_cfg5_build")]:
    p = os.path.join(src, rep)
    if not os.path.exists(p):
        continue
    res = ncu_summary.summarise(p)
    json.dump(res, open(os.path.join(dst, tag + ".json"), "w"), indent=1)
    with open(os.path.join(dst, tag + ".txt"), "w") as f:
        for d in res:
            f.write(d["kernel"][:110] + "\n")
            for k, v in d.items():
                if k != "kernel":
                    f.write(f"   {k:65s} {v[0]:>14s} {v[1]}\n")
    for d in res:
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if not rd:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = float(rd[0].replace(",", "")) * scale[rd[1]] + float(wr[0].replace(",", "")) * scale[wr[1]]
        k = d["kernel"]
        if tag in ("ncu_full_cfg2", "ncu_full_cfg3", "ncu_full_cfg4"):
            traffic.setdefault(tag[-4:], {})["build" if ("k1_" in k or "k_tile" in k) else "eval"] = b
        elif tag == "ncu_full_fused_cfg2":
            traffic.setdefault("cfg2", {})["fused"] = b
        elif tag == "ncu_full_cfg5_eval" and "k_eval_records" in k:
            traffic.setdefault("cfg5", {})["eval"] = b
traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
                    "(profiles/<round>/ncu_full_*.txt)")
json.dump(traffic, open(tp, "w"), indent=1)
print("saved to", dst)
