"""Copy the round's bench lines and launch list from gpurun_out/<tag>/ (scratch) into profiles/<round>/.
python tools/save_r02.py gpurun_out/r02f r02"""
import csv
import os
import sys

src, rnd = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)


def json_lines(p):
    return [ln for ln in open(p).read().splitlines() if ln.startswith("{")]


for log, out in [("bench_cfg4.log", "bench_cfg4.jsonl"), ("bench_reference.log", "bench_reference_cfg4.jsonl"),
                 ("bench_cfg3_xshared.log", "bench_cfg3_xshared.jsonl"), ("ablation.log", "ablation_sweep.jsonl")] + \
        [(f"bench_cfg{c}.log", f"bench_cfg{c}.jsonl") for c in (1, 2, 3, 5)]:
    p = os.path.join(src, log)
    if os.path.exists(p):
        ls = json_lines(p)
        if ls:
            keep = ls if log == "ablation.log" else ls[-1:]
            open(os.path.join(dst, out), "w").write("\n".join(keep) + "\n")
            print("saved", out, len(keep))
lp = os.path.join(src, "launches_cfg4.csv")
if os.path.exists(lp):
    rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per, cnt, tot = {}, {}, 0.0
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0].replace("void ", "").replace("fs::", "")[:70]
        per[k] = per.get(k, 0.0) + v
        cnt[k] = cnt.get(k, 0) + 1
        tot += v
    open(os.path.join(dst, "launches_cfg4.csv"), "w").write(open(lp).read())
    with open(os.path.join(dst, "launches_cfg4_shares.txt"), "w") as f:
        f.write("kernel  launches  total_us  share   (ncu launch list of python bench.py --steps 3 --warmup 3 "
                "--no-cpu-baseline --no-e2e; cold, serialised)\n")
        for k, v in sorted(per.items(), key=lambda kv: -kv[1]):
            f.write(f"{k:72s} {cnt[k]:4d} {v / 1e3:12.1f}  {v / tot:.3f}\n")
    print(open(os.path.join(dst, "launches_cfg4_shares.txt")).read())
