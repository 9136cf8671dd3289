"""Per kernel of an ncu report: the SASS lines with the most warp-stall samples and their top stall
reasons (from the source page), so the evidence travels without the .ncu-rep.
    python tools/ncu_hotspots.py REPORT [TOP] > hotspots.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
names = [r[r and list(csv.reader(io.StringIO(raw)))[0].index("Kernel Name")] for r in list(csv.reader(io.StringIO(raw)))[2:]]
for k, name in enumerate(names):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(k),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next((i for i, r in enumerate(rows) if r and r[0] == "Address"), None)
    print(f"=== {name[:150]}")
    if hi is None:
        print("   (no source page)")
        continue
    h = rows[hi]
    ix = {c: i for i, c in enumerate(h)}
    data = [r for r in rows[hi + 1:] if len(r) == len(h)]
    samp = "Warp Stall Sampling (All Samples)"
    tot = sum(int(r[ix[samp]] or 0) for r in data) or 1
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(r[ix[c]] or 0) for r in data) for c in stalls}
    print("   stall samples by reason: " + ", ".join(f"{c[6:]} {v / tot:.1%}" for c, v in
                                                    sorted(agg.items(), key=lambda kv: -kv[1])[:6]))
    print(f"   instructions executed: {sum(int(r[ix['Instructions Executed']] or 0) for r in data)}")
    for r in sorted(data, key=lambda r: -int(r[ix[samp]] or 0))[:top]:
        s = int(r[ix[samp]] or 0)
        why = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stalls), reverse=True)[:2]
        print(f"   {s / tot:6.1%}  {r[1].strip()[:70]:70s} " + " ".join(f"{n}={v}" for v, n in why if v))
