"""Per kernel of an ncu report: the SASS lines with the most warp-stall samples and their top stall
reasons (from the source page), so the evidence travels without the .ncu-rep.
    python tools/ncu_hotspots.py REPORT [TOP] > hotspots.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "?", "hdr": None, "data": []}
        blocks.append(cur)
    elif r and r[0] == "Address" and cur is not None:
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] is not None and len(r) == len(cur["hdr"]):
        cur["data"].append(r)
samp = "Warp Stall Sampling (All Samples)"
for b in blocks:
    print(f"=== {b['name'][:150]}")
    h, data = b["hdr"], b["data"]
    if not h or not data:
        print("   (no source page)")
        continue
    ix = {c: i for i, c in enumerate(h)}
    num = lambda r, c: int(r[ix[c]] or 0) if r[ix[c]].isdigit() else 0
    tot = sum(num(r, samp) for r in data) or 1
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(num(r, c) for r in data) for c in stalls}
    print("   stall samples by reason: " + ", ".join(f"{c[6:]} {v / tot:.1%}" for c, v in
                                                    sorted(agg.items(), key=lambda kv: -kv[1])[:6]))
    print(f"   instructions executed: {sum(num(r, 'Instructions Executed') for r in data)}")
    for r in sorted(data, key=lambda r: -num(r, samp))[:top]:
        s = num(r, samp)
        why = sorted(((num(r, c), c[6:]) for c in stalls), reverse=True)[:2]
        print(f"   {s / tot:6.1%}  {r[1].strip()[:70]:70s} " + " ".join(f"{n}={v}" for v, n in why if v))
