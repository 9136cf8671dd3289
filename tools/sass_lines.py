"""Map ncu per-SASS dynamic counts to CUDA source lines via nvdisasm line info.
python tools/sass_lines.py NCU_SASS_CSV CUBIN FUNC_MANGLED [TOP]"""
import collections
import csv
import re
import subprocess
import sys

csvp, cubin, func = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(csvp)))
hdr = rows[1]
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
dyn = []
for r in rows[2:]:
    try:
        dyn.append((int(r[0], 16), int(r[iE]), int(r[iW])))
    except Exception:
        pass
base = min(a for a, _, _ in dyn)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# keep only the requested function's section
secs = re.split(r"\n\s*\.section\s+", dis)
body = next((x for x in secs if x.startswith(".text." + func)), "")
line_of = {}
cur = "?"
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg_e, agg_w = collections.Counter(), collections.Counter()
seen = set()
for a, e, w in dyn:
    off = a - base
    if off in seen:
        continue
    seen.add(off)
    L = line_of.get(off, "?")
    agg_e[L] += e
    agg_w[L] += w
te, tw = sum(agg_e.values()), sum(agg_w.values())
print("total", te, tw)
for L, e in agg_e.most_common(top):
    print(f"{100 * e / te:5.1f}% instr {100 * agg_w[L] / max(tw, 1):5.1f}% stall  {L}")
