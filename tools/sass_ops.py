"""Opcode histogram (executed warp instructions + stall samples) from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops, st = collections.Counter(), collections.Counter()
tot = tots = 0
for r in data:
    try:
        e, w = int(r[iE]), int(r[iW])
    except Exception:
        continue
    toks = r[iS].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    ops[op] += e
    st[op] += w
    tot += e
    tots += w
print("total warp instr", tot, "stall samples", tots)
for op, c in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {c:12d} {100 * c / tot:5.1f}%  stalls {100 * st[op] / max(tots, 1):5.1f}%")
if len(sys.argv) > 3:  # top stall lines
    lines = sorted(((int(r[iW]) if r[iW].isdigit() else 0, r[0], r[iS]) for r in data), reverse=True)[:int(sys.argv[3])]
    for w, a, s in lines:
        print(w, a, s)
