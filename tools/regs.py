"""Print registers / spills per kernel from nvcc -Xptxas -v output on stdin."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        sp = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = re.sub(r"PKT_.*", "", cur.replace("_ZN2fs", ""))
        print(f"{m.group(1):>4} regs  spill {sp:>4}  {name}")
        cur = None
