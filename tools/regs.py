"""Registers / spills per kernel from `nvcc -Xptxas -v` output: python tools/regs.py [FILTER]"""
import re
import subprocess
import sys

sys.path.insert(0, '.')
from paper_2001_09253_b200 import _build  # noqa: E402

cmd = ["nvcc", *_build.NVCC_FLAGS, "-Xptxas", "-v", "-o", _build.LIB, _build.CSRC + "/spline_abi.cu"]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for ln in err.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur)
    m = re.search(r"(\d+) bytes spill stores", ln)
    if m and cur:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur and flt in cur:
        print(f"{m.group(1):>4} regs  spill {spill:>4}  {cur}")
