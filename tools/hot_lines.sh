# usage: bash tools/hot_lines.sh REPORT KREGEX MANGLED [TOP]
ncu -i $1 --page source --csv --print-source sass -k "regex:$2" 2>/dev/null > /tmp/_sass.csv
python tools/sass_lines.py /tmp/_sass.csv /tmp/cubin/spline_abi.sm_100a.cubin $3 ${4:-30} > /tmp/_lines.txt
python - <<'PY'
import re
src={f:open('paper_2001_09253_b200/csrc/'+f).read().split('\n') for f in ["eval.cuh","common.cuh","build_thomas.cuh","build_tile.cuh","fused.cuh"]}
for l in open('/tmp/_lines.txt'):
    m=re.search(r'(\S+\.cuh):(\d+)',l)
    if m and m.group(1) in src: print(l.rstrip()[:40], '|', m.group(2), src[m.group(1)][int(m.group(2))-1].strip()[:90])
    else: print(l.rstrip())
PY
