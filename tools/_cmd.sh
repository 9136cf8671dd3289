T=gpurun_out/r02ah; mkdir -p $T
python tools/pcie_probe.py > $T/pcie.json 2>&1; cat $T/pcie.json
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > $T/b$r.log 2>&1; python -c "
import json; d=json.loads(open('$T/b$r.log').read().strip().splitlines()[-1]); e=d['e2e']; print('e2e ms', e['ms_per_step'], 'Gq/s', e['value']/1e9, 'GB/s', (e['h2d_bytes_per_step']+e['d2h_bytes_per_step'])/e['ms_per_step']/1e6)"; done
