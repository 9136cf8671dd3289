# usage: bash tools/gpu_round.sh  -- tests, full-size parity, benches of all configs
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m "gpu" -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for c in 2 3 1 4 5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_cfg$c.log").read().strip().splitlines()[-1])
    print("cfg$c", "ms/step %.4f"%d["ms_per_step"], "build_ms %.4f"%d["build_ms"], "eval_ms %.4f"%d["eval_ms"], "eval frac %.3f"%d["roofline"]["frac"], "build frac %.3f"%d["roofline"]["build"]["frac"], "e2e", d["e2e"]["value"] if d["e2e"] else None)
except Exception as e: print("cfg$c parse fail", e)
PY
done
