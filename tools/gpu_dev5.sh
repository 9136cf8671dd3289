mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 > gpurun_out/pytest_dev.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_dev.log
timeout 300 python tools/time_paths.py 5 10 2>&1 | tail -5
python tools/prof.py 5 2 > gpurun_out/pp_5.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:records" -s 2 -c 2 -o gpurun_out/prof_cfg5r -f python tools/prof.py 5 2 > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc=$?"
