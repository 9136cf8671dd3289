T=gpurun_out/r02am; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x --timeout 600 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for r in 1 2; do for v in O A; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; for c in 4 5; do timeout 300 python tools/time_paths.py $c 10 2>&1 | grep -E " build |step" | sed "s/^/$v r$r /"; done; done; done
cp /tmp/live.so $L
