T=gpurun_out/r02bk; mkdir -p $T
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
cp $L paper_2001_09253_b200/csrc/libfastspline_C2.so
timeout 300 python tools/time_paths.py 1 50 2>&1 | grep -E "step|split" | sed "s/^/live /"
for r in 1 2; do for v in C2 C3 C4 C4S4; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 5 10 2>&1 | grep -E " eval " | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
