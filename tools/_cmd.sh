T=gpurun_out/r02x; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_ablation.py tests/test_gpu_determinism.py -q -x --timeout 600 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for r in 1 2; do for v in A F; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 4 20 2>&1 | grep -E " eval" | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
