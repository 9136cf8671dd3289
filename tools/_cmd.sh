T=gpurun_out/r02tt; mkdir -p $T
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_determinism.py tests/test_gpu_dist_nccl.py -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
cp $L paper_2001_09253_b200/csrc/libfastspline_T3.so
for r in 1 2; do for v in OLDP T3 T2 T3P; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; for c in 4 5; do timeout 300 python tools/time_paths.py $c 20 2>&1 | grep -E " build |step \(auto" | sed "s/^/$v r$r /"; done; done; done
cp /tmp/live.so $L
