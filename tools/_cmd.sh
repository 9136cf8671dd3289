T=gpurun_out/r02bw; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x --timeout 600 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
cp $L paper_2001_09253_b200/csrc/libfastspline_M3.so
for r in 1 2; do for v in M3 M2 M4; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 2 30 2>&1 | grep -E "step|split" | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
