T=gpurun_out/r02te; mkdir -p $T
timeout 1200 python -m pytest tests/test_gpu_fused.py -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
cp $L paper_2001_09253_b200/csrc/libfastspline_TE2.so
for r in 1 2; do for v in TE2 TE3; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 4 20 2>&1 | grep -E "step|fused|split" | sed "s/^/$v r$r /"; done; done
cp paper_2001_09253_b200/csrc/libfastspline_TE3.so $L
timeout 1200 python -m pytest tests/test_gpu_fused.py -q -x --timeout 900 -k tile > $T/pytest3.log 2>&1; echo "pytest TE3 rc=$?"; tail -2 $T/pytest3.log
cp /tmp/live.so $L
