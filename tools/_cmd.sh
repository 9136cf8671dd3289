T=gpurun_out/r02af; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x --timeout 600 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for r in 1 2; do for v in live A; do if [ $v = A ]; then cp paper_2001_09253_b200/csrc/libfastspline_A.so $L; else cp /tmp/live.so $L; fi; timeout 300 python tools/time_paths.py 4 20 2>&1 | grep -E "step|build\+eval" | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
