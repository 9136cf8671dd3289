T=gpurun_out/r02bk3; mkdir -p $T
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "bucket or cfg5 or long" > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for v in SM2S0 SM2S0O1; do echo "== $v"; cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 600 python tools/_diag.py 2>&1 | grep "^rep"; done
cp /tmp/live.so $L; echo "== live"; timeout 600 python tools/_diag.py 2>&1 | grep "^rep"
