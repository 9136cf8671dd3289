T=gpurun_out/r02p; mkdir -p $T
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $T/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $T/pytest.log
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for v in A B C; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 5 5 2>&1 | grep " eval" | sed "s/^/$v /"; done
cp /tmp/live.so $L
