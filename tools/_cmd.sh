T=gpurun_out/r02y; mkdir -p $T
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
timeout 300 python tools/time_paths.py 5 5 2>&1 | grep -E " eval" | sed "s/^/old /"
for r in 1 2; do for v in A E G; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 5 5 2>&1 | grep -E " eval" | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
