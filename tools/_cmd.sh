L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for r in 1 2; do for v in A W0 W4 W8; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L; timeout 300 python tools/time_paths.py 4 20 2>&1 | grep -E " eval" | sed "s/^/$v r$r /"; done; done
cp /tmp/live.so $L
