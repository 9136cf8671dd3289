T=gpurun_out/r02w; mkdir -p $T
L=paper_2001_09253_b200/csrc/libfastspline.so
cp $L /tmp/live.so
for v in A P; do cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L
  timeout 600 python tools/precision_report.py $T/precision_$v.json > $T/precision_$v.log 2>&1; echo "$v prec rc=$?"; tail -12 $T/precision_$v.log
  for c in 1 4 5; do timeout 300 python tools/time_paths.py $c 10 2>&1 | grep -E " build | build\+eval" | sed "s/^/$v /"; done
done
cp /tmp/live.so $L
