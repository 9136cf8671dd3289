# usage: [VARIANTS="A B C"] bash tools/ab.sh "CFGS" [ROUNDS] -- interleaved timing of builds of the library
# on one box: paper_2001_09253_b200/csrc/libfastspline_<V>.so (copied over the live .so in turn)
L=paper_2001_09253_b200/csrc/libfastspline.so
for r in $(seq ${2:-2}); do
  for v in ${VARIANTS:-A B}; do
    cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L
    for c in $1; do timeout 300 python tools/time_paths.py $c 30 2>&1 | sed -n 1,4p | sed "s/^/$v r$r /"; done
  done
done
