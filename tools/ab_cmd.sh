# usage: bash tools/ab_cmd.sh ROUNDS CMD... -- run CMD with libfastspline_A.so and _B.so alternately
L=paper_2001_09253_b200/csrc/libfastspline.so
R=$1; shift
for r in $(seq $R); do
  for v in A B; do
    cp paper_2001_09253_b200/csrc/libfastspline_$v.so $L
    "$@" 2>&1 | sed "s/^/$v r$r /"
  done
done
