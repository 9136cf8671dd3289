for e in 0 1 2; do
  if [ $e = 0 ]; then L=""; else L="SPLINE_LIB_OVERRIDE=$PWD/gpurun_exp$e.so"; fi
  for c in ${1:-2 3}; do echo "exp $e"; env $L timeout 300 python tools/time_paths.py $c 20 2>&1 | grep " eval "; done
done
