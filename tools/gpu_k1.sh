for c in 2; do timeout 300 python tools/time_paths.py $c 20 2>&1 | head -1; SPLINE_K1_BABE=1 timeout 300 python tools/time_paths.py $c 20 2>&1 | head -1; done
