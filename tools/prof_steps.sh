# the timed paths of every config, one process each (for one ncu --target-processes all capture)
set -e
for c in 1 2 3 4 5; do python tools/prof.py $c 1; done
python tools/prof.py 3 1 --x-shared
