#!/bin/bash
# usage: bash tools/oracle_mutations.sh -- each plausible oracle mistake below must fail >= 1 CPU pin
# (tests/test_oracle_pins.py).  Restores oracle/oracle.c afterwards.
set -u
cd "$(dirname "$0")/.."
cp oracle/oracle.c /tmp/oracle.c.orig
trap 'cp /tmp/oracle.c.orig oracle/oracle.c; touch oracle/oracle.c; python -c "import oracle; oracle.build(force=True)"' EXIT
muts=(
  's/J->yp1\[c\] : 0.0/J->yp1[0] : 0.0/'                         # batch build: curve 0's start slope
  's/J->ypn\[c\] : 0.0/J->ypn[0] : 0.0/'                         # batch build: curve 0's end slope
  's/J->y + c \* J->n, J->n, J->bc/J->y, J->n, J->bc/'           # batch build: y offset dropped
  's/J->y2 + c \* J->n);/J->y2);/'                               # batch build: y2 offset dropped
  's/\*xc = J->x + c \* J->n/*xc = J->x/'                        # batch eval: x offset dropped
  's/\*yc = J->y + c \* J->n/*yc = J->y/'                        # batch eval: y offset dropped
  's/\*zc = J->y2c + c \* J->n;/*zc = J->y2c;/'                  # batch eval: y2 offset dropped
  's/int64_t c = f \/ J->m;/int64_t c = f \/ (J->m + 1);/'       # batch eval: wrong curve of a query
  's/ypp\[0\] = 3 \* (new_dj - start_deriv) \/ cj;/ypp[0] = 3 * (start_deriv - new_dj) \/ cj;/'  # clamped start sign
  's/double bj = 2 \* (cj + aj);/double bj = 2 * cj + aj;/'      # diagonal term
  's/double dj = 6 \* (new_dj - old_dj);/double dj = 6 * (old_dj - new_dj);/'  # sign of d_j
  's/if (x\[mid\] <= q) lo = mid;/if (x[mid] < q) lo = mid;/'    # tie-break (reading c1)
  's/double D = (B \* B \* B - B) \* (h \* h) \/ 6;/double D = (B * B * B - B) * h \/ 6;/'  # dropped h in D
)
fail=0
for pat in "${muts[@]}"; do
  cp /tmp/oracle.c.orig oracle/oracle.c
  sed -i "$pat" oracle/oracle.c
  if cmp -s oracle/oracle.c /tmp/oracle.c.orig; then echo "NOT APPLIED: $pat"; fail=1; continue; fi
  r=$(timeout 600 python -m pytest tests/test_oracle_pins.py -q -x -p no:cacheprovider 2>&1 | tail -1)
  case "$r" in *failed*) echo "caught   : $pat";; *) echo "SURVIVED : $pat ($r)"; fail=1;; esac
done
exit $fail
