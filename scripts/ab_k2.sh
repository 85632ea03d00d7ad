#!/bin/bash
# A/B of library builds at K = 20 and K = 100 (quick_time short: 1 and 4 chains)
for rep in 1 2; do
  for lib in "$@"; do
    for K in 20 100; do
      echo "== $lib K=$K (rep $rep)"
      QT_K=$K CMC_LIB_OVERRIDE=$PWD/$lib python scripts/quick_time.py short 2>&1 | grep "chains="
    done
  done
done
