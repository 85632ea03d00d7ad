#!/bin/bash
# A/B of library builds: 4-chain sweep time (K = 20, 100) and whole run() wall
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    QT_K=20 CMC_LIB_OVERRIDE=$PWD/$lib python scripts/quick_time.py short 2>&1 | grep "chains=4"
    QT_K=100 CMC_LIB_OVERRIDE=$PWD/$lib python scripts/quick_time.py short 2>&1 | grep "chains=4"
    CMC_LIB_OVERRIDE=$PWD/$lib python scripts/e2e_phases.py 2>&1 | grep "run() e2e"
  done
done
