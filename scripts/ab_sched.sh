#!/bin/bash
# A/B of lane count x stagger at K = 20 and K = 100
for rep in 1 2; do
  for lib in exp/lanes2.so exp/lanes4.so; do
    for st in 0 1; do
      for K in 20 100; do
        echo "== $lib stagger=$st K=$K (rep $rep)"
        QT_K=$K CMC_STAGGER=$st CMC_LIB_OVERRIDE=$PWD/$lib python scripts/quick_time.py short 2>&1 | grep "chains=4"
      done
    done
  done
done
