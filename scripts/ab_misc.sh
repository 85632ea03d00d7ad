#!/bin/bash
# priorities (CMC_PRIO=<eps><gene><tail>) and graph chunk sizes
for rep in 1 2; do
  for pr in 001 011 000 101; do
    echo "== prio $pr (rep $rep)"; QT_K=100 CMC_PRIO=$pr CMC_LIB_OVERRIDE=$PWD/exp/prio.so python scripts/quick_time.py short 2>&1 | grep "chains=4"
  done
  for ch in ch25 ch50 ch100; do
    echo "== $ch e2e (rep $rep)"; CMC_LIB_OVERRIDE=$PWD/exp/$ch.so python scripts/e2e_breakdown.py 2>&1 | tail -2
  done
done
