#!/bin/bash
# A/B of the carried beta exps (CMC_BETA_CARRY), then parity of the carried build
for rep in 1 2 3; do
  for kv in CMC_BETA_CARRY=0 CMC_BETA_CARRY=1; do
    echo "== $kv (rep $rep)"
    env $kv python scripts/quick_time.py short 2>&1 | grep "G="
  done
done
for kv in CMC_BETA_CARRY=0 CMC_BETA_CARRY=1; do
  echo "== $kv (large)"; env $kv QT_K=20 python scripts/quick_time.py 2>&1 | grep "G=1000000\|G=200000"
done
