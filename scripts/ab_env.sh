#!/bin/bash
# A/B sweep timing of environment switches on the current build
# usage: scripts/ab_env.sh "VAR=a" "VAR=b" ...
for rep in 1 2; do
  for kv in "$@"; do
    echo "== $kv (rep $rep)"
    env $kv python scripts/quick_time.py short 2>&1 | grep "G="
  done
done
