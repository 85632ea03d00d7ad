#!/bin/bash
# A/B sweep timing of library builds under exp/ (development aid).
# usage: scripts/ab_time.sh exp/lib_a.so exp/lib_b.so ...
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    CMC_LIB_OVERRIDE=$PWD/$lib python scripts/quick_time.py short 2>&1 | grep "G="
  done
done
