#!/bin/bash
# A/B of xi-prior sweep timings over library builds and CMC_XI_TRIPS values
for rep in 1 2; do
  echo "== base (rep $rep)"; CMC_LIB_OVERRIDE=$PWD/exp/xi_base.so python scripts/xi_time.py horseshoe t
  for T in 4 8 16 32; do
    echo "== park T=$T (rep $rep)"; CMC_XI_TRIPS=$T CMC_LIB_OVERRIDE=$PWD/exp/xi_park.so python scripts/xi_time.py horseshoe t
  done
done
