#!/bin/bash
# A/B of xi-prior sweep timings over library builds in exp/ (and CMC_XI_TRIPS)
for rep in 1 2; do
  for lib in "$@"; do
    for T in ${TRIPS:-16}; do
      echo "== $lib T=$T (rep $rep)"; CMC_XI_TRIPS=$T CMC_LIB_OVERRIDE=$PWD/$lib python scripts/xi_time.py horseshoe t
    done
  done
done
