for rep in 1 2; do for T in 8 16 32 100000; do echo "== T=$T"; CMC_XI_TRIPS=$T python scripts/xi_time.py horseshoe; done; done
