#!/bin/bash
# per-launch ncu durations of the tail kernels (hyper_a, leaf_b) for library builds
for lib in "$@"; do
  CMC_LIB_OVERRIDE=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hyper_a|leaf_b|gene_sweep|eps_sweep" -s 400 -c 80 --csv python scripts/profile_sweep.py --chains 4 --burn 200 --sweeps 10 2>/dev/null > gpurun_out/tl_$(basename $lib .so).csv
  python - "$lib" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open("gpurun_out/tl_" + sys.argv[1].split("/")[-1][:-3] + ".csv")) if len(r) > 14 and r[0] != "ID"]
t = collections.defaultdict(list)
for r in rows: t[r[4].split("(")[0][-30:]].append(float(r[14].replace(",", "")) / 1000)
print(sys.argv[1], {k: round(sum(v) / len(v), 1) for k, v in t.items()})
PY
done
