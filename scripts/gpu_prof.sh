# timeline + ncu full capture of one steady-state sweep's kernels (both lanes)
set -x
python scripts/timeline.py > gpurun_out/timeline.txt 2>&1
python scripts/profile_sweep.py --chains 4 --burn 200 --sweeps 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-eps_sweep|gene_sweep|hyper_a|leaf_b}" -s ${SKIP:-1600} -c ${COUNT:-8} \
    -o gpurun_out/${REP:-prof} python scripts/profile_sweep.py --chains 4 --burn 200 --sweeps 2 > gpurun_out/ncu.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu.log
cat gpurun_out/timeline.txt | head -60
