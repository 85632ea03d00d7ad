# final round-2 evidence: launch list, whole-graph metrics, per-kernel full sets
set -x
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-xi --no-other-configs --no-e2e"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo launch rc=$?
python scripts/graph_sweeps.py > gpurun_out/plain_graph.log 2>&1 && \
ncu --graph-profiling graph --clock-control none --cache-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,lts__t_bytes.sum,sm__inst_executed_pipe_xu.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file gpurun_out/graph_metrics.csv python scripts/graph_sweeps.py > gpurun_out/ncu_graph.log 2>&1
echo graph rc=$?
python scripts/profile_sweep.py --chains 4 --burn 200 --sweeps 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"eps_sweep|gene_sweep|hyper_a|leaf_b" -s 1600 -c 8 \
    -o gpurun_out/prof_final python scripts/profile_sweep.py --chains 4 --burn 200 --sweeps 2 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
tail -2 gpurun_out/ncu_full.log
