# GPU parity tests + a short bench (development loop)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], "ms", d["ms_per_step"], "launches", d["gpu_launches"])
    print("roofline", json.dumps(d["roofline"].get("kernels")))
    print("burnin", json.dumps(d["burnin"]))
    print("xi", json.dumps(d.get("xi_priors")))
    print("other", json.dumps(d.get("other_configs"))[:600])
    print("e2e", d["e2e"]["value"] if d.get("e2e") else None, "cpu", (d.get("cpu_baseline") or {}).get("value"))
except Exception as ex:
    print("no bench line", ex)
PY
