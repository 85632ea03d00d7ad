# both bench arms as the driver runs them (reference first), N = 1
set -x
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo b200 rc=$?
tail -c 600 gpurun_out/bench_ref.json
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
r = json.loads(open("gpurun_out/bench_ref.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "post", d["e2e"]["post_burnin_value"])
print("ref", r["value"], "ratio", d["value"] / r["value"], "e2e ratio", d["e2e"]["value"] / r["value"])
print("roofline", d["roofline"]["frac"], d["roofline"]["traffic"], d["roofline"].get("issue_roofline", {}).get("frac"))
print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["single_core"]["value"])
print("other", {k: (v["value"], v.get("ratio_vs_cpu")) for k, v in d["other_configs"].items() if isinstance(v, dict)})
print("xi", {k: v["ms_per_step"] for k, v in d["xi_priors"].items() if isinstance(v, dict)})
print("burnin", d["burnin"]["ms_per_sweep"], d["burnin"]["first_ms_per_sweep"], "clocks", d["clocks"])
PY
