mkdir -p gpurun_out
timeout -s KILL 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_full.json"))
print({k:d[k] for k in ("value","ms_per_step","s_per_rl_step","e2e","gpu_launches","clocks","roofline","retained_tokens_per_s","speculation_waste")})
for r in d["rounds"]: print(r)
print(d["cpu_baseline"])
PY
tail -3 gpurun_out/bench_full.err
