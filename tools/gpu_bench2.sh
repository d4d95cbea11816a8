mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 900 python bench.py --config C2-7b --steps 1 --warmup 1 > gpurun_out/bench_7b.json 2> gpurun_out/bench_7b.err; echo 7b rc=$?
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_7b.json"))
print({k:d[k] for k in ("value","ms_per_step","s_per_rl_step","roofline")})
for k,v in d["kernel_profile"].items(): print(k, v)
PY
tail -3 gpurun_out/bench_7b.err
