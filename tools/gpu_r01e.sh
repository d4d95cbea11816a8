# round-1 closing call: full GPU test suite, cooperative split-K A/B, smoke and the default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -n 5 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
M="128 90 64 48 32 16"
for c in 96 48 1000; do
  echo "== coop_min=$c"
  RP_COOP_MIN=$c timeout -s KILL 400 python tools/step_profile.py $M 2>&1 | grep -o "B~[0-9]* rows/step=[0-9.]* ctx/row=[0-9]* eager_step_ms=[0-9.]* graph_step_ms=[0-9.]*"
done > gpurun_out/coop_ab.txt 2>&1
cat gpurun_out/coop_ab.txt
timeout -s KILL 1500 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; echo bench rc=$?
cat gpurun_out/bench_r01e.json | head -c 3000
