# round-1 closing call (2 GPUs): GPU suite incl. DP/TP parity at coop default 24, small-batch coop A/B, bench
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?
tail -n 3 gpurun_out/pytest_gpu3.log
M="40 32 24 20 16 12 8"
for rep in 1 2; do
for c in 24 16 8; do
  echo "== coop_min=$c rep=$rep"
  CUDA_VISIBLE_DEVICES=0 RP_COOP_MIN=$c timeout -s KILL 400 python tools/step_profile.py $M 2>&1 | grep -o "B~[0-9]* rows/step=[0-9.]* ctx/row=[0-9]* eager_step_ms=[0-9.]* graph_step_ms=[0-9.]*"
done; done > gpurun_out/coop_ab3.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 1500 python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01g.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
