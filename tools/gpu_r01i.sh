# N=2 bench line at coop default 16, and the CTA-pair GEMM A/B re-run at the new coop default
mkdir -p gpurun_out
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/bench_r01i_n2.json 2> gpurun_out/bench_r01i_n2.err; echo bench2 rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01i_n2.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
M="256 128 90 64 48 32 16"
for p in 0 1; do
  echo "== pair=$p"
  if [ $p = 1 ]; then export RP_GEMM_PAIR=1; fi
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 python tools/step_profile.py $M 2>&1 | grep -o "B~[0-9]* rows/step=[0-9.]* ctx/row=[0-9]* eager_step_ms=[0-9.]* graph_step_ms=[0-9.]*"
done > gpurun_out/pair_ab.txt 2>&1
cat gpurun_out/pair_ab.txt
