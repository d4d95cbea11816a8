#!/bin/bash
# 2 GPUs: real-NCCL DP / TP parity, the N=2 bench line, C3 at P0=128 with KV-pressure preemption (TP2)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -s -k "dp.py or tp.py" > gpurun_out/r02p_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_multi.log
timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --steps 6 --warmup 5 > gpurun_out/r02p_bench_n2.json 2> gpurun_out/r02p_bench_n2.err
timeout 2400 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
   tools/c3_long_round.py --p0 128 --preempt --kv-gb 40 --out gpurun_out/r02p_c3_tp2_preempt.json > gpurun_out/r02p_c3.log 2>&1
tail -3 gpurun_out/r02p_multi.log
python -c "
import json
d=json.loads(open('gpurun_out/r02p_bench_n2.json').read().strip().splitlines()[-1]); print('N=2', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('clocks'))
"
tail -2 gpurun_out/r02p_c3.log
