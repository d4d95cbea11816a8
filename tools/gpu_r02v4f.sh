#!/bin/bash
# 4 GPUs: real-NCCL DP, TP and DPxTP (2x2) parity, the N=4 bench line, C4 (32B) long round TP4
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -s > gpurun_out/r02v4f_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02v4f_multi.log
tail -3 gpurun_out/r02v4f_multi.log
timeout 1800 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
   bench.py --gpus 4 --steps 6 --warmup 5 > gpurun_out/r02v4f_bench_n4.json 2> gpurun_out/r02v4f_bench_n4.err
python -c "
import json
s=open('gpurun_out/r02v4f_bench_n4.json').read(); d=json.loads(s[s.index('{'):]); print('N=4', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('clocks'))
"
tail -3 gpurun_out/r02v4f_bench_n4.err
timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 \
   bench.py --gpus 2 --steps 6 --warmup 5 > gpurun_out/r02v4f_bench_n2.json 2> gpurun_out/r02v4f_bench_n2.err
python -c "
import json
s=open('gpurun_out/r02v4f_bench_n2.json').read(); d=json.loads(s[s.index('{'):]); print('N=2', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('clocks'))
"
