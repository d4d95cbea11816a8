#!/bin/bash
# DSMEM split-K: capacities, GEMM + decode parity, A/B vs the global-memory split-K paths, 7B parity, bench
cd $GRAFT_REPO_ROOT
RP_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "gemm or decode_step or split_kv or sibling_groups and auto or short_round" > gpurun_out/r02z_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_parity.log
grep -m2 "split-K qkv" gpurun_out/r02z_parity.log; tail -3 gpurun_out/r02z_parity.log
if grep -q "rc=0" gpurun_out/r02z_parity.log; then
for v in 1 0; do
  RP_GEMM_DSM=$v RP_VERBOSE=1 timeout 600 python tools/step_ab.py --tag dsm$v --batches 16,32,64,128,256 --ctx 1024 >> gpurun_out/r02z_ab.jsonl 2>> gpurun_out/r02z_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02z_ab.jsonl'):
    d=json.loads(l); c=d['cls']; print(d['tag'],d['B'],d['graph_step_ms'],{k:c.get(k) for k in ('gemm_qkv','gemm_o','gemm_down','gemm_gu','attention')})
"
grep -m2 "split-K" gpurun_out/r02z_ab.err; tail -3 gpurun_out/r02z_ab.err
timeout 1200 python -m pytest tests/test_gpu_7b.py tests/test_gpu_7b_decode.py -q -s > gpurun_out/r02z_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_7b.log
tail -2 gpurun_out/r02z_7b.log; grep -h "max-abs" gpurun_out/r02z_7b.log
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
python -c "
import json
s=open('gpurun_out/r02z_bench.json').read(); d=json.loads(s[s.index('{'):]); print('bench', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('kernel_profile',{}).get('attention'), d.get('clocks'))
"
fi
