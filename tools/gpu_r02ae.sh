#!/bin/bash
# O projection split-K through DSMEM (4 splits, clusters of 4): parity, step A/B, bench A/B
cd $GRAFT_REPO_ROOT
RP_VERBOSE=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_7b.py tests/test_gpu_local.py -q -x > gpurun_out/r02ae2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ae2_parity.log
grep -m1 "split-K qkv" gpurun_out/r02ae2_parity.log; tail -3 gpurun_out/r02ae2_parity.log
if grep -q "rc=0" gpurun_out/r02ae2_parity.log; then
for v in 1 0; do
  RP_GEMM_DSM_O=$v timeout 600 python tools/step_ab.py --tag o$v --batches 16,32,64,128,256 --ctx 1024 >> gpurun_out/r02ae2_ab.jsonl 2>> gpurun_out/r02ae2_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02ae2_ab.jsonl'):
    d=json.loads(l); c=d['cls']; print(d['tag'],d['B'],d['graph_step_ms'],{k:c.get(k) for k in ('gemm_qkv','gemm_o','gemm_down','attention')})
"
for v in 1 0; do
  RP_GEMM_DSM_O=$v timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02ae2_bench_o$v.json 2> gpurun_out/r02ae2_bench_o$v.err
  python -c "
import json
s=open('gpurun_out/r02ae2_bench_o$v.json').read(); d=json.loads(s[s.index('{'):]); kp=d.get('kernel_profile',{}); print('o$v', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], kp.get('gemm_o'), d.get('clocks'))
"
done
fi
