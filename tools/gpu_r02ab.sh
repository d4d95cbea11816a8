#!/bin/bash
# layer-major KV layout: parity (attention, fork, recompute, TP local groups), A/B points, bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_preempt.py tests/test_gpu_local.py -q -x > gpurun_out/r02ab_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ab_parity.log
tail -3 gpurun_out/r02ab_parity.log
if grep -q "rc=0" gpurun_out/r02ab_parity.log; then
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --batches 16,64,256 --ctx 1024 >> gpurun_out/r02ab_ab.jsonl 2>> gpurun_out/r02ab_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --batches 16 --ctx 3000 >> gpurun_out/r02ab_ab.jsonl 2>> gpurun_out/r02ab_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --G 1 --batches 8,32 --ctx 4096 >> gpurun_out/r02ab_ab.jsonl 2>> gpurun_out/r02ab_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02ab_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -2 gpurun_out/r02ab_ab.err
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02ab_bench_g$v.json 2> gpurun_out/r02ab_bench_g$v.err
  python -c "
import json
s=open('gpurun_out/r02ab_bench_g$v.json').read(); d=json.loads(s[s.index('{'):]); print('g$v', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('kernel_profile',{}).get('attention'), d.get('clocks'))
"
done
fi
