#!/bin/bash
# group attention only above 128 live rows (per-graph kernel choice): parity, 7B, bench A/B
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_preempt.py tests/test_gpu_7b_decode.py -q -x > gpurun_out/r02ad_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ad_parity.log
tail -3 gpurun_out/r02ad_parity.log
if grep -q "rc=0" gpurun_out/r02ad_parity.log; then
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02ad_bench_g$v.json 2> gpurun_out/r02ad_bench_g$v.err
  python -c "
import json
s=open('gpurun_out/r02ad_bench_g$v.json').read(); d=json.loads(s[s.index('{'):]); kp=d.get('kernel_profile',{}); print('g$v', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], kp.get('attention'), kp.get('ctl'), d.get('clocks'))
"
done
fi
