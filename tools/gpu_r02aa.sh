#!/bin/bash
# attention policy (fills-saved threshold) bench A/B vs the per-row kernel; parity of the group paths
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups or decode_step or dsm" > gpurun_out/r02aa_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02aa_parity.log
tail -3 gpurun_out/r02aa_parity.log
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02aa_bench_g$v.json 2> gpurun_out/r02aa_bench_g$v.err
  python -c "
import json
s=open('gpurun_out/r02aa_bench_g$v.json').read(); d=json.loads(s[s.index('{'):]); print('g$v', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('kernel_profile',{}).get('attention'), d.get('clocks'))
"
done
