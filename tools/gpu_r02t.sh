#!/bin/bash
# sibling-group decode attention: parity first, then A/B vs the per-row work list, suite, bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02t_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_parity.log
tail -3 gpurun_out/r02t_parity.log
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag grp$v --batches 16,64,256 --ctx 1024 >> gpurun_out/r02t_ab.jsonl 2>> gpurun_out/r02t_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag grp$v --batches 16 --ctx 3000 >> gpurun_out/r02t_ab.jsonl 2>> gpurun_out/r02t_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag grp$v --G 1 --batches 8,32 --ctx 4096 >> gpurun_out/r02t_ab.jsonl 2>> gpurun_out/r02t_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02t_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -3 gpurun_out/r02t_ab.err
timeout 2400 python -m pytest tests -q -s -m gpu --deselect tests/test_gpu_parity.py > gpurun_out/r02t_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_rest.log
tail -2 gpurun_out/r02t_rest.log; grep -h "max-abs" gpurun_out/r02t_rest.log
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
python -c "
import json
s=open('gpurun_out/r02t_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('roofline'))
"
