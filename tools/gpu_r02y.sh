#!/bin/bash
# power-of-two sibling groups: parity, A/B at full and partial groups, bench (auto) and bench (per-row kernel)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups" > gpurun_out/r02y_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_parity.log
tail -3 gpurun_out/r02y_parity.log
for v in 1 0; do
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --batches 16,32,48,128 --ctx 1024 >> gpurun_out/r02y_ab.jsonl 2>> gpurun_out/r02y_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --G 3 --batches 24,48,96 --ctx 1024 >> gpurun_out/r02y_ab.jsonl 2>> gpurun_out/r02y_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --G 2 --batches 32,64 --ctx 2048 >> gpurun_out/r02y_ab.jsonl 2>> gpurun_out/r02y_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02y_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -3 gpurun_out/r02y_ab.err
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
RP_ATTN_GROUP=0 timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02y_bench_rows.json 2> gpurun_out/r02y_bench_rows.err
for f in r02y_bench r02y_bench_rows; do python -c "
import json
s=open('gpurun_out/$f.json').read(); d=json.loads(s[s.index('{'):]); print('$f', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('kernel_profile',{}).get('attention'), d.get('clocks'))
"; done
