#!/bin/bash
# group attention auto policy: parity, crossover A/B (sibling groups / single rows / per-row kernel), suite, bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups" > gpurun_out/r02x_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_parity.log
tail -3 gpurun_out/r02x_parity.log
for v in 2 3 0; do
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --batches 16,24,32,48,64,128,256 --ctx 1024 >> gpurun_out/r02x_ab.jsonl 2>> gpurun_out/r02x_ab.err
  RP_ATTN_GROUP=$v timeout 600 python tools/step_ab.py --tag g$v --batches 16,32,64 --ctx 3000 >> gpurun_out/r02x_ab.jsonl 2>> gpurun_out/r02x_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02x_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -3 gpurun_out/r02x_ab.err
timeout 2400 python -m pytest tests -q -s -m gpu --deselect tests/test_gpu_parity.py > gpurun_out/r02x_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_rest.log
tail -2 gpurun_out/r02x_rest.log; grep -h "max-abs" gpurun_out/r02x_rest.log
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err
python -c "
import json
s=open('gpurun_out/r02x_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('roofline'), d.get('clocks'))
"
