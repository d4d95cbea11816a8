#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02q_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02q_parity.log
timeout 600 python tools/step_ab.py --tag fused > gpurun_out/r02q_ab.jsonl 2> gpurun_out/r02q_ab.err
RP_FUSE_QKV=0 timeout 600 python tools/step_ab.py --tag unfused >> gpurun_out/r02q_ab.jsonl 2>> gpurun_out/r02q_ab.err
timeout 1800 python -m pytest tests -q -s -m gpu --deselect tests/test_gpu_parity.py > gpurun_out/r02q_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02q_rest.log
timeout 900 python bench.py --steps 6 --warmup 5 --profile-steps 0 > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
tail -2 gpurun_out/r02q_parity.log; grep -n "assert\|Error" gpurun_out/r02q_parity.log | head -5
python -c "
import json
for l in open('gpurun_out/r02q_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['graph_step_ms'],d['cls'].get('gemm_qkv'),d['cls'].get('attention'))
"
tail -2 gpurun_out/r02q_rest.log; grep -h "max-abs" gpurun_out/r02q_rest.log
python -c "
import json
d=json.loads(open('gpurun_out/r02q_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'])
"
