#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k gemm > gpurun_out/r02o_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_gemm.log
timeout 600 python tools/step_ab.py --tag lo_pair > gpurun_out/r02o_ab.jsonl 2> gpurun_out/r02o_ab.err
timeout 900 python -m pytest tests/test_gpu_7b.py tests/test_gpu_7b_decode.py -q -s > gpurun_out/r02o_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_7b.log
timeout 900 python bench.py --steps 6 --warmup 5 --profile-steps 0 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
tail -2 gpurun_out/r02o_gemm.log; grep -n "assert\|Error" gpurun_out/r02o_gemm.log | head -5
python -c "
import json
for l in open('gpurun_out/r02o_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['graph_step_ms'],d['cls'].get('gemm_gu'),d['cls'].get('gemm_down'))
"
grep -h "max-abs\|passed\|failed" gpurun_out/r02o_7b.log
python -c "
import json
d=json.loads(open('gpurun_out/r02o_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'])
"
