#!/bin/bash
# fast Gumbel noise in the sampler: token parity, sampler time, bench
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_7b.py tests/test_gpu_7b_decode.py tests/test_gpu_preempt.py tests/test_gpu_migrate.py -q -x -s > gpurun_out/r02as_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02as_parity.log
tail -3 gpurun_out/r02as_parity.log; grep -h "max-abs\|in-gap" gpurun_out/r02as_parity.log | head
if grep -q "rc=0" gpurun_out/r02as_parity.log; then
timeout 600 python tools/step_ab.py --tag fastlog --batches 16,64,256 --ctx 1024 > gpurun_out/r02as_ab.jsonl 2> gpurun_out/r02as_ab.err
python -c "
import json
for l in open('gpurun_out/r02as_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['graph_step_ms'],d['cls'].get('sampler'))
"
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02as_bench.json 2> gpurun_out/r02as_bench.err
python -c "
import json
s=open('gpurun_out/r02as_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d['kernel_profile']['sampler'], d.get('clocks'))
"
fi
