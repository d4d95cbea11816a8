#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_preempt.py -q -x -s > gpurun_out/r02k_preempt.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_preempt.log
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_7b.py --deselect tests/test_gpu_7b_decode.py --deselect tests/test_gpu_preempt.py > gpurun_out/r02k_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_rest.log
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02k_bench_lo.json 2> gpurun_out/r02k_bench_lo.err
RP_ACT_LO=0 timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02k_bench_nolo.json 2> gpurun_out/r02k_bench_nolo.err
tail -3 gpurun_out/r02k_preempt.log; tail -2 gpurun_out/r02k_rest.log
python -c "
import json
for f in ['gpurun_out/r02k_bench_lo.json','gpurun_out/r02k_bench_nolo.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('roofline',{}).get('kernel'), d.get('roofline',{}).get('frac'))
    except Exception as e: print(f, 'ERR', e)
"
