#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_preempt.py -q -s > gpurun_out/r02m_preempt.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_preempt.log
for m in 30 26; do
  RP_LO_MASK=$m timeout 900 python -m pytest tests/test_gpu_7b.py -q -s -k teacher > gpurun_out/r02m_7b_m$m.log 2>&1
  RP_LO_MASK=$m timeout 900 python bench.py --steps 6 --warmup 5 --profile-steps 0 > gpurun_out/r02m_bench_m$m.json 2> gpurun_out/r02m_bench_m$m.err
done
tail -2 gpurun_out/r02m_preempt.log; grep -h "max-abs" gpurun_out/r02m_7b_m*.log
python -c "
import json
for m in (30, 26):
    f='gpurun_out/r02m_bench_m%d.json' % m
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(m, d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'])
    except Exception as e: print(f, 'ERR', e)
"
