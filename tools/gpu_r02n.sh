#!/bin/bash
cd $GRAFT_REPO_ROOT
for m in 31 27; do
  RP_LO_MASK=$m timeout 900 python -m pytest tests/test_gpu_7b.py -q -s -k teacher > gpurun_out/r02n_7b_m$m.log 2>&1
done
RP_LO_MASK=27 timeout 900 python bench.py --steps 6 --warmup 5 --profile-steps 0 > gpurun_out/r02n_bench_m27.json 2> gpurun_out/r02n_bench_m27.err
RP_LO_MASK=31 timeout 900 python bench.py --steps 6 --warmup 5 --profile-steps 0 > gpurun_out/r02n_bench_m31.json 2> gpurun_out/r02n_bench_m31.err
grep -h "max-abs" gpurun_out/r02n_7b_m*.log
python -c "
import json
for m in (27, 31):
    f='gpurun_out/r02n_bench_m%d.json' % m
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(m, d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'])
    except Exception as e: print(f, 'ERR', e)
"
