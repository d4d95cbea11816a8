#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02av_bench.json 2> gpurun_out/r02av_bench.err
python -c "
import json
s=open('gpurun_out/r02av_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['e2e']['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d['roofline']['frac'], d['step_roofline']['frac'], d.get('gpu_launches'), d.get('clocks'))
"
tail -2 gpurun_out/r02av_bench.err
