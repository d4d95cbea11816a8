#!/bin/bash
# final build: smoke, whole single-GPU suite, bench N=1
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ao_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_smoke.log
tail -2 gpurun_out/r02ao_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02ao_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_tests.log
tail -3 gpurun_out/r02ao_tests.log
timeout 900 python bench.py > gpurun_out/r02ao_bench.json 2> gpurun_out/r02ao_bench.err
python -c "
import json
s=open('gpurun_out/r02ao_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d['steps'], d['warmup'], d.get('roofline',{}).get('frac'), d.get('clocks'))
"
