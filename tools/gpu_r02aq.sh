#!/bin/bash
# kv_tokens_unique counters (schedule test) + the bench line with unique-KV roofline bytes
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "short_round_schedule or gemm_tcgen05_vs_fp32 or decode_step" > gpurun_out/r02aq_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02aq_parity.log
tail -3 gpurun_out/r02aq_parity.log; grep -m3 "assert\|Error" gpurun_out/r02aq_parity.log
timeout 900 python bench.py --steps 6 --warmup 5 > gpurun_out/r02aq_bench.json 2> gpurun_out/r02aq_bench.err
python -c "
import json
s=open('gpurun_out/r02aq_bench.json').read(); d=json.loads(s[s.index('{'):]); print(d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d['roofline']['frac'], d['step_roofline']['frac'], d['round_roofline']['frac'], d['kernel_profile']['attention'], d.get('clocks'))
"
tail -2 gpurun_out/r02aq_bench.err
