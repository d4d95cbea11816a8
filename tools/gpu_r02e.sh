#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_7b.py tests/test_gpu_7b_decode.py -q -s > gpurun_out/r02e_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_7b.log
timeout 600 python tools/step_ab.py --tag lo > gpurun_out/r02e_ab.jsonl 2> gpurun_out/r02e_ab.err
RP_ACT_LO=0 timeout 600 python tools/step_ab.py --tag nolo >> gpurun_out/r02e_ab.jsonl 2>> gpurun_out/r02e_ab.err
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_7b.py --deselect tests/test_gpu_7b_decode.py > gpurun_out/r02e_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_rest.log
grep -h "max-abs\|passed\|failed" gpurun_out/r02e_7b.log; cat gpurun_out/r02e_ab.jsonl; tail -3 gpurun_out/r02e_rest.log
