#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_preempt.py -q -s > gpurun_out/r02l_preempt.log 2>&1; echo "rc=$?" >> gpurun_out/r02l_preempt.log
timeout 600 python tools/step_ab.py --tag lo200 > gpurun_out/r02l_ab.jsonl 2> gpurun_out/r02l_ab.err
RP_ACT_LO=0 timeout 600 python tools/step_ab.py --tag nolo200 >> gpurun_out/r02l_ab.jsonl 2>> gpurun_out/r02l_ab.err
timeout 600 python tools/gemm_bench.py down > gpurun_out/r02l_gemm_down.txt 2>&1
tail -3 gpurun_out/r02l_preempt.log; grep -n "Error\|assert" gpurun_out/r02l_preempt.log | head; cut -c1-200 gpurun_out/r02l_ab.jsonl; cat gpurun_out/r02l_gemm_down.txt | tail -25
