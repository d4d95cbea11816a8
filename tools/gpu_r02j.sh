#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm" > gpurun_out/r02j_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_gemm.log
timeout 600 python tools/step_ab.py --tag lo > gpurun_out/r02j_ab.jsonl 2> gpurun_out/r02j_ab.err
RP_ACT_LO=0 timeout 600 python tools/step_ab.py --tag nolo >> gpurun_out/r02j_ab.jsonl 2>> gpurun_out/r02j_ab.err
timeout 1500 python -m pytest tests/test_gpu_7b.py tests/test_gpu_7b_decode.py -q -s > gpurun_out/r02j_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_7b.log
tail -3 gpurun_out/r02j_gemm.log; cut -c1-330 gpurun_out/r02j_ab.jsonl; grep -h "max-abs\|passed\|failed" gpurun_out/r02j_7b.log
