#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/step_ab.py --tag lo > gpurun_out/r02h_ab.jsonl 2> gpurun_out/r02h_ab.err
RP_ACT_LO=0 timeout 600 python tools/step_ab.py --tag nolo >> gpurun_out/r02h_ab.jsonl 2>> gpurun_out/r02h_ab.err
for sk in attention gemm_qkv gemm_o gemm_gu gemm_down gemm_lm sampler "gemm_qkv,gemm_o" ; do
  RP_SKIP=$sk timeout 600 python tools/step_ab.py --tag "skip:$sk" --batches 16,64 >> gpurun_out/r02h_ab.jsonl 2>> gpurun_out/r02h_ab.err
done
timeout 1500 python -m pytest tests/test_gpu_7b.py tests/test_gpu_7b_decode.py -q -s > gpurun_out/r02h_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_7b.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_7b.py --deselect tests/test_gpu_7b_decode.py > gpurun_out/r02h_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_rest.log
cut -c1-120 gpurun_out/r02h_ab.jsonl; grep -h "max-abs\|passed\|failed" gpurun_out/r02h_7b.log; tail -2 gpurun_out/r02h_rest.log
