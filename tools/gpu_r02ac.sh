#!/bin/bash
# GEMM phase timelines at decode sizes (where the small-batch GEMM time goes)
cd $GRAFT_REPO_ROOT
timeout 600 python tools/gemm_timeline.py 16 32 64 128 > gpurun_out/r02ac_gemm_tl.log 2>&1; echo "rc=$?" >> gpurun_out/r02ac_gemm_tl.log
cat gpurun_out/r02ac_gemm_tl.log | grep -v "^$" | tail -40
