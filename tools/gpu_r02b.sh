#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/local_diag.py 4 > gpurun_out/r02b_diag4.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_diag4.log
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python tools/local_diag.py 4 > gpurun_out/r02b_diag4_c32.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_diag4_c32.log
timeout 1500 python -m pytest tests/test_gpu_7b_decode.py tests/test_gpu_7b.py -q -s > gpurun_out/r02b_7b.log 2>&1
echo "7b rc=$?" >> gpurun_out/r02b_7b.log
tail -3 gpurun_out/r02b_*.log
