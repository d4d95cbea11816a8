#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_local.py -q -s > gpurun_out/r02c_local.log 2>&1
echo "local rc=$?" >> gpurun_out/r02c_local.log
tail -3 gpurun_out/r02c_local.log
