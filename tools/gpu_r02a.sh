#!/bin/bash
# round 2: new multi-context (local group) tests + full-width 7B decode parity + the rest of the GPU suite
cd $GRAFT_REPO_ROOT
python -c "from paper_2509_21009_b200 import build; build.build()" > gpurun_out/r02a_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_local.py -x -q -s > gpurun_out/r02a_local.log 2>&1
echo "local rc=$?" >> gpurun_out/r02a_local.log
timeout 1500 python -m pytest tests/test_gpu_7b_decode.py tests/test_gpu_7b.py -x -q -s > gpurun_out/r02a_7b.log 2>&1
echo "7b rc=$?" >> gpurun_out/r02a_7b.log
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_gpu_local.py --deselect tests/test_gpu_7b_decode.py --deselect tests/test_gpu_7b.py > gpurun_out/r02a_rest.log 2>&1
echo "rest rc=$?" >> gpurun_out/r02a_rest.log
tail -3 gpurun_out/r02a_*.log
