#!/bin/bash
# 2 GPUs: DP=2 -> 1 migration over NCCL, migration to the second GPU
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multi.py -q -s -k "migrate" > gpurun_out/r02al_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02al_multi.log
tail -5 gpurun_out/r02al_multi.log
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/test_gpu_migrate_nccl.py > gpurun_out/r02al_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/r02al_nccl.log
grep -h "migrate DP\|PASS\|Error" gpurun_out/r02al_nccl.log | head
timeout 900 python -m pytest tests/test_gpu_migrate.py -q > gpurun_out/r02al_migrate.log 2>&1; echo "rc=$?" >> gpurun_out/r02al_migrate.log
tail -3 gpurun_out/r02al_migrate.log
