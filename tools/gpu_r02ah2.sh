#!/bin/bash
# 2 GPUs: migration to the second GPU, real-NCCL DP/TP parity with the O-projection DSMEM split-K
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_migrate.py -q -x > gpurun_out/r02ah_migrate2.log 2>&1; echo "rc=$?" >> gpurun_out/r02ah_migrate2.log
tail -3 gpurun_out/r02ah_migrate2.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -s -k "dp.py or tp.py" > gpurun_out/r02ah_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r02ah_multi.log
tail -3 gpurun_out/r02ah_multi.log
