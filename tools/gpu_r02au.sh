#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_migrate.py -q -x > gpurun_out/r02au_migrate.log 2>&1; echo "rc=$?" >> gpurun_out/r02au_migrate.log
tail -25 gpurun_out/r02au_migrate.log
