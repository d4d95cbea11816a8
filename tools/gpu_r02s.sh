#!/bin/bash
cd $GRAFT_REPO_ROOT
bash tools/gpu_sanitize.sh > gpurun_out/r02s_sanitize.txt 2>&1
bash tools/gpu_r02r.sh > gpurun_out/r02s_ncu.txt 2>&1
tail -n 12 gpurun_out/r02s_sanitize.txt; tail -n 30 gpurun_out/r02s_ncu.txt
