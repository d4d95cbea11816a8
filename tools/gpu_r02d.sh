#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm or teacher or decode_step" > gpurun_out/r02d_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_parity.log
timeout 600 python tools/step_ab.py --tag tiled > gpurun_out/r02d_ab.jsonl 2> gpurun_out/r02d_ab.err
RP_W_ROWMAJOR=1 timeout 600 python tools/step_ab.py --tag rowmajor >> gpurun_out/r02d_ab.jsonl 2>> gpurun_out/r02d_ab.err
timeout 600 python tools/step_ab.py --tag tiled2 >> gpurun_out/r02d_ab.jsonl 2>> gpurun_out/r02d_ab.err
timeout 900 python -m pytest tests/test_gpu_7b_decode.py -q -x -s > gpurun_out/r02d_7b.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_7b.log
tail -2 gpurun_out/r02d_parity.log; cat gpurun_out/r02d_ab.jsonl; tail -4 gpurun_out/r02d_7b.log
