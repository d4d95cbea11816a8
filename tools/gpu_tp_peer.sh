mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
bash tools/gpu_dp.sh 2>&1 | grep -v "NCCL INFO" | grep "value\|short\|long" | cut -c1-300
