set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" 2>&1 | tail -30
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not gemm" 2>&1 | tail -40
