# parity + graph step times at several live-batch sizes
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 200 python tools/step_profile.py 256 128 64 48 40 32 16 2>&1 | grep -A1 "graph_step"
