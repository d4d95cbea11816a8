mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_7b.py -x -q -s 2>&1 | grep "max-abs\|passed\|failed"
timeout -s KILL 200 python tools/step_profile.py 256 128 64 16 2>&1 | grep "graph_step"
