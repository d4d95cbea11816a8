timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout -s KILL 200 python tools/gemm_timeline.py 2>&1 | grep -E "timeline M=(4608|3584)|^M=(4608|3584)"
timeout -s KILL 300 python tools/step_profile.py 256 128 32 16 2>&1 | grep -A1 B~
