timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout -s KILL 300 python tools/step_profile.py 256 128 32 16 2>&1 | grep -A1 B~
bash tools/gpu_bench_full.sh 2>&1 | head -3 | cut -c1-400
