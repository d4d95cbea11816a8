mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 1500 python tools/sweep_c5.py --steps 5 --ratios 25,32 --out gpurun_out/sweep_c5_pr.json 2>&1 | grep "^{"
