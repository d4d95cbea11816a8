# round-1 closing call (2 GPUs): GPU suite incl. DP/TP parity at coop default 16, smoke, bench, launch lists
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?
tail -n 3 gpurun_out/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke4.log 2>&1; echo smoke rc=$?
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 1500 python bench.py > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01h.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h_launches_b256.csv python tools/ncu_decode.py 0 1 > gpurun_out/ncu_l1.log 2>&1; echo launches256 rc=$?
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h_launches_b16.csv python tools/ncu_small_b.py 1 > gpurun_out/ncu_l2.log 2>&1; echo launches16 rc=$?
