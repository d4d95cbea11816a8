mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 300 python bench.py --config C1-tiny --steps 5 --warmup 3 > gpurun_out/bench_tiny.json 2> gpurun_out/bench_tiny.err; echo tiny rc=$?
tail -c 3000 gpurun_out/bench_tiny.json; tail -5 gpurun_out/bench_tiny.err
timeout -s KILL 900 python bench.py --config C2-7b --steps 1 --warmup 1 > gpurun_out/bench_7b.json 2> gpurun_out/bench_7b.err; echo 7b rc=$?
tail -c 4000 gpurun_out/bench_7b.json; tail -20 gpurun_out/bench_7b.err
