mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "streaming or speculation" 2>&1 | tail -2
timeout -s KILL 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 tools/c3_long_round.py --model qwen2.5-32b --p0 64 --out gpurun_out/c4_tp4.json > gpurun_out/c4_tp4.log 2> gpurun_out/c4_tp4.err; echo rc=$?
grep "^{" gpurun_out/c4_tp4.log | cut -c1-600; grep -v "^frame\|OMP_NUM\|^\*\*\*\|NCCL" gpurun_out/c4_tp4.err | tail -4
