mkdir -p gpurun_out
timeout -s KILL 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 3 --profile-steps 0 > gpurun_out/bench_dp2.json 2> gpurun_out/bench_dp2.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_dp2.json')); print({k:d[k] for k in ('value','n_gpus','per_gpu_tokens_per_s','s_per_rl_step','config')}); [print(r) for r in d['rounds']]"
grep -v "^frame\|Exception raised\|TCPStore\|should dump\|^NCCL" gpurun_out/bench_dp2.err | tail -3
