mkdir -p gpurun_out
timeout -s KILL 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 2 --warmup 3 --profile-steps 0 > gpurun_out/bench_dp4.json 2> gpurun_out/bench_dp4.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_dp4.json')); print({k:d[k] for k in ('value','n_gpus','s_per_rl_step','step_roofline')}); [print(r) for r in d['rounds']]"
grep -v "^frame\|Exception raised\|TCPStore\|should dump\|NCCL" gpurun_out/bench_dp4.err | tail -3
