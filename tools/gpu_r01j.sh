# N=4 bench line at coop default 16
mkdir -p gpurun_out
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 > gpurun_out/bench_r01j_n4.json 2> gpurun_out/bench_r01j_n4.err; echo bench4 rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01j_n4.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['s_per_rl_step'], d['clocks'])"
