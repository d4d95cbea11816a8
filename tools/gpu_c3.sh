mkdir -p gpurun_out
N=${1:-2}
timeout -s KILL 1200 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/c3_long_round.py --out gpurun_out/c3_tp$N.json $2 > gpurun_out/c3_tp$N.log 2> gpurun_out/c3_tp$N.err; echo rc=$?
grep "^{" gpurun_out/c3_tp$N.log; grep -v "^frame\|OMP_NUM\|^\*\*\*\|^NCCL" gpurun_out/c3_tp$N.err | tail -5
