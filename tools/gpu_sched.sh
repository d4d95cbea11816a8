# tail batching vs plain synchronous rollout on the same prompt stream, N GPUs (weak scaling)
mkdir -p gpurun_out
N=${1:-1}; STEPS=${2:-5}   # usage: gpu_sched.sh N STEPS "tail sync issue"
for S in ${3:-tail sync}; do
if [ "$N" = "1" ]; then
  timeout -s KILL 1500 python bench.py --schedule $S --steps $STEPS --warmup 3 --profile-steps 0 > gpurun_out/sched_${S}_n$N.json 2> gpurun_out/sched_${S}_n$N.err
else
  timeout -s KILL 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --schedule $S --steps $STEPS --warmup 3 --profile-steps 0 > gpurun_out/sched_${S}_n$N.json 2> gpurun_out/sched_${S}_n$N.err
fi
python -c "
import json; d=json.load(open('gpurun_out/sched_${S}_n$N.json')); print('$S', 'N=$N', d['value'], d['s_per_rl_step'], d['round_roofline']['frac'])"
done
