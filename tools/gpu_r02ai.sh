#!/bin/bash
# plain synchronous rollout (the veRL baseline) vs tail batching, final build, N=1 and N=2
cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --schedule sync --steps 4 --warmup 3 > gpurun_out/r02ai_sync_n1.json 2> gpurun_out/r02ai_sync_n1.err
timeout 1500 python bench.py --schedule tail --steps 4 --warmup 3 > gpurun_out/r02ai_tail_n1.json 2> gpurun_out/r02ai_tail_n1.err
timeout 2000 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
   bench.py --gpus 2 --schedule sync --steps 4 --warmup 3 > gpurun_out/r02ai_sync_n2.json 2> gpurun_out/r02ai_sync_n2.err
timeout 2000 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
   bench.py --gpus 2 --schedule tail --steps 4 --warmup 3 > gpurun_out/r02ai_tail_n2.json 2> gpurun_out/r02ai_tail_n2.err
for f in sync_n1 tail_n1 sync_n2 tail_n2; do python -c "
import json
s=open('gpurun_out/r02ai_$f.json').read(); d=json.loads(s[s.index('{'):]); print('$f', d['value'], d['decoded_tokens_per_s'], d['s_per_rl_step'], d.get('clocks',{}).get('reasons'))
"; done
