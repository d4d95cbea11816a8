#!/bin/bash
# group decode attention v2 (8 single-member warps, cooperative split merge): parity, then A/B vs the per-row list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups or decode_step or split_kv or sampled" > gpurun_out/r02w_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02w_parity.log
tail -3 gpurun_out/r02w_parity.log
for t in "1 0" "1 1" "0 0"; do set -- $t
  RP_ATTN_GROUP=$1 RP_AG_DBG=$2 timeout 600 python tools/step_ab.py --tag g$1d$2 --batches 16,64,256 --ctx 1024 >> gpurun_out/r02w_ab.jsonl 2>> gpurun_out/r02w_ab.err
  RP_ATTN_GROUP=$1 RP_AG_DBG=$2 timeout 600 python tools/step_ab.py --tag g$1d$2 --batches 16 --ctx 3000 >> gpurun_out/r02w_ab.jsonl 2>> gpurun_out/r02w_ab.err
  RP_ATTN_GROUP=$1 RP_AG_DBG=$2 timeout 600 python tools/step_ab.py --tag g$1d$2 --G 1 --batches 8,32 --ctx 4096 >> gpurun_out/r02w_ab.jsonl 2>> gpurun_out/r02w_ab.err
done
python -c "
import json
for l in open('gpurun_out/r02w_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -3 gpurun_out/r02w_ab.err
