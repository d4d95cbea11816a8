#!/bin/bash
# group vs per-row decode attention: parity of the new test, then a cost breakdown (RP_AG_DBG: 1 no MMAs, 2 no q_lo)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups or decode_step or split_kv" > gpurun_out/r02u_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_parity.log
tail -3 gpurun_out/r02u_parity.log
for v in 1 0; do for d in 0 1 2; do
  RP_ATTN_GROUP=$v RP_AG_DBG=$d timeout 600 python tools/step_ab.py --tag g${v}d$d --batches 64,256 --ctx 1024 >> gpurun_out/r02u_ab.jsonl 2>> gpurun_out/r02u_ab.err
  RP_ATTN_GROUP=$v RP_AG_DBG=$d timeout 600 python tools/step_ab.py --tag g${v}d$d --batches 16 --ctx 3000 >> gpurun_out/r02u_ab.jsonl 2>> gpurun_out/r02u_ab.err
done; done
python -c "
import json
for l in open('gpurun_out/r02u_ab.jsonl'):
    d=json.loads(l); print(d['tag'],d['B'],d['G'],d['ctx'],d['graph_step_ms'],d['cls'].get('attention'))
"
tail -3 gpurun_out/r02u_ab.err
