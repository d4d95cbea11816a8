#!/bin/bash
# group list split budget (waves) on the bench's live sets
cd $GRAFT_REPO_ROOT
for w in 2 3; do
  RP_ATTN_GROUP_MIN=0 RP_ATTN_GROUP_WAVES=$w timeout 900 python tools/attn_window_ab.py --tag group_w$w >> gpurun_out/r02ap.jsonl 2>> gpurun_out/r02ap.err
done
RP_ATTN_GROUP_MIN=0 RP_ATTN_GROUP=2 RP_ATTN_GROUP_WAVES=3 timeout 900 python tools/attn_window_ab.py --tag forced_w3 >> gpurun_out/r02ap.jsonl 2>> gpurun_out/r02ap.err
cat gpurun_out/r02ap.jsonl; tail -2 gpurun_out/r02ap.err
