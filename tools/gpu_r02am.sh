#!/bin/bash
cd $GRAFT_REPO_ROOT
RP_ATTN_GROUP=0 timeout 900 python tools/attn_window_ab.py --tag rows > gpurun_out/r02am.jsonl 2> gpurun_out/r02am.err
RP_ATTN_GROUP_MIN=0 timeout 900 python tools/attn_window_ab.py --tag group >> gpurun_out/r02am.jsonl 2>> gpurun_out/r02am.err
RP_ATTN_GROUP_MIN=0 RP_ATTN_GROUP=2 timeout 900 python tools/attn_window_ab.py --tag group_forced >> gpurun_out/r02am.jsonl 2>> gpurun_out/r02am.err
cat gpurun_out/r02am.jsonl; tail -3 gpurun_out/r02am.err
