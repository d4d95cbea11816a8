#!/bin/bash
# attn_group 4 (shared pages in group units, private pages per row, per-row merge): parity, windows A/B
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sibling_groups" > gpurun_out/r02an_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02an_parity.log
tail -3 gpurun_out/r02an_parity.log; grep -m5 "Error\|assert" gpurun_out/r02an_parity.log
if grep -q "rc=0" gpurun_out/r02an_parity.log; then
RP_ATTN_GROUP=4 RP_ATTN_GROUP_MIN=0 timeout 900 python tools/attn_window_ab.py --tag split > gpurun_out/r02an.jsonl 2> gpurun_out/r02an.err
RP_ATTN_GROUP=0 timeout 900 python tools/attn_window_ab.py --tag rows >> gpurun_out/r02an.jsonl 2>> gpurun_out/r02an.err
cat gpurun_out/r02an.jsonl; tail -3 gpurun_out/r02an.err
fi
