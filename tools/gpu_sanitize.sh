#!/bin/bash
# compute-sanitizer on the tiny config: memcheck, racecheck, synccheck over smoke()
# (teacher-forced logits + one short round in graphs) and a small KV-pressure round.
cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $S --tool $tool --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/preempt_small.py > gpurun_out/san_memcheck_preempt.log 2>&1
echo "memcheck preempt rc=$?" >> gpurun_out/san_memcheck_preempt.log
tail -n 4 gpurun_out/san_*.log
