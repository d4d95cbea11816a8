#!/bin/bash
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/r02f_smi.txt
for v in old new_lo new_nolo old2 new_lo2; do
  case $v in
    old*) RP_LIB=build/old/librollpacker.so timeout 600 python tools/step_ab.py --tag $v >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err ;;
    new_lo*) timeout 600 python tools/step_ab.py --tag $v >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err ;;
    new_nolo) RP_ACT_LO=0 timeout 600 python tools/step_ab.py --tag $v >> gpurun_out/r02f_ab.jsonl 2>> gpurun_out/r02f_ab.err ;;
  esac
done
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv >> gpurun_out/r02f_smi.txt
cut -c1-200 gpurun_out/r02f_ab.jsonl
