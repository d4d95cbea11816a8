#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in old A B C old2 A2; do
  case $v in
    old*) L=build/old/librollpacker.so ;;
    A*) L=paper_2509_21009_b200/librollpacker.so ;;
    B) L=build/vB/librollpacker.so ;;
    C) L=build/vC/librollpacker.so ;;
  esac
  RP_ACT_LO=0 RP_LIB=$L timeout 600 python tools/step_ab.py --tag $v --batches 16,256 >> gpurun_out/r02g_ab.jsonl 2>> gpurun_out/r02g_ab.err
done
cut -c1-300 gpurun_out/r02g_ab.jsonl
