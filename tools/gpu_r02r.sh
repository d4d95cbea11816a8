#!/bin/bash
# round-2 ncu evidence: (1) launch list of the bench command (gpu__time_duration per launch, from the middle of the
# first short round, ~38 live rows), (2) --set full of one layer's GEMMs + attention at ~38 rows (graph steps) and
# at 256 rows (first steps), (3) summaries under profiles/ (tools/make_profiles.py)
cd $GRAFT_REPO_ROOT
N=/usr/local/cuda/bin/ncu
timeout 1800 $N --metrics gpu__time_duration.sum --clock-control none --launch-skip 170000 --launch-count 2900 --csv \
   --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 1 --warmup 3 --profile-steps 0 > gpurun_out/r02r_bench_under_ncu.log 2>&1
# 141 matching launches per decode step (28 x 5 + LM head) and for the prefill; layer 10 of the first measured step
timeout 1800 $N --set full --clock-control none --import-source on -k regex:"gemm|attn" \
   --launch-skip $((141 * 1201 + 50)) --launch-count 6 -o gpurun_out/r02_ncu_b38 -f \
   python tools/ncu_step.py --skip 1200 --steps 1 --graph-steps 16 > gpurun_out/r02r_ncu_b38.log 2>&1
timeout 1800 $N --set full --clock-control none --import-source on -k regex:"gemm|attn" \
   --launch-skip $((141 * 2 + 50)) --launch-count 6 -o gpurun_out/r02_ncu_b256 -f \
   python tools/ncu_step.py --skip 0 --steps 2 > gpurun_out/r02r_ncu_b256.log 2>&1
ROWS_b38=38 ROWS_b256=256 SHAPE_b38="7B decode step ~1200 of the first bench round (38 live rows, ctx ~1270)" \
  SHAPE_b256="7B decode step 2 of the first bench round (256 live rows, ctx ~520)" \
  python tools/make_profiles.py r02 gpurun_out/r02_ncu_b38.ncu-rep:b38 gpurun_out/r02_ncu_b256.ncu-rep:b256 \
  --launches gpurun_out/r02_launches_bench.csv > gpurun_out/r02r_digest.txt 2>&1
cat gpurun_out/r02r_digest.txt | head -40
