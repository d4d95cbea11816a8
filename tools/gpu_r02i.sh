#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in lo nolo; do
  if [ $v = nolo ]; then export RP_ACT_LO=0; else unset RP_ACT_LO; fi
  timeout 900 ncu --set full --clock-control none -k regex:gemm_tcgen05 --launch-skip 2000 --launch-count 4 \
    -o gpurun_out/r02i_$v -f python tools/step_ab.py --tag $v --batches 16 > gpurun_out/r02i_$v.log 2>&1
  ncu -i gpurun_out/r02i_$v.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/r02i_$v.csv 2>&1
done
cat gpurun_out/r02i_lo.csv gpurun_out/r02i_nolo.csv | cut -c1-400
