mkdir -p gpurun_out
timeout -s KILL 300 python tools/ncu_step.py --steps 2 > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -s 113 -c 5 -o gpurun_out/prof_gemm -f python tools/ncu_step.py --steps 1 > gpurun_out/ncu_gemm.log 2>&1
echo rc=$?
tail -5 gpurun_out/ncu_gemm.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 28 -c 2 -o gpurun_out/prof_attn -f python tools/ncu_step.py --steps 1 > gpurun_out/ncu_attn.log 2>&1
echo rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_step.py --steps 2 > gpurun_out/ncu_launch.log 2>&1
echo rc=$?
ls -la gpurun_out
