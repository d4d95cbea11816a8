mkdir -p gpurun_out
# bash tools/gpu_bench_full.sh
timeout -s KILL 200 python tools/ncu_decode.py 0 1 > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b256.csv python tools/ncu_decode.py 0 1 > gpurun_out/ncu_l1.log 2>&1; echo launches rc=$?
timeout -s KILL 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm_tcgen05|attn_kernel" -c 6 -o gpurun_out/r01c_full_b256 -f python tools/ncu_decode.py 0 1 > gpurun_out/ncu_f1.log 2>&1; echo full256 rc=$?
timeout -s KILL 200 python tools/ncu_small_b.py 1 > gpurun_out/plain2.log 2>&1 && \
timeout -s KILL 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm_tcgen05|attn_kernel" -c 6 -o gpurun_out/r01c_full_b16 -f python tools/ncu_small_b.py 1 > gpurun_out/ncu_f2.log 2>&1; echo full16 rc=$?
timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b16.csv python tools/ncu_small_b.py 1 > gpurun_out/ncu_l2.log 2>&1; echo launches16 rc=$?
ls gpurun_out/*.ncu-rep gpurun_out/launches_*.csv
