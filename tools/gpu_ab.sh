mkdir -p gpurun_out
for i in 1 2; do
timeout -s KILL 200 python tools/step_profile.py 256 192 128 2>&1 | grep -A1 "graph_step"
RP_GEMM_NO_PAIR=1 timeout -s KILL 200 python tools/step_profile.py 256 192 128 2>&1 | grep -A1 "graph_step"
done
