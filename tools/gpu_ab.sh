mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do
timeout -s KILL 200 python tools/step_profile.py 256 192 128 16 2>&1 | grep -A1 "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*\|gemm_gu=[0-9.]*\|gemm_qkv=[0-9.]*\|rmsnorm=[0-9.]*" | paste -sd' '
RP_NO_FOLD=1 timeout -s KILL 200 python tools/step_profile.py 256 192 128 16 2>&1 | grep -A1 "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*\|gemm_gu=[0-9.]*\|gemm_qkv=[0-9.]*\|rmsnorm=[0-9.]*" | paste -sd' '
done
