mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 200 python tools/gemm_shapes.py 37888,3584,256 37888,3584,136 37888,3584,16 152064,3584,16 2>&1 | grep "splits=1"
RP_GEMM_NO_PAIR=1 timeout -s KILL 200 python tools/gemm_shapes.py 37888,3584,256 37888,3584,136 37888,3584,16 152064,3584,16 2>&1 | grep "splits=1"
for i in 1 2; do
timeout -s KILL 200 python tools/step_profile.py 256 128 64 16 2>&1 | grep -A1 "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*\|gemm_gu=[0-9.]*\|gemm_lm=[0-9.]*" | paste -sd' '
RP_GEMM_NO_PAIR=1 timeout -s KILL 200 python tools/step_profile.py 256 128 64 16 2>&1 | grep -A1 "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*\|gemm_gu=[0-9.]*\|gemm_lm=[0-9.]*" | paste -sd' '
done
