mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
timeout -s KILL 200 python tools/step_profile.py 256 64 16 2>&1 | grep "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*" | paste -sd' '
RP_NO_FUSED_SAMPLER=1 timeout -s KILL 200 python tools/step_profile.py 256 64 16 2>&1 | grep "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*" | paste -sd' '
done
