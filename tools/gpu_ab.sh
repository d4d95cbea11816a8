mkdir -p gpurun_out
for CW in 6 3 2; do
RP_ATTN_CW=$CW timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "decode or long_context or sampled" 2>&1 | tail -1
RP_ATTN_CW=$CW timeout -s KILL 200 python tools/step_profile.py 256 64 16 2>&1 | grep -A1 "graph_step" | grep -o "B~[0-9]*\|graph_step_ms=[0-9.]*\|attention=[0-9.]*" | paste -sd' ' | sed "s/^/CW=$CW /"
done
