mkdir -p gpurun_out
for U in 0 18 9 74; do echo "U=$U"; RP_ATTN_UNITS=$U timeout -s KILL 200 python tools/step_profile.py 256 64 16 2>&1 | grep -A1 "graph_step" | grep -o "graph_step_ms=[0-9.]*\|attention=[0-9.]*"; done
