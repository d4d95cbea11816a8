# A/B of the cooperative split-K threshold (RP_COOP_MIN): graph step ms at mid batches of the bench short round
mkdir -p gpurun_out
RP_COOP_MIN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm or logits" 2>&1 | tail -2
M="128 100 90 84 78 72 64 56 48 40 32 16"
for rep in 1 2; do
for c in 96 48 24; do
  echo "== coop_min=$c rep=$rep"
  RP_COOP_MIN=$c timeout -s KILL 600 python tools/step_profile.py $M 2>&1 | grep -o "B~[0-9]* rows/step=[0-9.]* ctx/row=[0-9]* eager_step_ms=[0-9.]* graph_step_ms=[0-9.]*"
done
done
