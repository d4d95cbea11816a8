# A/B of the k-wave attention split budget (RP_ATTN_WAVES=1, default) vs the one-wave floor (=0):
# graph step ms at several live batches of the first bench short round, alternating twice
mkdir -p gpurun_out
M="256 192 128 96 64 48 40 32 24 16"
for rep in 1 2; do
for w in 0 1; do
  echo "== waves=$w rep=$rep"
  RP_ATTN_WAVES=$w timeout -s KILL 600 python tools/step_profile.py $M 2>&1 | grep -o "B~[0-9]* rows/step=[0-9.]* ctx/row=[0-9]* eager_step_ms=[0-9.]* graph_step_ms=[0-9.]*\|attention=[0-9.]*"
done
done
