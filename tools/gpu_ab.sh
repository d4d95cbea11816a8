# A/B: folded RMSNorm vs the RMSNorm kernel, graph step times at several live-batch sizes
mkdir -p gpurun_out
for i in 1 2; do
timeout -s KILL 200 python tools/step_profile.py 256 128 64 16 2>&1 | grep -A1 "graph_step"
RP_NO_FOLD=1 timeout -s KILL 200 python tools/step_profile.py 256 128 64 16 2>&1 | grep -A1 "graph_step"
done
