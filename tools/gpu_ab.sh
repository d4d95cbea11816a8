# A/B of the small-footprint GEMM (co-resident PDL prefetch) vs the 192 KB ring
set -x
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout -s KILL 200 python tools/step_profile.py 256 128 64 48 32 16 2>&1 | grep "graph_step" 
RP_GEMM_BIGRING=1 timeout -s KILL 200 python tools/step_profile.py 256 128 64 48 32 16 2>&1 | grep "graph_step"
