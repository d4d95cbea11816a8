nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
for v in a b c a b c; do cp abtest/$v.so paper_2509_21009_b200/librollpacker.so; echo "== $v"; timeout -s KILL 200 python tools/gemm_bench.py lm gu 2>&1 | grep -E "auto" | grep -E "N= 16|N=256"; done
