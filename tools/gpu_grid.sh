# offline decode profile for the planner: TP 1, 2, 4 on one 4-GPU box (gpurun --gpus 4)
mkdir -p gpurun_out
timeout -s KILL 900 python tools/profile_grid.py --out gpurun_out/grid_tp1.json > gpurun_out/grid_tp1.log 2>&1; echo tp1 rc=$?
timeout -s KILL 900 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/profile_grid.py --out gpurun_out/grid_tp2.json > gpurun_out/grid_tp2.log 2>&1; echo tp2 rc=$?
timeout -s KILL 900 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/profile_grid.py --out gpurun_out/grid_tp4.json > gpurun_out/grid_tp4.log 2>&1; echo tp4 rc=$?
grep -h '"tp"' gpurun_out/grid_tp*.log | head -60
for f in gpurun_out/grid_tp*.log; do tail -n 3 $f; done
