timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout -s KILL 200 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tests/test_gpu_tp.py 2>&1 | grep -E "rank|PARITY|Error|error|watchdog" | head -20
timeout -s KILL 200 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tests/test_gpu_dp.py 2>&1 | grep -E "rank|PARITY|Error|error|watchdog" | head -20
