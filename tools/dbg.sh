timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 200 python tools/ncu_step.py --skip 3000 --steps 1 --graph-steps 16 > gpurun_out/dbg.log 2>&1; echo "rc=$?"
grep -a -E "stuck|watchdog|Error" gpurun_out/dbg.log | head; tail -2 gpurun_out/dbg.log
