#!/bin/bash
# final round-2 evidence on one B200: smoke, the whole single-GPU suite, ncu launch list + full-set digests
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_smoke.log
tail -2 gpurun_out/r02f_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_tests.log
tail -3 gpurun_out/r02f_tests.log
bash tools/gpu_r02r.sh > gpurun_out/r02f_ncu.txt 2>&1
tail -12 gpurun_out/r02f_ncu.txt
