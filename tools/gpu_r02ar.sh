#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ar_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02ar_smoke.log
tail -2 gpurun_out/r02ar_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r02ar_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ar_tests.log
tail -3 gpurun_out/r02ar_tests.log
python -c "
import json
"
