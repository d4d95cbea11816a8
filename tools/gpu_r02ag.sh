#!/bin/bash
# migration cost of a 7B round (export / import with KV recompute)
cd $GRAFT_REPO_ROOT
timeout 1500 python tools/migrate_bench.py --t 200 600 > gpurun_out/r02ag_migrate.jsonl 2> gpurun_out/r02ag_migrate.err
cat gpurun_out/r02ag_migrate.jsonl; tail -3 gpurun_out/r02ag_migrate.err
