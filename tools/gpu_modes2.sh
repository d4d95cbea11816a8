# the new bench modes at N=2: continuous issuance and the profile-driven long-round TP choice
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout -s KILL 1200 $R --master-port 29701 bench.py --gpus 2 --schedule issue --steps 4 --profile-steps 0 > gpurun_out/issue_n2.json 2> gpurun_out/issue_n2.err; echo issue rc=$?
timeout -s KILL 1200 $R --master-port 29702 bench.py --gpus 2 --long-tp profile --steps 4 --profile-steps 0 > gpurun_out/ltp_profile_n2.json 2> gpurun_out/ltp_profile_n2.err; echo profile rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/issue_n2.json", "gpurun_out/ltp_profile_n2.json"):
    try:
        d = json.load(open(f))
        print(f, d["value"], d["s_per_rl_step"], d["config"]["parallelism"], [(r["kind"], r.get("unissued")) for r in d["rounds"]])
    except Exception as e:
        print(f, "unreadable", e)
PY
