# end-of-round evidence on one GPU: smoke, the default bench line, the streaming-collect bench line,
# and ncu launch lists of one decode step at 256 and 16 live rows
mkdir -p gpurun_out
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout -s KILL 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
timeout -s KILL 1500 python bench.py --stream-collect 64 --profile-steps 0 > gpurun_out/bench_stream.json 2> gpurun_out/bench_stream.err; echo stream rc=$?
timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b256.csv python tools/ncu_decode.py 0 1 > gpurun_out/ncu_l1.log 2>&1; echo launches256 rc=$?
timeout -s KILL 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b16.csv python tools/ncu_small_b.py 1 > gpurun_out/ncu_l2.log 2>&1; echo launches16 rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_final.json", "gpurun_out/bench_stream.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "s_per_rl_step", "e2e", "gpu_launches", "clocks",
                                     "streamed_fraction")})
    print(" roofline", d.get("roofline"), "\n round_roofline", d.get("round_roofline", {}).get("frac"))
PY
tail -n 2 gpurun_out/smoke.log
