"""Turn ncu reports and launch lists from gpurun_out/ into the committed
summaries under profiles/ (named per round), and the per-kernel DRAM-traffic
table bench.py reads for roofline.traffic.

  python tools/make_profiles.py r01 gpurun_out/prof_gemm.ncu-rep:gemm_b256 \
         gpurun_out/prof_attn.ncu-rep:attn_b256 --launches gpurun_out/launches.csv
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_inst_executed_op_utcmma.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]].split("(")[0]}
        for key in KEYS:
            for h in hdr:
                if h.endswith(key):
                    v, u = d[idx[h]], units[idx[h]]
                    try:
                        val = float(v.replace(",", ""))
                        rec[key] = val * SCALE.get(u, 1.0) if u in SCALE else val
                        rec[key + ".unit"] = "SI" if u in SCALE else u
                    except ValueError:
                        rec[key] = v
                    break
        res.append(rec)
    return res


def launches(path):
    by = defaultdict(list)
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        name = r.get("Kernel Name", "").split("(")[0]
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            by[name].append(v * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3}.get(unit, 1e-9))
    tot = sum(sum(v) for v in by.values())
    return {k: {"launches": len(v), "total_s": sum(v), "share": sum(v) / tot if tot else 0.0,
                "mean_us": 1e6 * sum(v) / len(v)} for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1]))}


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    lfile = None
    if "--launches" in args:
        i = args.index("--launches")
        lfile = args[i + 1]
        args = args[:i] + args[i + 2:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary = {"round": tag, "reports": {}}
    for spec in args:
        path, label = spec.split(":")
        summary["reports"][label] = raw(path)
    if lfile:
        summary["launch_list"] = launches(lfile)
    out = os.path.join(ROOT, "profiles", "%s_ncu_summary.json" % tag)
    json.dump(summary, open(out, "w"), indent=1)
    # human-readable digest
    lines = ["# ncu digest %s (cold-cache, serialised replays: compare shares, not absolutes)" % tag]
    for label, recs in summary["reports"].items():
        lines.append("\n## %s" % label)
        for r in recs:
            t = r.get("gpu__time_duration.sum", 0)
            rd, wr = r.get("dram__bytes_read.sum", 0), r.get("dram__bytes_write.sum", 0)
            lines.append("%-28s %8.1f us  DRAM %7.1f MB (%5.1f%% of peak)  SM %5.1f%%  tcgen05 pipe %5.1f%%  "
                         "UTCMMA %8s  issue %5.1f%%  regs %s  grid %s" % (
                r["kernel"][:28], t * 1e6, (rd + wr) / 1e6,
                r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
                r.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0),
                r.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 0) or 0,
                r.get("smsp__sass_inst_executed_op_utcmma.sum", "?"),
                r.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
                r.get("launch__registers_per_thread", "?"), r.get("launch__grid_size", "?")))
    if lfile:
        lines.append("\n## launch list (%s)" % os.path.basename(lfile))
        for k, v in list(summary["launch_list"].items())[:20]:
            lines.append("%-40s %6d launches  %8.1f us mean  share %5.1f%%" % (k[:40], v["launches"], v["mean_us"],
                                                                             100 * v["share"]))
    open(os.path.join(ROOT, "profiles", "%s_ncu_digest.txt" % tag), "w").write("\n".join(lines) + "\n")
    # per-kernel DRAM traffic per launch (bench.py roofline.traffic): the
    # captures hold the first six GEMM/attention launches of one decode step
    order = ["gemm_qkv", "attention", "gemm_o", "gemm_gu", "gemm_down", "gemm_qkv_next_layer"]
    traffic = {}
    for label, recs in summary["reports"].items():
        shape = os.environ.get("SHAPE_" + label, label)
        traffic["%s_%s" % (tag, label)] = {
            "shape": shape, "rows": int(os.environ.get("ROWS_" + label, "0")),
            "source": "profiles/%s_ncu_summary.json (ncu --set full, one decode step)" % tag,
            "dram_bytes_per_launch": {k: r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
                                      for k, r in zip(order, recs)},
            "ncu_duration_us": {k: 1e6 * r.get("gpu__time_duration.sum", 0) for k, r in zip(order, recs)}}
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "%s_ncu_traffic.json" % tag), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
