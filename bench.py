"""Rollout benchmark: tail-batching RL steps on B200 through the C ABI.

One "step" = one RL step = one rollout round (SHORT or LONG, chosen by the
tail-batching planner, P:529-538 / S:271-279): submit -> prefill -> decode
steps on device -> collect.  Workload (N=1): BASELINE.json configs[1], the
Qwen2.5-7B-shaped random-init bf16 model, 32 prompts x G=8 per GPU (the
per-GPU share of "256 prompts x G=8 on DP=8"), short cap 8192, target
floor(n/1.25) (reading Z8), long rounds of P0 = target prompts from the FIFO;
synthetic prompts and a long-tail length trace.

Prints ONE JSON line (rank 0).  `--impl reference` times the oracle (plain
CPU fp64 decoder + integer scheduler) on a bounded sample of the same
workload on the host cores instead.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import configs, gen  # noqa: E402

ETA_NUM, ETA_DEN = 5, 4          # eta = 1.25
ETA = ETA_NUM / ETA_DEN
METRIC = "rollout retained tokens/s (whole job), plus s/RL-step short vs long"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2-7b", choices=list(configs.ROUNDS))
    ap.add_argument("--graph-steps", type=int, default=16)
    ap.add_argument("--profile-steps", type=int, default=1,
                    help="> 0: profile the first short and the first long warm-up round whole (per-kernel roofline)")
    ap.add_argument("--max-rounds-steps", type=int, default=0, help="debug: cap decode steps per round (invalid)")
    ap.add_argument("--out", default="")
    ap.add_argument("--stream-collect", type=int, default=0,
                    help="NEXT-3: rp_collect_ready every K decode steps during the round (0 = off)")
    ap.add_argument("--issue-cap", type=int, default=0,
                    help="--schedule issue: max active prompts per GPU (0 = ceil(P0 / n_gpus))")
    ap.add_argument("--schedule", default="tail", choices=["tail", "sync", "issue"],
                    help="tail batching (default) or the plain synchronous rollout baseline on the same stream")
    ap.add_argument("--long-tp", default="auto", choices=["auto", "1", "n", "profile"],
                    help="long-round tensor parallelism: auto = smallest TP whose worst-case KV fits (planner), "
                         "1 = data-parallel replicas, n = one TP group over all GPUs, profile = fastest "
                         "fitting size by the offline profile (tools/profile_grid.py)")
    return ap.parse_args()


# ------------------------------------------------------------------ workload
class Workload:
    """Deterministic prompt stream + length trace (the caller's dataset).  The
    tail-batching planner and the global long-prompt FIFO live in the library
    (rp_plan_round, rp_long_queue); `plan`/`commit` here are the plain
    synchronous baseline and the oracle-side bookkeeping of tools/tests."""

    def __init__(self, cfg_name, world, schedule="tail"):
        self.R = configs.ROUNDS[cfg_name]
        self.model = configs.model_config(self.R["model"])
        self.world = world
        self.n_submit = self.R["n_submit"] * world                       # weak scaling
        self.P0 = self.n_submit * ETA_DEN // ETA_NUM                      # floor(n / eta)
        self.G = self.R["G"]
        self.total = self.n_submit * 64
        self.prompts = gen.prompts(self.total, 0, self.model["eos_id"], self.R["prompt_len"], configs.PROMPT_SEED)
        tp = self.R["trace"]
        self.trace = gen.length_trace(self.total, self.G, tp["mu0"], tp["sigma_p"], tp["sigma_r"], tp["l_max"],
                                      configs.TRACE_SEED)
        from paper_2509_21009_b200.dp import GlobalQueue
        self.queue = GlobalQueue()            # oracle-side mirror (tools, tests); the bench uses the library's
        self.next_fresh = 0
        # "tail": the planner of S:271-279; "sync": plain synchronous rollout (the
        # veRL baseline): every RL step decodes P0 fresh prompts to completion
        self.schedule = schedule
        # "issue": tail batching with continuous issuance in the short rounds
        # (NEXT-4); prompts a round never issued return to the stream
        self.returned = []

    def plan(self):
        if self.schedule == "sync":
            ids = list(range(self.next_fresh, self.next_fresh + self.P0))
            return "long", ids, self.P0, self.R["long_cap"], self.trace[ids, 0, :]
        if len(self.queue) >= self.P0:
            ids = self.queue.ids[:self.P0]
            return "long", ids, self.P0, self.R["long_cap"], self.trace[ids, 1, :]
        ids = self.returned + list(range(self.next_fresh, self.next_fresh + self.n_submit - len(self.returned)))
        return "short", ids, self.P0, self.R["short_cap"], self.trace[ids, 0, :]

    def fresh(self, n):
        """The next n prompts of the stream: prompts a continuous-issuance
        round never issued come back first (NEXT-4)."""
        ids = self.returned[:n] + list(range(self.next_fresh, self.next_fresh + n - min(n, len(self.returned))))
        self.returned = self.returned[n:]
        self.next_fresh = max([self.next_fresh] + [i + 1 for i in ids])
        return ids

    def commit(self, kind, ids, accepted_ids, unissued=()):
        if self.schedule == "sync":
            self.next_fresh += len(ids)
            return
        if kind == "long":
            self.queue.pop(len(ids))
        else:
            self.next_fresh = max(self.next_fresh, max(ids) + 1)
            un = set(unissued)
            self.returned = [i for i in ids if i in un]
            self.queue.defer([i for i in ids if i not in un], accepted_ids)


# ------------------------------------------------------------------ clocks
class Clocks:
    def __init__(self, idx):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", "clocks_%d.csv" % os.getpid())
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(idx), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for k, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(k)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ ours
def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2509_21009_b200 import rp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # torch.distributed is host plumbing only (NCCL id broadcast, membership,
        # timing reductions); the data-path exchange is the library's own NCCL
        # communicator inside the CUDA graph (a second NCCL group in the same
        # process deadlocked at init on this image)
        dist.init_process_group("gloo")
    W = Workload(a.config, world, a.schedule)
    cfg, G = W.model, W.G
    # per-rank capacities
    n_loc = math.ceil(W.n_submit / world)
    lo, hi = W.R["prompt_len"]
    nccl_id = None
    if world > 1:
        obj = [rp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # Long-round parallelism (elastic TP; the static form of the
    # planner): the smallest TP size whose worst-case KV --
    # every sequence of a replica's share at prompt + cap tokens -- fits the
    # per-GPU pool without preemption.  TP=1 means the N GPUs run data-parallel
    # replicas of the long round (each decodes its slice of the P0 prompts).
    grid = json.load(open(TP_GRID)) if (a.long_tp == "profile" and os.path.exists(TP_GRID)) else None
    long_tp = plan_long_tp(a.long_tp, cfg, W, world, grid)
    # short rounds: data parallel over the N GPUs (prompts sharded by index)
    eng = rp.Engine(cfg, max_seqs=n_loc * G, max_prompts=n_loc, max_prompt_len=hi, max_prompt_tokens=n_loc * hi,
                    max_cap=max(W.R["short_cap"], W.R["long_cap"]), graph_steps=a.graph_steps, rank=rank,
                    world=world, nccl_id=nccl_id, sample_seed=configs.SAMPLE_SEED,
                    kv_fraction=0.85 if long_tp == 1 else 0.45)
    st_ev = eng.stream
    # long rounds (elastic TP): one TP=N group over the same GPUs,
    # holding only its weight shard; every rank decodes all P0 queued prompts
    eng_long = eng
    if long_tp > 1:
        obj = [rp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng_long = rp.Engine(cfg, max_seqs=W.P0 * G, max_prompts=W.P0, max_prompt_len=hi,
                             max_prompt_tokens=W.P0 * hi, max_cap=W.R["long_cap"], graph_steps=a.graph_steps,
                             tp=world, tp_rank=rank, nccl_id=obj[0], sample_seed=configs.SAMPLE_SEED,
                             kv_fraction=0.85, stream=st_ev)

    from paper_2509_21009_b200.dp import all_gather_ids as allgather_ids
    issue_cap = a.issue_cap or -(-W.P0 // world)
    W.issue_cap = issue_cap if W.schedule == "issue" else None

    def one_round(round_no, profile=False):
        """One RL step.  Tail batching: the library's planner (rp_plan_round)
        picks the round; a SHORT round takes ceil(eta * P0) fresh prompts of
        the stream, a LONG round pops P0 prompts off the library's global
        queue (submit with prompts == NULL; every DP rank pops the same)."""
        tr = W.trace
        if W.schedule == "sync":
            ids = W.fresh(W.P0)
            kind, e = "long", eng
            plist = [W.prompts[i] for i in ids]
            e.submit(plist, G, W.R["long_cap"], len(ids), long_round=True, trace=tr[ids, 0, :], round_id=round_no)
        else:
            kind, n = eng.plan(W.P0, ETA)
            if kind == "short":
                e = eng
                ids = W.fresh(n)
                plist = [W.prompts[i] for i in ids]
                if W.schedule == "issue":
                    e.issue_cap(issue_cap)
                e.submit(plist, G, W.R["short_cap"], W.P0, trace=tr[ids, 0, :], trace_retry=tr[ids, 1, :],
                         round_id=round_no)
            else:
                ids = eng.long_queue()[:n]
                plist = [W.prompts[i] for i in ids]
                if eng_long is eng:
                    e = eng
                    if W.schedule == "issue":
                        e.issue_cap(0)
                    e.submit(None, G, W.R["long_cap"], n, long_round=True, trace_mode=True, round_id=round_no)
                else:                       # TP context over the same GPUs: hand the queue head over
                    e = eng_long
                    e.submit(plist, G, W.R["long_cap"], n, long_round=True, trace=tr[ids, 1, :], round_id=round_no)
                    eng.long_queue_pop(n)
        h2d = sum(len(p["tokens"]) for p in plist) * 4 + len(plist) * G * 4 * (2 if kind == "short" else 1)
        if profile:
            e.debug_profile_arm(1 << 30)        # every decode step of this round, eagerly, events per launch
        streamed = 0
        if a.stream_collect > 0:
            # NEXT-3: stream the accepted prompts' responses every `stream_collect`
            # decode steps while the round runs (a reward stage would consume them)
            first = 0
            st = e.step(a.stream_collect)
            while not st.done:
                got, first = e.collect_ready(first)      # final: accepted before the round ended
                streamed += sum(r["len"] for r in got)
                st = e.step(a.stream_collect)
        else:
            st = e.run()
        prof = None
        hist = e.rows_histogram()
        if profile:
            prof = e.debug_profile_read()
            e.debug_profile_arm(-1)
            # bytes: each prompt's shared pages once per step (what HBM must deliver);
            # FLOPs: every row's full context
            prof.update(kind=kind, hist=hist.tolist(), kv_tokens=st.kv_tokens_unique,
                        kv_tokens_per_row=st.kv_tokens_read, tp=e.tp)
        res = e.collect()
        if W.schedule == "issue" and kind == "short":
            W.returned = allgather_ids(e.unissued()) + W.returned
        d2h = (sum(r["len"] for r in res) + streamed) * 4 + len(res) * 24
        retained = sum(r["len"] for r in res)
        decoded = st.decoded_tokens
        # algorithmic HBM bytes of this rank's decode steps (step 1 comes from the prefill)
        hbm = step_bytes(cfg, e.tp, max(0, st.t - 1), st.decoded_tokens, st.kv_tokens_unique)
        t_roof = round_t_roof(cfg, e.tp, hist, st.decoded_tokens, st.kv_tokens_unique)
        if e is not eng and rank != 0:
            # TP ranks decode the same tokens: count them once (on rank 0)
            decoded, retained, h2d, d2h = 0, 0, 0, 0
        info = dict(kind=kind, t_end=st.t, streamed=streamed, decoded=decoded, retained=retained, h2d=h2d,
                    d2h=d2h, accepted=st.accepted, underfilled=st.underfilled, tp=e.tp, hbm_bytes=hbm,
                    t_roof_s=t_roof)
        return info, prof

    # ---- warm-up.  The first SHORT and the first LONG warm-up round are
    # profiled whole (every decode step eager, CUDA events around every launch
    # on the engine stream): the per-kernel-class roofline covers the same
    # mix of live-batch sizes and contexts as the timed region.
    profs = []
    for r in range(a.warmup):
        kind_next = "long" if (W.schedule == "sync" or eng.plan(W.P0, ETA)[0] == "long") else "short"
        want = a.profile_steps > 0 and kind_next not in {p["kind"] for p in profs}
        _, prof = one_round(r, profile=want)
        if prof is not None:
            profs.append(prof)
    # ---- timed region
    clk = Clocks(local) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.launch_count() + (eng_long.launch_count() if eng_long is not eng else 0)
    w0 = time.perf_counter()
    e0.record(st_ev)
    rounds = []
    round_ms = []
    for r in range(a.steps):
        rs, re_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tr0 = time.perf_counter()
        rs.record(st_ev)
        info, _ = one_round(a.warmup + r)
        re_.record(st_ev)
        re_.synchronize()
        info["wall_s"] = time.perf_counter() - tr0
        info["dev_s"] = rs.elapsed_time(re_) / 1e3
        rounds.append(info)
    e1.record(st_ev)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    clocks = clk.stop() if clk else None
    dev_s = e0.elapsed_time(e1) / 1e3
    wall_s = w1 - w0
    launches = eng.launch_count() + (eng_long.launch_count() if eng_long is not eng else 0) - launches0
    # ---- reductions over ranks
    t = torch.tensor([dev_s, wall_s], dtype=torch.float64)
    tot = torch.tensor([sum(x["decoded"] for x in rounds), sum(x["retained"] for x in rounds),
                        sum(x["h2d"] for x in rounds), sum(x["d2h"] for x in rounds), launches,
                        sum(x["hbm_bytes"] for x in rounds)], dtype=torch.float64)
    t_roof_all = torch.tensor([sum(x["t_roof_s"] for x in rounds)], dtype=torch.float64)
    per_round = torch.tensor([x["dev_s"] for x in rounds], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(per_round, op=dist.ReduceOp.MAX)
        dist.all_reduce(t_roof_all, op=dist.ReduceOp.MAX)
    dev_s, wall_s = t.tolist()
    decoded, retained, h2d, d2h, launches_all, hbm_all = tot.tolist()
    per_round = per_round.tolist()
    def shutdown():
        if world > 1:
            dist.barrier()
        if eng_long is not eng:
            eng_long.close()
        eng.close()
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()

    if rank != 0:
        shutdown()
        return
    short = [s for s, x in zip(per_round, rounds) if x["kind"] == "short"]
    long_ = [s for s, x in zip(per_round, rounds) if x["kind"] == "long"]
    value = retained / dev_s
    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(1e3 * dev_s / a.steps, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp16",
        "data": "synthetic (random-init Qwen2.5-7B-shaped weights, seeded prompts, lognormal length trace)",
        "config": bench_config(W, "short rounds dp%d, long rounds %s" % (
            world, ("tp%d" % long_tp) if eng_long is not eng else ("dp%d (planner: TP=1 fits the worst-case KV)" % world if a.long_tp != "profile" else
                 "dp%d (planner: profile predicts DP replicas fastest among the fitting TP sizes)" % world)),
            a.graph_steps),
        "per_gpu_tokens_per_s": round(value / world, 1),
        "decoded_tokens_per_s": round(decoded / dev_s, 1),
        "decoded_per_gpu_tokens_per_s": round(decoded / dev_s / world, 1),
        "speculation_waste": round(decoded / max(1.0, retained), 3),
        "s_per_rl_step": {"short_mean": round(statistics.mean(short), 3) if short else None,
                          "long_mean": round(statistics.mean(long_), 3) if long_ else None,
                          "all_mean": round(dev_s / a.steps, 3)},
        "rounds": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in x.items()} for x in rounds],
        "e2e": {"value": round(retained / wall_s, 1), "unit": "tokens/s",
                "h2d_bytes_per_step": int(h2d / a.steps), "d2h_bytes_per_step": int(d2h / a.steps)},
        "gpu_launches": int(launches_all),
        "clocks": clocks,
    }
    if a.stream_collect:
        line["config"]["stream_collect_steps"] = a.stream_collect
        line["streamed_fraction"] = round(sum(x["streamed"] for x in rounds) / max(1, sum(x["retained"] for x in rounds)), 4)
    if profs:
        line["roofline"], line["kernel_profile"] = roofline(profs, cfg)
    peak_hbm = load_peaks()[0]
    line["round_roofline"] = {
        "t_roof_s": round(t_roof_all.item(), 3), "t_measured_s": round(dev_s, 3),
        "frac": round(t_roof_all.item() / dev_s, 4),
        "formula": "sum over decode steps t of max(W/BW, 2 P B_t / peak_tensor) + KV_t/BW + logits_t/BW "
                   "(SURVEY section 8(d)); B_t from the device histogram of live rows per step, "
                   "BW and peak_tensor (sustained) from MEASURED_PEAKS.json; max over ranks"}
    line["step_roofline"] = {
        "bound": "hbm", "unit": "GB/s", "achieved": round(hbm_all / dev_s / 1e9, 1), "peak": peak_hbm * world,
        "frac": round(hbm_all / dev_s / 1e9 / (peak_hbm * world), 4),
        "bytes_per_decode_step": round(hbm_all / max(1, sum(max(0, x["t_end"] - 1) for x in rounds)), 0),
        "scope": "whole timed rounds: every decode step streams all weights once, plus the KV context each "
                 "live row's attention reads and the logits write + sampler read (DESIGN.md section 7)"}
    if world == 1:
        line["cpu_baseline"] = cpu_baseline(W)
    emit(json.dumps(line))
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(line) + "\n")
    shutdown()


def bench_config(W, parallelism, graph_steps):
    """The workload description shared by both arms (BASELINE.json configs[1], per GPU)."""
    sched = {"tail": "tail batching (eta=1.25)",
             "sync": "plain synchronous rollout baseline: P0 fresh prompts per RL step decoded to completion",
             "issue": "tail batching (eta=1.25) with continuous issuance in the short rounds, at most %s prompts "
                      "active per GPU (NEXT-4)" % getattr(W, "issue_cap", None)}[W.schedule]
    return {"workload": "BASELINE configs[1]: Qwen2.5-7B-shaped, %d prompts x G=%d per GPU, short cap %d, "
                        "target floor(n/1.25), %s, trace mode" % (W.R["n_submit"], W.G, W.R["short_cap"], sched),
            "schedule": W.schedule,
            "global_prompts_per_short_round": W.n_submit, "P0": W.P0, "G": W.G,
            "short_cap": W.R["short_cap"], "long_cap": W.R["long_cap"], "parallelism": parallelism,
            "l2": "inputs larger than L2 (14 GB of weights streamed per decode step)", "graph_steps": graph_steps}


TP_GRID = os.path.join(ROOT, "profiles", "r01_tp_grid_7b.json")


def grid_step_ms(grid, tp, B, ctx):
    """Decode-step ms of the offline profile (tools/profile_grid.py) for TP
    size tp: the grid context nearest to ctx (log space), then linear in B
    between the bracketing grid batches (extrapolated past the ends), or
    None when the profile has no point of this TP size."""
    pts = [p for p in grid["points"] if p["tp"] == tp]
    if not pts:
        return None
    c = min({p["ctx"] for p in pts}, key=lambda c: abs(math.log(c / ctx)))
    row = sorted((p["B"], p["ms_per_step"]) for p in pts if p["ctx"] == c)
    if len(row) == 1:
        return row[0][1]
    k = next((i for i in range(1, len(row)) if row[i][0] >= B), len(row) - 1)
    (b0, m0), (b1, m1) = row[k - 1], row[k]
    return max(m0 + (m1 - m0) * (B - b0) / (b1 - b0), 0.0)


def plan_long_tp(choice, cfg, W, world, grid=None):
    """Long-round TP size: 1, the whole group, (auto) the smallest of {1,
    world} whose worst-case KV per GPU fits ~80% of the memory left after
    that TP size's weight shard, or (profile, A8/A9) among the sizes that fit,
    the one the offline profile predicts fastest per decode step for the
    long round's rows per replica at a representative context (mean prompt +
    a quarter of the long cap)."""
    can_tp = world > 1 and cfg["n_kv_heads"] % world == 0
    if choice == "1" or world == 1:
        return 1
    if choice == "n":
        return world if can_tp else 1
    import torch
    free, _ = torch.cuda.mem_get_info()
    hi = W.R["prompt_len"][1]
    per_tok = cfg["n_layers"] * cfg["n_kv_heads"] * cfg["head_dim"] * 2 * 2
    fits = []
    for t in ([1, world] if can_tp else [1]):
        prompts = -(-W.P0 // (world // t))
        need = prompts * W.G * (hi + W.R["long_cap"]) * per_tok / t
        # t = 1: one engine holds the full weights; t > 1: the DP engine's full
        # weights plus the TP shard
        full = weight_bytes(cfg, 1) + cfg["vocab"] * cfg["d_model"] * 2
        weights = full if t == 1 else full + weight_bytes(cfg, t)
        if need <= 0.8 * (free - weights):
            fits.append(t)
    if not fits:
        return world if can_tp else 1
    if choice == "profile" and grid is not None:
        ctx = sum(W.R["prompt_len"]) / 2 + W.R["long_cap"] / 4
        pred = {t: grid_step_ms(grid, t, -(-W.P0 // (world // t)) * W.G, ctx) for t in fits}
        pred = {t: v for t, v in pred.items() if v is not None}
        if pred:
            return min(pred, key=pred.get)
    return fits[0]


def weight_bytes(cfg, tp=1):
    """bf16 weight bytes one rank streams per decode step (all GEMMs + LM head shard)."""
    d, H, KV, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff", "vocab",
                                              "n_layers"))
    per_layer = ((H + 2 * KV) * hd * d + d * H * hd + 2 * F * d + d * F) * 2 // tp
    return L * per_layer + V * d * 2 // tp


def step_bytes(cfg, tp, steps, rows, kv_tokens):
    """Algorithmic HBM bytes of `steps` decode steps over `rows` decoded rows
    reading `kv_tokens` context tokens (per layer and KV head) in total:
    weights once per step + K and V of every context token in every layer and
    local KV head + fp32 logits written by the LM head and read by the sampler."""
    L, KV, hd, V = cfg["n_layers"], cfg["n_kv_heads"] // tp, cfg["head_dim"], cfg["vocab"] // tp
    return steps * weight_bytes(cfg, tp) + kv_tokens * L * KV * hd * 2 * 2 + rows * V * 4 * 2


def round_t_roof(cfg, tp, hist, rows, kv_tokens):
    """Roofline time of one round's decode steps on one rank:
    every step streams the weight shard or runs its GEMM FLOPs at the tensor
    peak, whichever is longer, plus the KV reads and the logits traffic."""
    bw, _, tf_sus, _ = load_peaks()
    w = weight_bytes(cfg, tp)
    p = w / 2                                           # parameters streamed per step (16-bit)
    L, KV, hd, V = cfg["n_layers"], cfg["n_kv_heads"] // tp, cfg["head_dim"], cfg["vocab"] // tp
    t = 0.0
    for r, steps in enumerate(hist):
        if steps:
            t += steps * max(w / (bw * 1e9), 2.0 * p * r / (tf_sus * 1e12))
    t += kv_tokens * L * KV * hd * 2 * 2 / (bw * 1e9) + rows * V * 4 * 2 / (bw * 1e9)
    return t


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    (and the capture's live batch) from the newest committed ncu --set full
    summary, profiles/rNN_ncu_traffic.json, written by tools/make_profiles.py
    from a capture of this bench command's decode steps."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_traffic.json")))
    if not files:
        return None, None
    d = json.load(open(files[-1]))
    best = None
    for tag, ent in d.items():
        if kernel in ent.get("dram_bytes_per_launch", {}):
            b = int(ent["dram_bytes_per_launch"][kernel])
            if best is None or ent.get("rows", 0) < best[2]:      # the smallest captured batch: the common case
                best = (b, "%s [%s] %s" % (os.path.relpath(files[-1], ROOT), tag, ent.get("shape", "")),
                        ent.get("rows", 0))
    return (best[0], best[1]) if best else (None, None)


def launch_work(cfg, tp, cls, B):
    """Algorithmic (bytes, FLOPs) of ONE launch of kernel class `cls` at B live
    rows: a GEMM streams its weights once and reads /
    writes its activations (M*K*2 + B*K*2 + B*M*out, + B*M*4 for residual
    read-modify-write), FLOPs 2*B*M*K; the sampler reads the fp32 logits;
    RMSNorm / embedding read and write one row each.  Attention is counted
    from the context separately (attn_work)."""
    d, H, KV, hd, F, V = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ff", "vocab"))
    H, KV, F, V = H // tp, KV // tp, F // tp, V // tp
    qkvw = (H + 2 * KV) * hd
    g = {"gemm_qkv": (qkvw, d, 2, 0),          # fused RoPE epilogue: q -> fp16, k/v -> their KV page (fp16)
         "gemm_o": (d, H * hd, 4, 4), "gemm_gu": (2 * F, d, 1, 0), "gemm_down": (d, F, 4, 4),
         "gemm_lm": (V, d, 4, 0)}
    if cls in g:
        M, K, ob, rd = g[cls]
        return M * K * 2 + B * K * 2 + B * M * ob + B * M * rd, 2.0 * B * M * K
    if cls == "sampler":
        return B * V * 4, 0.0
    if cls in ("rmsnorm", "embed"):
        return B * d * 6, 0.0
    return 0, 0.0


LAUNCHES_PER_STEP = {"gemm_qkv": "L", "gemm_o": "L", "gemm_gu": "L", "gemm_down": "L", "attention": "L",
                     "gemm_lm": 1, "sampler": 1, "embed": 1, "ctl": 1}


def roofline(profs, cfg):
    """Per-kernel-class roofline over whole profiled rounds (the first short
    and the first long round of the run, every decode step): algorithmic
    bytes and FLOPs summed over every launch at its live batch (device
    histogram of rows per step) and the attention context (bytes: each
    prompt's shared pages once per step, kv_tokens_unique; FLOPs: every row's
    context, kv_tokens_read), divided by the class's summed CUDA-event time.  The
    `roofline` object is the dominant class (largest share of the profiled
    time): bound = hbm if its launches' byte time exceeds their FLOP time at
    the peaks, achieved = algorithmic bytes (FLOPs) / time."""
    hbm, tf_burst, tf_sus, src = load_peaks()
    L = cfg["n_layers"]
    tot_ms, tot_cnt, by, fl, t_roof, steps, rows_sum, ctx_sum = {}, {}, {}, {}, {}, 0, 0, 0
    for p in profs:
        tp = p.get("tp", 1)
        hd, KV, H = cfg["head_dim"], cfg["n_kv_heads"] // tp, cfg["n_heads"] // tp
        hist = p["hist"]
        steps += sum(hist)
        rows_sum += sum(B * n for B, n in enumerate(hist))
        kv_rows = p.get("kv_tokens_per_row", p["kv_tokens"])
        ctx_sum += kv_rows
        for k, v in p["ms"].items():
            tot_ms[k] = tot_ms.get(k, 0.0) + v
            tot_cnt[k] = tot_cnt.get(k, 0) + p["launches"][k]
        for cls in ("gemm_qkv", "gemm_o", "gemm_gu", "gemm_down", "gemm_lm", "sampler", "embed"):
            nl = L if LAUNCHES_PER_STEP[cls] == "L" else 1
            for B, n in enumerate(hist):
                if n:
                    b, f = launch_work(cfg, tp, cls, B)
                    by[cls] = by.get(cls, 0) + n * nl * b
                    fl[cls] = fl.get(cls, 0) + n * nl * f
                    t_roof[cls] = t_roof.get(cls, 0) + n * nl * max(b / (hbm * 1e9), f / (tf_sus * 1e12))
        ab = p["kv_tokens"] * L * KV * hd * 2 * 2 + sum(B * n for B, n in enumerate(hist)) * L * H * hd * 2 * 2
        by["attention"] = by.get("attention", 0) + ab
        fl["attention"] = fl.get("attention", 0) + 4.0 * kv_rows * L * H * hd
        t_roof["attention"] = t_roof.get("attention", 0) + ab / (hbm * 1e9)
    total = sum(tot_ms.values())
    detail = {}
    for k, v in sorted(tot_ms.items(), key=lambda kv: -kv[1]):
        if not tot_cnt.get(k):
            continue
        dd = {"ms_per_step": round(v / max(1, steps), 4), "share": round(v / total, 4),
              "launches_per_step": round(tot_cnt[k] / max(1, steps), 2)}
        if k in by:
            t = v / 1e3
            dd["hbm_gbs"] = round(by[k] / t / 1e9, 1)
            if fl.get(k):
                dd["tflops"] = round(fl[k] / t / 1e12, 1)
            dd["roofline_frac"] = round(t_roof[k] / t, 4)
        detail[k] = dd
    dom = max(tot_ms, key=lambda k: tot_ms[k])
    t = tot_ms[dom] / 1e3
    tensor = fl.get(dom, 0) / (tf_sus * 1e12) > by.get(dom, 0) / (hbm * 1e9)
    if tensor:
        ach = fl[dom] / t / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 1), "peak": tf_sus, "unit": "TFLOP/s",
                "frac": round(ach / tf_sus, 4)}
    else:
        ach = by.get(dom, 0) / t / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4)}
    traffic, traffic_src = ncu_traffic(dom)
    roof.update({"kernel": dom, "traffic": traffic, "traffic_source": traffic_src,
                 "peak_source": src + (" sustained cuBLAS bf16 dense (fp16 runs at the same tensor rate)"
                                       if tensor else " HBM copy bandwidth"),
                 "share_of_profiled_time": round(tot_ms[dom] / total, 4),
                 "roofline_time_frac": round(t_roof.get(dom, 0) / t, 4),
                 "launches": tot_cnt[dom], "mean_live_rows": round(rows_sum / max(1, steps), 1),
                 "mean_ctx_per_row": round(ctx_sum / max(1, rows_sum), 1),
                 "measured": "CUDA events around every launch of every decode step of whole rounds (%s; %d "
                             "steps), step enqueued behind a host gate so no host gap is timed" % (
                                 " + ".join("%s round of %d steps" % (p["kind"], sum(p["hist"])) for p in profs),
                                 steps)})
    return roof, detail


# ------------------------------------------------------------------ oracle (CPU)
class OracleSample:
    """The oracle as it stands, on the bounded sample of BASELINE.md section 4:
    B = 8 sequences (one prompt's G = 8 responses) at context ~512, decoded
    one token at a time with the fp64 KVDecoder, on the Qwen2.5-7B shape cut
    to ONE full-width layer + the full 152 064-row LM head.  Setup (weight
    formula, widening to fp64, the shared 512-token prefill) is not timed; a
    timed step feeds one token to each of the 8 sequences.  Per-token time is
    extrapolated to the full depth as t_layer * n_layers + t_lm."""

    def __init__(self, W, B=8, ctx=512):
        from oracle import decoder, weights
        self.decoder = decoder
        cfg1 = dict(W.model, n_layers=1)
        self.L = W.model["n_layers"]
        w = weights.Weights(cfg1, configs.WEIGHT_SEED, use_c=True)
        w.layer(0)
        for k in list(w._c):
            w._c[k] = np.asarray(w._c[k], np.float64)
        self.lm = np.asarray(w.lm_head(), np.float64)
        self.w = w
        prompt = np.resize(W.prompts[0]["tokens"], ctx)            # ~512 prompt tokens
        root = decoder.KVDecoder(w)
        root.step(prompt, head=False)
        self.decs = [root.fork() for _ in range(B)]
        self.tok = [int(prompt[-1 - b]) for b in range(B)]
        self.B, self.ctx = B, ctx
        self.t_layer = self.t_lm = 0.0
        self.n = 0

    def step(self):
        """One decode step of the B sequences; returns seconds per token
        extrapolated to the full depth."""
        tl = tm = 0.0
        for b, d in enumerate(self.decs):
            t0 = time.perf_counter()
            h = d.step([self.tok[b]], head=False)
            t1 = time.perf_counter()
            z = h @ self.lm.T
            t2 = time.perf_counter()
            self.tok[b] = int(np.argmax(z[0]))
            tl += t1 - t0
            tm += t2 - t1
        self.t_layer += tl
        self.t_lm += tm
        self.n += self.B
        return (tl * self.L + tm) / self.B

    def per_token(self):
        return (self.t_layer * self.L + self.t_lm) / max(1, self.n)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return {i.get("internal_api", "?"): i.get("num_threads") for i in threadpool_info()}
    except Exception:
        return {}


def sample_text(o):
    return ("fp64 NumPy oracle (KVDecoder), Qwen2.5-7B shape cut to 1 full-width layer + the full LM head, "
            "B=%d sequences (one prompt's G=8 responses forked from a shared %d-token prefill), %d decode "
            "tokens timed; per-token time extrapolated to %d layers (t_layer=%.3fs, t_lm=%.3fs per token); "
            "BLAS threads %s" % (o.B, o.ctx, o.n, o.L, o.t_layer / max(1, o.n), o.t_lm / max(1, o.n),
                                 blas_threads()))


def cpu_baseline(W, steps=8):
    o = OracleSample(W)
    for _ in range(steps):
        o.step()
    return {"value": round(1.0 / o.per_token(), 4), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": sample_text(o)}


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = Workload(a.config, 1)
    o = OracleSample(W)
    for _ in range(a.warmup):
        o.step()
    o.t_layer = o.t_lm = 0.0
    o.n = 0
    t0 = time.perf_counter()
    for _ in range(a.steps):
        o.step()
    wall = time.perf_counter() - t0
    value = 1.0 / o.per_token()
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * wall / a.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (random-init Qwen2.5-7B-shaped weights, seeded prompts)",
            "config": bench_config(W, "fp64 NumPy oracle on the host cores, rank 0 only (bounded sample)", 0),
            "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": "per step: one decode token for each of the 8 sequences; " + sample_text(o)},
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(json.dumps(line))


_STDOUT_FD = None


def emit(text):
    """Write the result line to the real stdout (fd 1 is redirected to stderr
    while the libraries run, so NCCL/CUDA banners cannot pollute it)."""
    os.write(_STDOUT_FD if _STDOUT_FD is not None else 1, (text + "\n").encode())


def main():
    global _STDOUT_FD
    _STDOUT_FD = os.dup(1)
    sys.stdout.flush()
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
