"""The rollout GPU set shrinks mid-round (NEXT-3; reading
Z27) on real GPUs: run under torchrun with 2 GPUs (gpurun --gpus 2):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/test_gpu_migrate_nccl.py
A DP=2 round (NCCL cutoff exchange inside the decode graphs) is stepped to
step ~60 on both GPUs; each rank exports its state, rank 0 gathers them,
re-shards them to one rank (rp_round_reshard), frees nothing on GPU 1 but its
engine, and finishes the round alone on GPU 0 after recomputing the KV of
the responses that lived on GPU 1.  The schedule after the cut, the
acceptance order, the lengths and the tokens (gap rule) must be the
single-rank oracle's."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from oracle import decoder, sampler, sched, weights
    from paper_2509_21009_b200 import rp
    from synth import configs, gen
    world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [rp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = configs.model_config("tiny")
    n, G, cap, target, rid = 12, 3, 250, 9, 6
    ps = gen.prompts(n, 0, cfg["eos_id"], (5, 100), 91)
    L = np.random.default_rng(55).integers(20, 300, size=(n, G)).astype(np.int64)
    kw = dict(max_seqs=64, max_prompts=16, max_prompt_len=128, max_prompt_tokens=1024, max_cap=512,
              kv_pool_bytes=64 << 20, graph_steps=4, sample_seed=configs.SAMPLE_SEED)
    eng = rp.Engine(cfg, rank=rank, world=world, nccl_id=obj[0], **kw)
    eng.submit(ps, G, cap, target, trace=L, round_id=rid)
    st = eng.step(60)
    state = eng.export_round()
    eng.close()
    states = [None] * world
    dist.all_gather_object(states, (st.t, state))
    if rank == 0:
        cut = states[0][0]
        ok = all(s[0] == cut for s in states)
        new = rp.reshard_round_states([s[1] for s in states], n, 1)
        e1 = rp.Engine(cfg, **kw)
        ref = sched.closed_form(L, cap, target, sched.SHORT, with_steps=True)
        e1.debug_trace_enable(ref.t_end + 8)
        e1.import_round(new[0], ps, G, cap, target, trace=L, round_id=rid)
        st1 = e1.run()
        got = e1.debug_trace(ref.t_end + 8, start=cut + 1)
        res = e1.collect()
        e1.close()
        ok = ok and st1.t == ref.t_end and st1.accepted == len(ref.accepted) and len(got) == ref.t_end - cut
        for x in got:
            want = ref.steps[x["t"] - 1]
            ok = ok and np.array_equal(x["live"], want["live"]) and x["accepted"] == want["accepted"]
        order = list(dict.fromkeys(r["prompt_id"] - ps[0]["prompt_id"] for r in res))
        ok = ok and order == list(ref.accepted)
        w = weights.Weights(cfg, configs.WEIGHT_SEED)
        checked = mism = bad = 0
        for r in res:
            i = r["prompt_id"] - ps[0]["prompt_id"]
            ok = ok and r["len"] == L[i, r["j"]]
            seq = np.concatenate([ps[i]["tokens"], r["tokens"]])
            lg = decoder.logits(w, seq[:-1], rows=np.arange(len(ps[i]["tokens"]) - 1, len(seq) - 1))
            for t in range(1, r["len"] + 1):
                tok, gap = sampler.sample(lg[t - 1], t, r["prompt_id"] * G + r["j"], rid, configs.SAMPLE_SEED,
                                          eos_id=cfg["eos_id"], trace_len=L[i, r["j"]])
                checked += 1
                if tok != r["tokens"][t - 1]:
                    mism += 1
                    bad += gap > 1e-2
        ok = ok and bad == 0 and checked > 500 and mism <= checked // 50
        print("migrate DP=2 -> 1 at step %d: t_end %d/%d accepted %d/%d tokens %d (%d in-gap) ok=%s" % (
            cut, st1.t, ref.t_end, st1.accepted, len(ref.accepted), checked, mism, ok), flush=True)
        if ok:
            print("MIGRATE NCCL PASS", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
