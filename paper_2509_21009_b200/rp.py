"""Thin ctypes binding of librollpacker.so (include/rollpacker.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  PyTorch provides device memory (weights, KV pool, workspace) and
the stream.  There is no CPU fallback: if the library is missing, importing
this module raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RP_LIB: load another build of the same ABI (A/B measurements of two builds in one box)
LIB_PATH = os.environ.get("RP_LIB") or os.path.join(_HERE, "librollpacker.so")

RP_OK, RP_EINVAL, RP_EBUSY, RP_ESTATE, RP_ENOMEM_KV, RP_ECUDA, RP_ENCCL, RP_ENOSPC = 0, -1, -2, -3, -4, -5, -6, -7
RP_SHORT, RP_LONG, RP_TRACE, RP_PREEMPT = 0, 1, 4, 8
RP_FINISH_EOS, RP_FINISH_CAP = 1, 2
RP_IPC_HANDLE_BYTES = 64


class ModelDesc(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("d_ff", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("eos_id", ctypes.c_int32), ("qkv_bias", ctypes.c_int32),
                ("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float), ("weight_seed", ctypes.c_uint64)]


class RuntimeDesc(ctypes.Structure):
    _fields_ = [("weights", ctypes.c_void_p), ("weights_bytes", ctypes.c_size_t),
                ("kv_pool", ctypes.c_void_p), ("kv_pool_bytes", ctypes.c_size_t),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("max_seqs", ctypes.c_int32), ("max_prompts", ctypes.c_int32), ("max_prompt_len", ctypes.c_int32),
                ("max_prompt_tokens", ctypes.c_int32), ("max_cap", ctypes.c_int32),
                ("sample_seed", ctypes.c_uint64), ("temperature", ctypes.c_float), ("graph_steps", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("tp", ctypes.c_int32), ("tp_rank", ctypes.c_int32),
                ("tp_nccl_id", ctypes.c_void_p), ("local_group", ctypes.c_void_p)]


class Sizes(ctypes.Structure):
    _fields_ = [("weights_bytes", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t),
                ("page_bytes", ctypes.c_size_t)]


class Prompt(ctypes.Structure):
    _fields_ = [("prompt_id", ctypes.c_int32), ("len", ctypes.c_int32),
                ("tokens", ctypes.POINTER(ctypes.c_int32)), ("trace_lens", ctypes.POINTER(ctypes.c_int32)),
                ("trace_lens_retry", ctypes.POINTER(ctypes.c_int32))]


class Status(ctypes.Structure):
    _fields_ = [("round_id", ctypes.c_int64), ("kind", ctypes.c_int32), ("t", ctypes.c_int32),
                ("n_live", ctypes.c_int32), ("accepted", ctypes.c_int32), ("accepted_local", ctypes.c_int32),
                ("done", ctypes.c_int32), ("underfilled", ctypes.c_int32), ("n_prompts_local", ctypes.c_int32),
                ("decoded_tokens", ctypes.c_int64), ("kv_tokens_read", ctypes.c_int64),
                ("preemptions", ctypes.c_int32), ("kv_tokens_unique", ctypes.c_int64)]


class Response(ctypes.Structure):
    _fields_ = [("prompt_id", ctypes.c_int32), ("j", ctypes.c_int32), ("len", ctypes.c_int32),
                ("finish", ctypes.c_int32), ("tok_off", ctypes.c_int64)]


EXPORTS = ["rp_query_sizes", "rp_init_model", "rp_submit_round", "rp_step", "rp_collect", "rp_long_queue",
           "rp_free", "rp_last_error", "rp_launch_count", "rp_debug_logits", "rp_debug_trace_enable",
           "rp_debug_trace_get", "rp_debug_last_logits", "rp_debug_gemm", "rp_debug_profile", "rp_nccl_unique_id",
           "rp_tp_ipc_handle", "rp_tp_ipc_open", "rp_collect_ready", "rp_round_rows_histogram",
           "rp_round_issue_cap", "rp_round_unissued", "rp_plan_round", "rp_long_queue_pop",
           "rp_local_group_create", "rp_local_group_free", "rp_plan_tp", "rp_round_state_bytes", "rp_round_export", "rp_round_import",
           "rp_round_reshard"]


def load_library(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError("librollpacker.so not built (run __graft_entry__.build()); no CPU fallback exists")
    lib = ctypes.CDLL(path)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.rp_query_sizes.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(RuntimeDesc), ctypes.POINTER(Sizes)]
    lib.rp_init_model.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(RuntimeDesc), ctypes.POINTER(P)]
    lib.rp_submit_round.argtypes = [P, ctypes.POINTER(Prompt), I32, I32, I32, I32, I32, I32, I64]
    lib.rp_step.argtypes = [P, I32, ctypes.POINTER(Status)]
    lib.rp_collect.argtypes = [P, ctypes.POINTER(Response), I32, ctypes.POINTER(I32), I64, ctypes.POINTER(I32),
                               ctypes.POINTER(I64)]
    lib.rp_long_queue.argtypes = [P, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)]
    lib.rp_free.argtypes = [P]
    lib.rp_free.restype = None
    lib.rp_last_error.argtypes = [P]
    lib.rp_last_error.restype = ctypes.c_char_p
    lib.rp_launch_count.argtypes = [P]
    lib.rp_launch_count.restype = I64
    lib.rp_debug_logits.argtypes = [P, ctypes.POINTER(I32), I32, ctypes.POINTER(ctypes.c_float)]
    lib.rp_debug_trace_enable.argtypes = [P, I32]
    lib.rp_debug_trace_get.argtypes = [P, ctypes.POINTER(I32), I32]
    lib.rp_debug_last_logits.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(I32), I32,
                                         ctypes.POINTER(I32)]
    lib.rp_debug_gemm.argtypes = [P, P, P, I32, P, I32, I32, I32, I32, I32, I32, ctypes.POINTER(ctypes.c_float)]
    lib.rp_debug_profile.argtypes = [P, I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64),
                                     ctypes.POINTER(I64)]
    lib.rp_nccl_unique_id.argtypes = [P]
    lib.rp_tp_ipc_handle.argtypes = [P, P]
    lib.rp_tp_ipc_open.argtypes = [P, P]
    lib.rp_round_rows_histogram.argtypes = [P, ctypes.POINTER(I64), I32]
    lib.rp_round_state_bytes.argtypes = [P, ctypes.POINTER(I64)]
    lib.rp_round_export.argtypes = [P, P, I64]
    lib.rp_round_import.argtypes = [P, ctypes.POINTER(Prompt), I32, I32, I32, I32, I32, I32, I64, P, I64]
    lib.rp_round_reshard.argtypes = [ctypes.POINTER(P), ctypes.POINTER(I64), I32, I32, I32, I32, P, I64,
                                     ctypes.POINTER(I64)]
    lib.rp_round_issue_cap.argtypes = [P, I32]
    lib.rp_round_unissued.argtypes = [P, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)]
    lib.rp_collect_ready.argtypes = [P, I32, ctypes.POINTER(Response), I32, ctypes.POINTER(I32), I64,
                                     ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I32)]
    lib.rp_plan_round.argtypes = [P, I32, ctypes.c_float, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.rp_long_queue_pop.argtypes = [P, I32]
    lib.rp_local_group_create.argtypes = [I32, I32, ctypes.POINTER(P)]
    lib.rp_local_group_free.argtypes = [P]
    lib.rp_local_group_free.restype = None
    lib.rp_plan_tp.argtypes = [I32, I32, I64, I64, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    for name in EXPORTS:
        if name not in ("rp_free", "rp_last_error", "rp_launch_count", "rp_local_group_free"):
            getattr(lib, name).restype = I32
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    rc = lib().rp_nccl_unique_id(buf)
    if rc != RP_OK:
        raise RuntimeError("rp_nccl_unique_id failed: %d" % rc)
    return buf.raw


class RPError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("rollpacker error %d: %s" % (code, msg))
        self.code = code


def plan_tp(tp, tp_max, prev_preemptions, preemptions, zero_streak):
    """rp_plan_tp: the planner's TP adaptation -> (tp, streak)."""
    a, b = ctypes.c_int32(), ctypes.c_int32()
    rc = lib().rp_plan_tp(int(tp), int(tp_max), int(prev_preemptions), int(preemptions), int(zero_streak),
                          ctypes.byref(a), ctypes.byref(b))
    if rc != RP_OK:
        raise RPError(rc, "rp_plan_tp")
    return a.value, b.value


class LocalGroup:
    """Single-GPU local group (rp_local_group_create): the world x tp ranks of
    a job as contexts of this process on the current device, exchanging
    through device memory.  Create one Engine per rank, each from its own
    thread (rp_init_model waits for every member); close the engines first."""

    def __init__(self, world, tp=1):
        self.L = lib()
        h = ctypes.c_void_p()
        rc = self.L.rp_local_group_create(world, tp, ctypes.byref(h))
        if rc != RP_OK:
            raise RPError(rc, "rp_local_group_create(%d, %d)" % (world, tp))
        self.h, self.world, self.tp = h, world, tp

    def close(self):
        if getattr(self, "h", None):
            self.L.rp_local_group_free(self.h)
            self.h = None


def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def model_desc(cfg, weight_seed=0):
    return ModelDesc(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"],
                     cfg["d_ff"], cfg["vocab"], cfg["eos_id"], cfg.get("qkv_bias", 1), cfg["rope_theta"],
                     cfg["rms_eps"], weight_seed)


def reshard_round_states(states, n_prompts, new_world):
    """Exported states of every rank of a DP job (rank order) -> the states of
    new_world ranks (rp_round_reshard), for Engine.import_round."""
    L = lib()
    n = len(states)
    bufs = [ctypes.create_string_buffer(bytes(s), len(s)) for s in states]
    ptrs = (ctypes.c_void_p * n)(*[ctypes.cast(b, ctypes.c_void_p) for b in bufs])
    sizes = (ctypes.c_int64 * n)(*[len(s) for s in states])
    need = ctypes.c_int64()
    rc = L.rp_round_reshard(ptrs, sizes, n, n_prompts, new_world, 0, None, 0, ctypes.byref(need))
    if rc != RP_OK:
        raise RPError(rc, L.rp_last_error(None).decode())
    out = []
    for r in range(new_world):
        buf = ctypes.create_string_buffer(need.value)
        rc = L.rp_round_reshard(ptrs, sizes, n, n_prompts, new_world, r, ctypes.cast(buf, ctypes.c_void_p),
                                need.value, ctypes.byref(need))
        if rc != RP_OK:
            raise RPError(rc, L.rp_last_error(None).decode())
        out.append(buf.raw)
    return out


class Engine:
    """One rollout context on the current CUDA device.

    cfg: model shape dict (synth.configs).  Device buffers are torch tensors
    owned by this object and borrowed by the library."""

    def __init__(self, cfg, max_seqs, max_prompts, max_prompt_len, max_prompt_tokens, max_cap, kv_pool_bytes=None,
                 kv_fraction=0.85, weight_seed=0, sample_seed=3, temperature=1.0, graph_steps=16, rank=0, world=1,
                 nccl_id=None, stream=None, tp=1, tp_rank=0, tp_peer=True, tp_nccl_id=None, local_group=None):
        import torch
        self.torch = torch
        self.L = lib()
        self.cfg = dict(cfg)
        self.md = model_desc(cfg, weight_seed)
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self._nccl_id = self._tp_nccl_id = None
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
        if tp_nccl_id is not None:
            self._tp_nccl_id = ctypes.create_string_buffer(bytes(tp_nccl_id), 128)
        self.local_group = local_group
        rd = RuntimeDesc()
        rd.rank, rd.world = rank, world
        rd.tp, rd.tp_rank = tp, tp_rank
        self.tp, self.tp_rank = tp, tp_rank
        rd.max_seqs, rd.max_prompts, rd.max_prompt_len = max_seqs, max_prompts, max_prompt_len
        rd.max_prompt_tokens, rd.max_cap = max_prompt_tokens, max_cap
        rd.sample_seed, rd.temperature, rd.graph_steps = sample_seed, temperature, graph_steps
        rd.stream = self.stream.cuda_stream
        rd.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None
        rd.tp_nccl_id = ctypes.cast(self._tp_nccl_id, ctypes.c_void_p) if self._tp_nccl_id is not None else None
        rd.local_group = local_group.h if local_group is not None else None
        sz = Sizes()
        rd.kv_pool_bytes = 1 << 30
        self._check(self.L.rp_query_sizes(ctypes.byref(self.md), ctypes.byref(rd), ctypes.byref(sz)), None)
        self.sizes = sz
        dev = torch.cuda.current_device()
        self.weights = torch.empty(sz.weights_bytes, dtype=torch.uint8, device=dev)
        if kv_pool_bytes is None:
            free, _ = torch.cuda.mem_get_info(dev)
            kv_pool_bytes = int((free - sz.workspace_bytes * 1.2) * kv_fraction)
        kv_pool_bytes = max(int(kv_pool_bytes) // sz.page_bytes, 2) * sz.page_bytes
        rd.kv_pool_bytes = kv_pool_bytes
        self._check(self.L.rp_query_sizes(ctypes.byref(self.md), ctypes.byref(rd), ctypes.byref(sz)), None)
        self.sizes = sz
        self.workspace = torch.empty(sz.workspace_bytes, dtype=torch.uint8, device=dev)
        self.kv_pool = torch.empty(kv_pool_bytes, dtype=torch.uint8, device=dev)
        rd.weights, rd.weights_bytes = self.weights.data_ptr(), sz.weights_bytes
        rd.workspace, rd.workspace_bytes = self.workspace.data_ptr(), sz.workspace_bytes
        rd.kv_pool, rd.kv_pool_bytes = self.kv_pool.data_ptr(), kv_pool_bytes
        self.rd = rd
        self.n_pages = kv_pool_bytes // sz.page_bytes
        self.max_seqs, self.max_cap = max_seqs, max_cap
        h = ctypes.c_void_p()
        torch.cuda.synchronize()
        self._check(self.L.rp_init_model(ctypes.byref(self.md), ctypes.byref(rd), ctypes.byref(h)), None)
        self.h = h
        self.tp_peer = local_group is not None and tp > 1       # local groups map the peers at init
        if tp > 1 and tp_peer and local_group is None:
            self._open_tp_peers()

    def _open_tp_peers(self):
        """TP decode over NVLink peer memory: gather every rank's IPC handle
        of its receive block over the host process group (which must be the
        TP group, ranks in TP order) and map the peers."""
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size() != self.tp:
            return
        hb = ctypes.create_string_buffer(RP_IPC_HANDLE_BYTES)
        if self.L.rp_tp_ipc_handle(self.h, hb) != RP_OK:
            return                                   # shape without a peer block: NCCL all-reduce path
        allh = [None] * self.tp
        dist.all_gather_object(allh, hb.raw)
        joined = ctypes.create_string_buffer(b"".join(allh), RP_IPC_HANDLE_BYTES * self.tp)
        self._check(self.L.rp_tp_ipc_open(self.h, joined))
        self.tp_peer = True

    # ------------------------------------------------------------------ utils
    def _check(self, rc, h="self"):
        if rc != RP_OK:
            hh = self.h if h == "self" else None
            msg = self.L.rp_last_error(hh)
            raise RPError(rc, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "h", None):
            self.L.rp_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self):
        return int(self.L.rp_launch_count(self.h))

    # --------------------------------------------------------------- the ABI
    def submit(self, prompts, G, cap, target, long_round=False, trace=None, round_id=0, keep=0, trace_retry=None,
               trace_mode=None, preempt=False):
        """prompts: list of dicts {prompt_id, tokens} (None -> pop `target`
        prompts off the long-prompt queue; pass trace_mode=True for a trace-mode
        round over queued prompts); trace: None or int array [n, G] of response
        lengths (trace mode); trace_retry: [n, G] lengths of the re-roll used if
        a prompt is deferred (reading Z5); keep: responses retained per prompt
        (R0 < G: response-level speculation; 0 -> G)."""
        tm = trace is not None if trace_mode is None else trace_mode
        flags = (RP_LONG if long_round else RP_SHORT) | (RP_TRACE if tm else 0) | (RP_PREEMPT if preempt else 0)
        if prompts is None:
            n = target
            rc = self.L.rp_submit_round(self.h, None, n, G, keep, cap, target, flags, round_id)
            self._check(rc)
            return
        arr, n = self._prompt_array(prompts, trace, trace_retry)
        self._check(self.L.rp_submit_round(self.h, arr, n, G, keep, cap, target, flags, round_id))

    def _prompt_array(self, prompts, trace, trace_retry=None):
        n = len(prompts)
        arr = (Prompt * n)()
        self._keep = []
        for i, p in enumerate(prompts):
            toks = np.ascontiguousarray(p["tokens"], dtype=np.int32)
            self._keep.append(toks)
            arr[i].prompt_id = int(p["prompt_id"])
            arr[i].len = len(toks)
            arr[i].tokens = _i32p(toks)
            if trace is not None:
                tl = np.ascontiguousarray(trace[i], dtype=np.int32)
                self._keep.append(tl)
                arr[i].trace_lens = _i32p(tl)
            if trace_retry is not None:
                tr = np.ascontiguousarray(trace_retry[i], dtype=np.int32)
                self._keep.append(tr)
                arr[i].trace_lens_retry = _i32p(tr)
        return arr, n

    def export_round(self):
        """The in-flight round's step state (bytes; NEXT-3 migration, see
        rp_round_export).  The KV cache is not part of it."""
        nb = ctypes.c_int64()
        self._check(self.L.rp_round_state_bytes(self.h, ctypes.byref(nb)))
        buf = ctypes.create_string_buffer(nb.value)
        self._check(self.L.rp_round_export(self.h, ctypes.cast(buf, ctypes.c_void_p), nb.value))
        return buf.raw

    def import_round(self, state, prompts, G, cap, target, long_round=False, trace=None, round_id=0, keep=0,
                     trace_retry=None, preempt=False):
        """Continue a round exported by export_round on this (idle) engine:
        the original submit arguments plus the state; the live responses' KV
        is recomputed (rp_round_import)."""
        flags = (RP_LONG if long_round else RP_SHORT) | (RP_TRACE if trace is not None else 0) | \
            (RP_PREEMPT if preempt else 0)
        arr, n = self._prompt_array(prompts, trace, trace_retry)
        buf = ctypes.create_string_buffer(bytes(state), len(state))
        self._check(self.L.rp_round_import(self.h, arr, n, G, keep, cap, target, flags, round_id,
                                           ctypes.cast(buf, ctypes.c_void_p), len(state)))

    def step(self, max_steps=1 << 30):
        st = Status()
        self._check(self.L.rp_step(self.h, max_steps, ctypes.byref(st)))
        return st

    def run(self):
        st = self.step()
        while not st.done:
            st = self.step()
        return st

    def collect(self):
        n, nt = ctypes.c_int32(), ctypes.c_int64()
        self._check(self.L.rp_collect(self.h, None, 0, None, 0, ctypes.byref(n), ctypes.byref(nt)))
        out = (Response * max(1, n.value))()
        toks = np.zeros(max(1, nt.value), dtype=np.int32)
        self._check(self.L.rp_collect(self.h, out, n.value, _i32p(toks), nt.value, ctypes.byref(n), ctypes.byref(nt)))
        res = []
        for i in range(n.value):
            r = out[i]
            res.append(dict(prompt_id=r.prompt_id, j=r.j, len=r.len, finish=r.finish,
                            tokens=toks[r.tok_off:r.tok_off + r.len].copy()))
        return res

    def collect_ready(self, first):
        """Streaming collect: responses of the prompts accepted with local
        acceptance index >= first so far (the round stays active).  Returns
        (responses, accepted count to pass as `first` next time)."""
        n, nt, na = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
        self._check(self.L.rp_collect_ready(self.h, first, None, 0, None, 0, ctypes.byref(n), ctypes.byref(nt),
                                            ctypes.byref(na)))
        out = (Response * max(1, n.value))()
        toks = np.zeros(max(1, nt.value), dtype=np.int32)
        self._check(self.L.rp_collect_ready(self.h, first, out, n.value, _i32p(toks), nt.value, ctypes.byref(n),
                                            ctypes.byref(nt), ctypes.byref(na)))
        res = [dict(prompt_id=out[i].prompt_id, j=out[i].j, len=out[i].len, finish=out[i].finish,
                    tokens=toks[out[i].tok_off:out[i].tok_off + out[i].len].copy()) for i in range(n.value)]
        return res, na.value

    def rows_histogram(self):
        """Decode steps of the current/last round by live-row count (index = rows)."""
        out = np.zeros(self.max_seqs + 1, dtype=np.int64)
        self._check(self.L.rp_round_rows_histogram(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                   len(out)))
        return out

    def issue_cap(self, max_active):
        """Continuous issuance for the next rounds (NEXT-4): at most
        `max_active` prompts of this rank active; 0 turns it off."""
        self._check(self.L.rp_round_issue_cap(self.h, int(max_active)))

    def unissued(self):
        """Global ids of this rank's prompts the finished round never issued."""
        n = ctypes.c_int32()
        self._check(self.L.rp_round_unissued(self.h, None, 0, ctypes.byref(n)))
        ids = np.zeros(max(1, n.value), dtype=np.int32)
        self._check(self.L.rp_round_unissued(self.h, _i32p(ids), n.value, ctypes.byref(n)))
        return ids[:n.value].tolist()

    def plan(self, P0, eta=1.25, drain=False):
        """The library's tail-batching planner: ('long', P0) when the queue
        holds >= P0 prompts, else ('short', ceil(eta * P0))."""
        k, n = ctypes.c_int32(), ctypes.c_int32()
        self._check(self.L.rp_plan_round(self.h, int(P0), float(eta), 1 if drain else 0, ctypes.byref(k),
                                         ctypes.byref(n)))
        return ("long" if k.value == RP_LONG else "short"), n.value

    def long_queue_pop(self, n):
        self._check(self.L.rp_long_queue_pop(self.h, int(n)))

    def long_queue(self):
        n = ctypes.c_int32()
        self._check(self.L.rp_long_queue(self.h, None, 0, ctypes.byref(n)))
        ids = np.zeros(max(1, n.value), dtype=np.int32)
        self._check(self.L.rp_long_queue(self.h, _i32p(ids), n.value, ctypes.byref(n)))
        return ids[:n.value].tolist()

    # ------------------------------------------------------------ test-only
    def debug_logits(self, tokens):
        """Teacher-forced logits (under TP: this rank's vocab shard)."""
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        out = np.zeros((len(toks), self.cfg["vocab"] // max(1, self.tp)), dtype=np.float32)
        self._check(self.L.rp_debug_logits(self.h, _i32p(toks), len(toks),
                                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return out

    def debug_trace_enable(self, steps):
        self._check(self.L.rp_debug_trace_enable(self.h, steps))
        self._trace_steps = steps

    def debug_trace(self, steps=None, start=1):
        """Per-step records from step `start` (1-based) up to the first step
        without live rows (an imported round records from its import step)."""
        steps = steps or self._trace_steps
        buf = np.zeros((steps, 2 + self.max_seqs), dtype=np.int32)
        self._check(self.L.rp_debug_trace_get(self.h, _i32p(buf), steps))
        out = []
        for t in range(start - 1, steps):
            n = int(buf[t, 0])
            if n == 0:
                break
            out.append(dict(t=t + 1, live=buf[t, 2:2 + n].copy(), accepted=int(buf[t, 1] & ((1 << 30) - 1)),
                            done=int(buf[t, 1] >> 30)))
        return out

    def debug_last_logits(self):
        out = np.zeros((self.max_seqs, self.cfg["vocab"] // max(1, self.tp)), dtype=np.float32)
        slots = np.zeros(self.max_seqs, dtype=np.int32)
        n = ctypes.c_int32()
        self._check(self.L.rp_debug_last_logits(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                                _i32p(slots), self.max_seqs, ctypes.byref(n)))
        return out[:n.value], slots[:n.value]

    PROF_NAMES = ["embed", "rmsnorm", "gemm_qkv", "rope_append", "attention", "attn_merge", "gemm_o", "gemm_gu",
                  "gemm_down", "gemm_lm", "sampler", "ctl", "nccl"]

    def debug_profile_arm(self, steps):
        self._check(self.L.rp_debug_profile(self.h, steps, None, None, None))

    def debug_profile_read(self):
        n = len(self.PROF_NAMES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        rcs = (ctypes.c_int64 * 3)()
        self._check(self.L.rp_debug_profile(self.h, 0, ms, cnt, rcs))
        return dict(ms={k: ms[i] for i, k in enumerate(self.PROF_NAMES)},
                    launches={k: int(cnt[i]) for i, k in enumerate(self.PROF_NAMES)},
                    rows=int(rcs[0]), ctx=int(rcs[1]), steps=int(rcs[2]))

    def debug_gemm(self, W, X, N, splits=0, iters=1, timed=False, tiled=False, X_lo=None):
        """W: torch fp16 [M, K] cuda, X: torch fp16 [rows_cap, K] cuda -> Y fp32 [N, M]
        (and the mean ms per launch when timed).  tiled=True hands W to the
        kernel in the 128 x 64 tiled layout the model's weights use (the
        rearrangement is argument marshalling: the same values).  X_lo: the
        fp16 rounding residuals of X (split precision): Y = W (X + X_lo)^T."""
        torch = self.torch
        M, K = W.shape
        flags = (1 if tiled else 0) | (2 if X_lo is not None else 0)
        if X_lo is not None:
            X = torch.cat([X, X_lo]).contiguous()
        if tiled:
            W = W.reshape(M // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous()
        Y = torch.zeros((max(N, 1), M), dtype=torch.float32, device=W.device)
        torch.cuda.synchronize()
        ms = ctypes.c_float()
        self._check(self.L.rp_debug_gemm(self.h, W.data_ptr(), X.data_ptr(), X.shape[0] // (2 if X_lo is not None else 1),
                                         Y.data_ptr(), M, N, K, splits, iters, flags, ctypes.byref(ms)))
        return (Y[:N], ms.value) if timed else Y[:N]
