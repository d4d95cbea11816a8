// Host engine behind the C ABI (include/rollpacker.h): weight layout, TMA
// descriptors, workspace carving, the round state machine (submit -> prefill
// -> device-resident decode steps in CUDA graphs -> collect), the long-prompt
// FIFO and the DP cutoff exchange over NCCL.  Every arithmetic step of the
// path runs in the kernels of this directory; the host only plans, launches
// and copies.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <climits>
#include <condition_variable>
#include <chrono>
#include <mutex>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "../../include/rollpacker.h"
#include "common.cuh"
#include "gemm.h"
#include "kernels.h"

using namespace rp;

namespace {

constexpr int kSMs = 148;
constexpr size_t kAlign = 1024;

size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct Carver {
  uint8_t* base;
  size_t off = 0;
  explicit Carver(void* b) : base((uint8_t*)b) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off);
    T* p = base ? (T*)(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct LayerW {
  __half *wqkv, *wo, *wgu, *wd;           // fp16 re-encodings of the bf16 formula values (Z20)
  float *bqkv, *ln1, *ln2;
  GemmPlan p_qkv, p_o, p_gu, p_down;
};

struct QueuedPrompt {
  int32_t id;
  std::vector<int32_t> tokens;
  std::vector<int32_t> trace;        // lengths of this round's attempt (trace mode)
  std::vector<int32_t> trace_retry;  // lengths of the re-roll if deferred (reading Z5; empty -> trace)
};

struct Sizes {
  int S, P, maxp, Tcap, max_items_dec, max_items_pre, pt_rows, max_items_g;
  size_t part_floats, apart_floats;
};

// Exchange buffers of one communicator of a single-GPU local group
// (k_comm.cu): slots[2][size][slot_bytes] and the members' epochs gen[size].
struct LocalComm {
  int size = 0;
  size_t slot_bytes = 0;
  uint8_t* slots = nullptr;
  unsigned long long* gen = nullptr;
};

// One communicator of a context: NCCL, or the device-memory exchange of a
// local group (then `state` = this member's {epoch, ticket} on the device).
struct CommCtx {
  ncclComm_t nccl = nullptr;
  LocalComm* local = nullptr;
  int size = 1, rank = 0;
  int* state = nullptr;
};

}  // namespace

// Single-GPU local group (rp_local_group_create): world x tp contexts of one
// process on one device.  DP communicator d_t = {(r, t) : r < world} per
// tp rank t, TP communicator t_r = {(r, q) : q < tp} per replica r.
struct RpLocalGroup {
  int world = 1, tp = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, barrier_gen = 0;
  std::vector<LocalComm> dp, tpc;     // [tp], [world]
  std::vector<void*> tp_blocks;       // [world * tp] TP peer receive blocks
  bool alloc_ok = false;
  std::string alloc_err;

  // host barrier over every member context (rp_init_model); false after
  // 300 s without every member (one of them failed before the barrier)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int g = barrier_gen;
    if (++arrived == world * tp) {
      arrived = 0;
      ++barrier_gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(300), [&] { return barrier_gen != g; });
  }
};

struct RpCtx {
  rp_model_desc md{};
  rp_runtime_desc rd{};
  ModelDims m{};
  cudaStream_t st = nullptr;
  std::string err;
  Sizes z{};
  int n_pages = 0;
  long long launches = 0;

  // weights
  std::vector<LayerW> layers;
  __nv_bfloat16* emb = nullptr;            // gathered by the embedding kernel only
  __half* lm = nullptr;
  float* lnf = nullptr;
  GemmPlan p_lm{};
  int s_qkv = 1, s_o = 1, s_gu = 1, s_down = 1, s_lm = 1;
  // tensor-parallel peer all-reduce (decode): this rank's IPC-exported block
  // = recv [2 slots][tp][S][d] fp32 + flags [2][tp] u64, the peers' blocks
  // mapped through CUDA IPC, per-slot use generations and CTA tickets
  void* tp_ipc = nullptr;
  size_t tp_recv_floats = 0;      // floats of one [tp][S][d] slot
  void* tp_peer_base[8] = {nullptr};
  bool tp_peer = false;
  unsigned long long* tp_gen = nullptr;   // [2]
  int* tp_done = nullptr;                 // [2]
  bool peer_decode = false;               // the current forward pushes partials (final norm owes a tp_norm)
  long long* attn_tl = nullptr;           // debug (RP_ATTN_TIMELINE): last attention launch's CTA marks

  // activations / workspace
  float* x = nullptr;
  float* ssq = nullptr;         // [rows][d / 128] per-tile sums of squares of x (folded RMSNorm)
  float* ar = nullptr;          // TP: all-reduced partial of a row-parallel GEMM
  __half *h = nullptr, *q = nullptr, *att = nullptr, *mid = nullptr;   // activations (Z20)
  // split-precision residuals of the activations (reading Z22); the
  // producers write them and the consumers read them only while act_lo is set
  __half *h_lo = nullptr, *q_lo = nullptr, *att_lo = nullptr, *mid_lo = nullptr;
  bool act_lo = true;
  int lo_mask = 0;
  // decode attention sums the QKV split partials (RP_FUSE_QKV=1; off by
  // default: measured slower, profiles/r02_fused_qkv_ab.txt)
  bool fuse_qkv = false;
  int ag_dbg = 0;
  bool o_dsm = false;                     // O projection split-K through DSMEM
  int gemm_rows_max = 0;                  // rows bound of the current forward (decode bucket / prefill tokens)
  bool cur_gmode = false;                 // the decode step being captured / launched uses the group attention
  int* gmode_dev = nullptr;               // RoundDev.gmode
  int* gmode_h = nullptr;                 // pinned staging of it
  int gmode_last = -1;                         // RP_AG_DBG: group-attention measurement knobs (k_attn_group.cu)
  float *qkv = nullptr, *logits = nullptr, *gpart = nullptr, *apart = nullptr;
  int* gctr = nullptr;
  int* atickets = nullptr;
  float* rowpart = nullptr;   // group attention: member-row split partials (attn_group 4)
  int* rtickets = nullptr;
  double* inv_freq = nullptr;
  float2* rope_cs = nullptr;    // [pos][hd/2] (cos, sin) of pos * theta^(-2i/hd), from fp64
  AttnItem *items_pre = nullptr;
  int *pre_tok = nullptr, *pre_pos = nullptr, *pre_pt = nullptr, *pre_last = nullptr, *fork_jobs = nullptr;
  int *col_meta = nullptr, *col_tok = nullptr;
  int* identity_pages = nullptr;
  RoundDev R{};
  CtlBlock* h_ctl = nullptr;   // pinned mirror
  CUtensorMap kv_map{};        // the KV pool as [token rows, head_dim] for TMA

  // graphs
  struct Graph { int bucket; bool gmode; cudaGraphExec_t exec; int nodes; };
  std::vector<Graph> graphs;    // per live-row bucket, valid for the current round
  cudaGraphExec_t gexec = nullptr;
  int graph_nodes = 0;
  bool graph_dirty = true;
  int tp = 1;
  bool own_stream = false;

  // communicators: data-parallel (the cutoff exchange and round membership)
  // and tensor-parallel (all-reduces); NCCL or a local group's device memory
  CommCtx dp, tpc;
  RpLocalGroup* lg = nullptr;
  int coop_min = 16;          // cooperative split-K from this chunk width (no_spin: never)
  int* memb = nullptr;        // [P + 1] local membership, then [world][P + 1] gathered (rp_collect)
  int* memb_h = nullptr;      // pinned host staging of memb
  int* rejobs_h = nullptr;    // pinned host copy of the recompute jobs (KV pressure)

  // round state (host)
  bool active = false, collected = true;
  int kind = 0, trace = 0, G = 0, keep = 0, cap = 0, target = 0, n_glob = 0, lo = 0, n_loc = 0;
  int issue_cap = 0;       // rp_round_issue_cap: applies to the next submitted rounds
  int max_active = 0;      // of the current round (0 = every prompt issued at submit)
  int64_t round_id = 0;
  std::vector<QueuedPrompt> round_prompts;  // this rank's slice
  std::vector<QueuedPrompt> round_all;      // the whole submitted list (the global FIFO needs every prompt)
  int fifo_pop = 0;                         // queue entries the active round consumes (popped at submit success)
  std::deque<QueuedPrompt> fifo;
  int trace_steps = 0;
  int* trace_dev = nullptr;
  bool step_logits_valid = false;

  // per-kernel-class profiling of eager decode steps (rp_debug_profile)
  int prof_steps_left = 0;
  bool capturing = false;
  std::vector<cudaEvent_t> ev, ev_pool;   // events of the current profiled step (from the pool)
  std::vector<int> ev_cls;
  volatile int* gate_h = nullptr;         // host-mapped flag that holds a profiled step until it is enqueued
  // measurement only (RP_SKIP=attention,gemm_qkv,...): kernel classes left
  // out of decode steps, so a graph step's time without them is its exposed cost
  unsigned skip_mask = 0;
  int cur_cls = -1;
  int* gate_d = nullptr;
  double prof_ms[RP_PROF_N] = {0};
  long long prof_cnt[RP_PROF_N] = {0};
  long long prof_rows = 0, prof_ctx = 0, prof_step_count = 0;

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
};

static std::string g_init_err;

// split-precision operands (reading Z22)
enum { LO_QKV = 1, LO_O = 2, LO_GU = 4, LO_DOWN = 8, LO_Q = 16 };
static const int kDefaultLoMask = LO_QKV | LO_O | LO_GU | LO_DOWN | LO_Q;

// Programmatic dependent launch is off while a local-group context issues
// work from this thread (common.cuh g_no_pdl).
static inline void pdl_mode(const RpCtx* c) { g_no_pdl = c->lg != nullptr; }
static inline bool skipped(const RpCtx* c) { return c->cur_cls >= 0 && ((c->skip_mask >> c->cur_cls) & 1u); }

// Local groups: a pageable-memory copy is staged by the driver in order
// across the whole CUDA context, so one queued behind this stream's spinning
// collective would also hold up the other members' copies -- a deadlock.
// Pageable copies are therefore only issued on an idle stream.
static inline cudaError_t idle(RpCtx* c) { return c->lg ? cudaStreamSynchronize(c->st) : cudaSuccess; }

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return c->fail(RP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define CKN(call)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) return c->fail(RP_ENCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------------ sizing
static int tp_of(const rp_runtime_desc* rd) { return rd->tp > 1 ? rd->tp : 1; }

// Dimensions of this rank's shard: heads, KV heads, d_ff and vocab are split
// over the TP group (column-parallel QKV / gate||up / LM head, row-parallel
// O / down); d_model, layers and the embedding stay whole.
static ModelDims local_dims(const rp_model_desc* md, const rp_runtime_desc* rd) {
  const int T = tp_of(rd), r = T > 1 ? rd->tp_rank : 0;
  ModelDims m{};
  m.L = md->n_layers; m.d = md->d_model; m.hd = md->head_dim; m.eos = md->eos_id; m.eps = md->rms_eps;
  m.H = md->n_heads / T; m.KV = md->n_kv_heads / T; m.F = md->d_ff / T; m.V = md->vocab / T; m.v0 = r * m.V;
  m.page_bytes = (size_t)m.L * m.KV * 2 * kPage * m.hd * 2;
  return m;
}

static Sizes compute_sizes(const rp_model_desc* md, const rp_runtime_desc* rd) {
  Sizes z{};
  z.S = rd->max_seqs;
  z.P = rd->max_prompts;
  z.maxp = (rd->max_prompt_len + rd->max_cap + kPage - 1) / kPage + 1;
  z.Tcap = std::max(rd->max_seqs, rd->max_prompt_tokens);
  z.pt_rows = z.S + z.P;
  // Decode attention work list (ctl phase B): row r gets ns_r <= want_r key
  // splits with sum_r want_r <= rows + U, U <= 3 * U1 (k-wave budget, k <= 3)
  // and U1 = 148 / KV (or the RP_ATTN_UNITS override): at most S + 3 * U1.
  const int kv_loc = md->n_kv_heads / tp_of(rd);
  const int units_env = getenv("RP_ATTN_UNITS") ? atoi(getenv("RP_ATTN_UNITS")) : 0;
  const int U1max = std::max(std::max(1, 148 / std::max(1, kv_loc)), units_env);
  z.max_items_dec = z.S + 3 * U1max;
  // sibling-group list: group units + per-row private units (attn_group 4) + splits
  z.max_items_g = 2 * z.S + 3 * U1max;
  z.max_items_pre = rd->max_prompt_tokens * ((rd->max_prompt_len + kAttnChunk - 1) / kAttnChunk) + z.P;
  // split-K partials: worst GEMM at the decode sizes
  const ModelDims lm = local_dims(md, rd);
  const int d = lm.d, qkvw = (lm.H + 2 * lm.KV) * lm.hd, F = lm.F;
  const int hid = lm.H * lm.hd;
  const int shapes[5][2] = {{qkvw, d}, {d, hid}, {2 * F, d}, {d, F}, {lm.V, d}};
  size_t mx = 0;
  const int nch = z.S <= 128 ? 1 : (z.S + 255) / 256;   // narrow split-precision chunks: N <= 128
  for (auto& s : shapes) {
    const int sp = gemm_pick_splits(s[0], s[1], kSMs);
    if (sp > 1) mx = std::max(mx, (size_t)(s[0] / 128) * nch * sp * 256 * 128);
  }
  // rp_debug_gemm may request splits of an arbitrary shape: keep >= 16M floats
  z.part_floats = std::max(mx, (size_t)1 << 24);
  // attention split partials: per-row items (16 rows of (m, l, O)) or
  // sibling-group items (8 members x 8 rows)
  z.apart_floats = std::max((size_t)z.max_items_dec * lm.KV * std::max((size_t)16 * (lm.hd + 2),
                                                                       attn_group_partial_floats(lm.hd)),
                            (size_t)z.max_items_pre * lm.KV * 16 * (lm.hd + 2));
  return z;
}

struct WeightLayout {
  size_t total;
  std::vector<size_t> off;  // per layer: wqkv, bqkv, wo, wgu, wd, ln1, ln2 (7 entries); then emb, lm, lnf
};

static WeightLayout weight_layout(const rp_model_desc* md, const rp_runtime_desc* rd) {
  WeightLayout w;
  const ModelDims lm = local_dims(md, rd);
  const size_t d = lm.d, hd = lm.hd, H = lm.H, KV = lm.KV, F = lm.F, V = lm.V, Vfull = md->vocab;
  const size_t qkvw = (H + 2 * KV) * hd;
  size_t off = 0;
  auto put = [&](size_t bytes) {
    off = align_up(off);
    w.off.push_back(off);
    off += bytes;
  };
  for (int l = 0; l < md->n_layers; ++l) {
    put(qkvw * d * 2);
    put(qkvw * 4);
    put(d * H * hd * 2);
    put(2 * F * d * 2);
    put(d * F * 2);
    put(d * 4);
    put(d * 4);
  }
  put(Vfull * d * 2);   // embedding (whole on every rank)
  put(V * d * 2);       // LM head shard
  put(d * 4);
  w.total = align_up(off);
  return w;
}

static size_t workspace_bytes(const rp_model_desc* md, const rp_runtime_desc* rd, RpCtx* c /*nullable*/) {
  const Sizes z = compute_sizes(md, rd);
  const ModelDims lm = local_dims(md, rd);
  const size_t d = lm.d, hd = lm.hd, H = lm.H, KV = lm.KV, F = lm.F, V = lm.V;
  Carver cv(c ? rd->workspace : nullptr);
  auto x = cv.take<float>((size_t)z.Tcap * d);
  auto ar = cv.take<float>(tp_of(rd) > 1 ? (size_t)z.Tcap * d : 1);
  auto h = cv.take<__half>((size_t)z.Tcap * d);
  auto h_lo = cv.take<__half>((size_t)z.Tcap * d);         // split-precision residuals (reading Z22)
  auto ssq = cv.take<float>((size_t)z.Tcap * std::max<size_t>(1, d / 128));   // folded-RMSNorm partial sums
  auto qkv = cv.take<float>((size_t)z.Tcap * (H + 2 * KV) * hd);
  auto q = cv.take<__half>((size_t)z.Tcap * H * hd);
  auto q_lo = cv.take<__half>((size_t)z.Tcap * H * hd);
  auto att = cv.take<__half>((size_t)z.Tcap * H * hd);
  auto att_lo = cv.take<__half>((size_t)z.Tcap * H * hd);
  auto mid = cv.take<__half>((size_t)z.Tcap * F);
  auto mid_lo = cv.take<__half>((size_t)z.Tcap * F);
  auto logits = cv.take<float>((size_t)std::max(z.S, std::max(z.P, rd->max_prompt_len)) * V);
  auto gpart = cv.take<float>(z.part_floats);
  auto gctr = cv.take<int>(1 << 16);
  auto apart = cv.take<float>(z.apart_floats);
  auto atick = cv.take<int>((size_t)std::max(z.max_items_dec, z.max_items_pre) * KV);
  auto invf = cv.take<double>(hd / 2);
  auto rope_cs = cv.take<float2>((size_t)(rd->max_prompt_len + rd->max_cap + 2) * (hd / 2));
  auto items_dec = cv.take<AttnItem>(z.max_items_dec);
  auto gitems_dec = cv.take<AttnGroupItem>(z.max_items_g);   // sibling-group list (RoundDev.attn_group)
  auto rowpart = cv.take<float>((size_t)z.S * KV * kRowSplits * (attn_group_partial_floats(hd) / 8));
  auto rtick = cv.take<int>((size_t)z.S * KV);
  auto gmode = cv.take<int>(1);
  auto grp_key = cv.take<int>(z.S);
  auto grp_start = cv.take<int>((size_t)z.S + 1);
  auto rows_hist = cv.take<unsigned long long>((size_t)z.S + 1);
  auto items_pre = cv.take<AttnItem>(z.max_items_pre);
  auto pre_tok = cv.take<int>(rd->max_prompt_tokens);
  auto pre_pos = cv.take<int>(rd->max_prompt_tokens);
  auto pre_pt = cv.take<int>(rd->max_prompt_tokens);
  auto pre_last = cv.take<int>(std::max(z.P, rd->max_prompt_len));
  auto fork_jobs = cv.take<int>((size_t)3 * z.S);
  auto col_meta = cv.take<int>((size_t)5 * z.S + 1);
  auto col_tok = cv.take<int>((size_t)z.S * rd->max_cap);
  // round state
  auto slot_prompt = cv.take<int>(z.S);
  auto slot_j = cv.take<int>(z.S);
  auto kv_len = cv.take<int>(z.S);
  auto gen = cv.take<int>(z.S);
  auto trace_L = cv.take<int>(z.S);
  auto status = cv.take<int>(z.S);
  auto own0 = cv.take<int>(z.S);
  auto t0 = cv.take<int>(z.S);
  auto p_last_tok = cv.take<int>(z.P);
  auto p_stamp = cv.take<int>(z.P);
  auto tok_out = cv.take<int>((size_t)z.S * rd->max_cap);
  auto page_table = cv.take<int>((size_t)z.pt_rows * z.maxp);
  auto p_cnt = cv.take<int>(z.P);
  auto p_state = cv.take<int>(z.P);
  auto p_gid = cv.take<int>(z.P);
  auto comp_list = cv.take<int>(z.P);
  auto accept_order = cv.take<int>(z.P);
  auto live = cv.take<int>(z.S);
  auto live_next = cv.take<int>(z.S);
  auto tok_in = cv.take<int>(z.S);
  auto row_pos = cv.take<int>(z.S);
  auto row_pt = cv.take<int>(z.S);
  auto best = cv.take<unsigned long long>(std::max(z.S, 1));
  auto ks_local = cv.take<int>(4);
  auto ks = cv.take<int>((size_t)4 * std::max(1, rd->world));
  // KV pressure (NEXT-2): per-prompt admission / wait state, scratch sums, the wait FIFO, recompute jobs
  auto p_plen = cv.take<int>(z.P);
  auto p_adm = cv.take<int>(z.P);
  auto p_wait = cv.take<int>(z.P);
  auto p_live = cv.take<int>(z.P);
  auto p_pfree = cv.take<int>(z.P);
  auto p_pneed = cv.take<int>(z.P);
  auto wait_q = cv.take<int>(z.P);
  auto rejobs = cv.take<int>((size_t)5 * z.S);
  auto memb = cv.take<int>((size_t)(z.P + 1) * (1 + std::max(1, rd->world)));
  auto ctl = cv.take<CtlBlock>(1);
  const size_t page_bytes = lm.page_bytes;
  const size_t max_pages = rd->kv_pool_bytes / page_bytes;
  auto free_stack = cv.take<int>(max_pages + 1);
  auto ident = cv.take<int>(max_pages + 1);
  if (c) {
    c->x = x; c->ar = ar; c->h = h; c->ssq = ssq; c->qkv = qkv; c->q = q; c->att = att; c->mid = mid; c->logits = logits;
    c->h_lo = h_lo; c->q_lo = q_lo; c->att_lo = att_lo; c->mid_lo = mid_lo;
    c->gpart = gpart; c->gctr = gctr; c->apart = apart; c->atickets = atick; c->inv_freq = invf;
    c->rope_cs = rope_cs;
    c->items_pre = items_pre; c->pre_tok = pre_tok; c->pre_pos = pre_pos; c->pre_pt = pre_pt;
    c->pre_last = pre_last; c->fork_jobs = fork_jobs; c->col_meta = col_meta; c->col_tok = col_tok;
    c->identity_pages = ident;
    c->memb = memb;
    RoundDev& R = c->R;
    R.S = z.S; R.P = z.P; R.maxp = z.maxp; R.kv_heads = (int)KV; R.eos = md->eos_id;
    R.world = rd->world; R.rank = rd->rank;
    R.attn_units = getenv("RP_ATTN_UNITS") ? atoi(getenv("RP_ATTN_UNITS")) : 0;   // measurement override
    R.attn_waves = getenv("RP_ATTN_WAVES") ? atoi(getenv("RP_ATTN_WAVES")) : 1;   // A/B switch
    R.slot_prompt = slot_prompt; R.slot_j = slot_j; R.kv_len = kv_len; R.gen = gen; R.trace_L = trace_L;
    R.status = status; R.own0 = own0; R.t0 = t0; R.p_last_tok = p_last_tok; R.p_stamp = p_stamp; R.tok_out = tok_out; R.page_table = page_table; R.p_cnt = p_cnt;
    R.p_state = p_state; R.p_gid = p_gid; R.comp_list = comp_list; R.accept_order = accept_order;
    R.live = live; R.live_next = live_next; R.tok_in = tok_in; R.row_pos = row_pos; R.row_pt = row_pt;
    R.max_items = z.max_items_dec;
    R.p_plen = p_plen; R.p_adm = p_adm; R.p_wait = p_wait; R.p_live = p_live; R.p_pfree = p_pfree;
    R.p_pneed = p_pneed; R.wait_q = wait_q; R.rejobs = rejobs;
    R.grp_key = grp_key; R.grp_start = grp_start;
    R.best = best; R.items = items_dec; R.gitems = gitems_dec; R.gmode = gmode; c->gmode_dev = gmode;
    R.max_items_g = z.max_items_g; c->rowpart = rowpart; c->rtickets = rtick; R.rows_hist = rows_hist; R.free_stack = free_stack; R.ks_local = ks_local; R.ks = ks;
    R.ctl = ctl; R.cap = rd->max_cap;
  }
  return align_up(cv.off);
}

static int validate(const rp_model_desc* md, const rp_runtime_desc* rd, std::string& e) {
  auto bad = [&](const char* f) { e = std::string("invalid field: ") + f; return RP_EINVAL; };
  if (!md || !rd) return bad("desc (null)");
  if (md->n_layers < 1) return bad("n_layers");
  if (md->head_dim != 64 && md->head_dim != 128) return bad("head_dim (64 or 128)");
  if (md->d_model % 128) return bad("d_model (multiple of 128)");
  if ((md->n_heads * md->head_dim) % 128) return bad("n_heads*head_dim (multiple of 128)");
  if (md->d_ff % 64) return bad("d_ff (multiple of 64)");
  if (md->vocab % 128) return bad("vocab (multiple of 128)");
  if (md->n_kv_heads < 1 || md->n_heads % md->n_kv_heads) return bad("n_kv_heads");
  if (md->n_heads / md->n_kv_heads > 8) return bad("n_heads/n_kv_heads (<= 8)");
  if (((md->n_heads + 2 * md->n_kv_heads) * md->head_dim) % 128) return bad("qkv width (multiple of 128)");
  if (md->eos_id < 0 || md->eos_id >= md->vocab) return bad("eos_id");
  const RpLocalGroup* lg = (const RpLocalGroup*)rd->local_group;
  if (lg && (lg->world != std::max(1, rd->world) || lg->tp != std::max(1, rd->tp)))
    return bad("local_group (created for another world / tp)");
  if (rd->tp > 1) {
    const int T = rd->tp;
    if (rd->tp_rank < 0 || rd->tp_rank >= T) return bad("tp_rank");
    if (!lg && !rd->tp_nccl_id && !(rd->world == 1 && rd->nccl_id)) return bad("tp_nccl_id (tp > 1)");
    if (md->n_kv_heads % T || md->n_heads % T) return bad("tp (must divide n_heads and n_kv_heads)");
    if ((md->d_ff / T) % 64 || md->d_ff % T) return bad("tp (d_ff / tp multiple of 64)");
    if (md->vocab % T || (md->vocab / T) % 128) return bad("tp (vocab / tp multiple of 128)");
    if (((md->n_heads + 2 * md->n_kv_heads) / T * md->head_dim) % 128) return bad("tp (local qkv width)");
    if ((md->n_heads / T * md->head_dim) % 64) return bad("tp (local attention width)");
  }
  if (rd->world < 1 || rd->rank < 0 || rd->rank >= rd->world) return bad("rank/world");
  if (rd->world > 1 && !rd->nccl_id && !lg) return bad("nccl_id (world > 1)");
  if (rd->tp < 0 || rd->tp > 8) return bad("tp (1..8)");
  if (rd->max_seqs < 1 || rd->max_seqs > 1 << 16) return bad("max_seqs");
  if (rd->max_prompts < 1 || rd->max_prompts > rd->max_seqs) return bad("max_prompts");
  if (rd->max_prompt_len < 1 || rd->max_prompt_tokens < rd->max_prompt_len) return bad("max_prompt_len/tokens");
  if (rd->max_cap < 1) return bad("max_cap");
  if (rd->temperature <= 0.f) return bad("temperature");
  return RP_OK;
}

// ------------------------------------------------------------------ model forward
// Profiling brackets: when an eager decode step is profiled, every launch is
// bracketed by CUDA events on the launching stream.
static cudaEvent_t prof_event(RpCtx* c) {
  if (c->ev.size() == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  cudaEvent_t e = c->ev_pool[c->ev.size()];
  c->ev.push_back(e);
  return e;
}
struct ProfScope {
  RpCtx* c; int cls; bool on;
  ProfScope(RpCtx* c_, int cls_) : c(c_), cls(cls_), on(c_->prof_steps_left > 0 && !c_->capturing) {
    c->cur_cls = cls;
    if (on) { cudaEventRecord(prof_event(c), c->st); c->ev_cls.push_back(-1); }
  }
  ~ProfScope() {
    if (on) { cudaEventRecord(prof_event(c), c->st); c->ev_cls.push_back(cls); }
  }
};
// Folded RMSNorm (DESIGN.md §5 K6): FOLD_PRODUCE on a RESID GEMM also writes
// fp16(x) into c->h and per-tile sums of squares into c->ssq; FOLD_CONSUME
// scales each output row of a GEMM reading c->h by 1/rms.  The norm gains are
// folded into the consuming weights at init (rp_init_model), so every norm
// runs with unit gain; under TP the RMSNorm kernel runs instead.
enum { FOLD_NONE = 0, FOLD_PRODUCE = 1, FOLD_CONSUME = 2 };

// Tensor-parallel peer push of a row-parallel GEMM's fp32 output: rank q's
// receive slot `slot` for source rank `src`, inside rank q's IPC block `base`.
static float* tp_slot(RpCtx* c, void* base, int slot, int src) {
  return (float*)base + (size_t)slot * c->tp_recv_floats + (size_t)src * (c->tp_recv_floats / c->tp);
}
static unsigned long long* tp_flags(RpCtx* c, void* base, int slot) {
  return (unsigned long long*)((float*)base + 2 * c->tp_recv_floats) + (size_t)slot * c->tp;
}

// ---------------------------------------------------------------- collectives
// NCCL (one process per GPU) or the device-memory exchange of a single-GPU
// local group; both carry the same message and combine it in rank order.
static void local_coll(RpCtx* c, CommCtx& cm, int op, const void* send, void* recv, size_t bytes) {
  launch_local_publish(send, bytes, cm.local->slots, cm.local->slot_bytes, cm.size, cm.rank, cm.local->gen, cm.state,
                       c->st);
  launch_local_reduce(op, recv, bytes, cm.local->slots, cm.local->slot_bytes, cm.size, cm.local->gen, cm.state, c->st);
  c->launches += 2;
}
static void coll_allgather_i32(RpCtx* c, CommCtx& cm, const int* send, int* recv, size_t count) {
  if (cm.local) local_coll(c, cm, LOP_GATHER, send, recv, count * 4);
  else ncclAllGather(send, recv, count, ncclInt32, cm.nccl, c->st);
}
static void coll_allreduce_sum_f32(RpCtx* c, CommCtx& cm, float* buf, size_t count) {
  if (cm.local) local_coll(c, cm, LOP_SUM_F32, buf, buf, count * 4);
  else ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, cm.nccl, c->st);
}
static void coll_allreduce_max_u64(RpCtx* c, CommCtx& cm, unsigned long long* buf, size_t count) {
  if (cm.local) local_coll(c, cm, LOP_MAX_U64, buf, buf, count * 8);
  else ncclAllReduce(buf, buf, count, ncclUint64, ncclMax, cm.nccl, c->st);
}

static void gemm(RpCtx* c, const GemmPlan& p, int M, int K, const int* n_dev, int n_host, int splits, int epi,
                 void* out, int ldo, const float* bias, const RopeArgs* rope = nullptr, int fold = FOLD_NONE,
                 int push_slot = -1, __half* out_lo = nullptr, bool dsm = false) {
  if (skipped(c)) return;
  GemmArgs a{};
  if (push_slot >= 0) {
    const int me = c->rd.tp_rank;
    a.push_n = c->tp;
    for (int q = 0; q < c->tp; ++q) {
      a.push_dst[q] = tp_slot(c, c->tp_peer_base[q], push_slot, me);
      a.push_flag[q] = tp_flags(c, c->tp_peer_base[q], push_slot) + me;
    }
  }
  if (rope) a.rope = *rope;
  a.M = M; a.K = K; a.n_dev = n_dev; a.n_host = n_host; a.splits = splits; a.epi = epi; a.out = out; a.ldo = ldo;
  a.bias = bias; a.partial = c->gpart; a.counters = c->gctr;
  a.no_spin = c->lg ? 1 : 0;
  a.dsm = (gemm_dsm_enabled() || dsm) && c->gemm_rows_max > 0 && c->gemm_rows_max <= 256 ? 1 : 0;
  a.lo = c->act_lo ? 1 : 0;
  a.out_lo = c->act_lo ? out_lo : nullptr;
  a.ssq_stride = c->m.d / 128; a.ssq_parts = c->m.d / 128;
  a.norm_inv_d = 1.0f / (float)c->m.d; a.norm_eps = c->m.eps;
  if (fold == FOLD_PRODUCE) { a.xb_out = c->h; a.xb_lo = c->h_lo; a.ldxb = c->m.d; a.ssq_out = c->ssq; }
  if (fold == FOLD_CONSUME) a.ssq_in = c->ssq;
  gemm_launch(p, a, kSMs, c->st);
  c->launches++;
}

// TP all-reduce (sum) of the row-parallel partial in c->ar over `rows` rows
// (a host count: the graph bucket at decode, the prompt tokens at prefill).
static void tp_allreduce_rows(RpCtx* c, int rows) {
  ProfScope ps(c, RP_PROF_NCCL);
  coll_allreduce_sum_f32(c, c->tpc, c->ar, (size_t)rows * c->m.d);
}

// Transformer body over `n` rows (n_dev on device or n_host): decode (one token
// per live sequence) or prefill (all prompt tokens).  Under tensor
// parallelism the O and down GEMMs write their partial sums to c->ar, which
// is all-reduced and added to the residual stream by the next RMSNorm
// (`*pending` tells the caller the final norm still owes that add).
static void forward_layers(RpCtx* c, const int* tok, const int* n_dev, int n_host, const int* row_pos,
                           const int* row_pt, const AttnItem* items, const int* n_items_dev, int n_items_host,
                           bool decode, int ar_rows, bool* pending) {
  const ModelDims& m = c->m;
  const bool tp = c->tp > 1;
  const float* delta = nullptr;
  const int qkvw = (m.H + 2 * m.KV) * m.hd;
  c->gemm_rows_max = decode ? ar_rows : n_host;   // DSMEM split-K needs one activation chunk (<= 256 rows)
  const int sp_qkv = decode ? c->s_qkv : 1, sp_o = decode ? c->s_o : 1, sp_gu = decode ? c->s_gu : 1,
            sp_down = decode ? c->s_down : 1;
  // folded RMSNorm on a single rank: only layer 0's input norm is a kernel
  static const bool no_fold = getenv("RP_NO_FOLD") != nullptr;   // A/B switch for measurements
  const bool fold = !tp && m.d % 128 == 0 && !no_fold;
  const int f_prod = fold ? FOLD_PRODUCE : FOLD_NONE, f_cons = fold ? FOLD_CONSUME : FOLD_NONE;
  // TP decode over NVLink peer memory: the O/down GEMMs push their partials
  // into every rank (slots 0/1) and tp_norm adds them and normalizes
  const bool peer = tp && decode && c->tp_peer;
  c->peer_decode = peer;
  auto tp_norm = [&](int slot, const float* gamma, int splits) {
    ProfScope ps(c, RP_PROF_RMSNORM);
    void* own = c->tp_peer_base[c->rd.tp_rank];
    launch_tp_norm(c->x, tp_slot(c, own, slot, 0), c->tp, c->tp_recv_floats / c->tp, tp_flags(c, own, slot),
                   c->tp_gen + slot, c->tp_done + slot, m.d / 128, splits, c->coop_min, c->lg ? 8 : 0, n_dev, n_host,
                   gamma, c->h, m.d, m.eps, c->st, c->h_lo);
    c->launches++;
  };
  { ProfScope ps(c, RP_PROF_EMBED); if (!skipped(c)) launch_embed(tok, n_dev, n_host, c->emb, c->x, m.d, c->st); c->launches++; }
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = c->layers[l];
    const int f_in = (fold && l > 0) ? FOLD_CONSUME : FOLD_NONE;
    // the norm gains are folded into the consuming weights at init (unit gain here)
    if (peer && l > 0) {
      tp_norm(1, nullptr, sp_down);
    } else if (f_in == FOLD_NONE) {
      ProfScope ps(c, RP_PROF_RMSNORM);
      if (!skipped(c)) launch_rmsnorm(c->x, delta, nullptr, n_dev, n_host, nullptr, c->h, m.d, m.eps, c->st, c->h_lo); c->launches++;
    }
    QkvFuse fz{};
    const bool fuse = decode && sp_qkv > 1 && m.hd % 64 == 0 && c->fuse_qkv;
    if (fuse) {
      // the QKV GEMM writes its split-K partials; the decode attention sums
      // them per row, applies the folded norm, bias and RoPE, and appends k / v
      ProfScope ps(c, RP_PROF_GEMM_QKV);
      gemm(c, w.p_qkv, qkvw, m.d, n_dev, n_host, sp_qkv, EPI_PARTIAL, c->qkv, qkvw, w.bqkv, nullptr, f_in);
      fz.part = c->gpart; fz.splits = sp_qkv; fz.m_tiles = qkvw / 128;
      fz.gemm_lo = c->act_lo && (c->lo_mask & LO_QKV) ? 1 : 0;
      fz.n_rows = n_dev; fz.bias = w.bqkv;
      fz.ssq = f_in == FOLD_CONSUME ? c->ssq : nullptr; fz.ssq_parts = m.d / 128; fz.ssq_stride = m.d / 128;
      fz.inv_d = 1.0f / (float)m.d; fz.eps = m.eps;
      fz.cs = c->rope_cs; fz.kv_pool = (uint8_t*)c->rd.kv_pool; fz.page_bytes = m.page_bytes;
      fz.n_pages = m.n_pages;
    } else if (decode && sp_qkv > 1 && m.hd % 64 == 0) {
      // RoPE + KV append fused into the split-K reduction of the QKV GEMM
      ProfScope ps(c, RP_PROF_GEMM_QKV);
      RopeArgs ra{c->q, c->q_lo, (uint8_t*)c->rd.kv_pool, c->R.page_table, row_pos, row_pt, c->rope_cs, m.page_bytes,
                  c->R.maxp, l, m.H, m.KV, m.hd, m.n_pages};
      gemm(c, w.p_qkv, qkvw, m.d, n_dev, n_host, sp_qkv, EPI_QKV_ROPE, c->qkv, qkvw, w.bqkv, &ra, f_in);
    } else {
      { ProfScope ps(c, RP_PROF_GEMM_QKV);
        gemm(c, w.p_qkv, qkvw, m.d, n_dev, n_host, sp_qkv, EPI_F32, c->qkv, qkvw, w.bqkv, nullptr, f_in); }
      { ProfScope ps(c, RP_PROF_ROPE);
        launch_rope_append(c->qkv, n_dev, n_host, row_pos, row_pt, c->R.page_table, c->R.maxp, c->q,
                           c->rd.kv_pool, m, l, c->inv_freq, c->st, c->q_lo); c->launches++; }
    }
    { ProfScope ps(c, RP_PROF_ATTN);
      if (skipped(c)) {
      } else if (decode && c->cur_gmode) {
        launch_attention_group(c->kv_map, c->q, c->q_lo, c->R.page_table, c->R.maxp, c->R.gitems,
                               &c->R.ctl->n_gitems, c->att, c->att_lo, c->apart, c->atickets, m, l, c->st, c->ag_dbg,
                               c->lg ? 0 : 1, c->rowpart, c->rtickets);
      } else {
        fz.dbg = c->ag_dbg;
        launch_attention(c->kv_map, c->q, c->R.page_table, c->R.maxp, items, n_items_dev, n_items_host, c->att,
                         c->apart, c->atickets, m, l, decode, c->st, c->q_lo, c->att_lo,
                         fuse || c->ag_dbg ? &fz : nullptr);
      }
      c->launches++; }
    { ProfScope ps(c, RP_PROF_GEMM_O);
      gemm(c, w.p_o, m.d, m.H * m.hd, n_dev, n_host, sp_o, tp ? EPI_F32 : EPI_RESID, tp ? c->ar : c->x, m.d,
           nullptr, nullptr, f_prod, peer ? 0 : -1, nullptr, decode && c->o_dsm && !tp); }
    if (peer) {
      tp_norm(0, nullptr, sp_o);
    } else if (tp) {
      tp_allreduce_rows(c, ar_rows);
    }
    if (!fold && !peer) {
      ProfScope ps(c, RP_PROF_RMSNORM);
      launch_rmsnorm(c->x, tp ? c->ar : nullptr, nullptr, n_dev, n_host, nullptr, c->h, m.d, m.eps, c->st, c->h_lo);
      c->launches++;
    }
    { ProfScope ps(c, RP_PROF_GEMM_GU);
      gemm(c, w.p_gu, 2 * m.F, m.d, n_dev, n_host, sp_gu, EPI_SWIGLU, c->mid, m.F, nullptr, nullptr, f_cons, -1,
           c->mid_lo); }
    { ProfScope ps(c, RP_PROF_GEMM_DOWN);
      gemm(c, w.p_down, m.d, m.F, n_dev, n_host, sp_down, tp ? EPI_F32 : EPI_RESID, tp ? c->ar : c->x, m.d,
           nullptr, nullptr, f_prod, peer ? 1 : -1); }
    if (tp && !peer) {
      tp_allreduce_rows(c, ar_rows);
      delta = c->ar;
    }
  }
  *pending = tp;
}

// LM head over this rank's vocab shard + sampling; under TP the packed
// per-row argmax is MAX-all-reduced (exact: the order of maxima is irrelevant).
static void lm_head_sample(RpCtx* c, const int* n_dev, int n_host, const int* gather, int rows_out, int row_div,
                           int best_rows, bool pending, int splits) {
  RoundDev& R = c->R;
  // folded final norm when the rows are the residual rows in place (decode)
  const bool fold = c->tp <= 1 && !gather && c->m.d % 128 == 0 && !getenv("RP_NO_FOLD");
  if (c->peer_decode && !gather) {
    ProfScope ps(c, RP_PROF_RMSNORM);
    void* own = c->tp_peer_base[c->rd.tp_rank];
    launch_tp_norm(c->x, tp_slot(c, own, 1, 0), c->tp, c->tp_recv_floats / c->tp, tp_flags(c, own, 1),
                   c->tp_gen + 1, c->tp_done + 1, c->m.d / 128, c->s_down, c->coop_min, c->lg ? 8 : 0, n_dev, n_host,
                   nullptr, c->h, c->m.d, c->m.eps, c->st, c->h_lo);
    c->launches++;
  } else if (!fold) {
    ProfScope ps(c, RP_PROF_RMSNORM);
    launch_rmsnorm(c->x, pending ? c->ar : nullptr, gather, n_dev, n_host, nullptr, c->h, c->m.d, c->m.eps, c->st,
                   c->h_lo);
    c->launches++;
  }
  { ProfScope ps(c, RP_PROF_GEMM_LM);
    gemm(c, c->p_lm, c->m.V, c->m.d, n_dev, rows_out, splits, EPI_F32, c->logits, c->m.V, nullptr, nullptr,
         fold ? FOLD_CONSUME : FOLD_NONE); }
  { ProfScope ps(c, RP_PROF_SAMPLER);
    if (!skipped(c)) launch_sampler(c->logits, c->m.V, c->m.v0, row_div, R, c->rd.sample_seed, 1.0f / c->rd.temperature,
                   (uint32_t)c->round_id, c->st); c->launches++; }
  if (c->tp > 1) {
    ProfScope ps(c, RP_PROF_NCCL);
    coll_allreduce_max_u64(c, c->tpc, R.best, (size_t)best_rows);
  }
}

static void decode_step(RpCtx* c, int bucket) {
  RoundDev& R = c->R;
  const int* n_dev = &R.ctl->n_live;
  bool pending = false;
  forward_layers(c, R.tok_in, n_dev, 0, R.row_pos, R.row_pt, R.items, &R.ctl->n_items, 0, true, bucket, &pending);
  lm_head_sample(c, n_dev, 0, nullptr, 0, 1, bucket, pending, c->s_lm);
  if (c->rd.world == 1) {
    ProfScope ps(c, RP_PROF_CTL);
    launch_ctl(R, 1, 0, c->st); c->launches++;
  } else {
    { ProfScope ps(c, RP_PROF_CTL); launch_ctl(R, 1, 1, c->st); c->launches++; }
    { ProfScope ps(c, RP_PROF_NCCL); coll_allgather_i32(c, c->dp, R.ks_local, R.ks, 4); }
    { ProfScope ps(c, RP_PROF_CTL); launch_ctl(R, 1, 2, c->st); c->launches++; }
  }
}

// (Re)capture graph_steps decode steps.  Kernel parameters (the RoundDev
// scalars: cap, G, target, kind, trace, round id) are baked into the graph, so
// it is rebuilt once per round, before its first decode step.
// Live-row bucket of a decode step: the kernels read the live count on the
// device, but NCCL counts are host values, so under TP the graphs are keyed
// by a power-of-two bucket >= the live count (the count only shrinks).
static int bucket_for(const RpCtx* c, int n) {
  if (c->tp <= 1) return c->z.S;
  int b = 16;
  while (b < n) b *= 2;
  return std::min(b, c->z.S);
}

// Decode attention of the next steps: the sibling-group kernel while the
// live batch exceeds group_rows_min (wide steps: siblings mostly alive, the
// shared prompt pages dominate the reads; 45 vs 67 us per layer at the
// bench's 255-row steps), the per-row kernel below (profiles/r02_attn_group_ab.txt).  The device flag
// tells ctl to keep building the group list while a group-mode graph runs.
static int set_gmode(RpCtx* c) {
  // (an imported / re-sharded step carries no group list: n_gitems == 0)
  const bool mode = c->R.attn_group && c->h_ctl->n_live > c->R.group_rows_min && c->h_ctl->n_gitems > 0;
  if ((int)mode != c->gmode_last) {
    *c->gmode_h = mode ? 1 : 0;
    CK(cudaMemcpyAsync(c->gmode_dev, c->gmode_h, sizeof(int), cudaMemcpyHostToDevice, c->st));
    c->gmode_last = mode;
  }
  c->cur_gmode = mode;
  return RP_OK;
}

static int ensure_graph(RpCtx* c, int bucket) {
  if (c->graph_dirty) {
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
    c->graph_dirty = false;
  }
  for (auto& g : c->graphs)
    if (g.bucket == bucket && g.gmode == c->cur_gmode) { c->gexec = g.exec; c->graph_nodes = g.nodes; return RP_OK; }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  const long long before = c->launches;
  c->capturing = true;
  for (int i = 0; i < c->rd.graph_steps; ++i) decode_step(c, bucket);
  c->capturing = false;
  cudaError_t e = cudaStreamEndCapture(c->st, &g);
  if (e != cudaSuccess) return c->fail(RP_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  RpCtx::Graph entry{bucket, c->cur_gmode, nullptr, (int)(c->launches - before)};
  c->launches = before;
  CK(cudaGraphInstantiate(&entry.exec, g, 0));
  CK(cudaGraphDestroy(g));
  c->graphs.push_back(entry);
  c->gexec = entry.exec;
  c->graph_nodes = entry.nodes;
  return RP_OK;
}


// ------------------------------------------------------------------ C ABI
extern "C" {

int rp_query_sizes(const rp_model_desc* md, const rp_runtime_desc* rd, rp_sizes* out) {
  std::string e;
  int r = validate(md, rd, e);
  if (r) { g_init_err = e; return r; }
  if (!out) { g_init_err = "invalid field: out"; return RP_EINVAL; }
  out->weights_bytes = weight_layout(md, rd).total;
  out->workspace_bytes = workspace_bytes(md, rd, nullptr);
  out->page_bytes = local_dims(md, rd).page_bytes;
  return RP_OK;
}

static int init_impl(RpCtx* c) {
  const rp_model_desc* md = &c->md;
  const rp_runtime_desc* rd = &c->rd;
  c->st = (cudaStream_t)rd->stream;
  if (!c->st) {   // graphs cannot be captured on the legacy stream: own one
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  ModelDims& m = c->m;
  m = local_dims(md, rd);
  c->tp = tp_of(rd);
  c->z = compute_sizes(md, rd);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  int sms = 0, cc_major = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, dev));
  if (cc_major != 10) return c->fail(RP_ECUDA, "device is not sm_100 (compute capability %d.x)", cc_major);
  const WeightLayout wl = weight_layout(md, rd);
  if (rd->weights_bytes < wl.total) return c->fail(RP_ENOSPC, "weights buffer too small: %zu < %zu", rd->weights_bytes, wl.total);
  const size_t ws = workspace_bytes(md, rd, nullptr);
  if (rd->workspace_bytes < ws) return c->fail(RP_ENOSPC, "workspace too small: %zu < %zu", rd->workspace_bytes, ws);
  c->n_pages = (int)(rd->kv_pool_bytes / m.page_bytes);
  if (c->n_pages < 2) return c->fail(RP_ENOSPC, "kv pool holds %d pages", c->n_pages);
  m.n_pages = c->n_pages;   // layer-major KV layout (kv_block_elems)
  if (make_kv_map(&c->kv_map, rd->kv_pool, (size_t)c->n_pages, m))
    return c->fail(RP_ECUDA, "KV tensor map (pool too large for 2^31 token rows?)");
  // stale rows of a page are masked in attention but multiplied by P = 0:
  // they must be finite, so the pool starts zeroed (all later writes are finite)
  CK(cudaMemsetAsync(rd->kv_pool, 0, (size_t)c->n_pages * m.page_bytes, c->st));
  workspace_bytes(md, rd, c);
  if (gemm_init_attrs()) return c->fail(RP_ECUDA, "gemm smem attribute");
  if (attn_init_attrs() || attn_group_init_attrs()) return c->fail(RP_ECUDA, "attention smem attribute");

  // ---- weights (formula Z12), layout per layer
  uint8_t* wb = (uint8_t*)rd->weights;
  const size_t d = m.d, hd = m.hd, H = m.H, KV = m.KV, F = m.F, V = m.V;
  const uint64_t seed = md->weight_seed;
  c->layers.resize(m.L);
  size_t k = 0;
  // split-precision activations (reading Z22); RP_ACT_LO=0 turns them off (A/B)
  c->act_lo = !(getenv("RP_ACT_LO") && atoi(getenv("RP_ACT_LO")) == 0);
  if (const char* sk = getenv("RP_SKIP")) {
    static const char* names[RP_PROF_N] = {"embed", "rmsnorm", "gemm_qkv", "rope_append", "attention", "attn_merge",
                                           "gemm_o", "gemm_gu", "gemm_down", "gemm_lm", "sampler", "ctl", "nccl"};
    for (int i = 0; i < RP_PROF_N; ++i)
      if (i != RP_PROF_CTL && i != RP_PROF_NCCL && strstr(sk, names[i])) c->skip_mask |= 1u << i;
  }
  // which operands carry their residual: bit 0 QKV input, 1 O input (attention
  // output), 2 gate/up input, 3 down input (SwiGLU output), 4 the attention
  // query; RP_LO_MASK overrides, RP_ACT_LO=0 clears it (A/B)
  c->lo_mask = getenv("RP_LO_MASK") ? (int)strtol(getenv("RP_LO_MASK"), nullptr, 0) : kDefaultLoMask;
  if (!c->act_lo) c->lo_mask = 0;
  c->act_lo = c->lo_mask != 0;
  c->fuse_qkv = getenv("RP_FUSE_QKV") && atoi(getenv("RP_FUSE_QKV")) != 0;
  // decode attention over sibling groups (k_attn_group.cu; g <= 8 query heads
  // per KV head fit one n-tile per member): RP_ATTN_GROUP=1 auto, 2 / 3 force
  // sibling groups / single rows.  Off by default: 1.9x faster attention at
  // 256 rows x 1K context, but on the bench rounds (fragmented groups, long
  // private tails) 2.5% slower overall than the per-row kernel
  // (profiles/r02_attn_group_ab.txt)
  c->ag_dbg = getenv("RP_AG_DBG") ? atoi(getenv("RP_AG_DBG")) : 0;
  c->R.attn_group = c->fuse_qkv || m.H / m.KV > 8 ? 0 : (getenv("RP_ATTN_GROUP") ? atoi(getenv("RP_ATTN_GROUP")) : 1);
  // the group kernel wins on the bench's own live sets only while nearly
  // every sibling is alive and the private tails are short (above ~200 of
  // 256 rows; tools/attn_window_ab.py, profiles/r02_attn_group_ab.txt)
  c->R.group_rows_min = getenv("RP_ATTN_GROUP_MIN") ? atoi(getenv("RP_ATTN_GROUP_MIN")) : 200;
  c->R.group_waves = getenv("RP_ATTN_GROUP_WAVES") ? std::max(1, atoi(getenv("RP_ATTN_GROUP_WAVES"))) : 1;
  // producers skip the residuals nobody reads; plans without one map hi only
  if (!(c->lo_mask & (LO_QKV | LO_GU))) c->h_lo = nullptr;
  if (!(c->lo_mask & LO_O)) c->att_lo = nullptr;
  if (!(c->lo_mask & LO_DOWN)) c->mid_lo = nullptr;
  if (!(c->lo_mask & LO_Q)) c->q_lo = nullptr;
  // GEMM weights in 128 x 64 tiles: every weight TMA box is one contiguous
  // 16 KB read (RP_W_ROWMAJOR=1: plain row-major, an A/B switch)
  const int wt = getenv("RP_W_ROWMAJOR") ? 0 : 1;
  std::vector<float> ones(std::max(d, (size_t)1), 1.0f);
  for (int l = 0; l < m.L; ++l) {
    LayerW& w = c->layers[l];
    w.wqkv = (__half*)(wb + wl.off[k++]);
    w.bqkv = (float*)(wb + wl.off[k++]);
    w.wo = (__half*)(wb + wl.off[k++]);
    w.wgu = (__half*)(wb + wl.off[k++]);
    w.wd = (__half*)(wb + wl.off[k++]);
    w.ln1 = (float*)(wb + wl.off[k++]);
    w.ln2 = (float*)(wb + wl.off[k++]);
    const uint32_t base = 0x100u * (uint32_t)(l + 1);
    // this rank's shard = a block of each full tensor (rank r of T: q rows
    // [r*H*hd, ...), k/v rows [r*KV*hd, ...), o columns [r*H*hd, ...), gate/up
    // rows [r*F, ...), down columns [r*F, ...); H, KV, F are local here)
    const int tr = c->tp > 1 ? rd->tp_rank : 0;
    const size_t Hf = (size_t)md->n_heads, Ff = (size_t)md->d_ff;
    // GEMM weights are stored in 128 x 64 tiles (weight_tiled_index, k_model.cu)
    launch_init_weights(w.wqkv, (long long)(H * hd), (int)d, (long long)tr * H * hd, 0, (int)d, base + 0, seed, 0, 0,
                        c->st, 1, 0, wt);
    launch_init_weights(w.wqkv, (long long)(KV * hd), (int)d, (long long)tr * KV * hd, 0, (int)d, base + 1, seed, 0, 0,
                        c->st, 1, (long long)(H * hd), wt);
    launch_init_weights(w.wqkv, (long long)(KV * hd), (int)d, (long long)tr * KV * hd, 0, (int)d, base + 2, seed, 0, 0,
                        c->st, 1, (long long)((H + KV) * hd), wt);
    if (md->qkv_bias) {
      launch_init_weights(w.bqkv, (long long)(H * hd), 1, (long long)tr * H * hd, 0, 1, base + 3, seed, 1, 0, c->st);
      launch_init_weights(w.bqkv + H * hd, (long long)(KV * hd), 1, (long long)tr * KV * hd, 0, 1, base + 4, seed, 1,
                          0, c->st);
      launch_init_weights(w.bqkv + (H + KV) * hd, (long long)(KV * hd), 1, (long long)tr * KV * hd, 0, 1, base + 5,
                          seed, 1, 0, c->st);
    } else {
      CK(cudaMemsetAsync(w.bqkv, 0, (H + 2 * KV) * hd * 4, c->st));
    }
    launch_init_weights(w.wo, (long long)d, (int)(H * hd), 0, (int)(tr * H * hd), (int)(Hf * hd), base + 6, seed, 0, 0,
                        c->st, 1, 0, wt);
    launch_init_weights(w.wgu, (long long)F, (int)d, (long long)tr * F, 0, (int)d, base + 7, seed, 2, 0, c->st, 1, 0, wt);
    launch_init_weights(w.wgu, (long long)F, (int)d, (long long)tr * F, 0, (int)d, base + 8, seed, 2, 1, c->st, 1, 0, wt);
    launch_init_weights(w.wd, (long long)d, (int)F, 0, (int)(tr * F), (int)Ff, base + 9, seed, 0, 0, c->st, 1, 0, wt);
    CK(cudaMemcpyAsync(w.ln1, ones.data(), d * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(w.ln2, ones.data(), d * 4, cudaMemcpyHostToDevice, c->st));
  }
  c->emb = (__nv_bfloat16*)(wb + wl.off[k++]);
  c->lm = (__half*)(wb + wl.off[k++]);
  c->lnf = (float*)(wb + wl.off[k++]);
  launch_init_weights(c->emb, (long long)md->vocab, (int)d, 0, 0, (int)d, 0x10000000u, seed, 0, 0, c->st, 0, 0, 0);
  launch_init_weights(c->lm, (long long)V, (int)d, (long long)m.v0, 0, (int)d, 0x10000001u, seed, 0, 0, c->st, 1, 0, wt);
  CK(cudaMemcpyAsync(c->lnf, ones.data(), d * 4, cudaMemcpyHostToDevice, c->st));
  // RMSNorm gains folded into the consuming GEMMs' weight columns (QKV <- ln1,
  // gate||up <- ln2, LM head <- final norm): RMSNorm(x) * g . W^T =
  // (x / rms) . (W diag g)^T, so every norm kernel and folded norm runs with
  // unit gain.  The Z12 gains are 1, for which the fold is exact.
  for (auto& w : c->layers) {
    launch_scale_cols(w.wqkv, (long long)((H + 2 * KV) * hd), (int)d, w.ln1, c->st, wt);
    launch_scale_cols(w.wgu, (long long)(2 * F), (int)d, w.ln2, c->st, wt);
  }
  launch_scale_cols(c->lm, (long long)V, (int)d, c->lnf, c->st, wt);
  CK(cudaGetLastError());

  // ---- RoPE frequencies theta^(-2i/hd) in fp64
  std::vector<double> invf(hd / 2);
  for (size_t i = 0; i < hd / 2; ++i) invf[i] = std::pow((double)md->rope_theta, -2.0 * (double)i / (double)hd);
  CK(cudaMemcpyAsync(c->inv_freq, invf.data(), invf.size() * 8, cudaMemcpyHostToDevice, c->st));
  {
    const size_t npos = (size_t)rd->max_prompt_len + rd->max_cap + 2;
    std::vector<float2> cs(npos * (hd / 2));
    for (size_t p = 0; p < npos; ++p)
      for (size_t i = 0; i < hd / 2; ++i) {
        const double ang = std::fmod((double)p * invf[i], 6.283185307179586);
        cs[p * (hd / 2) + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    CK(cudaMemcpyAsync(c->rope_cs, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
  }

  // ---- TMA descriptors
  const int Tcap = c->z.Tcap;
  const int qkvw = (int)((H + 2 * KV) * hd);
  for (auto& w : c->layers) {
    if (make_plan(&w.p_qkv, w.wqkv, qkvw, (int)d, c->h, Tcap, wt, (c->lo_mask & LO_QKV) ? c->h_lo : nullptr) ||
        make_plan(&w.p_o, w.wo, (int)d, (int)(H * hd), c->att, Tcap, wt, c->att_lo) ||
        make_plan(&w.p_gu, w.wgu, (int)(2 * F), (int)d, c->h, Tcap, wt, (c->lo_mask & LO_GU) ? c->h_lo : nullptr) ||
        make_plan(&w.p_down, w.wd, (int)d, (int)F, c->mid, Tcap, wt, c->mid_lo))
      return c->fail(RP_ECUDA, "cuTensorMapEncodeTiled failed");
  }
  // the LM head reads the final-norm activations in fp16 only: its split
  // precision moves the 28-layer logits error by < 1e-4 (0.0155 vs 0.0154,
  // profiles/r02_emulate_fp16_points.txt) at 65% more LM-head time at 256 rows
  if (make_plan(&c->p_lm, c->lm, (int)V, (int)d, c->h, Tcap, wt, nullptr))
    return c->fail(RP_ECUDA, "cuTensorMapEncodeTiled failed (lm head)");
  c->s_qkv = gemm_pick_splits(qkvw, (int)d, kSMs);
  // the O projection reduces its split-K through DSMEM (4 splits in clusters
  // of 4 beat 5 splits over global memory: profiles/r02_gemm_dsm_ab.txt);
  // RP_GEMM_DSM_O=0 keeps the global paths
  // (single rank only: under TP the O partials are pushed to the peers and
  // tp_norm counts the split CTAs' signals by the global-path rules)
  c->o_dsm = c->tp <= 1 && !(getenv("RP_GEMM_DSM_O") && atoi(getenv("RP_GEMM_DSM_O")) == 0);
  c->s_o = c->o_dsm ? gemm_pick_splits_dsm((int)d, (int)(H * hd), kSMs) : gemm_pick_splits((int)d, (int)(H * hd), kSMs);
  c->s_gu = gemm_pick_splits((int)(2 * F), (int)d, kSMs);
  c->s_down = gemm_pick_splits((int)d, (int)F, kSMs);
  c->s_lm = gemm_pick_splits((int)V, (int)d, kSMs);
  CK(cudaMemsetAsync(c->gctr, 0, (1 << 16) * sizeof(int), c->st));
  CK(cudaMemsetAsync(c->atickets, 0, (size_t)std::max(c->z.max_items_dec, c->z.max_items_pre) * KV * sizeof(int),
                     c->st));
  CK(cudaMemsetAsync(c->rtickets, 0, (size_t)c->z.S * KV * sizeof(int), c->st));

  // ---- identity free list (page ids 0..n_pages-1)
  {
    std::vector<int> idp(c->n_pages);
    for (int i = 0; i < c->n_pages; ++i) idp[i] = i;
    CK(cudaMemcpyAsync(c->identity_pages, idp.data(), idp.size() * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  CK(cudaMallocHost(&c->h_ctl, sizeof(CtlBlock)));
  CK(cudaMallocHost(&c->gmode_h, sizeof(int)));
  *c->gmode_h = 0;
  CK(cudaMemcpyAsync(c->gmode_dev, c->gmode_h, sizeof(int), cudaMemcpyHostToDevice, c->st));
  c->gmode_last = 0;
  if (rd->world > 1) CK(cudaMallocHost(&c->memb_h, (size_t)(c->z.P + 1) * (rd->world + 1) * 4));
  CK(cudaMallocHost(&c->rejobs_h, (size_t)5 * c->z.S * 4));
  memset(c->h_ctl, 0, sizeof(CtlBlock));
  c->h_ctl->done = 1;
  CK(cudaMemcpyAsync(c->R.ctl, c->h_ctl, sizeof(CtlBlock), cudaMemcpyHostToDevice, c->st));

  if (getenv("RP_VERBOSE"))
    fprintf(stderr, "rollpacker: decode split-K qkv %d o %d gu %d down %d lm %d; dsm %d, cluster capacity 2..8: %d %d %d %d %d %d %d\n",
            c->s_qkv, c->s_o, c->s_gu, c->s_down, c->s_lm, (int)gemm_dsm_enabled(), gemm_cluster_cap(2),
            gemm_cluster_cap(3), gemm_cluster_cap(4), gemm_cluster_cap(5), gemm_cluster_cap(6), gemm_cluster_cap(7),
            gemm_cluster_cap(8));
  if (getenv("RP_ATTN_TIMELINE")) {
    CK(cudaMalloc(&c->attn_tl, (size_t)kSMs * 8 * sizeof(long long)));
    CK(cudaMemset(c->attn_tl, 0, (size_t)kSMs * 8 * sizeof(long long)));
    attn_set_timeline(c->attn_tl);
  }

  // ---- TP peer block (exported with CUDA IPC; rp_tp_ipc_open enables it)
  if (c->tp > 1 && c->tp <= 8 && d % 128 == 0) {
    c->tp_recv_floats = (size_t)c->tp * c->z.S * d;
    const size_t bytes = 2 * c->tp_recv_floats * sizeof(float) + 2 * (size_t)c->tp * sizeof(unsigned long long);
    CK(cudaMalloc(&c->tp_ipc, bytes));
    CK(cudaMemset(c->tp_ipc, 0, bytes));
    CK(cudaMalloc(&c->tp_gen, 2 * sizeof(unsigned long long) + 2 * sizeof(int)));
    CK(cudaMemset(c->tp_gen, 0, 2 * sizeof(unsigned long long) + 2 * sizeof(int)));
    c->tp_done = (int*)(c->tp_gen + 2);
  }

  // ---- communicators: DP group (the ranks with this tp_rank, one per
  // replica) and TP group (this replica's tp ranks)
  c->lg = (RpLocalGroup*)rd->local_group;
  c->coop_min = c->lg ? 0x7FFFFFFF : gemm_coop_min();
  c->dp.size = std::max(1, rd->world); c->dp.rank = rd->world > 1 ? rd->rank : 0;
  c->tpc.size = c->tp; c->tpc.rank = c->tp > 1 ? rd->tp_rank : 0;
  if (c->lg) {
    RpLocalGroup* g = c->lg;
    {
      // the first member sizes and allocates the exchange buffers
      std::lock_guard<std::mutex> lk(g->mu);
      if (!g->alloc_ok && g->alloc_err.empty()) {
        const size_t dp_slot = align_up((size_t)(c->z.P + 1) * 4 + 16, 256);
        const size_t tp_slot = align_up(std::max((size_t)c->z.Tcap * m.d * 4, (size_t)c->z.S * 8) + 16, 256);
        auto mk = [&](LocalComm& lc, int size, size_t slot) -> bool {
          lc.size = size; lc.slot_bytes = slot;
          if (cudaMalloc(&lc.slots, 2 * (size_t)size * slot) != cudaSuccess) return false;
          if (cudaMalloc(&lc.gen, (size_t)size * 8) != cudaSuccess) return false;
          return cudaMemset(lc.gen, 0, (size_t)size * 8) == cudaSuccess;
        };
        g->dp.resize(g->tp); g->tpc.resize(g->world);
        bool ok = true;
        if (g->world > 1) for (auto& lc : g->dp) ok = ok && mk(lc, g->world, dp_slot);
        if (g->tp > 1) for (auto& lc : g->tpc) ok = ok && mk(lc, g->tp, tp_slot);
        g->tp_blocks.assign((size_t)g->world * g->tp, nullptr);
        if (ok) g->alloc_ok = true; else g->alloc_err = "local group exchange buffers: cudaMalloc failed";
      }
      if (!g->alloc_ok) return c->fail(RP_ECUDA, "%s", g->alloc_err.c_str());
      if (c->tp > 1) g->tp_blocks[(size_t)c->dp.rank * c->tp + c->tpc.rank] = c->tp_ipc;
    }
    CK(cudaMalloc(&c->dp.state, 8 * sizeof(int)));
    CK(cudaMemset(c->dp.state, 0, 8 * sizeof(int)));
    c->tpc.state = c->dp.state + 4;
    if (c->dp.size > 1) {
      c->dp.local = &g->dp[c->tpc.rank];
      if ((size_t)(c->z.P + 1) * 4 + 16 > c->dp.local->slot_bytes) return c->fail(RP_EINVAL, "local group: max_prompts differ");
    }
    if (c->tp > 1) {
      c->tpc.local = &g->tpc[c->dp.rank];
      if ((size_t)c->z.Tcap * m.d * 4 > c->tpc.local->slot_bytes) return c->fail(RP_EINVAL, "local group: capacities differ");
    }
    CK(cudaStreamSynchronize(c->st));
    if (!g->barrier()) return c->fail(RP_ESTATE, "local group: not every member reached rp_init_model");
    if (c->tp > 1 && c->tp_ipc) {
      for (int q = 0; q < c->tp; ++q) c->tp_peer_base[q] = g->tp_blocks[(size_t)c->dp.rank * c->tp + q];
      c->tp_peer = true;   // plain device pointers: the peers live on this device
    }
  } else {
    if (rd->world > 1) {
      ncclUniqueId id;
      memcpy(&id, rd->nccl_id, sizeof id);
      CKN(ncclCommInitRank(&c->dp.nccl, rd->world, id, rd->rank));
    }
    if (c->tp > 1) {
      ncclUniqueId id;
      memcpy(&id, rd->tp_nccl_id ? rd->tp_nccl_id : rd->nccl_id, sizeof id);
      CKN(ncclCommInitRank(&c->tpc.nccl, c->tp, id, rd->tp_rank));
    }
  }

  c->graph_dirty = true;
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

int rp_init_model(const rp_model_desc* md, const rp_runtime_desc* rd, void** out) {
  std::string e;
  int r = validate(md, rd, e);
  if (r) { g_init_err = e; return r; }
  if (!out) { g_init_err = "invalid field: out"; return RP_EINVAL; }
  RpCtx* c = new RpCtx();
  c->md = *md;
  c->rd = *rd;
  c->lg = (RpLocalGroup*)rd->local_group;
  pdl_mode(c);
  r = init_impl(c);
  if (r) {
    g_init_err = c->err;
    rp_free(c);
    *out = nullptr;
    return r;
  }
  *out = c;
  return RP_OK;
}

int rp_nccl_unique_id(void* out) {
  if (!out) return RP_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) { g_init_err = "ncclGetUniqueId failed"; return RP_ENCCL; }
  memcpy(out, &id, sizeof id);
  return RP_OK;
}

void rp_free(void* ctx) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return;
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->gate_h) cudaFreeHost((void*)c->gate_h);
  if (c->memb_h) cudaFreeHost(c->memb_h);
  if (c->rejobs_h) cudaFreeHost(c->rejobs_h);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  if (c->gmode_h) cudaFreeHost(c->gmode_h);
  if (c->trace_dev) cudaFree(c->trace_dev);
  if (c->dp.nccl) ncclCommDestroy(c->dp.nccl);
  if (c->tpc.nccl) ncclCommDestroy(c->tpc.nccl);
  if (c->dp.state) cudaFree(c->dp.state);
  if (!c->lg)
    for (int q = 0; q < 8; ++q)
      if (c->tp_peer_base[q] && c->tp_peer_base[q] != c->tp_ipc) cudaIpcCloseMemHandle(c->tp_peer_base[q]);
  if (c->tp_ipc) cudaFree(c->tp_ipc);
  if (c->tp_gen) cudaFree(c->tp_gen);
  if (c->attn_tl) { attn_set_timeline(nullptr); cudaFree(c->attn_tl); }
  if (c->own_stream) cudaStreamDestroy(c->st);
  delete c;
}

const char* rp_last_error(const void* ctx) {
  return ctx ? ((const RpCtx*)ctx)->err.c_str() : g_init_err.c_str();
}

int64_t rp_launch_count(const void* ctx) { return ctx ? ((const RpCtx*)ctx)->launches : 0; }

// Prefill attention work list: query blocks of floor(16/g) tokens x key splits.
static int build_prefill_items(RpCtx* c, const std::vector<int>& plen, const std::vector<int>& poff,
                               std::vector<AttnItem>& items) {
  const int g = c->m.H / c->m.KV, tpb = 16 / g;
  items.clear();
  for (size_t p = 0; p < plen.size(); ++p) {
    for (int b0 = 0; b0 < plen[p]; b0 += tpb) {
      const int nq = std::min(tpb, plen[p] - b0);
      const int hi = b0 + nq;  // keys [0, hi)
      const int ns = (hi + kAttnChunk - 1) / kAttnChunk;
      const int item0 = (int)items.size();
      for (int s = 0; s < ns; ++s) {
        AttnItem I;
        I.q_row0 = poff[p] + b0; I.n_qtok = nq; I.pos0 = b0; I.pt_row = c->z.S + (int)p;
        I.kv_lo = s * kAttnChunk; I.kv_hi = std::min(hi, (s + 1) * kAttnChunk);
        I.nsplit = ns; I.item0 = item0;
        items.push_back(I);
      }
    }
  }
  return (int)items.size() <= c->z.max_items_pre ? 0 : -1;
}

// Allocate prompt pages (host mirror of the LIFO free list: ids top-1, top-2, ...)
// and run the prefill forward of `plen` prompts whose tokens are concatenated in
// `toks`.  Writes KV into pages of page-table rows S + p; leaves the final-norm
// hidden state of the rows listed in `out_rows` in h[0..).
static int prefill(RpCtx* c, const std::vector<int>& toks, const std::vector<int>& plen, int& top,
                   std::vector<std::vector<int>>& prompt_pages, const std::vector<int>& out_rows) {
  const int maxp = c->z.maxp, S = c->z.S;
  const int T = (int)toks.size();
  std::vector<int> poff(plen.size()), pos(T), pt(T);
  int o = 0;
  prompt_pages.assign(plen.size(), {});
  std::vector<int> ptab((size_t)plen.size() * maxp, 0);
  for (size_t p = 0; p < plen.size(); ++p) {
    poff[p] = o;
    const int np = (plen[p] + kPage - 1) / kPage;
    if (np > maxp) return c->fail(RP_EINVAL, "prompt %zu longer than max_prompt_len", p);
    for (int k = 0; k < np; ++k) {
      if (top <= 0) return c->fail(RP_ENOMEM_KV, "KV pool exhausted during prefill");
      const int page = --top;
      prompt_pages[p].push_back(page);
      ptab[p * maxp + k] = page;
    }
    for (int i = 0; i < plen[p]; ++i) { pos[o + i] = i; pt[o + i] = S + (int)p; }
    o += plen[p];
  }
  std::vector<AttnItem> items;
  if (build_prefill_items(c, plen, poff, items)) return c->fail(RP_ENOSPC, "prefill attention items exceed capacity");
  CK(idle(c));
  CK(cudaMemcpyAsync(c->R.page_table + (size_t)S * maxp, ptab.data(), ptab.size() * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->pre_tok, toks.data(), T * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->pre_pos, pos.data(), T * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->pre_pt, pt.data(), T * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->items_pre, items.data(), items.size() * sizeof(AttnItem), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->pre_last, out_rows.data(), out_rows.size() * 4, cudaMemcpyHostToDevice, c->st));
  bool pending = false;
  forward_layers(c, c->pre_tok, nullptr, T, c->pre_pos, c->pre_pt, c->items_pre, nullptr, (int)items.size(), false,
                 T, &pending);
  launch_rmsnorm(c->x, pending ? c->ar : nullptr, c->pre_last, nullptr, (int)out_rows.size(), nullptr, c->h, c->m.d,
                 c->m.eps, c->st, c->h_lo);
  c->launches++;
  gemm(c, c->p_lm, c->m.V, c->m.d, nullptr, (int)out_rows.size(), 1, EPI_F32, c->logits, c->m.V, nullptr);
  CK(cudaGetLastError());
  return RP_OK;
}

int rp_submit_round(void* ctx, const rp_prompt* prompts, int32_t n, int32_t G, int32_t keep, int32_t cap,
                    int32_t target, int32_t flags, int64_t round_id) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (c->active) return c->fail(RP_EBUSY, "a round is active (collect it first)");
  const int kind = flags & RP_LONG ? 1 : 0;
  const int trace = flags & RP_TRACE ? 1 : 0;
  const int preempt = flags & RP_PREEMPT ? 1 : 0;
  if (preempt && c->issue_cap > 0)
    return c->fail(RP_EINVAL, "invalid field: flags (RP_PREEMPT with continuous issuance is not supported)");
  if (G < 1) return c->fail(RP_EINVAL, "invalid field: G (>= 1)");
  if (keep == 0) keep = G;
  if (keep < 1 || keep > G) return c->fail(RP_EINVAL, "invalid field: keep (1..G, 0 = G)");
  if (kind == 1 && keep != G) return c->fail(RP_EINVAL, "invalid field: keep (RP_LONG needs keep == G)");
  if (n < 1) return c->fail(RP_EINVAL, "invalid field: n_prompts (>= 1)");
  if (cap < 1 || cap > c->rd.max_cap) return c->fail(RP_EINVAL, "invalid field: cap (1..max_cap)");
  if (target < 1 || target > n) return c->fail(RP_EINVAL, "invalid field: target (1..n_prompts)");
  if (kind == 1 && target != n) return c->fail(RP_EINVAL, "invalid field: target (RP_LONG needs target == n_prompts)");
  // the full list (this rank's slice is decoded).  A NULL list takes the head
  // of the (global) long-prompt queue; the entries leave the queue only once
  // the round has started, so a failed submit loses no prompt
  std::vector<QueuedPrompt> all;
  int pop = 0;
  if (!prompts) {
    if ((int)c->fifo.size() < n) return c->fail(RP_EINVAL, "invalid field: n_prompts (queue holds %zu)", c->fifo.size());
    all.assign(c->fifo.begin(), c->fifo.begin() + n);
    for (auto& q : all)   // the long round re-rolls the prompt (reading Z5)
      if (!q.trace_retry.empty()) q.trace = q.trace_retry;
    pop = n;
  } else {
    all.resize(n);
    for (int i = 0; i < n; ++i) {
      const rp_prompt& p = prompts[i];
      if (p.len < 1 || !p.tokens) return c->fail(RP_EINVAL, "invalid field: prompts[%d].len/tokens", i);
      if (p.len > c->rd.max_prompt_len) return c->fail(RP_EINVAL, "invalid field: prompts[%d].len > max_prompt_len", i);
      all[i].id = p.prompt_id;
      all[i].tokens.assign(p.tokens, p.tokens + p.len);
      for (int t : all[i].tokens)
        if (t < 0 || t >= c->md.vocab || t == c->m.eos) return c->fail(RP_EINVAL, "invalid field: prompts[%d].tokens", i);
      if (trace) {
        if (!p.trace_lens) return c->fail(RP_EINVAL, "invalid field: prompts[%d].trace_lens (RP_TRACE)", i);
        all[i].trace.assign(p.trace_lens, p.trace_lens + G);
        for (int L : all[i].trace)
          if (L < 1) return c->fail(RP_EINVAL, "invalid field: prompts[%d].trace_lens (>= 1)", i);
        if (p.trace_lens_retry) {
          all[i].trace_retry.assign(p.trace_lens_retry, p.trace_lens_retry + G);
          for (int L : all[i].trace_retry)
            if (L < 1) return c->fail(RP_EINVAL, "invalid field: prompts[%d].trace_lens_retry (>= 1)", i);
        }
      }
    }
  }
  if (trace)
    for (auto& p : all) {
      if ((int)p.trace.size() < G) return c->fail(RP_EINVAL, "invalid field: trace_lens (queued prompt lacks a trace)");
      p.trace.resize(G);   // a queued prompt re-runs with the long round's G (= R0)
    }
  // contiguous slice of this rank
  const int W = c->rd.world, r = c->rd.rank;
  const int base = n / W, extra = n % W;
  const int lo = r * base + std::min(r, extra);
  const int n_loc = base + (r < extra ? 1 : 0);
  if (n_loc > c->z.P) return c->fail(RP_ENOSPC, "prompts on this rank %d > max_prompts %d", n_loc, c->z.P);
  if (n_loc * G > c->z.S) return c->fail(RP_ENOSPC, "sequences on this rank %d > max_seqs %d", n_loc * G, c->z.S);
  long long T = 0;
  for (int i = 0; i < n_loc; ++i) T += (long long)all[lo + i].tokens.size();
  if (T > c->rd.max_prompt_tokens) return c->fail(RP_ENOSPC, "prompt tokens %lld > max_prompt_tokens", T);

  // continuous issuance: the first min(A, n_loc) prompts start at step 1, the
  // others are prefilled without their last token, which they decode as their
  // first step once issued (oracle sched.issue_step_loop)
  const int A = c->issue_cap > 0 ? std::min(c->issue_cap, n_loc) : 0;
  if (A > 0)
    for (int i = A; i < n_loc; ++i)
      if (all[lo + i].tokens.size() < 2)
        return c->fail(RP_EINVAL, "invalid field: prompts[%d].len (continuous issuance needs >= 2)", lo + i);
  c->kind = kind; c->trace = trace; c->G = G; c->keep = keep; c->cap = cap; c->target = target; c->n_glob = n;
  c->max_active = A;
  c->lo = lo; c->n_loc = n_loc; c->round_id = round_id;
  c->round_prompts.assign(all.begin() + lo, all.begin() + lo + n_loc);
  c->round_all = all;
  RoundDev& R = c->R;
  R.cap = cap; R.G = G; R.keep = keep; R.target = target; R.kind = kind; R.trace = trace; R.n_prompts = n_loc;
  R.max_active = A;
  R.preempt = preempt;
  const int n_first = A > 0 ? A : n_loc;   // prompts live at step 1
  R.trace_buf = c->trace_dev; R.trace_steps = c->trace_steps;

  // ---- host plan: prompt pages, sibling page tables, fork jobs
  const int S = c->z.S, maxp = c->z.maxp;
  int top = c->n_pages;
  std::vector<int> toks, plen(n_loc), last(n_first), last_tok(n_loc);
  for (int p = 0; p < n_loc; ++p) {
    const auto& tk = c->round_prompts[p].tokens;
    plen[p] = (int)tk.size() - (p >= n_first ? 1 : 0);
    last_tok[p] = tk.back();
    toks.insert(toks.end(), tk.begin(), tk.begin() + plen[p]);
    if (p < n_first) last[p] = (int)toks.size() - 1;
  }
  std::vector<std::vector<int>> ppages;
  if (n_loc > 0) {
    int rc = prefill(c, toks, plen, top, ppages, last);
    if (rc) return rc;
  }
  const int nS = n_loc * G;
  std::vector<int> slot_prompt(nS), slot_j(nS), kv_len(nS), zeros(std::max(nS, n_loc), 0), trL(nS, 0), own0(nS),
      live(n_first * G), gid(n_loc), ptab((size_t)std::max(nS, 1) * maxp, 0), jobs;
  for (int p = 0; p < n_loc; ++p) {
    gid[p] = c->round_prompts[p].id;
    for (int j = 0; j < G; ++j) {
      const int s = p * G + j;
      slot_prompt[s] = p; slot_j[s] = j; kv_len[s] = plen[p];
      if (p < n_first) live[s] = s;
      trL[s] = trace ? c->round_prompts[p].trace[j] : 0;
      const int full = plen[p] / kPage;
      for (int k = 0; k < full; ++k) ptab[(size_t)s * maxp + k] = ppages[p][k];
      own0[s] = full;
      if (plen[p] % kPage) {
        if (top <= 0) return c->fail(RP_ENOMEM_KV, "KV pool exhausted forking prompt pages");
        const int pg = --top;
        ptab[(size_t)s * maxp + full] = pg;
        jobs.push_back(ppages[p][full]); jobs.push_back(pg); jobs.push_back(plen[p] % kPage);
      }
    }
  }
  auto up = [&](int* dst, const std::vector<int>& v, size_t count) {
    return cudaMemcpyAsync(dst, v.data(), count * 4, cudaMemcpyHostToDevice, c->st);
  };
  CK(idle(c));   // the prefill may end in (TP) collectives
  if (nS > 0) {
    CK(up(R.slot_prompt, slot_prompt, nS)); CK(up(R.slot_j, slot_j, nS)); CK(up(R.kv_len, kv_len, nS));
    CK(up(R.gen, zeros, nS)); CK(up(R.status, zeros, nS)); CK(up(R.trace_L, trL, nS)); CK(up(R.own0, own0, nS));
    CK(up(R.live, live, (size_t)n_first * G)); CK(up(R.page_table, ptab, (size_t)nS * maxp)); CK(up(R.t0, zeros, nS));
    CK(cudaMemsetAsync(R.best, 0, (size_t)nS * 8, c->st));
  }
  if (n_loc > 0) {
    CK(up(R.p_gid, gid, n_loc)); CK(up(R.p_cnt, zeros, n_loc)); CK(up(R.p_state, zeros, n_loc));
    std::vector<int> ident(n_loc);
    for (int p = 0; p < n_loc; ++p) ident[p] = p;                  // admission stamps: index order
    CK(up(R.p_plen, plen, n_loc)); CK(up(R.p_adm, ident, n_loc)); CK(up(R.p_wait, zeros, n_loc));
    CK(up(R.p_last_tok, last_tok, n_loc)); CK(up(R.p_stamp, zeros, n_loc));
  }
  if (!jobs.empty()) {
    CK(up(c->fork_jobs, jobs, jobs.size()));
    launch_kv_fork(c->fork_jobs, (int)jobs.size() / 3, c->rd.kv_pool, c->m, c->st);
    c->launches++;
  }
  CK(cudaMemcpyAsync(R.free_stack, c->identity_pages, (size_t)c->n_pages * 4, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemsetAsync(R.rows_hist, 0, ((size_t)c->z.S + 1) * sizeof(unsigned long long), c->st));
  CtlBlock cb{};
  cb.n_live = n_first * G; cb.t = 1; cb.free_top = top; cb.n_issued = n_first;
  cb.adm_ctr = n_loc - 1;
  *c->h_ctl = cb;
  CK(cudaMemcpyAsync(R.ctl, c->h_ctl, sizeof(CtlBlock), cudaMemcpyHostToDevice, c->st));
  if (c->trace_dev) CK(cudaMemsetAsync(c->trace_dev, 0, (size_t)c->trace_steps * (2 + S) * 4, c->st));
  // ---- step 1: token 1 of every sibling from its prompt's prefill logits
  launch_sampler(c->logits, c->m.V, c->m.v0, G, R, c->rd.sample_seed, 1.0f / c->rd.temperature, (uint32_t)round_id,
                 c->st);
  c->launches++;
  if (c->tp > 1 && nS > 0) coll_allreduce_max_u64(c, c->tpc, R.best, (size_t)n_first * G);
  if (c->rd.world == 1) {
    launch_ctl(R, 0, 0, c->st); c->launches++;
  } else {
    launch_ctl(R, 0, 1, c->st); c->launches++;
    coll_allgather_i32(c, c->dp, R.ks_local, R.ks, 4);
    launch_ctl(R, 0, 2, c->st); c->launches++;
  }
  CK(cudaGetLastError());
  for (int i = 0; i < pop; ++i) c->fifo.pop_front();
  c->active = true;
  c->collected = false;
  c->step_logits_valid = false;
  c->graph_dirty = true;
  return RP_OK;
}

static int read_ctl(RpCtx* c) {
  CK(cudaMemcpyAsync(c->h_ctl, c->R.ctl, sizeof(CtlBlock), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

static void fill_status(RpCtx* c, rp_status* st) {
  if (!st) return;
  const CtlBlock& b = *c->h_ctl;
  st->round_id = c->round_id; st->kind = c->kind;
  st->t = b.done ? b.t_end : b.t - 1;
  st->n_live = b.done ? 0 : b.n_live;
  st->accepted = b.acc; st->accepted_local = b.acc_local; st->done = b.done; st->underfilled = b.underfilled;
  st->n_prompts_local = c->n_loc; st->decoded_tokens = b.decoded;
  st->kv_tokens_read = b.kv_read;
  st->kv_tokens_unique = b.kv_read_unique;
  st->preemptions = b.preemptions;
}

// KV recompute of response tokens (re-admission after preemption, Z26;
// migration of an in-flight round, Z27): for each segment the decoder runs
// the prefill kernels over tokens k0 .. k1-1 of slot s's response (positions
// plen + k), reading their keys from the slot's own page table and writing
// their KV; no LM head.  Pieces bounded by the prefill buffers.
struct RecomputeSeg { int s, plen, k0, k1; };
static int recompute_segments(RpCtx* c, std::vector<RecomputeSeg>& segs) {
  const int g_heads = c->m.H / c->m.KV, tpb = 16 / g_heads;
  const int tok_cap = c->rd.max_prompt_tokens;
  size_t si = 0;
  while (si < segs.size()) {
    // one piece: whole or partial segments within the token and item capacities
    std::vector<int> pos, pt;
    std::vector<AttnItem> items;
    std::vector<std::array<int, 4>> copies;   // dst offset, slot, k0, count
    int T = 0;
    while (si < segs.size() && T < tok_cap) {
      RecomputeSeg& sg = segs[si];
      int take = std::min(sg.k1 - sg.k0, tok_cap - T);
      // items of these tokens: ceil(nq / tpb) blocks x ceil(keys / chunk) splits each
      auto n_items_for = [&](int k0, int cnt) {
        int it = 0;
        for (int b0 = 0; b0 < cnt; b0 += tpb) {
          const int hi = sg.plen + k0 + std::min(b0 + tpb, cnt);
          it += (hi + kAttnChunk - 1) / kAttnChunk;
        }
        return it;
      };
      while (take > 0 && (int)items.size() + n_items_for(sg.k0, take) > c->z.max_items_pre) take /= 2;
      if (take <= 0) break;
      const int off = T;
      for (int k = 0; k < take; ++k) { pos.push_back(sg.plen + sg.k0 + k); pt.push_back(sg.s); }
      for (int b0 = 0; b0 < take; b0 += tpb) {
        const int nq = std::min(tpb, take - b0);
        const int p0 = sg.plen + sg.k0 + b0, hi = p0 + nq;
        const int ns = (hi + kAttnChunk - 1) / kAttnChunk, item0 = (int)items.size();
        for (int sp = 0; sp < ns; ++sp) {
          AttnItem I;
          I.q_row0 = off + b0; I.n_qtok = nq; I.pos0 = p0; I.pt_row = sg.s;
          I.kv_lo = sp * kAttnChunk; I.kv_hi = std::min(hi, (sp + 1) * kAttnChunk);
          I.nsplit = ns; I.item0 = item0;
          items.push_back(I);
        }
      }
      copies.push_back({off, sg.s, sg.k0, take});
      T += take;
      sg.k0 += take;
      if (sg.k0 >= sg.k1) ++si;
    }
    if (T == 0) return c->fail(RP_ENOSPC, "recompute: prefill buffers too small for one token");
    CK(idle(c));
    for (auto& cp : copies)
      CK(cudaMemcpyAsync(c->pre_tok + cp[0], c->R.tok_out + (size_t)cp[1] * c->R.cap + cp[2],   // row stride: the round's cap
                         (size_t)cp[3] * 4, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->pre_pos, pos.data(), T * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->pre_pt, pt.data(), T * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->items_pre, items.data(), items.size() * sizeof(AttnItem), cudaMemcpyHostToDevice, c->st));
    bool pending = false;
    forward_layers(c, c->pre_tok, nullptr, T, c->pre_pos, c->pre_pt, c->items_pre, nullptr, (int)items.size(), false,
                   T, &pending);
    CK(cudaGetLastError());
  }
  return RP_OK;
}

// Recompute of re-admitted responses (KV pressure, reading Z26), between
// two decode steps while the round is paused: copy the prompt's partial page
// into each response's first private page, then run the decoder over the
// response's tokens 1 .. g-1 at positions plen .. plen + g - 2 (prefill
// kernels; keys from the response's own page table), writing their KV; no LM
// head.  Pieces bounded by the prefill buffers.  Then resume the step.
static int recompute_paused(RpCtx* c) {
  CtlBlock& b = *c->h_ctl;
  const int nj = b.n_rejobs;
  if (nj > 0) {
    CK(cudaMemcpyAsync(c->rejobs_h, c->R.rejobs, (size_t)5 * nj * 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::vector<int> jobs;
    for (int j = 0; j < nj; ++j) {
      const int* J = c->rejobs_h + 5 * j;
      if (J[4] > 0) { jobs.push_back(J[2]); jobs.push_back(J[3]); jobs.push_back(J[4]); }
    }
    if (!jobs.empty()) {
      CK(idle(c));
      CK(cudaMemcpyAsync(c->fork_jobs, jobs.data(), jobs.size() * 4, cudaMemcpyHostToDevice, c->st));
      launch_kv_fork(c->fork_jobs, (int)jobs.size() / 3, c->rd.kv_pool, c->m, c->st);
      c->launches++;
    }
    // continuation segments (slot, first token index, end) in job order
    std::vector<RecomputeSeg> segs;
    for (int j = 0; j < nj; ++j) {
      const int* J = c->rejobs_h + 5 * j;
      const int s = J[0], g = J[1], plen = (int)c->round_prompts[s / c->G].tokens.size();
      if (g >= 2) segs.push_back({s, plen, 0, g - 1});
    }
    const int rc = recompute_segments(c, segs);
    if (rc) return rc;
  }
  // resume the held step
  b.pause = 0;
  b.n_live = b.n_live_saved;
  b.n_items = b.n_items_saved;
  b.n_gitems = b.n_gitems_saved;
  CK(cudaMemcpyAsync(c->R.ctl, c->h_ctl, sizeof(CtlBlock), cudaMemcpyHostToDevice, c->st));
  return RP_OK;
}

int rp_step(void* ctx, int32_t max_steps, rp_status* st) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (!c->active) return c->fail(RP_ESTATE, "no active round");
  int rc = read_ctl(c);
  if (rc) return rc;
  int steps = 0;
  while (!c->h_ctl->done && steps < max_steps) {
    if (c->h_ctl->pause) {                 // re-admitted responses wait for their KV
      if ((rc = recompute_paused(c))) return rc;
      continue;
    }
    // rows can grow inside a graph of graph_steps steps when prompts are issued
    const int grow = c->max_active ? std::min(c->max_active * c->G, c->h_ctl->n_live +
                                              (c->n_loc - c->h_ctl->n_issued) * c->G) : 0;
    const int bucket = bucket_for(c, std::max(c->h_ctl->n_live, grow));
    if ((rc = set_gmode(c))) return rc;
    if (c->prof_steps_left > 0) {
      const int rows = c->h_ctl->n_live;
      const long long ctx = c->h_ctl->ctx_sum;
      // the step is enqueued behind a gate kernel and released once every
      // launch is queued, so the kernels run back to back and no event
      // bracket contains host launch latency
      if (!c->gate_h) {
        int* hp = nullptr;
        CK(cudaHostAlloc(&hp, sizeof(int), cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(&c->gate_d, hp, 0));
        c->gate_h = hp;
      }
      *c->gate_h = 0;
      launch_host_gate(c->gate_d, c->st);
      decode_step(c, bucket);
      __sync_synchronize();
      *c->gate_h = 1;
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(c->st));
      for (size_t i = 0; i + 1 < c->ev.size(); i += 2) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]);
        c->prof_ms[c->ev_cls[i + 1]] += ms;
        c->prof_cnt[c->ev_cls[i + 1]] += 1;
      }
      c->ev.clear(); c->ev_cls.clear();
      c->prof_rows += rows; c->prof_ctx += ctx; c->prof_step_count += 1;
      c->prof_steps_left -= 1;
      steps += 1;
    } else if (c->rd.graph_steps > 0) {
      if ((rc = ensure_graph(c, bucket))) return rc;
      CK(cudaGraphLaunch(c->gexec, c->st));
      c->launches += c->graph_nodes;
      steps += c->rd.graph_steps;
      c->step_logits_valid = true;   // logits of the graph's last decoded step
    } else {
      decode_step(c, bucket);
      CK(cudaGetLastError());
      steps += 1;
      c->step_logits_valid = true;
    }
    if ((rc = read_ctl(c))) return rc;
  }
  fill_status(c, st);
  if (c->attn_tl) {   // debug: marks of the last attention launch, us from the earliest CTA start
    std::vector<long long> h((size_t)kSMs * 8);
    CK(cudaMemcpy(h.data(), c->attn_tl, h.size() * 8, cudaMemcpyDeviceToHost));
    long long t0 = LLONG_MAX;
    for (int b = 0; b < kSMs; ++b) if (h[(size_t)b * 8]) t0 = std::min(t0, h[(size_t)b * 8]);
    const char* nm[7] = {"start", "depwait", "page0", "lastpage", "written", "merged", "end"};
    fprintf(stderr, "attn timeline (n_live %d):", c->h_ctl->n_live);
    for (int k = 0; k < 7; ++k) {
      double sum = 0, mx = -1e30; int n = 0;
      for (int b = 0; b < kSMs; ++b) {
        const long long v = h[(size_t)b * 8 + k];
        if (v && v >= t0) { const double u = (v - t0) / 1e3; sum += u; mx = std::max(mx, u); ++n; }
      }
      if (n) fprintf(stderr, " %s=%.2f/%.2f(%d)", nm[k], sum / n, mx, n);
    }
    fprintf(stderr, "\n");
    CK(cudaMemset(c->attn_tl, 0, h.size() * 8));
  }
  if (c->h_ctl->err == 1) return c->fail(RP_ENOMEM_KV, "KV page pool exhausted (no preemption; reading Z17)");
  if (c->h_ctl->err == 2) return c->fail(RP_ENOSPC, "page table overflow (max_prompt_len + max_cap)");
  if (c->h_ctl->err == 3) return c->fail(RP_ENOSPC, "decode attention work list overflow (capacity %d)", c->z.max_items_dec);
  return RP_OK;
}

// Pack the responses of this rank's accepted prompts with acceptance index
// in [first, accepted so far) and copy them to the host (shared by rp_collect
// and rp_collect_ready).  n_out / n_tok may be queried with out == NULL.
static int collect_range(RpCtx* c, int first, rp_response* out, int32_t max_out, int32_t* tok_buf, int64_t tok_cap,
                         int32_t* n_out, int64_t* n_tok, std::vector<char>* accepted) {
  const int acc = c->h_ctl->acc_local;
  const int nr = std::max(0, acc - first) * c->keep;
  launch_collect_pack(c->R, first, c->col_meta, c->col_tok, c->st);
  c->launches += 2;
  std::vector<int> meta((size_t)4 * nr + nr + 1);
  CK(cudaMemcpyAsync(meta.data(), c->col_meta, (size_t)4 * nr * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(meta.data() + 4 * nr, c->col_meta + 4 * c->z.S, (size_t)(nr + 1) * 4,
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const int64_t total = meta[4 * nr + nr];
  if (n_out) *n_out = nr;
  if (n_tok) *n_tok = total;
  if (!out) return RP_OK;
  if (max_out < nr || tok_cap < total || !tok_buf) return c->fail(RP_ENOSPC, "collect buffers too small");
  if (total > 0) CK(cudaMemcpyAsync(tok_buf, c->col_tok, total * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (int r = 0; r < nr; ++r) {
    const int p = meta[4 * r];
    if (accepted) (*accepted)[p] = 1;
    out[r].prompt_id = c->round_prompts[p].id;
    out[r].j = meta[4 * r + 1];
    out[r].len = meta[4 * r + 2];
    out[r].finish = meta[4 * r + 3] == ST_CAPPED ? RP_FINISH_CAP : RP_FINISH_EOS;
    out[r].tok_off = meta[4 * nr + r];
  }
  return RP_OK;
}

int rp_collect(void* ctx, rp_response* out, int32_t max_out, int32_t* tok_buf, int64_t tok_cap, int32_t* n_out,
               int64_t* n_tok) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (!c->active) return c->fail(RP_ESTATE, "no active round");
  int rc = read_ctl(c);
  if (rc) return rc;
  if (!c->h_ctl->done) return c->fail(RP_ESTATE, "round not done");
  std::vector<char> accepted(c->n_loc, 0);
  if ((rc = collect_range(c, 0, out, max_out, tok_buf, tok_cap, n_out, n_tok, &accepted))) return rc;
  if (!out) return RP_OK;
  if (c->kind == 0) {
    // Deferral (reading Z7): every issued, unaccepted prompt of the
    // round joins the long-prompt queue in submission order.  Under DP the
    // ranks all-gather {accepted flags of their slice, prompts issued}, so
    // every rank appends the same prompts: the queue is global.
    const int W = c->rd.world, P1 = c->z.P + 1;
    std::vector<int> memb((size_t)P1 * W, 0);
    for (int p = 0; p < c->n_loc; ++p) memb[p] = accepted[p];
    memb[P1 - 1] = std::min(c->h_ctl->n_issued, c->n_loc);
    if (W > 1) {
      // pinned staging: the copy back is queued behind the collective
      memcpy(c->memb_h, memb.data(), (size_t)P1 * 4);
      CK(cudaMemcpyAsync(c->memb, c->memb_h, (size_t)P1 * 4, cudaMemcpyHostToDevice, c->st));
      coll_allgather_i32(c, c->dp, c->memb, c->memb + P1, (size_t)P1);
      CK(cudaMemcpyAsync(c->memb_h + P1, c->memb + P1, (size_t)P1 * W * 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      memcpy(memb.data(), c->memb_h + P1, (size_t)P1 * W * 4);
    }
    const int n = c->n_glob, base = n / W, extra = n % W;
    for (int q = 0; q < W; ++q) {
      const int lo_q = q * base + std::min(q, extra), n_q = base + (q < extra ? 1 : 0);
      const int* mq = memb.data() + (size_t)q * P1;
      for (int i = 0; i < n_q; ++i)
        if (!mq[i] && i < mq[P1 - 1]) c->fifo.push_back(c->round_all[lo_q + i]);
    }
  }
  c->active = false;
  c->collected = true;
  return RP_OK;
}

int rp_collect_ready(void* ctx, int32_t first, rp_response* out, int32_t max_out, int32_t* tok_buf, int64_t tok_cap,
                     int32_t* n_out, int64_t* n_tok, int32_t* n_accepted) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (!c->active) return c->fail(RP_ESTATE, "no active round");
  int rc = read_ctl(c);
  if (rc) return rc;
  if (first < 0 || first > c->h_ctl->acc_local) return c->fail(RP_EINVAL, "invalid field: first");
  if (n_accepted) *n_accepted = c->h_ctl->acc_local;
  return collect_range(c, first, out, max_out, tok_buf, tok_cap, n_out, n_tok, nullptr);
}

int rp_tp_ipc_handle(void* ctx, void* out) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c || !out) return RP_EINVAL;
  if (!c->tp_ipc) return c->fail(RP_ESTATE, "no TP peer block (tp == 1 or d % 128 != 0)");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->tp_ipc));
  memcpy(out, &h, sizeof h);
  return RP_OK;
}

int rp_tp_ipc_open(void* ctx, const void* handles) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c || !handles) return RP_EINVAL;
  if (!c->tp_ipc) return c->fail(RP_ESTATE, "no TP peer block");
  if (c->active) return c->fail(RP_EBUSY, "a round is active");
  for (int q = 0; q < c->tp; ++q) {
    if (q == c->rd.tp_rank) { c->tp_peer_base[q] = c->tp_ipc; continue; }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)q * RP_IPC_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return c->fail(RP_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
    c->tp_peer_base[q] = p;
  }
  c->tp_peer = true;
  c->graph_dirty = true;
  return RP_OK;
}

int rp_round_rows_histogram(void* ctx, int64_t* out, int32_t n) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c || !out || n < 1) return RP_EINVAL;
  const int m = std::min(n, c->z.S + 1);
  std::vector<unsigned long long> h(m);
  CK(cudaMemcpyAsync(h.data(), c->R.rows_hist, (size_t)m * 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (int i = 0; i < n; ++i) out[i] = i < m ? (int64_t)h[i] : 0;
  return RP_OK;
}

// ---- migration of an in-flight round (reading Z27) --------
// The device state a round carries from one decode step to the next, in a
// fixed order; the KV cache is not part of it (recomputed on import).
struct StateSec { void* dev; size_t bytes; };
static std::vector<StateSec> round_sections(RpCtx* c) {
  RoundDev& R = c->R;
  const size_t S = c->z.S, P = c->z.P, MI = c->z.max_items_dec;
  return {{R.ctl, sizeof(CtlBlock)},       {R.live, S * 4},           {R.tok_in, S * 4},
          {R.row_pos, S * 4},              {R.row_pt, S * 4},         {R.items, MI * sizeof(AttnItem)},
          {R.gitems, (size_t)c->z.max_items_g * sizeof(AttnGroupItem)}, {R.kv_len, S * 4}, {R.gen, S * 4},
          {R.status, S * 4},               {R.t0, S * 4},             {R.tok_out, S * (size_t)R.cap * 4},
          {R.p_state, P * 4},              {R.p_cnt, P * 4},          {R.accept_order, P * 4},
          {R.rows_hist, (S + 1) * 8},      {R.p_adm, P * 4},          {R.p_wait, P * 4},
          {R.wait_q, P * 4}};
}
constexpr int64_t kStateMagic = 0x3153525052LL;   // "RPRS1"
constexpr int kStateHdr = 13;                      // int64 header words
static void state_header(RpCtx* c, int64_t* h) {
  const int64_t v[kStateHdr] = {kStateMagic, c->z.S, c->z.P, c->R.cap, c->z.max_items_dec, (int64_t)sizeof(CtlBlock),
                                c->G, c->n_loc, c->kind, c->keep, c->rd.world, c->tp, c->rd.rank};
  for (int i = 0; i < kStateHdr; ++i) h[i] = v[i];
}

int rp_round_state_bytes(void* ctx, int64_t* bytes) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c || !bytes) return RP_EINVAL;
  size_t b = kStateHdr * 8;
  for (auto& sec : round_sections(c)) b += sec.bytes;
  *bytes = (int64_t)b;
  return RP_OK;
}

int rp_round_export(void* ctx, void* buf, int64_t bytes) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (!buf) return c->fail(RP_EINVAL, "invalid field: buf");
  if (!c->active) return c->fail(RP_ESTATE, "no active round");
  // (a TP group's ranks hold identical round state: each exports its own copy)
  if (c->max_active) return c->fail(RP_EINVAL, "round export: continuous issuance is not supported");
  int64_t need = 0;
  rp_round_state_bytes(ctx, &need);
  if (bytes < need) return c->fail(RP_ENOSPC, "round export: buffer of %lld bytes < %lld", (long long)bytes, (long long)need);
  int rc = read_ctl(c);
  if (rc) return rc;
  const CtlBlock& b = *c->h_ctl;
  if (b.done) return c->fail(RP_ESTATE, "round export: the round is done (collect it)");
  if (b.pause) return c->fail(RP_ESTATE, "round export: a re-admission is pausing the round (step once more)");
  uint8_t* out = (uint8_t*)buf;
  state_header(c, (int64_t*)out);
  size_t off = kStateHdr * 8;
  for (auto& sec : round_sections(c)) {
    CK(cudaMemcpyAsync(out + off, sec.dev, sec.bytes, cudaMemcpyDeviceToHost, c->st));
    off += sec.bytes;
  }
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

// Import: the round is submitted again with the caller's original arguments
// (prompts, G, keep, cap, target, flags, round_id: prefill, page tables and
// step 1 are deterministic), then the exported step state replaces the
// device state, the page tables are grown / shrunk to the live responses'
// contexts, and the KV of every live response's generated tokens 1 .. g-1 is
// recomputed (prefill kernels), so the next decode step continues the round
// exactly where the exporting engine left it.
int rp_round_import(void* ctx, const rp_prompt* prompts, int32_t n, int32_t G, int32_t keep, int32_t cap,
                    int32_t target, int32_t flags, int64_t round_id, const void* buf, int64_t bytes) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (!buf || !prompts) return c->fail(RP_EINVAL, "invalid field: buf / prompts");
  // (TP: every rank of the group imports at the same step -- submit and the
  // recompute run the TP collectives)
  if (c->issue_cap > 0) return c->fail(RP_EINVAL, "round import: continuous issuance is not supported");
  if (bytes < kStateHdr * 8) return c->fail(RP_EINVAL, "round import: state of %lld bytes", (long long)bytes);
  const int64_t* hdr = (const int64_t*)buf;
  int64_t mine[kStateHdr];
  int rc = rp_submit_round(ctx, prompts, n, G, keep, cap, target, flags, round_id);
  if (rc) return rc;
  int64_t need = 0;
  rp_round_state_bytes(ctx, &need);   // the token rows follow this round's cap
  if (bytes != need) {
    c->active = false;
    return c->fail(RP_EINVAL, "round import: state of %lld bytes, this round needs %lld", (long long)bytes,
                   (long long)need);
  }
  state_header(c, mine);
  for (int i = 0; i < kStateHdr; ++i)
    if (hdr[i] != mine[i]) {
      c->active = false;
      return c->fail(RP_EINVAL, "round import: state header word %d is %lld, this round has %lld", i,
                     (long long)hdr[i], (long long)mine[i]);
    }
  const std::vector<StateSec> secs = round_sections(c);
  std::vector<const uint8_t*> src(secs.size());
  size_t off = kStateHdr * 8;
  for (size_t i = 0; i < secs.size(); ++i) { src[i] = (const uint8_t*)buf + off; off += secs[i].bytes; }
  const CtlBlock& ex = *(const CtlBlock*)src[0];
  const int* ex_kv = (const int*)src[7];
  const int* ex_gen = (const int*)src[8];
  const int* ex_status = (const int*)src[9];
  if (ex.done || ex.pause) return c->fail(RP_EINVAL, "round import: the exported round is done or paused");
  // after submit: step 1 decoded, private pages for positions <= plen of the live responses
  if ((rc = read_ctl(c))) return rc;
  const int S = c->z.S, maxp = c->z.maxp, nS = c->n_loc * c->G;
  std::vector<int> st_now(S), kv_now(S), ptab((size_t)S * maxp), fstack(c->n_pages);
  CK(cudaMemcpyAsync(st_now.data(), c->R.status, (size_t)S * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(kv_now.data(), c->R.kv_len, (size_t)S * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(ptab.data(), c->R.page_table, ptab.size() * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(fstack.data(), c->R.free_stack, fstack.size() * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  int top = c->h_ctl->free_top;
  auto pages_of = [](int tokens) { return (tokens + kPage - 1) / kPage; };
  std::vector<RecomputeSeg> segs;
  // private pages: release those of responses that are no longer live (all
  // slots first, so a tight pool is not exhausted by the order), then grow
  // the live ones to their exported contexts
  for (int pass = 0; pass < 2; ++pass)
    for (int s = 0; s < nS; ++s) {
      const int plen = (int)c->round_prompts[s / c->G].tokens.size(), own0 = plen / kPage;
      const int cur = st_now[s] == ST_LIVE ? pages_of(kv_now[s] + 1) - own0 : 0;
      const int want = ex_status[s] == ST_LIVE ? pages_of(ex_kv[s] + 1) - own0 : 0;
      if (pass == 0) {
        for (int k = want; k < cur; ++k) fstack[top++] = ptab[(size_t)s * maxp + own0 + k];
        continue;
      }
      for (int k = cur; k < want; ++k) {
        if (top <= 0) { c->active = false; return c->fail(RP_ENOMEM_KV, "round import: KV pool exhausted"); }
        ptab[(size_t)s * maxp + own0 + k] = fstack[--top];
      }
      if (ex_status[s] == ST_LIVE && ex_gen[s] >= 2) segs.push_back({s, plen, 0, ex_gen[s] - 1});
    }
  CK(idle(c));
  CK(cudaMemcpyAsync(c->R.page_table, ptab.data(), ptab.size() * 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->R.free_stack, fstack.data(), (size_t)top * 4, cudaMemcpyHostToDevice, c->st));
  for (size_t i = 1; i < secs.size(); ++i)
    CK(cudaMemcpyAsync(secs[i].dev, src[i], secs[i].bytes, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->R.best, 0, (size_t)S * 8, c->st));
  // the KV of the generated tokens (the next step appends token g itself)
  if ((rc = recompute_segments(c, segs))) { c->active = false; return rc; }
  *c->h_ctl = ex;
  c->h_ctl->free_top = top;
  c->h_ctl->err = 0;
  CK(cudaMemcpyAsync(c->R.ctl, c->h_ctl, sizeof(CtlBlock), cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->step_logits_valid = false;
  c->graph_dirty = true;
  return RP_OK;
}

// Re-shard exported DP rank states to another world size (the rollout GPU
// set shrinks or grows mid-round, Z27).  The prompts are split contiguously by
// global index on both sides (as rp_submit_round does), so every prompt's
// per-response and per-prompt state moves whole; the next step's inputs are
// rebuilt from the live responses in slot order with one attention item per
// row (ctl re-balances the splits from the step after), the local acceptance
// order is the accepted prompts ordered by (completion step, index) -- the
// order the cutoff admitted them in -- and the measurement counters land on
// the new rank 0.
static std::vector<size_t> state_sizes(int64_t S, int64_t P, int64_t cap, int64_t MI) {
  return {sizeof(CtlBlock), (size_t)S * 4, (size_t)S * 4, (size_t)S * 4, (size_t)S * 4, (size_t)MI * sizeof(AttnItem),
          (size_t)(S + MI) * sizeof(AttnGroupItem),   // max_items_g = 2 S + 3 U1 = S + max_items_dec
          (size_t)S * 4, (size_t)S * 4, (size_t)S * 4, (size_t)S * 4,
          (size_t)S * cap * 4, (size_t)P * 4, (size_t)P * 4, (size_t)P * 4, (size_t)(S + 1) * 8,
          (size_t)P * 4, (size_t)P * 4, (size_t)P * 4};
}

int rp_round_reshard(const void* const* states, const int64_t* bytes, int32_t n_states, int32_t n_prompts,
                     int32_t new_world, int32_t new_rank, void* out, int64_t out_bytes, int64_t* need) {
  auto bad = [](const char* m) { g_init_err = m; return RP_EINVAL; };
  if (!states || !bytes || n_states < 1 || new_world < 1 || new_rank < 0 || new_rank >= new_world || n_prompts < 1)
    return bad("round reshard: invalid arguments");
  const int64_t* h0 = (const int64_t*)states[0];
  if (bytes[0] < kStateHdr * 8 || h0[0] != kStateMagic) return bad("round reshard: not a round state");
  const int64_t S = h0[1], P = h0[2], cap = h0[3], MI = h0[4], G = h0[6], kind = h0[8], keep = h0[9];
  if (h0[5] != (int64_t)sizeof(CtlBlock)) return bad("round reshard: state from another library version");
  const std::vector<size_t> sz = state_sizes(S, P, cap, MI);
  size_t total = kStateHdr * 8;
  for (size_t x : sz) total += x;
  if (need) *need = (int64_t)total;
  if (!out) return RP_OK;
  if (out_bytes < (int64_t)total) return bad("round reshard: output buffer too small");
  if (h0[10] != n_states) return bad("round reshard: need one state per old rank");
  auto part = [&](int world, int r, int& lo, int& nl) {
    const int base = n_prompts / world, extra = n_prompts % world;
    lo = r * base + std::min(r, extra);
    nl = base + (r < extra ? 1 : 0);
  };
  // section pointers of every old rank
  std::vector<std::vector<const uint8_t*>> sec(n_states);
  for (int r = 0; r < n_states; ++r) {
    const int64_t* h = (const int64_t*)states[r];
    if (bytes[r] != (int64_t)total || h[0] != kStateMagic || h[1] != S || h[2] != P || h[3] != cap || h[4] != MI ||
        h[6] != G || h[10] != n_states || h[11] != 1 || h[12] != r)
      return bad("round reshard: states of different shapes or ranks");
    int lo, nl;
    part(n_states, r, lo, nl);
    if (h[7] != nl) return bad("round reshard: state slice does not match n_prompts");
    const CtlBlock& cb = *(const CtlBlock*)((const uint8_t*)states[r] + kStateHdr * 8);
    if (cb.done || cb.pause || cb.wait_head != cb.wait_tail || cb.preemptions)
      return bad("round reshard: done, paused or preempted rounds are not supported");
    size_t off = kStateHdr * 8;
    for (size_t x : sz) { sec[r].push_back((const uint8_t*)states[r] + off); off += x; }
  }
  int nlo, nn;
  part(new_world, new_rank, nlo, nn);
  if ((int64_t)nn > P || (int64_t)nn * G > S) return bad("round reshard: the new slice exceeds max_prompts / max_seqs");
  std::vector<uint8_t> buf(total, 0);
  int64_t* ho = (int64_t*)buf.data();
  const int64_t hv[kStateHdr] = {kStateMagic, S, P, cap, MI, (int64_t)sizeof(CtlBlock), G, nn, kind, keep,
                                 new_world, 1, new_rank};
  for (int i = 0; i < kStateHdr; ++i) ho[i] = hv[i];
  std::vector<uint8_t*> o;
  {
    size_t off = kStateHdr * 8;
    for (size_t x : sz) { o.push_back(buf.data() + off); off += x; }
  }
  auto I32 = [](const uint8_t* p) { return (const int*)p; };
  auto O32 = [](uint8_t* p) { return (int*)p; };
  struct Acc { int step, gidx, nli; };
  std::vector<Acc> acc;
  for (int nli = 0; nli < nn; ++nli) {
    const int gi = nlo + nli;
    int r = 0, lo = 0, nl = 0;
    for (r = 0; r < n_states; ++r) {
      part(n_states, r, lo, nl);
      if (gi < lo + nl) break;
    }
    const int li = gi - lo;
    O32(o[12])[nli] = I32(sec[r][12])[li];
    O32(o[13])[nli] = I32(sec[r][13])[li];
    std::vector<int> fin;
    int t0 = 0;
    for (int j = 0; j < G; ++j) {
      const int os = li * (int)G + j, ns = nli * (int)G + j;
      for (int k : {7, 8, 9, 10}) O32(o[k])[ns] = I32(sec[r][k])[os];
      memcpy(o[11] + (size_t)ns * cap * 4, sec[r][11] + (size_t)os * cap * 4, (size_t)cap * 4);
      const int st = I32(sec[r][9])[os];
      t0 = I32(sec[r][10])[os];
      if (st == ST_FINISHED || st == ST_CAPPED || st == ST_DROPPED) fin.push_back(I32(sec[r][8])[os]);
    }
    if (O32(o[12])[nli] == PS_ACCEPTED) {
      std::sort(fin.begin(), fin.end());
      const int k = (int)std::min<int64_t>(keep, (int64_t)fin.size());
      acc.push_back({t0 + (k > 0 ? fin[k - 1] : 0), gi, nli});
    }
  }
  std::sort(acc.begin(), acc.end(), [](const Acc& a, const Acc& b) {
    return a.step != b.step ? a.step < b.step : a.gidx < b.gidx;
  });
  for (size_t k = 0; k < acc.size(); ++k) O32(o[14])[k] = acc[k].nli;
  // next-step inputs: the live responses in slot order
  int n_live = 0;
  long long ctx_sum = 0;
  AttnItem* items = (AttnItem*)o[5];
  for (int ns = 0; ns < nn * (int)G; ++ns) {
    if (O32(o[9])[ns] != ST_LIVE) continue;
    const int kv = O32(o[7])[ns], g = O32(o[8])[ns];
    O32(o[1])[n_live] = ns;
    O32(o[2])[n_live] = I32(o[11] + (size_t)ns * cap * 4)[g - 1];
    O32(o[3])[n_live] = kv;
    O32(o[4])[n_live] = ns;
    AttnItem I;
    I.q_row0 = n_live; I.n_qtok = 1; I.pos0 = kv; I.pt_row = ns;
    I.kv_lo = 0; I.kv_hi = kv + 1; I.nsplit = 1; I.item0 = n_live;
    items[n_live] = I;
    ctx_sum += kv + 1;
    ++n_live;
  }
  CtlBlock cb = *(const CtlBlock*)sec[0][0];     // global fields: t, acc, ...
  long long decoded = 0, kv_read = 0, kv_unique = 0;
  std::vector<unsigned long long> hist(S + 1, 0);
  for (int r = 0; r < n_states; ++r) {
    const CtlBlock& x = *(const CtlBlock*)sec[r][0];
    decoded += x.decoded;
    kv_read += x.kv_read;
    kv_unique += x.kv_read_unique;
    const unsigned long long* hx = (const unsigned long long*)sec[r][15];
    for (int64_t i = 0; i <= S; ++i) hist[i] += hx[i];
  }
  cb.n_live = n_live; cb.n_next = n_live; cb.n_items = n_live; cb.n_gitems = 0; cb.ctx_sum = ctx_sum;
  cb.acc_local = (int)acc.size(); cb.n_issued = nn; cb.issue_n = 0; cb.k_step = 0; cb.need_pages = 0;
  cb.decoded = new_rank == 0 ? decoded : 0;
  cb.kv_read = new_rank == 0 ? kv_read : 0;
  cb.kv_read_unique = new_rank == 0 ? kv_unique : 0;
  cb.err = 0; cb.underfilled = 0; cb.n_rejobs = 0; cb.readmit_n = cb.readmit_rows = cb.readmit_pages = 0;
  memcpy(o[0], &cb, sizeof(CtlBlock));
  if (new_rank == 0) memcpy(o[15], hist.data(), (size_t)(S + 1) * 8);
  for (int nli = 0; nli < nn; ++nli) O32(o[16])[nli] = nli;   // admission stamps: index order (as submit)
  cb.adm_ctr = nn - 1;
  memcpy(o[0], &cb, sizeof(CtlBlock));
  memcpy(out, buf.data(), total);
  return RP_OK;
}

int rp_round_issue_cap(void* ctx, int32_t max_active) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (max_active < 0) return c->fail(RP_EINVAL, "invalid field: max_active (>= 0)");
  if (c->active) return c->fail(RP_EBUSY, "a round is active (collect it first)");
  c->issue_cap = max_active;
  return RP_OK;
}

int rp_round_unissued(void* ctx, int32_t* ids_out, int32_t max, int32_t* n_out) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (c->active) {
    int rc = read_ctl(c);
    if (rc) return rc;
    if (!c->h_ctl->done) return c->fail(RP_ESTATE, "round not done");
  }
  const int n_is = c->round_prompts.empty() ? 0 : std::min(c->h_ctl->n_issued, c->n_loc);
  const int n = c->n_loc - n_is;
  if (n_out) *n_out = n;
  if (!ids_out) return RP_OK;
  if (max < n) return c->fail(RP_ENOSPC, "ids_out too small");
  for (int i = 0; i < n; ++i) ids_out[i] = c->round_prompts[n_is + i].id;
  return RP_OK;
}

int rp_long_queue(void* ctx, int32_t* ids_out, int32_t max, int32_t* n_out) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (n_out) *n_out = (int)c->fifo.size();
  if (!ids_out) return RP_OK;
  if (max < (int)c->fifo.size()) return c->fail(RP_ENOSPC, "ids_out too small");
  int i = 0;
  for (auto& q : c->fifo) ids_out[i++] = q.id;
  return RP_OK;
}

int rp_long_queue_pop(void* ctx, int32_t n) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (n < 0 || n > (int)c->fifo.size()) return c->fail(RP_EINVAL, "invalid field: n (queue holds %zu)", c->fifo.size());
  for (int i = 0; i < n; ++i) c->fifo.pop_front();
  return RP_OK;
}

// The tail-batching planner ("once the long-prompt queue reaches
// P0, a long round ... otherwise a short round over eta P0 fresh prompts";
// SPEC S:271-279 plan_round, S:277 ceil(eta * P0); reading Z7 for the drain).
int rp_plan_round(void* ctx, int32_t P0, float eta, int32_t drain, int32_t* kind, int32_t* n_prompts) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (P0 < 1) return c->fail(RP_EINVAL, "invalid field: P0 (>= 1)");
  if (!(eta >= 1.0f)) return c->fail(RP_EINVAL, "invalid field: eta (>= 1)");
  if (!kind || !n_prompts) return c->fail(RP_EINVAL, "invalid field: kind/n_prompts (NULL)");
  const int q = (int)c->fifo.size();
  if (q >= P0 || (drain && q > 0)) {
    *kind = RP_LONG;
    *n_prompts = std::min(q, P0);
  } else {
    *kind = RP_SHORT;
    // ceil in exact arithmetic: eta is a float (1.25 exactly); the tiny
    // margin keeps a product that lands on an integer from rounding up
    *n_prompts = (int)std::ceil((double)eta * (double)P0 - 1e-9);
  }
  return RP_OK;
}

// The parallelism planner's heuristic (oracle sched.plan_tp).
int rp_plan_tp(int32_t tp, int32_t tp_max, int64_t prev_preemptions, int64_t preemptions, int32_t zero_streak,
               int32_t* tp_next, int32_t* zero_streak_next) {
  if (!tp_next || !zero_streak_next || tp < 1 || tp_max < tp || preemptions < 0 || prev_preemptions < 0 ||
      zero_streak < 0) {
    g_init_err = "invalid field: rp_plan_tp arguments";
    return RP_EINVAL;
  }
  const int streak = preemptions == 0 ? zero_streak + 1 : 0;
  // a sudden rise (> 1.05x the previous round of this kind) doubles the TP size
  if (preemptions > 0 && (double)preemptions > 1.05 * (double)prev_preemptions) {
    *tp_next = std::min(2 * tp, tp_max);
    *zero_streak_next = 0;
  } else if (streak >= 4) {          // four rounds without preemption halve it
    *tp_next = std::max(tp / 2, 1);
    *zero_streak_next = 0;
  } else {
    *tp_next = tp;
    *zero_streak_next = streak;
  }
  return RP_OK;
}

int rp_local_group_create(int32_t world, int32_t tp, void** out) {
  if (!out || world < 1 || tp < 1 || tp > 8 || world * tp > 64) {
    g_init_err = "invalid field: world/tp/out";
    return RP_EINVAL;
  }
  RpLocalGroup* g = new RpLocalGroup();
  g->world = world;
  g->tp = tp;
  *out = g;
  return RP_OK;
}

void rp_local_group_free(void* group) {
  RpLocalGroup* g = (RpLocalGroup*)group;
  if (!g) return;
  for (auto& lc : g->dp) { if (lc.slots) cudaFree(lc.slots); if (lc.gen) cudaFree(lc.gen); }
  for (auto& lc : g->tpc) { if (lc.slots) cudaFree(lc.slots); if (lc.gen) cudaFree(lc.gen); }
  delete g;
}

int rp_debug_logits(void* ctx, const int32_t* tokens, int32_t n, float* logits_out) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (c->active) return c->fail(RP_EBUSY, "a round is active");
  if (n < 1 || n > c->rd.max_prompt_len || n > c->rd.max_prompt_tokens) return c->fail(RP_EINVAL, "invalid field: n");
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= c->md.vocab) return c->fail(RP_EINVAL, "invalid field: tokens[%d]", i);
  std::vector<int> toks(tokens, tokens + n), plen{n}, rows(n);
  for (int i = 0; i < n; ++i) rows[i] = i;
  int top = c->n_pages;
  std::vector<std::vector<int>> pp;
  int rc = prefill(c, toks, plen, top, pp, rows);
  if (rc) return rc;
  CK(idle(c));
  CK(cudaMemcpyAsync(logits_out, c->logits, (size_t)n * c->m.V * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

int rp_debug_trace_enable(void* ctx, int32_t steps) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (c->active) return c->fail(RP_EBUSY, "a round is active");
  if (c->trace_dev) { cudaFree(c->trace_dev); c->trace_dev = nullptr; }
  c->trace_steps = 0;
  if (steps > 0) {
    CK(cudaMalloc(&c->trace_dev, (size_t)steps * (2 + c->z.S) * 4));
    c->trace_steps = steps;
  }
  c->R.trace_buf = c->trace_dev; c->R.trace_steps = c->trace_steps;
  c->graph_dirty = true;
  return RP_OK;
}

int rp_debug_trace_get(void* ctx, int32_t* buf, int32_t steps) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (!c->trace_dev) return c->fail(RP_ESTATE, "trace not enabled");
  const int s = std::min(steps, c->trace_steps);
  CK(cudaMemcpyAsync(buf, c->trace_dev, (size_t)s * (2 + c->z.S) * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

int rp_debug_last_logits(void* ctx, float* logits_out, int32_t* slots_out, int32_t max_rows, int32_t* n_rows) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (!c->step_logits_valid) return c->fail(RP_ESTATE, "no decode step ran since submit");
  // rows of the last step were the live list before compaction: trace row t-1 holds it
  if (!c->trace_dev) return c->fail(RP_ESTATE, "needs rp_debug_trace_enable");
  int rc = read_ctl(c);
  if (rc) return rc;
  const int t = c->h_ctl->done ? c->h_ctl->t_end : c->h_ctl->t - 1;
  if (t < 1 || t > c->trace_steps) return c->fail(RP_ESTATE, "step outside the trace");
  std::vector<int> row(2 + c->z.S);
  CK(cudaMemcpyAsync(row.data(), c->trace_dev + (size_t)(t - 1) * (2 + c->z.S), row.size() * 4,
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const int n = row[0];
  if (n > max_rows) return c->fail(RP_ENOSPC, "max_rows too small");
  *n_rows = n;
  memcpy(slots_out, row.data() + 2, n * 4);
  CK(cudaMemcpyAsync(logits_out, c->logits, (size_t)n * c->m.V * 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return RP_OK;
}

int rp_debug_profile(void* ctx, int32_t steps, double* ms_out, int64_t* counts_out, int64_t* rows_ctx_steps) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  if (steps < 0) { c->prof_steps_left = 0; return RP_OK; }
  if (steps > 0) {   // arm: the next `steps` decode steps run eagerly, bracketed by events
    c->prof_steps_left = steps;
    for (int i = 0; i < RP_PROF_N; ++i) { c->prof_ms[i] = 0; c->prof_cnt[i] = 0; }
    c->prof_rows = c->prof_ctx = c->prof_step_count = 0;
    return RP_OK;
  }
  for (int i = 0; i < RP_PROF_N; ++i) {
    if (ms_out) ms_out[i] = c->prof_ms[i];
    if (counts_out) counts_out[i] = c->prof_cnt[i];
  }
  if (rows_ctx_steps) { rows_ctx_steps[0] = c->prof_rows; rows_ctx_steps[1] = c->prof_ctx; rows_ctx_steps[2] = c->prof_step_count; }
  return RP_OK;
}

int rp_debug_gemm(void* ctx, const void* W, const void* X, int32_t rows_cap, float* Y, int32_t M, int32_t N,
                  int32_t K, int32_t splits, int32_t iters, int32_t w_tiled, float* ms_out) {
  RpCtx* c = (RpCtx*)ctx;
  if (!c) return RP_EINVAL;
  pdl_mode(c);
  if (M % 128 || K % 64 || M <= 0 || K <= 0 || N < 0 || N > rows_cap) return c->fail(RP_EINVAL, "invalid GEMM shape");
  if (splits <= 0) splits = gemm_pick_splits(M, K, kSMs);
  splits = std::min(splits, K / 64);
  const int chunk = (w_tiled & 2) && N <= 128 ? 128 : 256;   // narrow split-precision chunks are 128 wide
  const size_t need = (size_t)(M / 128) * ((N + chunk - 1) / chunk) * splits * 256 * 128;
  if (splits > 1 && need > c->z.part_floats) return c->fail(RP_ENOSPC, "split-K workspace too small");
  if ((M / 128) * ((N + 255) / 256) > (1 << 15)) return c->fail(RP_ENOSPC, "too many tiles");
  GemmPlan p;
  // w_tiled bit 1: X holds [2][rows_cap][K] -- fp16 rows, then their residuals (split precision)
  const void* X_lo = (w_tiled & 2) ? (const void*)((const __half*)X + (size_t)rows_cap * K) : nullptr;
  if (make_plan(&p, W, M, K, X, rows_cap, w_tiled & 1, X_lo)) return c->fail(RP_ECUDA, "tensor map");
  iters = std::max(iters, 1);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const bool lo_saved = c->act_lo;
  c->act_lo = X_lo != nullptr;
  gemm(c, p, M, K, nullptr, N, splits, EPI_F32, Y, M, nullptr);   // warm
  if (getenv("RP_GEMM_TIMELINE")) {   // debug: per-CTA phase timeline of one launch, to stderr
    long long* tl = nullptr;
    CK(cudaMalloc(&tl, kSMs * 16 * sizeof(long long)));
    CK(cudaMemsetAsync(tl, 0, kSMs * 16 * sizeof(long long), c->st));
    GemmArgs a{};
    a.M = M; a.K = K; a.n_host = N; a.splits = splits; a.epi = EPI_F32; a.out = Y; a.ldo = M;
    a.dsm = gemm_dsm_enabled() && N <= 256 ? 1 : 0;   // taken when the split count fits a resident cluster grid
    a.partial = c->gpart; a.counters = c->gctr; a.timeline = tl;
    gemm_launch(p, a, kSMs, c->st);
    std::vector<long long> h(kSMs * 16);
    CK(cudaMemcpyAsync(h.data(), tl, h.size() * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    cudaFree(tl);
    long long t0 = LLONG_MAX, tend = 0;
    for (int b = 0; b < kSMs; ++b) if (h[b * 16]) t0 = std::min(t0, h[b * 16]);
    double acc[16] = {0}; int cnt[16] = {0};
    for (int b = 0; b < kSMs; ++b)
      for (int k = 0; k < 16; ++k)
        if (h[b * 16 + k]) { acc[k] += (h[b * 16 + k] - t0) / 1e3; cnt[k]++; tend = std::max(tend, h[b * 16 + k]); }
    fprintf(stderr, "gemm timeline M=%d N=%d K=%d splits=%d (us from first CTA start, mean over CTAs):", M, N, K, splits);
    const char* nm[16] = {"start", "setup", "it0_first", "it0_lastmma", "it1_first", "it1_lastmma", "it2_first",
                          "it2_lastmma", "it0_epi", "it1_epi", "it2_epi", "sk_partials", "sk_ticket", "sk_reduced", "sk_loaded", ""};
    for (int k = 0; k < 15; ++k) if (cnt[k]) fprintf(stderr, " %s=%.2f(%d)", nm[k], acc[k] / cnt[k], cnt[k]);
    fprintf(stderr, " end=%.2f\n", (tend - t0) / 1e3);
  }
  CK(cudaEventRecord(e0, c->st));
  for (int i = 0; i < iters; ++i) gemm(c, p, M, K, nullptr, N, splits, EPI_F32, Y, M, nullptr);
  c->act_lo = lo_saved;
  CK(cudaEventRecord(e1, c->st));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms_out) *ms_out = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return RP_OK;
}

}  // extern "C"
