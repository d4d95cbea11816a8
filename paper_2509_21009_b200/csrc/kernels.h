// Device data structures and launchers of the non-GEMM kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace rp {

// ST_DROPPED: finished (EOS) at the step its prompt completed but beyond the
// first `keep` (response-level speculation, ties to the lower j).
// ST_PREEMPTED: KV pressure (NEXT-2, reading Z26): the response's private
// pages were freed and its prompt waits for re-admission (recompute).
enum SeqStatus { ST_LIVE = 0, ST_FINISHED = 1, ST_CAPPED = 2, ST_ABORTED = 3, ST_DROPPED = 4, ST_PREEMPTED = 5 };
enum PromptState { PS_RUNNING = 0, PS_ACCEPTED = 1, PS_COMPLETE = 2 };
// per-prompt wait state (KV pressure): none / waiting / re-admitted at this step
enum WaitState { PW_NONE = 0, PW_WAITING = 1, PW_READMIT = 2, PW_VICTIM = 3 };

// One unit of attention work: a block of query tokens (decode: 1 token; the
// g query heads of a KV head form the MMA rows) against a key range.
struct AttnItem {
  int q_row0;   // first query row in q/attn_out
  int n_qtok;   // query tokens in the block
  int pos0;     // position of the first query token (token k may see keys <= pos0+k)
  int pt_row;   // page-table row
  int kv_lo, kv_hi;  // key range [lo, hi) of this split (lo multiple of kPage)
  int nsplit;   // splits of this query block (1 -> write output directly)
  int item0;    // index of the block's first item (partials of split s at item0+s)
};

// Decode attention over a group of <= 8 live siblings of one prompt
// (k_attn_group.cu): the shared prompt pages are read once for every member.
struct AttnGroupItem {
  int n_mem;        // members (live rows), <= 8
  int shared_np;    // leading pages shared by every member (identical page ids)
  int pg_lo, pg_hi; // page-index range of this split
  int nsplit;       // splits of the group (1 -> outputs written directly)
  int item0;        // the group's first item (split s: partials at item0 + s)
  int rep;          // consumer warps per member: 1 (5-8 members), 2 (3-4), 4 (2), 8 (1)
  int rowmerge;     // 1: partials per member row (sidx / nspl below), merged per row (attn_group 4)
  int q_row[8];     // members' rows in q / attn_out (next-step live positions)
  int pt_row[8];    // members' page-table rows (slots)
  int pos0[8];      // members' current positions (keys <= pos0 visible)
  int sidx[8];      // rowmerge: this unit's split index in each member row's partial list
  int nspl[8];      // rowmerge: each member row's number of partials (1 -> written directly)
};
constexpr int kRowSplits = 32;   // rowmerge: partials per (row, KV head)

struct CtlBlock {
  int n_live;       // rows decoded by the next step on this rank (0 => idle)
  int t;            // step index the next decode step produces
  int acc;          // accepted prompts (global under DP)
  int acc_local;    // accepted prompts of this rank's slice
  int done;         // round finished (identical on every rank)
  int err;          // 1 = KV pool exhausted, 2 = page table overflow, 3 = attention work list overflow (any rank)
  int n_final;      // live rows at the end (aborted in short rounds)
  int t_end;        // last decoded step
  int underfilled;
  int k_step;       // prompts of this rank completed at the last step
  int n_next;       // rows of this rank still live after the last step
  int n_items;      // attention items of the next step
  int free_top;     // KV free-list top
  int need_pages;   // pages the next step allocates
  long long decoded;  // tokens decoded this round on this rank
  long long ctx_sum;  // sum over next-step rows of the attention context (kv_len + 1)
  long long kv_read;  // sum over decode steps so far of the decoded rows' attention context
  int n_issued;     // continuous issuance: prompts of this rank issued so far (committed)
  int issue_n;      // prompts phase A issues after this step (committed by phase B unless done)
  // KV pressure (NEXT-2, reading Z26)
  int preemptions;  // prompts preempted this round on this rank
  int wait_head, wait_tail;   // FIFO of waiting prompts in wait_q[head .. tail)
  int adm_ctr;      // last admission stamp
  int readmit_n;    // prompts phase A re-admits after this step
  int readmit_rows; // their responses (rows appended by phase B)
  int readmit_pages;  // pages they take
  int pause;        // 1: re-admitted responses await their KV recompute (the host runs it between steps)
  int n_live_saved, n_items_saved;  // the next step's rows / attention items while paused
  int n_gitems;     // sibling-group attention items of the next step (RoundDev.gitems)
  int n_gitems_saved;
  int n_rejobs;     // recompute jobs written by phase B
  long long kv_read_unique;  // as kv_read with each prompt's shared full pages counted once per step
};

struct RoundDev {
  int S, P, maxp, cap, G, target, kind /*0 short 1 long*/, trace, eos, n_prompts, kv_heads;
  int keep;           // responses retained per prompt (R0 <= G; == G in long rounds)
  int max_active;     // continuous issuance (NEXT-4): max prompts with a live response; 0 = off
  int preempt;        // KV-pressure preemption with recompute (NEXT-2); 0 = exhaustion is an error
  int* p_plen;        // [P] prompt lengths (the KV a response starts from)
  int* p_adm;         // [P] admission stamps (LIFO victims: the largest)
  int* p_wait;        // [P] WaitState
  int* p_live;        // [P] scratch: live responses this step
  int* p_pfree;       // [P] scratch: their private pages
  int* p_pneed;       // [P] scratch: their next-step page needs
  int* wait_q;        // [P] FIFO ring of waiting prompts
  int* rejobs;        // [S][5] recompute jobs: slot, g, fork src page, fork dst page, fork rows
  int attn_units;     // decode-attention split budget per KV head (0: 148 / KV)
  int attn_waves;     // 1: budget whole waves of attention units (k-wave fill), 0: one-wave floor
  int attn_group;     // sibling-group work list (gitems, k_attn_group.cu) besides the per-row one: 0 off;
                      // 1 sibling groups unless too few (then single rows), 2 always sibling groups, 3 always single rows
  int group_rows_min; // build gitems when the next step has more rows (or *gmode: the running graph uses them)
  int group_waves;    // split budget of the group list: at least this many waves of units (A/B)
  const int* gmode;   // [1] 1 while the host runs decode steps with the group kernel
  AttnGroupItem* gitems;
  int* grp_key;       // [S] scratch: (prompt, j / 8) of each next-step row
  int* grp_start;     // [S + 1] scratch: first row of each group
  int world, rank;
  int max_items;      // capacity of `items` (ctl flags err 3 rather than overflow it)
  int max_items_g;    // capacity of `gitems`
  int* slot_prompt; int* slot_j; int* kv_len; int* gen; int* trace_L; int* status; int* own0;
  int* t0;            // [S] step before the sequence's first token: local token index = t - t0 (0 unless issued late)
  int* p_last_tok;    // [P] last prompt token (a late-issued prompt decodes it as its first step)
  int* p_stamp;       // [P] last step the prompt had a live response (active-prompt count)
  int* tok_out;       // [S][cap]
  int* page_table;    // [(S + P)][maxp]
  int* p_cnt; int* p_state; int* p_gid; int* comp_list; int* accept_order;
  int* live; int* live_next;
  int* tok_in; int* row_pos; int* row_pt;
  unsigned long long* best;
  AttnItem* items;
  unsigned long long* rows_hist;  // [S + 1] decode steps of this round by live rows (measurement)
  int* free_stack;
  int* ks_local;      // [4]: prompts completed at this step, rows still live, error, re-admission pause
  int* ks;            // [4 * world] all-gathered ks_local (== ks_local when world == 1)
  CtlBlock* ctl;
  int* trace_buf; int trace_steps;   // debug: [steps][2 + S] (n, acc|done<<30, live...)
};

// Per-rank model dimensions: under tensor parallelism H, KV, F and V are the
// local shard sizes (vocab rows [v0, v0 + V) of the LM head live here).
struct ModelDims {
  int L, d, H, KV, hd, F, V, eos;
  int v0;                  // first vocab id of this rank's LM-head shard
  float eps;
  size_t page_bytes;       // one page: L x KV x 2 x kPage x hd fp16 (reading Z20)
  int n_pages;             // pages in the KV pool (layout: kv_block_elems, common.cuh)
};

// weights
void launch_init_weights(void* out, long long rows, int cols, long long r0, int c0, int in_full, uint32_t tid,
                         uint64_t seed, int mode, int up, cudaStream_t st, int f16 = 1, long long dst_row0 = 0,
                         int tiled = 1);
// forward pieces (n = n_dev ? *n_dev : n_host)
void launch_embed(const int* tok, const int* n_dev, int n_host, const void* emb, float* x, int d, cudaStream_t st);
void launch_rmsnorm(float* x, const float* delta, const int* gather, const int* n_dev, int n_host,
                    const float* gamma, void* h, int d, float eps, cudaStream_t st, void* h_lo = nullptr);
void launch_tp_norm(float* x, const float* recv /* [tp][rows][d] slot base */, int tp, size_t src_stride,
                    const unsigned long long* flags /* [tp] */, unsigned long long* gen, int* done, int m_tiles,
                    int splits, int coop_min, int max_grid, const int* n_dev, int n_rows_grid, const float* gamma,
                    void* h, int d, float eps, cudaStream_t st, void* h_lo = nullptr);
// w[m][k] *= gamma[k] for an fp16 [rows, cols] weight (an RMSNorm gain folded
// into the GEMM that consumes the normalised activations)
void launch_scale_cols(void* w, long long rows, int cols, const float* gamma, cudaStream_t st, int tiled = 1);

// Device-memory collectives of a single-GPU local group (several contexts of
// one process on one device): rank `me` of a group of
// `size` copies `bytes` of src into its slot of the exchange buffer
// slots[2][size][slot_bytes] and publishes epoch e = state[0] + 1 in gen[me];
// the reduce kernel waits until every gen[q] >= e and combines the slots in
// rank order.  state = {epoch, ticket} per (context, group), zero-initialised.
enum LocalOp { LOP_GATHER = 0, LOP_SUM_F32 = 1, LOP_MAX_U64 = 2 };
void launch_local_publish(const void* src, size_t bytes, uint8_t* slots, size_t slot_bytes, int size, int me,
                          unsigned long long* gen, int* state, cudaStream_t st);
void launch_local_reduce(int op, void* dst, size_t bytes, const uint8_t* slots, size_t slot_bytes, int size,
                         const unsigned long long* gen, const int* state, cudaStream_t st);
void launch_rope_append(const float* qkv, const int* n_dev, int n_host, const int* row_pos, const int* row_pt,
                        const int* page_table, int maxp, void* q_out, void* kv_pool, const ModelDims& m, int layer,
                        const double* inv_freq, cudaStream_t st, void* q_lo = nullptr);
int make_kv_map(CUtensorMap* map, const void* pool, size_t n_pages, const ModelDims& m);
// Decode attention fused with the QKV GEMM's split-K reduction (EPI_PARTIAL):
// each work unit sums its row's q partials (and, for the unit holding the
// current token, k and v) in split order, applies the folded RMSNorm scale,
// the bias and RoPE, appends k / v to the KV page and uses q directly.
struct QkvFuse {
  const float* part;      // split partials [(chunk * m_tiles + tile) * splits + split][256][128]; nullptr = off
  int splits, m_tiles;
  int gemm_lo;            // the QKV GEMM ran split precision: 128-column chunks while the live count <= 128
  const int* n_rows;      // live rows of the step (device)
  const float* bias;      // bqkv [M]
  const float* ssq; int ssq_parts, ssq_stride; float inv_d, eps;   // folded RMSNorm (ssq == nullptr: none)
  const float2* cs;       // RoPE (cos, sin) [pos][hd / 2]
  uint8_t* kv_pool; size_t page_bytes;
  int n_pages;
  int dbg;                // RP_AG_DBG measurement knobs (also without the fusion): 1 no MMAs, 2 no q_lo MMAs
};

void launch_attention(const CUtensorMap& kv_map, const void* q, const int* page_table, int maxp,
                      const AttnItem* items, const int* n_items_dev, int n_items_host, void* out, float* partial,
                      int* tickets /* [items x KV], zero, self-resetting */, const ModelDims& m, int layer,
                      bool decode /* <= 8 query rows per unit */, cudaStream_t st, const void* q_lo = nullptr,
                      void* out_lo = nullptr, const QkvFuse* fuse = nullptr);
// sibling-group decode attention (RoundDev.attn_group; g = H / KV <= 8)
void launch_attention_group(const CUtensorMap& kv_map, const void* q, const void* q_lo, const int* page_table,
                            int maxp, const AttnGroupItem* items, const int* n_items_dev, void* out, void* out_lo,
                            float* partial, int* tickets, const ModelDims& m, int layer, cudaStream_t st,
                            int dbg = 0, int may_spin = 1 /* 0 in single-GPU local groups */,
                            float* rowpart = nullptr /* [S][KV][kRowSplits] member-row partials */,
                            int* rtickets = nullptr /* [S][KV], zero, self-resetting */);
int attn_group_init_attrs();
size_t attn_group_partial_floats(int hd);   // per (item, KV head)
void launch_kv_fork(const int* jobs /*[n][3] src,dst,rows*/, int n, void* kv_pool, const ModelDims& m,
                    cudaStream_t st);
void launch_sampler(const float* logits, int V, int v0, int row_div, const RoundDev& R, uint64_t seed,
                    float inv_temp, uint32_t round_id, cudaStream_t st);
void launch_ctl(const RoundDev& R, int appended, int mode /*0 all, 1 phase A, 2 phase B*/, cudaStream_t st);
// spin until the host-mapped *flag != 0 (profiling: release a fully enqueued step)
void launch_host_gate(const int* flag, cudaStream_t st);
// responses of the accepted prompts with acceptance index >= first (local)
void launch_collect_pack(const RoundDev& R, int first, int* meta /*[acc*keep][4]*/, int* tokens, cudaStream_t st);
int attn_smem_bytes(int hd);
void attn_set_timeline(long long* p /* [148][8] or nullptr */);
int attn_init_attrs();

}  // namespace rp
