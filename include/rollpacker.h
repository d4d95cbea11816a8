/*
 * rollpacker.h -- C ABI of the B200-native tail-batching rollout path
 * (RollPacker, arXiv 2509.21009).  Library: librollpacker.so (sm_100a).
 *
 * The path is the rollout stage of synchronous GRPO-style RL under tail
 * batching:
 *   - a SHORT round launches more prompts than it keeps ("launches more than
 *     P0 prompts but retains only the first P0 that finish"),
 *     decodes G responses per prompt under a per-round length cap, and stops
 *     once `target` prompts have all G responses finished;
 *   - prompts not accepted are deferred to a FIFO long-prompt queue ("added to
 *     a long-prompt queue");
 *   - a LONG round decodes queued prompts with speculation disabled, every
 *     response retained and truncated at the cap ("capped at the same
 *     maximum").
 * Paper notation: P0 = target prompts, R0 = G responses per prompt, eta =
 * over-provisioning (n_prompts = ceil(eta * P0)).
 *
 * Conventions
 *   - Every call returns 0 (RP_OK) or a negative RP_E* code; rp_last_error()
 *     gives a one-line reason.  No C++ exception crosses the ABI.
 *   - Device memory (weights, KV pool, workspace) is allocated by the caller
 *     (PyTorch) and BORROWED for the lifetime of the context.  Host arrays
 *     passed to calls are copied before the call returns (except where noted).
 *   - A context is bound to one CUDA device and one stream; it is
 *     thread-compatible, not thread-safe (one context per rank / thread).
 *   - Data-parallel short rounds (world > 1): every rank submits the SAME
 *     full prompt list; rank r decodes the contiguous slice of prompt indices
 *     partition(n, world)[r] and the per-step acceptance cutoff is exchanged
 *     with an NCCL all-gather.  Membership (which prompts are
 *     accepted / deferred) is identical for every world size, and so is the
 *     global long-prompt queue every rank keeps.
 */
#ifndef ROLLPACKER_H
#define ROLLPACKER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ error codes */
#define RP_OK 0
#define RP_EINVAL -1     /* bad argument (the message names the field)          */
#define RP_EBUSY -2      /* a round is active: submit while not collected        */
#define RP_ESTATE -3     /* wrong state: step/collect without an active round    */
#define RP_ENOMEM_KV -4  /* KV page pool exhausted (no preemption, reading Z17)  */
#define RP_ECUDA -5      /* CUDA runtime / driver error                          */
#define RP_ENCCL -6      /* NCCL error                                           */
#define RP_ENOSPC -7     /* caller buffer too small / capacity exceeded          */

/* ----------------------------------------------------------- round flags */
#define RP_SHORT 0       /* speculative short round: stop at `target` accepted   */
#define RP_LONG 1        /* long round: target must equal n_prompts, no aborts   */
#define RP_TRACE 4       /* trace mode: EOS masked before and forced at L (Z15)  */
#define RP_PREEMPT 8     /* KV pressure: recompute preemption instead of RP_ENOMEM_KV (Z26) */

/* ------------------------------------------------- finish codes (rp_response) */
#define RP_FINISH_EOS 1  /* ended with EOS (natural or trace-forced)             */
#define RP_FINISH_CAP 2  /* truncated at the cap (long rounds only)              */

/* Qwen2-shaped decoder ("Qwen2.5 family").  Weights are
 * the random-init formula of DESIGN.md reading Z12, generated on device from
 * weight_seed by rp_init_model.  Constraints: head_dim in {64, 128};
 * d_model, n_heads*head_dim and d_ff multiples of 128; vocab multiple of 128;
 * n_heads % n_kv_heads == 0 and n_heads / n_kv_heads <= 8. */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab, eos_id;
  int32_t qkv_bias;          /* 1 = q/k/v projections carry a bias (Qwen2)     */
  float rope_theta, rms_eps;
  uint64_t weight_seed;
} rp_model_desc;

typedef struct {
  void* weights;             /* device, >= rp_query_sizes().weights_bytes      */
  size_t weights_bytes;
  void* kv_pool;             /* device; n_pages = kv_pool_bytes / page_bytes   */
  size_t kv_pool_bytes;
  void* workspace;           /* device, >= rp_query_sizes().workspace_bytes    */
  size_t workspace_bytes;
  void* stream;              /* cudaStream_t all work is issued on (NULL = 0)  */
  int32_t rank, world;       /* data-parallel rank / size (world 1 = no NCCL)  */
  int32_t max_seqs;          /* max sequences (n_prompts_local * G) per round  */
  int32_t max_prompts;       /* max prompts per round on this rank             */
  int32_t max_prompt_len;    /* max tokens of one prompt                       */
  int32_t max_prompt_tokens; /* max total prompt tokens per round on this rank */
  int32_t max_cap;           /* max length cap of any round                    */
  uint64_t sample_seed;      /* Philox key of the sampler (reading Z10)        */
  float temperature;         /* T of the Gumbel-max sampler (reading Z9: 1.0)  */
  int32_t graph_steps;       /* decode steps per captured CUDA graph (0 = no graphs) */
  const void* nccl_id;       /* 128-byte ncclUniqueId of the DP group (world > 1): the ranks
                                with this context's tp_rank, one per replica; with world == 1
                                and tp > 1 it may instead name the TP group.  NULL otherwise */
  int32_t tp;                /* tensor-parallel size of this context (0/1 = none).  With
                                tp > 1 the context holds only its shard:
                                heads, KV heads, d_ff and vocab / tp (column-parallel QKV,
                                gate||up and LM head, row-parallel O and down with an fp32
                                all-reduce after each -- NCCL, or at decode the NVLink peer
                                push of rp_tp_ipc_open; vocab-sharded sampling with a
                                MAX all-reduce of the packed argmax).  Every TP rank submits
                                the same prompts and keeps identical round state. */
  int32_t tp_rank;           /* rank inside the TP group */
  const void* tp_nccl_id;    /* ncclUniqueId of this replica's TP group (tp > 1; NULL with
                                world == 1 -> nccl_id).  world > 1 with tp > 1 is DP x TP:
                                `world` replicas of `tp` ranks each (the C4 short rounds) */
  void* local_group;         /* NULL, or a handle of rp_local_group_create: every rank of
                                the job (world x tp) is a context of THIS process on THIS
                                device, created concurrently from one thread per rank;
                                collectives run through device memory (no NCCL, no IPC)
                                and nccl ids are ignored (a test mode, not a fast path) */
} rp_runtime_desc;

typedef struct {
  size_t weights_bytes, workspace_bytes, page_bytes;
} rp_sizes;

/* One prompt of a round.  `tokens` (len ids in [0, vocab), none == eos),
 * `trace_lens` (G response lengths >= 1, trace mode only, else NULL) and
 * `trace_lens_retry` are host pointers, copied by rp_submit_round.  prompt_id is the caller's global id:
 * it seeds the sampler stream uid = prompt_id * G + j (reading Z10). */
typedef struct {
  int32_t prompt_id;
  int32_t len;
  const int32_t* tokens;
  const int32_t* trace_lens;
  const int32_t* trace_lens_retry; /* trace mode: G lengths of the re-roll (reading Z5) used if
                                      this prompt is deferred and later popped by a NULL-prompt
                                      LONG round; NULL -> trace_lens again */
} rp_prompt;

typedef struct {
  int64_t round_id;
  int32_t kind;              /* RP_SHORT / RP_LONG                             */
  int32_t t;                 /* decode steps completed (t_end when done)      */
  int32_t n_live;            /* sequences still decoding on this rank          */
  int32_t accepted;          /* accepted prompts (global under DP)             */
  int32_t accepted_local;    /* accepted prompts decoded on this rank          */
  int32_t done;              /* 1 once the round reached target or ran dry     */
  int32_t underfilled;       /* done with accepted < target (reading Z4)       */
  int32_t n_prompts_local;
  int64_t decoded_tokens;    /* tokens decoded on this rank this round (incl. aborted) */
  int64_t kv_tokens_read;    /* sum over decode steps and decoded rows of the attention context
                                (KV tokens read per layer and KV head); measurement only   */
  int32_t preemptions;       /* prompts preempted by KV pressure this round on this rank */
  int64_t kv_tokens_unique;  /* kv_tokens_read with each prompt's shared full prompt pages counted
                                once per step (the bytes HBM must deliver); measurement only */
} rp_status;

typedef struct {
  int32_t prompt_id;         /* global prompt id                               */
  int32_t j;                 /* response index 0..G-1                          */
  int32_t len;               /* tokens, including the EOS (reading Z16)        */
  int32_t finish;            /* RP_FINISH_EOS / RP_FINISH_CAP                  */
  int64_t tok_off;           /* offset of the tokens in the collect token buffer */
} rp_response;

/* Size query: bytes the caller must provide for weights and workspace, and the
 * size of one KV page (64 tokens x all layers x KV heads x {K,V} x head_dim
 * fp16, reading Z20).  Pure host computation. */
int rp_query_sizes(const rp_model_desc* md, const rp_runtime_desc* rd, rp_sizes* out);

/* Create a context: validates the descriptors, generates the weights into
 * rd->weights on rd->stream (formula Z12), builds TMA descriptors, and
 * creates the NCCL communicator when world > 1.  *out receives the context. */
int rp_init_model(const rp_model_desc* md, const rp_runtime_desc* rd, void** out);

/* Plan the next round (the tail-batching planner; SPEC S:271-279
 * plan_round): if the long-prompt queue holds >= P0 prompts, *kind = RP_LONG
 * and *n_prompts = P0 (submit it with prompts == NULL: the first P0 queued
 * prompts, target = P0); otherwise *kind = RP_SHORT and *n_prompts =
 * ceil(eta * P0) (submit that many fresh prompts with target = P0).
 * drain != 0 (end of the prompt stream, reading Z7) plans a LONG round over
 * a non-empty queue shorter than P0.  Host only; identical on every rank.
 * Errors: RP_EINVAL (P0 < 1, eta < 1). */
int rp_plan_round(void* ctx, int32_t P0, float eta, int32_t drain, int32_t* kind, int32_t* n_prompts);

/* Start a round.  prompts: the FULL
 * prompt list of the round (every rank passes the same list); NULL pops
 * n_prompts entries from the head of the long-prompt queue (every DP rank
 * holds the same global queue, so every rank pops the same prompts and
 * decodes its slice).  The queue is popped only once the round has started:
 * a submit that fails leaves it unchanged.
 * G: responses launched per prompt.  keep: responses retained per prompt
 * (R0), 1 <= keep <= G, or 0 for keep = G.  keep < G is response-level
 * speculation ("each prompt produces more than R0
 * responses, finishing after the first R0 complete"): a prompt completes at
 * the step its keep-th response emits EOS (ties at that step go to the lower
 * j), its other responses are aborted at once, and only the keep finished
 * ones are collected.  RP_LONG requires keep == G (speculation disabled,
 * P:124).  cap: length cap of every response (>= 1).
 * target: prompts to accept (P0), 1 <= target <= n_prompts; RP_LONG requires
 * target == n_prompts.  flags: RP_SHORT|RP_LONG [|RP_TRACE] [|RP_PREEMPT].
 * RP_PREEMPT (reading Z26): when the next
 * step's KV pages exceed the free pages, the most recently admitted prompt
 * with a live response (never the last one) is preempted -- its responses'
 * private pages freed -- and waits in a FIFO; a step that preempts nothing
 * re-admits waiting prompts while they fit, and the library recomputes
 * their KV (prefill kernels over the response's own tokens) before the next
 * step, which continues them at their next token.  The schedule is exact
 * (oracle sched.kv_step_loop); rp_status.preemptions counts the victims.
 * Not combinable with continuous issuance.  Without it, exhaustion is
 * RP_ENOMEM_KV.  round_id seeds
 * the sampler counter (reading Z5: re-rolls draw fresh noise).  Runs the
 * prefill and decode step 1 (the token sampled from the prefill logits).
 * Errors: RP_EINVAL, RP_EBUSY (round active), RP_ENOMEM_KV, RP_ENOSPC. */
int rp_submit_round(void* ctx, const rp_prompt* prompts, int32_t n_prompts, int32_t G, int32_t keep, int32_t cap,
                    int32_t target, int32_t flags, int64_t round_id);

/* Run up to max_steps decode steps (or until the round is done) and report
 * the status.  Each step: embed -> L x (RMSNorm, QKV, RoPE+KV append,
 * attention, O, RMSNorm, gate||up+SwiGLU, down) -> LM head -> sampler ->
 * round control, all on device (captured in CUDA graphs of graph_steps
 * steps).  Errors: RP_ESTATE (no round), RP_ENOMEM_KV, RP_ECUDA, RP_ENCCL. */
int rp_step(void* ctx, int32_t max_steps, rp_status* st);

/* Collect a finished round.  Fills out[0..n) with the accepted responses of
 * the prompts decoded on this rank, in acceptance order (prompt-major, j
 * minor), and their tokens into tok_buf (host, int32).  Pass out == NULL to
 * query *n_out and *n_tok only (the round stays collectable).  A successful
 * collect with out != NULL closes the round: every unaccepted prompt of this
 * rank's slice is appended, in submission order, to the long-prompt queue
 * (SHORT rounds), and all KV pages return to the pool.
 * Errors: RP_ESTATE (round not done), RP_ENOSPC (buffers too small). */
int rp_collect(void* ctx, rp_response* out, int32_t max_out, int32_t* tok_buf, int64_t tok_cap, int32_t* n_out,
               int64_t* n_tok);

/* Streaming collect (completed prompts go to the
 * reward / trainer stages while the round continues).  Between rp_step calls
 * of an active round (or after it is done, before rp_collect), fills out[]
 * with the retained responses of this rank's accepted prompts whose
 * acceptance index (local, 0-based) is in [first, accepted so far), in the
 * order rp_collect would return them; *n_accepted receives the accepted
 * count (pass it as `first` next time).  An accepted prompt's responses are
 * final, so a streamed response never changes; the round stays active and
 * rp_collect still returns everything and closes it.  out == NULL queries
 * sizes.  Errors: RP_ESTATE (no round), RP_EINVAL (first), RP_ENOSPC. */
int rp_collect_ready(void* ctx, int32_t first, rp_response* out, int32_t max_out, int32_t* tok_buf, int64_t tok_cap,
                     int32_t* n_out, int64_t* n_tok, int32_t* n_accepted);

/* Measurement: out[r] = decode steps of the current (or last) round on this
 * rank that decoded r live rows, r = 0..n-1 (rows above max_seqs read 0).
 * Lets the caller compute the per-round roofline of SURVEY §8(d). */
int rp_round_rows_histogram(void* ctx, int64_t* out, int32_t n);

/* Migration of an in-flight round by recompute (PAPER.md
 * when rollout GPUs are handed to training, their
 * unfinished responses move to the remaining instances and their KV is
 * recomputed there; reading Z27).  Between two rp_step calls,
 * rp_round_export writes the round's step state -- control block, live list
 * and next-step inputs, attention work lists, per-response lengths, status,
 * tokens and issue offsets, per-prompt counters, acceptance order -- into a
 * caller buffer of rp_round_state_bytes bytes (host memory; the KV cache is
 * not exported).  rp_round_import, on an idle context created with the same
 * model and runtime sizes (on this or another GPU), takes the round's
 * ORIGINAL rp_submit_round arguments plus that buffer: it re-submits the round
 * (prefill and step 1 are deterministic), installs the exported state, sizes
 * the live responses' page tables and recomputes the KV of their generated
 * tokens with the prefill kernels, so rp_step continues at the exported step
 * with the same schedule (live lists, acceptance, cutoff) and the same
 * sampling counters.  DP jobs migrate rank by rank into contexts of the
 * same world and rank, TP groups rank by rank into groups of the same size
 * (every rank imports at the same step: the re-submit and the recompute run
 * the collectives); prompts preempted by KV pressure move with their
 * admission stamps and wait queue (re-admitted and recomputed there); not
 * at a step a re-admission paused, no continuous issuance; the exporting context keeps
 * its round (collect or drop it).  Errors: RP_ESTATE (no active round / done
 * / waiting prompts), RP_ENOSPC (buffer too small), RP_EINVAL (size or header
 * mismatch, unsupported mode), RP_ENOMEM_KV (the pool cannot hold the live
 * contexts), RP_ECUDA. */
int rp_round_state_bytes(void* ctx, int64_t* bytes);
int rp_round_export(void* ctx, void* buf, int64_t bytes);
int rp_round_import(void* ctx, const rp_prompt* prompts, int32_t n_prompts, int32_t G, int32_t keep, int32_t cap,
                    int32_t target, int32_t flags, int64_t round_id, const void* buf, int64_t bytes);

/* Re-shard the exported states of all W ranks of a DP job (rank order) to
 * new_world ranks, for rp_round_import into contexts of that world: the
 * rollout GPU set shrinks (or grows) mid-round (NEXT-3; Z27).
 * Host only (no context).  Prompts are re-split contiguously by global
 * index, each prompt's state moves whole; the next step's inputs are rebuilt
 * from the live responses in slot order (one attention item per row); the
 * local acceptance order is (completion step, index).  out == NULL returns
 * the state size in *need.  RP_EINVAL: mismatched / unsupported states
 * (done, paused, preempted), slice too large for the engine sizes. */
int rp_round_reshard(const void* const* states, const int64_t* bytes, int32_t n_states, int32_t n_prompts,
                     int32_t new_world, int32_t new_rank, void* out, int64_t out_bytes, int64_t* need);

/* Continuous issuance (DAPO integration:
 * "set a maximum number of active requests for each LLM instance and
 * continuously issue new requests"; readings Z21).  Applies to the rounds
 * submitted after the call; max_active = 0 (the default) turns it off.  With
 * max_active = A > 0 at most A of this rank's prompts have a live response at
 * any step: the first min(A, n_local) start at step 1, and after every step
 * the lowest-index unissued prompts are issued while fewer than A are active
 * (a prompt stays active until none of its responses is live).  A prompt
 * issued after step t decodes its last prompt token at step t + 1 and emits
 * its k-th token at step t + k (the sampler counter is the response's token
 * index k, so its tokens do not depend on when it was issued); its other
 * plen - 1 tokens are prefilled at submit, so every prompt of such a round
 * needs len >= 2 beyond the first A.  Acceptance, the cutoff, keep and the
 * cap are unchanged.  Prompts never issued when the round ends are neither
 * accepted nor deferred: rp_round_unissued lists them.  Errors: RP_EINVAL
 * (max_active < 0), RP_EBUSY (a round is active). */
int rp_round_issue_cap(void* ctx, int32_t max_active);

/* Global ids of this rank's prompts the finished round never issued
 * (continuous issuance; in submission order).  ids_out may be NULL to query
 * *n_out.  Errors: RP_ESTATE (round not done), RP_ENOSPC (max too small). */
int rp_round_unissued(void* ctx, int32_t* ids_out, int32_t max, int32_t* n_out);

/* Snapshot of the long-prompt queue (global prompt ids, oldest first); no
 * drain.  Under data parallelism the queue is global: rp_collect gathers
 * every rank's accepted prompts (DP collective) and every rank appends all
 * unaccepted prompts of the round in submission order, so all ranks hold
 * the same queue.  ids_out may be NULL to query *n_out. */
int rp_long_queue(void* ctx, int32_t* ids_out, int32_t max, int32_t* n_out);

/* Drop the first n entries of the long-prompt queue (they were submitted
 * explicitly on another context, e.g. a TP context of the same GPUs).
 * Errors: RP_EINVAL (n < 0 or n > queue length). */
int rp_long_queue_pop(void* ctx, int32_t n);

/* The parallelism planner's adaptation rule (SURVEY
 * NEXT-2): "a sudden rise in preemptions (e.g., >1.05x) triggers an increase
 * in TP (doubling the size), while sustained zero preemptions across four
 * steps trigger a decrease (halving the size)".  Given the current TP size of
 * a round kind, the largest allowed (the GPUs of one server), the previous
 * and the latest round's preemption counts (rp_status.preemptions summed
 * over the replica) and the count of consecutive zero-preemption rounds so
 * far, writes the next TP size and streak.  Host only, no context.
 * Errors: RP_EINVAL. */
int rp_plan_tp(int32_t tp, int32_t tp_max, int64_t prev_preemptions, int64_t preemptions, int32_t zero_streak,
               int32_t* tp_next, int32_t* zero_streak_next);

/* Single-GPU local group: a host object shared by the
 * world x tp contexts of one process on one device, holding the exchange
 * buffers of the device-memory collectives (k_comm.cu) and the TP peer
 * blocks.  Create it once, pass it in rp_runtime_desc.local_group of every
 * rank's context, create the contexts concurrently (rp_init_model waits for
 * all of them), free it after the contexts.  Errors: RP_EINVAL. */
int rp_local_group_create(int32_t world, int32_t tp, void** out);
void rp_local_group_free(void* group);

/* Tensor-parallel decode over NVLink peer memory.  A
 * context created with tp > 1 (d a multiple of 128) owns a device block of
 * receive slots [2][tp][max_seqs][d] fp32 plus arrival counters.
 * rp_tp_ipc_handle writes its CUDA IPC handle (RP_IPC_HANDLE_BYTES bytes) to
 * `out`; after every rank of the TP group has gathered all handles (rank
 * order, e.g. with torch.distributed), rp_tp_ipc_open maps the peers' blocks
 * and switches decode steps to the peer path: the row-parallel O/down GEMMs
 * push their fp32 partial tiles into every rank's slot with NVLink stores and
 * count them with system-scope release adds, and one kernel per norm adds
 * the partials in rank order and applies the RMSNorm (no NCCL call).  Prefill
 * and the LM-head argmax keep NCCL.  Errors: RP_ESTATE (no peer block),
 * RP_EBUSY (round active), RP_ECUDA (IPC mapping failed). */
#define RP_IPC_HANDLE_BYTES 64
int rp_tp_ipc_handle(void* ctx, void* out);
int rp_tp_ipc_open(void* ctx, const void* handles /* tp x RP_IPC_HANDLE_BYTES */);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 of a DP group creates it
 * and broadcasts it, e.g. with torch.distributed, before rp_init_model). */
int rp_nccl_unique_id(void* out);

/* Destroy a context (does not free caller-owned device memory). */
void rp_free(void* ctx);

/* Last error message of the context (or of the last failed rp_init_model
 * when ctx is NULL).  Valid until the next call on the context. */
const char* rp_last_error(const void* ctx);

/* Kernel launches issued by this context since creation (evidence for the
 * bench's gpu_launches; graph launches count their kernel nodes). */
int64_t rp_launch_count(const void* ctx);

/* ---------------------------------------------------------------- test-only */
/* Teacher-forced logits of one token sequence (host tokens[n], n <=
 * max_prompt_tokens and <= max_prompt_len) through the prefill path: writes
 * n x vocab fp32 to logits_out (host); under TP, n x (vocab / tp) of this
 * rank's vocab shard.  Requires no active round. */
int rp_debug_logits(void* ctx, const int32_t* tokens, int32_t n, float* logits_out);

/* Enable (steps > 0) or disable the per-step schedule trace of the next
 * round: for every decode step t, the list of sequences decoded at t (slot =
 * local_prompt * G + j, stable order), the accepted count and done flag. */
int rp_debug_trace_enable(void* ctx, int32_t steps);
/* Copy the trace out: buf[t][0] = n decoded, buf[t][1] = accepted | done << 30,
 * buf[t][2 .. 2 + n) = slots.  Row stride = 2 + max_seqs. */
int rp_debug_trace_get(void* ctx, int32_t* buf, int32_t steps);

/* Logits of the most recent decode step (rows in the live order of that step;
 * eager or the last step of a CUDA graph) and the slots of those rows;
 * requires rp_debug_trace_enable. */
int rp_debug_last_logits(void* ctx, float* logits_out, int32_t* slots_out, int32_t max_rows, int32_t* n_rows);

/* Kernel classes of rp_debug_profile. */
#define RP_PROF_EMBED 0
#define RP_PROF_RMSNORM 1
#define RP_PROF_GEMM_QKV 2
#define RP_PROF_ROPE 3
#define RP_PROF_ATTN 4
#define RP_PROF_MERGE 5
#define RP_PROF_GEMM_O 6
#define RP_PROF_GEMM_GU 7
#define RP_PROF_GEMM_DOWN 8
#define RP_PROF_GEMM_LM 9
#define RP_PROF_SAMPLER 10
#define RP_PROF_CTL 11
#define RP_PROF_NCCL 12
#define RP_PROF_N 13
/* Per-kernel-class timing.  steps > 0 arms profiling: the next `steps` decode
 * steps run eagerly (no graph) with every launch bracketed by CUDA events on
 * the context's stream.  steps == 0 reads the totals: ms_out[RP_PROF_N]
 * (summed milliseconds), counts_out[RP_PROF_N] (launches),
 * rows_ctx_steps[3] = {sum of live rows, sum of attention context tokens,
 * profiled steps}; steps < 0 disarms.  Any pointer may be NULL. */
int rp_debug_profile(void* ctx, int32_t steps, double* ms_out, int64_t* counts_out, int64_t* rows_ctx_steps);

/* Run the tcgen05 GEMM alone on device pointers: Y[n][m] = sum_k W[m][k] X[n][k]
 * (W fp16 [M,K], X fp16 [N,K] with N <= rows_cap rows allocated, Y fp32 [N,M]);
 * w_tiled bit 0: W is stored in 128 x 64 tiles, tile (m / 128, k / 64) at
 * element ((m / 128) * (K / 64) + k / 64) * 8192, row-major inside (the layout
 * rp_init_model generates the model's GEMM weights in); else row-major.
 * w_tiled bit 1: split-precision activations -- X holds 2 * rows_cap rows,
 * the fp16 values and then their fp16 rounding residuals, and Y = W (X_hi +
 * X_lo)^T (reading Z22).
 * splits = split-K factor (0 = automatic).  Runs once to warm up, then `iters`
 * back-to-back launches timed with CUDA events; *ms_out (may be NULL) gets the
 * mean milliseconds per launch. */
int rp_debug_gemm(void* ctx, const void* W, const void* X, int32_t rows_cap, float* Y, int32_t M, int32_t N,
                  int32_t K, int32_t splits, int32_t iters, int32_t w_tiled, float* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* ROLLPACKER_H */
