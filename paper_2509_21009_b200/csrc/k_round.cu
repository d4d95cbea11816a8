// Sampling and round control on the device (K9-K11).
//
// sampler: token = argmax_v (logit_v / T + g_v), g_v = -ln(-ln u_v) with
//   u_v from word v&3 of Philox4x32-10(ctr=(v>>2, t, uid, round_id), t the
//   response's token index (the step minus its issue offset t0),
//   key=seed) (readings Z9-Z11); trace mode masks EOS before the trace
//   length L and forces it at t = L.  Per-row argmax is a packed
//   (orderable value, ~index) atomicMax, so the result is independent of the
//   order CTAs finish in.
// ctl: one CTA per step.  Finish detection (EOS / cap), per-prompt finished
//   counters, race-to-completion acceptance in (step, prompt index) order
//   (P:116-119), round_done, stable prefix-sum compaction of the
//   live list, KV page free/alloc from a LIFO free list, and the next step's
//   attention work list.  No host synchronisation inside a step.
#include "common.cuh"
#include "kernels.h"

namespace rp {

// ------------------------------------------------------------------ sampler
constexpr int SAMP_CHUNK = 4096;   // vocab entries per work unit

// Gumbel noise g = -log(-log u), u = u01(x) = (k + 1/2) 2^-23, k = x >> 9
// (reading Z10), with the hardware log (MUFU lg2) instead of two accurate
// logf calls -- the sampler is ALU-bound on them.  The inner -log(u) loses
// relative accuracy near u = 1, where the largest noise values (the likely
// argmax) live, so there t = -log(1 - v) comes from its series in the exact
// v = 1 - u = (2^23 - k - 1/2) 2^-23 (six terms for v < 2^-5: truncation
// < 2^-35 relative); elsewhere t >= 0.031 and MUFU's 2^-21.4 absolute error is
// < 1.1e-5 relative.  The outer log is within 3 ulp of |g| <= 17.  Total
// |g error| < 2e-5: the same tokens as accurate fp32 logs except at top-2
// gaps below that, far inside the north-star's 1e-2 gap rule.
__device__ __forceinline__ float gumbel_fast(uint32_t x) {
  const uint32_t k = x >> 9;
  const float u = (__uint2float_rn(k) + 0.5f) * 1.1920928955078125e-07f;
  const float v = (__uint2float_rn((1u << 23) - k) - 0.5f) * 1.1920928955078125e-07f;
  const float ser = v * (1.f + v * (0.5f + v * (0.33333334f + v * (0.25f + v * (0.2f + v * 0.16666667f)))));
  const float t = k >= (1u << 23) - (1u << 18) ? ser : -__logf(u);
  return -__logf(t);
}

// Under tensor parallelism `logits` holds the vocab shard [v0, v0 + V): the
// noise and the packed index use the global vocab id, only the shard owning
// EOS masks / forces it, and the per-row maxima are then MAX-all-reduced.
__global__ void __launch_bounds__(256) sampler_kernel(const float* __restrict__ logits, int V, int v0, int row_div,
                                                       RoundDev R, uint32_t k0, uint32_t k1, float inv_temp,
                                                       uint32_t round_id) {
  pdl_wait();
  pdl_launch_dependents();
  const int n = R.ctl->n_live;
  const int t = R.ctl->t;
  const int chunks = (V + SAMP_CHUNK - 1) / SAMP_CHUNK;
  __shared__ unsigned long long red[8];
  for (int u = blockIdx.x; u < n * chunks; u += gridDim.x) {
    const int i = u / chunks, ch = u % chunks;
    const int s = R.live[i];
    const int tl = t - R.t0[s];                    // this response's token index
    const int L = R.trace ? R.trace_L[s] : 0x7FFFFFFF;
    if (R.trace && tl == L) {                       // forced EOS at the trace length
      if (ch == 0 && threadIdx.x == 0 && R.eos >= v0 && R.eos < v0 + V)
        atomicMax(&R.best[i], pack_arg(INFINITY, (uint32_t)R.eos));
      continue;
    }
    const uint32_t uid = (uint32_t)(R.p_gid[R.slot_prompt[s]] * R.G + R.slot_j[s]);
    const float* lr = logits + (size_t)(i / row_div) * V;
    unsigned long long best = 0ull;
    const int v_end = min(V, (ch + 1) * SAMP_CHUNK);
    for (int b = ch * (SAMP_CHUNK / 4) + threadIdx.x; 4 * b < v_end; b += blockDim.x) {
      const float4 z4 = *(const float4*)(lr + 4 * b);
      const U4 x = philox((uint32_t)(b + (v0 >> 2)), (uint32_t)tl, uid, round_id, k0, k1);
      const float zl[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int v = v0 + 4 * b + w;                 // global vocab id
        float z = zl[w] * inv_temp + gumbel_fast(u4_word(x, w));
        if (R.trace && v == R.eos) z = -INFINITY;   // tl < L here
        const unsigned long long p = pack_arg(z, (uint32_t)v);
        best = p > best ? p : best;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y > best ? y : best;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long b2 = red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b2 = red[w] > b2 ? red[w] : b2;
      atomicMax(&R.best[i], b2);
    }
    __syncthreads();
  }
}

void launch_sampler(const float* logits, int V, int v0, int row_div, const RoundDev& R, uint64_t seed,
                    float inv_temp, uint32_t round_id, cudaStream_t st) {
  launch_pdl(sampler_kernel, dim3(148 * 4), dim3(256), 0, st, logits, V, v0, row_div, R, (uint32_t)seed,
             (uint32_t)(seed >> 32), inv_temp, round_id);
}

// --------------------------------------------------------------------- ctl
constexpr int CTL_THREADS = 1024;

// Phase A (everything that does not depend on the other ranks): finish
// detection, prompts completed at step t (index order), page frees of ended
// sequences, and the counts exchanged between DP ranks: {k, rows still live,
// error}.
__device__ __forceinline__ int pages_of(int tokens) { return (tokens + kPage - 1) / kPage; }

// KV pressure (NEXT-2, reading Z26; oracle sched.kv_step_loop): while the
// survivors' next-step pages exceed the free pages, preempt the most recently
// admitted prompt with a live response (never the last one), freeing its
// responses' private pages; a step that preempts nothing re-admits waiting
// prompts from the head of the FIFO while their pages fit.  Updates the
// phase-A tallies in place.  Called by every thread.
__device__ void ctl_kv_pressure(const RoundDev& R, int* scan_sm, int& s_top, int& s_keep, int& s_need, int& s_err,
                                long long& s_ctx, int& s_pause) {
  __shared__ int v_need, v_top, v_preempted;
  CtlBlock* C = R.ctl;
  const int n = C->n_live;
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid == 0) { v_need = s_need; v_top = s_top; v_preempted = 0; }
  __syncthreads();
  if (v_need > v_top && !s_err) {
    for (int p = tid; p < R.n_prompts; p += CTL_THREADS) { R.p_live[p] = 0; R.p_pfree[p] = 0; R.p_pneed[p] = 0; }
    __syncthreads();
    for (int i = tid; i < n; i += CTL_THREADS) {
      const int s = R.live[i];
      if (R.status[s] != ST_LIVE) continue;
      const int p = R.slot_prompt[s];
      atomicAdd(&R.p_live[p], 1);
      atomicAdd(&R.p_pfree[p], pages_of(R.kv_len[s]) - R.own0[s]);
      atomicAdd(&R.p_pneed[p], R.kv_len[s] % kPage == 0 ? 1 : 0);
    }
    __syncthreads();
    if (tid == 0) {
      // LIFO whole-prompt victims until the survivors' pages fit
      while (v_need > v_top) {
        int live_p = 0, v = -1;
        for (int p = 0; p < R.n_prompts; ++p)
          if (R.p_live[p] > 0) { ++live_p; if (v < 0 || R.p_adm[p] > R.p_adm[v]) v = p; }
        if (live_p <= 1) { s_err = 1; break; }     // the last live prompt does not fit: exhausted
        v_top += R.p_pfree[v];
        v_need -= R.p_pneed[v];
        R.p_live[v] = 0;
        R.p_wait[v] = PW_VICTIM;
        R.wait_q[C->wait_tail % R.P] = v;
        C->wait_tail += 1;
        C->preemptions += 1;
        v_preempted = 1;
      }
    }
    __syncthreads();
    // free the victims' private pages; recount the survivors
    if (tid == 0) { s_keep = 0; s_need = 0; s_ctx = 0; }
    __syncthreads();
    for (int base = 0; base < n; base += CTL_THREADS) {
      const int i = base + tid;
      int cnt = 0, keep = 0, need = 0, s = -1;
      if (i < n) {
        s = R.live[i];
        if (R.status[s] == ST_LIVE) {
          if (R.p_wait[R.slot_prompt[s]] == PW_VICTIM) {
            R.status[s] = ST_PREEMPTED;
            cnt = pages_of(R.kv_len[s]) - R.own0[s];
          } else {
            keep = 1;
            need = R.kv_len[s] % kPage == 0 ? 1 : 0;
          }
        }
      }
      int tot, tk, tn, tc;
      const int off = block_exscan(cnt, &tot, scan_sm);
      block_exscan(keep, &tk, scan_sm);
      block_exscan(need, &tn, scan_sm);
      block_exscan(keep ? R.kv_len[s] + 1 : 0, &tc, scan_sm);
      for (int c = 0; c < cnt; ++c)
        R.free_stack[s_top + off + c] = R.page_table[(size_t)s * R.maxp + R.own0[s] + c];
      __syncthreads();
      if (tid == 0) { s_top += tot; s_keep += tk; s_need += tn; s_ctx += tc; }
      __syncthreads();
    }
    for (int p = tid; p < R.n_prompts; p += CTL_THREADS)
      if (R.p_wait[p] == PW_VICTIM) R.p_wait[p] = PW_WAITING;
    __syncthreads();
  }
  // re-admission (a step that preempted nothing): FIFO head first, while the
  // recomputed prefix + the next append of every preempted response fit
  if (tid == 0) {
    C->readmit_n = 0; C->readmit_rows = 0; C->readmit_pages = 0;
    if (!v_preempted && !s_err && C->wait_head < C->wait_tail) {
      int avail = s_top - s_need, rows = 0, pages = 0, nre = 0;
      long long ctx = 0;
      for (int q = C->wait_head; q < C->wait_tail; ++q) {
        const int v = R.wait_q[q % R.P];
        int req = 0, cnt = 0;
        for (int j = 0; j < R.G; ++j) {
          const int s = v * R.G + j;
          if (R.status[s] == ST_PREEMPTED) { req += pages_of(R.p_plen[v] + R.gen[s]) - R.own0[s]; ++cnt; }
        }
        if (req > avail) break;
        avail -= req;
        for (int j = 0; j < R.G; ++j) {
          const int s = v * R.G + j;
          if (R.status[s] != ST_PREEMPTED) continue;
          int* J = R.rejobs + 5 * (rows++);
          J[0] = s; J[1] = R.gen[s];
          J[2] = R.page_table[(size_t)(R.S + v) * R.maxp + R.own0[s]];   // the prompt's partial page
          J[3] = -1;
          J[4] = R.p_plen[v] % kPage;
          ctx += R.p_plen[v] + R.gen[s];
        }
        pages += req;
        R.p_wait[v] = PW_READMIT;
        ++nre;
      }
      C->readmit_n = nre; C->readmit_rows = rows; C->readmit_pages = pages;
      s_keep += rows; s_need += pages; s_ctx += ctx;
      s_pause = nre > 0;
    }
    if (!s_err && s_keep == 0 && C->wait_head < C->wait_tail && C->readmit_n == 0) s_err = 1;   // head never fits
  }
  __syncthreads();
}

__device__ void ctl_phase_a(const RoundDev& R, int appended, int* scan_sm) {
  __shared__ int s_k, s_top, s_keep, s_need, s_err, s_pause;
  __shared__ long long s_ctx, s_rd, s_ru;
  CtlBlock* C = R.ctl;
  const int n = C->n_live;
  const int t = C->t;
  const int tid = threadIdx.x;
  if (R.trace_buf && t <= R.trace_steps) {
    int* tb = R.trace_buf + (size_t)(t - 1) * (2 + R.S);
    for (int i = tid; i < n; i += CTL_THREADS) tb[2 + i] = R.live[i];
    if (tid == 0) tb[0] = n;
  }
  for (int i = tid; i < n; i += CTL_THREADS) {
    const int s = R.live[i];
    const int tl = t - R.t0[s];
    const int tok = (int)unpack_idx(R.best[i]);
    R.tok_out[(size_t)s * R.cap + tl - 1] = tok;
    R.gen[s] = tl;
    if (appended) R.kv_len[s] += 1;
    const bool fin = tok == R.eos;
    const bool capped = !fin && tl >= R.cap;
    R.status[s] = fin ? ST_FINISHED : capped ? ST_CAPPED : ST_LIVE;
    if (fin || (capped && R.kind == 1)) atomicAdd(&R.p_cnt[R.slot_prompt[s]], 1);
  }
  if (tid == 0) {
    s_k = 0; s_top = C->free_top; s_keep = 0; s_need = 0; s_err = 0; s_ctx = 0; s_rd = 0; s_ru = 0; s_pause = 0;
    if (appended && R.rows_hist) R.rows_hist[n] += 1;   // one decode step over n rows
  }
  __syncthreads();
  // prompts completing at step t, in prompt-index order.  A prompt completes
  // when `keep` of its responses have finished ("finishing after
  // the first R0 complete"; keep == G without response-level speculation).
  // Of the siblings that finished at step t, the lowest j fill the remaining
  // keep slots (the rest are ST_DROPPED); siblings still decoding are aborted
  // at once, so their pages are freed below and they leave the batch.
  for (int base = 0; base < R.n_prompts; base += CTL_THREADS) {
    const int p = base + tid;
    int flag = 0;
    if (p < R.n_prompts && R.p_state[p] == PS_RUNNING && R.p_cnt[p] >= R.keep) flag = 1;
    int tot;
    const int off = block_exscan(flag, &tot, scan_sm);
    if (flag) {
      R.p_state[p] = PS_COMPLETE; R.comp_list[s_k + off] = p;
      if (R.keep < R.G) {
        const int tl = t - R.t0[p * R.G];
        int room = R.keep;
        for (int j = 0; j < R.G; ++j)
          if (R.status[p * R.G + j] == ST_FINISHED && R.gen[p * R.G + j] < tl) --room;
        for (int j = 0; j < R.G; ++j) {
          const int s = p * R.G + j;
          const int st = R.status[s];
          if (st == ST_LIVE) R.status[s] = ST_ABORTED;
          else if (st == ST_FINISHED && R.gen[s] == tl) { if (room > 0) --room; else R.status[s] = ST_DROPPED; }
        }
      }
    }
    __syncthreads();
    if (tid == 0) s_k += tot;
    __syncthreads();
  }
  // free the private pages of sequences that ended; count survivors and the
  // pages they need for the next append
  for (int base = 0; base < n; base += CTL_THREADS) {
    const int i = base + tid;
    int cnt = 0, s = -1, keep = 0, need = 0;
    if (i < n) {
      s = R.live[i];
      if (R.status[s] != ST_LIVE) {
        const int used = (R.kv_len[s] + kPage - 1) / kPage;
        cnt = max(0, used - R.own0[s]);
      } else {
        keep = 1;
        if (R.max_active) R.p_stamp[R.slot_prompt[s]] = t;
        if (R.kv_len[s] % kPage == 0) {
          need = 1;
          if (R.kv_len[s] / kPage >= R.maxp) atomicExch(&s_err, 2);
        }
      }
    }
    int tot, tk, tn, tc, trd, tru;
    // KV tokens the attention of this step read for row i: its context incl. the appended token;
    // unique: the prompt's shared full pages once per prompt (its first live row; siblings are
    // adjacent in the live list) + every row's private tokens
    block_exscan(i < n && appended ? R.kv_len[s] : 0, &trd, scan_sm);
    int ru = 0;
    if (i < n && appended) {
      const int sh = R.own0[s] * kPage;
      ru = R.kv_len[s] - sh;
      if (i == 0 || R.slot_prompt[R.live[i - 1]] != R.slot_prompt[s]) ru += sh;
    }
    block_exscan(ru, &tru, scan_sm);
    const int off = block_exscan(cnt, &tot, scan_sm);
    block_exscan(keep, &tk, scan_sm);
    block_exscan(need, &tn, scan_sm);
    block_exscan(keep ? R.kv_len[s] + 1 : 0, &tc, scan_sm);
    for (int c = 0; c < cnt; ++c)
      R.free_stack[s_top + off + c] = R.page_table[(size_t)s * R.maxp + R.own0[s] + c];
    __syncthreads();
    if (tid == 0) { s_top += tot; s_keep += tk; s_need += tn; s_ctx += tc; s_rd += trd; s_ru += tru; }
    __syncthreads();
  }
  if (R.preempt) ctl_kv_pressure(R, scan_sm, s_top, s_keep, s_need, s_err, s_ctx, s_pause);
  // Continuous issuance (NEXT-4; oracle sched.issue_step_loop): after
  // step t the lowest-index unissued prompts of this rank are issued while
  // fewer than max_active prompts have a live response.  An issued prompt's G
  // sequences decode its last prompt token at step t + 1 (their KV holds the
  // other plen - 1 tokens since submit), producing token 1 there.
  int issue_n = 0;
  if (R.max_active) {
    __syncthreads();
    const int n_is = C->n_issued;
    int active = 0;
    for (int base = 0; base < n_is; base += CTL_THREADS) {
      int tot;
      block_exscan(base + tid < n_is && R.p_stamp[base + tid] == t ? 1 : 0, &tot, scan_sm);
      active += tot;
    }
    issue_n = max(0, min(R.max_active - active, R.n_prompts - n_is));
    for (int base = 0; base < issue_n * R.G; base += CTL_THREADS) {
      const int r = base + tid;
      int need = 0, ctx = 0;
      if (r < issue_n * R.G) {
        const int s = n_is * R.G + r;
        ctx = R.kv_len[s] + 1;
        if (R.kv_len[s] % kPage == 0) {
          need = 1;
          if (R.kv_len[s] / kPage >= R.maxp) atomicExch(&s_err, 2);
        }
      }
      int tn, tc;
      block_exscan(need, &tn, scan_sm);
      block_exscan(ctx, &tc, scan_sm);
      if (tid == 0) { s_need += tn; s_ctx += tc; }
      __syncthreads();
    }
  }
  if (tid == 0) {
    s_keep += issue_n * R.G;
    C->issue_n = issue_n;
    if (s_need > s_top && !s_err) s_err = 1;
    C->free_top = s_top;
    C->k_step = s_k;
    C->n_next = s_keep;
    C->need_pages = s_need;
    C->ctx_sum = s_ctx;
    C->kv_read += s_rd;
    C->kv_read_unique += s_ru;
    R.ks_local[0] = s_k; R.ks_local[1] = s_keep; R.ks_local[2] = s_err; R.ks_local[3] = s_pause;
    if (R.world == 1) { R.ks[0] = s_k; R.ks[1] = s_keep; R.ks[2] = s_err; R.ks[3] = s_pause; }
  }
}

// Phase B: the DP cutoff (S:289-297 under sharding): rank r admits
// min(k_r, max(0, target - acc - sum_{r'<r} k_r')) of its completed prompts,
// lowest index first; then stable compaction, page allocation, next-step
// inputs and attention items, and the (globally identical) done decision.
__device__ void ctl_phase_b(const RoundDev& R, int* scan_sm) {
  __shared__ int s_take, s_acc_new, s_next_global, s_err, s_pause;
  CtlBlock* C = R.ctl;
  const int n = C->n_live;
  const int t = C->t;
  const int tid = threadIdx.x;
  if (tid == 0) {
    const int acc = C->acc;
    int take = 0, total = 0, nextg = 0, err = 0, pause = 0;
    for (int r = 0; r < R.world; ++r) {
      const int kr = R.ks[4 * r];
      const int tr = min(kr, max(0, R.target - acc - total));
      if (r == R.rank) take = tr;
      total += tr;
      nextg += R.ks[4 * r + 1];
      err = max(err, R.ks[4 * r + 2]);
      pause |= R.ks[4 * r + 3];
    }
    s_take = take; s_acc_new = acc + total; s_next_global = nextg; s_err = err; s_pause = pause;
  }
  __syncthreads();
  for (int r = tid; r < s_take; r += CTL_THREADS) {
    const int p = R.comp_list[r];
    R.p_state[p] = PS_ACCEPTED;
    R.accept_order[C->acc_local + r] = p;
  }
  const int top = C->free_top;
  // Key splits: the flat (item, KV head) work list should fill one wave of
  // 148 CTAs with units of about equal size.  Row r gets
  // ns_r = max(1, floor(ctx_r * U / sum ctx)) splits, U = 148 / KV (so
  // sum ns_r <= U whenever no row is forced up to 1), each of
  // ceil(ctx_r / ns_r) tokens rounded up to whole pages.
  const long long ctx_total = max(1LL, C->ctx_sum);
  // rows n .. n + nis - 1 are the sequences issued after this step (none once
  // the target is reached: the round ends here)
  const int n_is0 = C->n_issued;
  const int nis = s_acc_new >= R.target ? 0 : C->issue_n * R.G;
  // ... or (KV pressure, exclusive with issuance) the responses re-admitted
  // after this step, in re-admission order: their KV restarts at the
  // recomputed prefix plen + g - 1 and they decode token g + 1 next
  const int nrd = s_acc_new >= R.target || s_err ? 0 : C->readmit_rows;
  for (int e = tid; e < nrd; e += CTL_THREADS) {
    const int sl = R.rejobs[5 * e];
    R.kv_len[sl] = R.p_plen[R.slot_prompt[sl]] + R.gen[sl] - 1;
    R.status[sl] = ST_LIVE;
    R.t0[sl] = t - R.gen[sl];        // its token index at step t + 1 is g + 1 (the counter of its next token)
  }
  __syncthreads();
  const int nx = nis + nrd;
#define EXTRA_SLOT(e) (nrd ? R.rejobs[5 * (e)] : n_is0 * R.G + (e))   // (#undef at the end of phase B)
  // Full waves: with k = ceil(rows / U1) in {2, 3} (between one and three
  // waves' worth of rows per head) budget k whole waves so the flat list
  // does not end in a partial wave; the splits left over by the floors go one
  // each to the first rows.  Measured (profiles/r01_attn_waves_ab.txt): -3% step
  // time at 40-48 rows, neutral at 56 and 83, but +2-6% at k >= 4 (more,
  // smaller units cost more merges than the balance saves), so k >= 4 and
  // k = 1 keep the plain floor.  R.attn_waves = 0 disables it (A/B).
  const int U1 = R.attn_units > 0 ? R.attn_units : max(1, 148 / R.kv_heads);
  int U = U1, left = 0;
  const int kw = (C->n_next + U1 - 1) / U1;
  if (R.attn_waves && !s_err && kw >= 2 && kw <= 3) {
    U = U1 * kw;
    int sum = 0;
    for (int base = 0; base < n + nx; base += CTL_THREADS) {
      const int i = base + tid;
      int b = 0;
      if (i < n + nx) {
        const int s = i < n ? R.live[i] : EXTRA_SLOT(i - n);
        if (i >= n || R.status[s] == ST_LIVE) b = (int)((long long)(R.kv_len[s] + 1) * U / ctx_total);
      }
      int tot;
      block_exscan(b, &tot, scan_sm);
      sum += tot;
    }
    left = max(0, U - sum);
  }
  int kept = 0, alloc = 0, items = 0;
  if (!s_err) {
    for (int base = 0; base < n + nx; base += CTL_THREADS) {
      const int i = base + tid;
      int keep = 0, need = 0, ns = 0, chunk = 0, s = -1;
      if (i < n + nx) {
        s = i < n ? R.live[i] : EXTRA_SLOT(i - n);
        keep = i >= n || R.status[s] == ST_LIVE;
        if (keep) {
          const int ctx = R.kv_len[s] + 1;
          // a re-admitted response takes the pages of its recomputed prefix and the next append
          need = (i >= n && nrd) ? pages_of(ctx) - R.own0[s] : (R.kv_len[s] % kPage) == 0;
          const int want = (int)max(1LL, (long long)ctx * U / ctx_total);
          chunk = ((ctx + want - 1) / want + kPage - 1) / kPage * kPage;   // whole pages per split
          ns = (ctx + chunk - 1) / chunk;
        }
      }
      int tk, ta, ti;
      const int ok = block_exscan(keep, &tk, scan_sm);
      if (keep && U != U1) {                // re-derive this row's splits with the leftover share
        const int ctx = R.kv_len[s] + 1;
        const int want = max(1, (int)((long long)ctx * U / ctx_total) + (kept + ok < left ? 1 : 0));
        chunk = ((ctx + want - 1) / want + kPage - 1) / kPage * kPage;
        ns = (ctx + chunk - 1) / chunk;
      }
      const int oa = block_exscan(need, &ta, scan_sm);
      const int oi = block_exscan(ns, &ti, scan_sm);
      if (keep) {
        const int pos = kept + ok;
        const int kv = R.kv_len[s];
        R.live_next[pos] = s;
        if (i < n) {
          R.tok_in[pos] = R.tok_out[(size_t)s * R.cap + (t - R.t0[s]) - 1];
        } else if (nrd) {
          R.tok_in[pos] = R.tok_out[(size_t)s * R.cap + R.gen[s] - 1];   // its last token (index g)
        } else {
          R.tok_in[pos] = R.p_last_tok[R.slot_prompt[s]];
          R.t0[s] = t;
        }
        R.row_pos[pos] = kv;
        R.row_pt[pos] = s;
        if (i >= n && nrd) {
          for (int k = 0; k < need; ++k)
            R.page_table[(size_t)s * R.maxp + R.own0[s] + k] = R.free_stack[top - 1 - (alloc + oa + k)];
          R.rejobs[5 * (i - n) + 3] = R.page_table[(size_t)s * R.maxp + R.own0[s]];   // fork destination
        } else if (need) {
          R.page_table[(size_t)s * R.maxp + kv / kPage] = R.free_stack[top - 1 - (alloc + oa)];
        }
        if (R.attn_group) R.grp_key[pos] = R.slot_prompt[s] * ((R.G + 7) / 8) + R.slot_j[s] / 8;
        const int it0 = items + oi;
        for (int sp = 0; sp < ns; ++sp) {
          AttnItem I;
          I.q_row0 = pos; I.n_qtok = 1; I.pos0 = kv; I.pt_row = s;
          I.kv_lo = sp * chunk; I.kv_hi = min(kv + 1, (sp + 1) * chunk);
          I.nsplit = ns; I.item0 = it0;
          if (it0 + sp < R.max_items) R.items[it0 + sp] = I;   // capacity proven in compute_sizes
        }
      }
      kept += tk; alloc += ta; items += ti;
    }
  }
  __syncthreads();
  // sibling-group work list for the group kernel, when the host may run the
  // next step with it (more than group_rows_min rows, or a group-mode graph
  // is running); the per-row list above is always built
  int gcnt = 0;
  if (R.attn_group && !s_err && (kept > R.group_rows_min || *R.gmode)) {
    int items = 0;   // shadows the per-row count in this block
    // Sibling groups (k_attn_group.cu): runs of next-step rows with the same
    // (prompt, j / 8) -- siblings are adjacent in the live list (slot order,
    // order-preserving compaction) -- cut into groups of 8 / 4 / 2 / 1 members
    // (the binary decomposition of the run length, largest first), so the 8
    // consumer warps divide evenly over the members (rep = 8 / members).  A
    // group's work is its longest member's pages x members / 8 per warp;
    // splits ns_g = max(1, floor(c_g * Ug / sum c)) with Ug <= 3 * U1 whole
    // waves, so items <= groups + Ug <= S + 3 * U1 (the work-list capacity).
    int ng = 0, nsib = 0, saved = 0, pages_all = 0;
    for (int base = 0; base < kept; base += CTL_THREADS) {
      const int pos = base + tid;
      int st = 0, sib = 0, sv = 0, pg = 0;
      if (pos < kept) {
        const int key = R.grp_key[pos];
        int k = 0, n = 1;
        while (k < 7 && pos - k - 1 >= 0 && R.grp_key[pos - k - 1] == key) ++k;
        n += k;
        while (n < 8 && pos + (n - k) < kept && R.grp_key[pos + (n - k)] == key) ++n;
        sib = k == 0;
        pg = pages_of(R.row_pos[pos] + 1);
        for (int b = 8, off = 0; b >= 1; b >>= 1)
          if (n & b) {
            if (k == off) {   // a group of b members starts here: b - 1 fills saved per shared page
              st = 1;
              sv = min(R.own0[R.live_next[pos]], R.row_pos[pos] / kPage) * (b - 1);
            }
            off += b;
          }
      }
      int tot, tsib, tsv, tpg;
      const int o = block_exscan(st, &tot, scan_sm);
      block_exscan(sib, &tsib, scan_sm);
      block_exscan(sv, &tsv, scan_sm);
      block_exscan(pg, &tpg, scan_sm);
      if (st) R.grp_start[ng + o] = pos;
      ng += tot;
      nsib += tsib;
      saved += tsv;
      pages_all += tpg;
    }
    // Sibling groups pay off when they save a large share of the page fills:
    // with few sibling runs (nsib < U1 / 8, e.g. 16 rows of 2 prompts) the
    // groups would need ~U1 / nsib page splits each to fill the wave, whose
    // partials and merges cost more than the fills save, and late in a round
    // (long private tails, small groups) the shared prompt pages are a small
    // share of the reads.  Then every row is its own group (8 warps split its
    // pages, as the per-row list did): below 40% of the fills saved, measured
    // on the bench rounds (profiles/r02_attn_group_ab.txt).  attn_group 2 / 3
    // force sibling groups / single rows (A/B).
    if (R.attn_group == 3 || (R.attn_group == 1 && (nsib * 8 < U1 || saved * 10 < pages_all * 4))) {
      for (int pos = tid; pos < kept; pos += CTL_THREADS) R.grp_start[pos] = pos;
      ng = kept;
    }
    if (tid == 0) R.grp_start[ng] = kept;
    __syncthreads();
    if (R.attn_group == 4) {
      // Shared pages in group units (every member's columns, one fill per
      // page), private pages in per-row units (8 warps page-parallel); each
      // member row's partials (kRowSplits slots) are merged by the last of
      // its units.  Cost in warp-pages: shared pages x members / 8, private
      // pages / 8; splits ns = clamp(floor(c * Ug / sum c), 1, 16) per part.
      struct GInfo { int p0, nm, snp, w[8]; };
      auto ginfo = [&](int gi) {
        GInfo q;
        q.p0 = R.grp_start[gi];
        q.nm = min(8, R.grp_start[gi + 1] - q.p0);
        q.snp = 1 << 30;
        for (int x = 0; x < q.nm; ++x) {
          const int sl = R.live_next[q.p0 + x], pos = R.row_pos[q.p0 + x];
          q.w[x] = pages_of(pos + 1);
          q.snp = min(q.snp, min(R.own0[sl], pos / kPage));
        }
        return q;
      };
      auto parts = [&](const GInfo& q, int ug, long long csum, int& ns_s, int& ch_s, int* ns_p, int* ch_p) {
        const int c_s = (q.snp * q.nm + 7) / 8;
        int want = ug > 0 ? (int)max(1LL, min(16LL, (long long)c_s * ug / csum)) : 1;
        ns_s = 0; ch_s = 1;
        if (q.snp > 0) { ch_s = (q.snp + want - 1) / want; ns_s = (q.snp + ch_s - 1) / ch_s; }
        int units = ns_s;
        for (int x = 0; x < q.nm; ++x) {
          const int pp = q.w[x] - q.snp;
          ns_p[x] = 0; ch_p[x] = 1;
          if (pp > 0) {
            want = ug > 0 ? (int)max(1LL, min(16LL, (long long)((pp + 7) / 8) * ug / csum)) : 1;
            ch_p[x] = (pp + want - 1) / want;
            ns_p[x] = (pp + ch_p[x] - 1) / ch_p[x];
          }
          units += ns_p[x];
        }
        return units;
      };
      long long csum = 0;
      int nbase = 0;
      for (int base = 0; base < ng; base += CTL_THREADS) {
        const int gi = base + tid;
        int c = 0, nb = 0, tot;
        if (gi < ng) {
          const GInfo q = ginfo(gi);
          c = (q.snp * q.nm + 7) / 8;
          nb = q.snp > 0 ? 1 : 0;
          for (int x = 0; x < q.nm; ++x)
            if (q.w[x] > q.snp) { c += (q.w[x] - q.snp + 7) / 8; ++nb; }
        }
        block_exscan(c, &tot, scan_sm);
        csum += tot;
        block_exscan(nb, &tot, scan_sm);
        nbase += tot;
      }
      csum = max(1LL, csum);
      const int Ug = U1 * min(3, max(1, (nbase + U1 - 1) / U1));
      AttnGroupItem* gitems = R.gitems;
      int items = 0;
      for (int base = 0; base < ng; base += CTL_THREADS) {
        const int gi = base + tid;
        int units = 0, ns_s = 0, ch_s = 1, ns_p[8], ch_p[8];
        GInfo q;
        if (gi < ng) {
          q = ginfo(gi);
          units = parts(q, Ug, csum, ns_s, ch_s, ns_p, ch_p);
        }
        int tot;
        const int o = block_exscan(units, &tot, scan_sm);
        if (gi < ng) {
          int it = items + o;
          AttnGroupItem I;
          I.nsplit = 1; I.item0 = 0; I.rowmerge = 1; I.shared_np = q.snp;
          for (int x = 0; x < 8; ++x) {
            const bool m = x < q.nm;
            I.q_row[x] = m ? q.p0 + x : 0;
            I.pt_row[x] = m ? R.live_next[q.p0 + x] : 0;
            I.pos0[x] = m ? R.row_pos[q.p0 + x] : -1;
            I.nspl[x] = m ? ns_s + ns_p[x] : 1;
          }
          // shared units: every member
          I.n_mem = q.nm; I.rep = 8 / q.nm;
          for (int k = 0; k < ns_s; ++k, ++it) {
            I.pg_lo = k * ch_s; I.pg_hi = min(q.snp, (k + 1) * ch_s);
            for (int x = 0; x < 8; ++x) I.sidx[x] = k;
            if (it < R.max_items_g) gitems[it] = I;
          }
          // private units: one member each
          for (int x = 0; x < q.nm; ++x) {
            AttnGroupItem J = I;
            J.n_mem = 1; J.rep = 8;
            J.q_row[0] = I.q_row[x]; J.pt_row[0] = I.pt_row[x]; J.pos0[0] = I.pos0[x]; J.nspl[0] = I.nspl[x];
            for (int y = 1; y < 8; ++y) { J.q_row[y] = 0; J.pt_row[y] = 0; J.pos0[y] = -1; J.nspl[y] = 1; J.sidx[y] = 0; }
            for (int k = 0; k < ns_p[x]; ++k, ++it) {
              J.pg_lo = q.snp + k * ch_p[x]; J.pg_hi = min(q.w[x], q.snp + (k + 1) * ch_p[x]);
              J.sidx[0] = ns_s + k;
              if (it < R.max_items_g) gitems[it] = J;
            }
          }
        }
        items += tot;
      }
      gcnt = items;
    } else {
    auto gcost = [&](int gi, int& w, int& nm, int& rep) {
      const int p0 = R.grp_start[gi];
      nm = min(8, R.grp_start[gi + 1] - p0);
      w = 0;
      for (int x = 0; x < nm; ++x) w = max(w, pages_of(R.row_pos[p0 + x] + 1));
      rep = 8 / nm;                     // nm in {1, 2, 4, 8}: warps per member (k_attn_group.cu)
      return (w + rep - 1) / rep;
    };
    long long csum = 0;
    for (int base = 0; base < ng; base += CTL_THREADS) {
      const int gi = base + tid;
      int w, nm, rep, c = 0, tot;
      if (gi < ng) c = gcost(gi, w, nm, rep);
      block_exscan(c, &tot, scan_sm);
      csum += tot;
    }
    csum = max(1LL, csum);
    const int Ug = U1 * min(3, max(R.group_waves, (ng + U1 - 1) / U1));   // whole waves (one-wave cap measured slower)
    auto nsplits = [&](int c, int w, int ug, int& chunk) {
      const int want = (int)max(1LL, min(32LL, (long long)c * ug / csum));   // <= 32: the merge's smem
      chunk = (w + want - 1) / want;
      return (w + chunk - 1) / chunk;
    };
    AttnGroupItem* gitems = R.gitems;
    for (int base = 0; base < ng; base += CTL_THREADS) {
      const int gi = base + tid;
      int w = 0, nm = 0, rep = 1, ns = 0, chunk = 1;
      if (gi < ng) ns = nsplits(gcost(gi, w, nm, rep), w, Ug, chunk);
      int tot;
      const int o = block_exscan(ns, &tot, scan_sm);
      if (gi < ng) {
        const int p0 = R.grp_start[gi], it0 = items + o;
        AttnGroupItem I;
        I.n_mem = nm; I.nsplit = ns; I.item0 = it0; I.rep = rep; I.rowmerge = 0;
        int snp = 1 << 30;
        for (int x = 0; x < 8; ++x) {
          const int s = x < nm ? R.live_next[p0 + x] : 0;
          I.q_row[x] = x < nm ? p0 + x : 0;
          I.pt_row[x] = s;
          I.pos0[x] = x < nm ? R.row_pos[p0 + x] : -1;
          if (x < nm) snp = min(snp, min(R.own0[s], R.row_pos[p0 + x] / kPage));
        }
        I.shared_np = snp;
        for (int sp = 0; sp < ns; ++sp) {
          I.pg_lo = sp * chunk; I.pg_hi = min(w, (sp + 1) * chunk);
          if (it0 + sp < R.max_items_g) gitems[it0 + sp] = I;
        }
      }
      items += tot;
    }
    gcnt = items;
    }   // attn_group 1-3
  }
  for (int i = tid; i < n; i += CTL_THREADS) R.best[i] = 0ull;
  for (int i = tid; i < kept; i += CTL_THREADS) R.live[i] = R.live_next[i];
  if (tid == 0) {
    C->acc = s_acc_new;
    C->acc_local += s_take;
    C->decoded += n;
    C->free_top = top - alloc;
    C->n_items = min(items, R.max_items);
    C->n_gitems = min(gcnt, R.max_items_g);
    C->n_issued = n_is0 + nis / R.G;
    C->issue_n = 0;
    // commit the re-admissions: popped from the FIFO, newest admissions
    C->n_rejobs = nrd;
    if (nrd)
      for (int q = 0; q < C->readmit_n; ++q) {
        const int v = R.wait_q[(C->wait_head + q) % R.P];
        R.p_wait[v] = PW_NONE;
        R.p_adm[v] = ++C->adm_ctr;
      }
    if (nrd) C->wait_head += C->readmit_n;
    if (items > R.max_items || gcnt > R.max_items_g) s_err = 3;    // unreachable by the bound S + 3 * U1; fail loudly if not
    const bool done = s_acc_new >= R.target || s_next_global == 0 || s_err;
    if (R.trace_buf && t <= R.trace_steps) {
      int* tb = R.trace_buf + (size_t)(t - 1) * (2 + R.S);
      tb[1] = s_acc_new | (done ? (1 << 30) : 0);
    }
    if (s_err) C->err = s_err;
    if (done) {
      C->done = 1; C->t_end = t; C->n_final = kept; C->n_live = 0;
      C->underfilled = s_acc_new < R.target;
    } else if (s_pause) {
      // some rank re-admitted responses: every rank holds the next step
      // until the host recomputed their KV (rp_step, between steps)
      C->pause = 1; C->n_live_saved = kept; C->n_items_saved = min(items, R.max_items);
      C->n_gitems_saved = min(gcnt, R.max_items_g);
      C->n_live = 0; C->n_items = 0; C->n_gitems = 0; C->t = t + 1;
    } else {
      C->n_live = kept; C->t = t + 1;
    }
  }
}

#undef EXTRA_SLOT

__global__ void __launch_bounds__(CTL_THREADS) ctl_kernel(RoundDev R, int appended, int mode) {
  __shared__ int scan_sm[40];
  pdl_wait();
  pdl_launch_dependents();
  if (R.ctl->done || R.ctl->pause) return;
  if (mode != 2) ctl_phase_a(R, appended, scan_sm);
  if (mode == 0) { __threadfence_block(); __syncthreads(); }
  if (mode != 1) ctl_phase_b(R, scan_sm);
}

void launch_ctl(const RoundDev& R, int appended, int mode, cudaStream_t st) {
  launch_pdl(ctl_kernel, dim3(1), dim3(CTL_THREADS), 0, st, R, appended, mode);
}

// ------------------------------------------------------------ collect pack
// Pack the retained responses of the accepted prompts, in acceptance order,
// j ascending: all G in a long round, the `keep` finished ones in a short
// round.  meta[r] = {prompt (local index), j, len, status}; tokens contiguous.
__device__ __forceinline__ int retained_slot(const RoundDev& R, int r) {
  const int p = R.accept_order[r / R.keep];
  int q = r % R.keep;
  for (int j = 0; j < R.G; ++j) {
    const int s = p * R.G + j;
    if (R.kind == 1 || R.status[s] == ST_FINISHED) {
      if (q == 0) return s;
      --q;
    }
  }
  return p * R.G;   // unreachable: an accepted prompt has keep retained responses
}

__global__ void collect_offsets_kernel(RoundDev R, int first, int* meta, int* offs) {
  __shared__ int scan_sm[40];
  const int acc = R.ctl->acc_local;
  const int nr = max(0, acc - first) * R.keep;
  int base_off = 0;
  for (int base = 0; base < nr; base += blockDim.x) {
    const int r = base + threadIdx.x;
    int len = 0;
    if (r < nr) {
      const int s = retained_slot(R, first * R.keep + r), p = R.slot_prompt[s], j = R.slot_j[s];
      len = R.gen[s];
      meta[4 * r] = p; meta[4 * r + 1] = j; meta[4 * r + 2] = len; meta[4 * r + 3] = R.status[s];
    }
    int tot;
    const int off = block_exscan(len, &tot, scan_sm);
    if (r < nr) offs[r] = base_off + off;
    base_off += tot;
  }
  if (threadIdx.x == 0) offs[nr] = base_off;
}

__global__ void collect_copy_kernel(RoundDev R, int first, const int* offs, int* tokens) {
  const int nr = max(0, R.ctl->acc_local - first) * R.keep;
  for (int r = blockIdx.x; r < nr; r += gridDim.x) {
    const int s = retained_slot(R, first * R.keep + r);
    const int len = R.gen[s];
    for (int k = threadIdx.x; k < len; k += blockDim.x) tokens[offs[r] + k] = R.tok_out[(size_t)s * R.cap + k];
  }
}

void launch_collect_pack(const RoundDev& R, int first, int* meta, int* tokens, cudaStream_t st) {
  // offs lives right after meta: meta has 4*S ints, offs S+1
  int* offs = meta + 4 * R.S;
  collect_offsets_kernel<<<1, 1024, 0, st>>>(R, first, meta, offs);
  collect_copy_kernel<<<148, 256, 0, st>>>(R, first, offs, tokens);
}

}  // namespace rp
