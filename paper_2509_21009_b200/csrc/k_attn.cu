// Paged-KV GQA attention for decode and prefill (K4/K5).
//
// The KV pool is addressed by TMA as a 2-D tensor of token rows x head_dim
// (fp16, reading Z20): page p, layer l, KV head h, K|V is the 64-row block starting at row
// (((p*L + l)*KV + h)*2 + kv)*64.  One CTA = 1 producer warp + 3 consumer
// warps.  The producer streams whole pages (K and V, SWIZZLE_128B boxes of 64
// columns) into a 6-stage mbarrier ring; consumer warp w (of 3) owns the
// pages with global index = w mod 3 and therefore always the same 2 stages.  Work item = (query block, KV head, key
// split): the 16 MMA rows are the (query token, query head) pairs served by
// one KV head -- decode: 1 token x g heads (g = H/KV <= 8); prefill:
// floor(16/g) tokens x g heads with per-row causal limits.  S = Q K^T and
// O += P V run on mma.sync m16n8k16 (fp16, fp32 accumulate; a 16-row MMA is
// the natural shape for g <= 8 query rows) with an online softmax in the
// log2 domain; the warps merge in shared memory; multi-split blocks write
// (m, l, O) partials and the last split to finish (atomic ticket) combines
// them in split order.
// Decode attention moves g FLOP per KV byte, far below the ridge point: the
// design goal is bytes in flight (6 x 32 KB per SM) and few instructions per
// byte (one TMA per 8 KB box, 128 MMAs per 64-token page per warp).
#include <cuda.h>
#include "common.cuh"
#include "kernels.h"
#include "attn_mma.cuh"

namespace rp {

constexpr int AT_STAGES = 6;   // 64-token stages.  Stage s is always consumed by warp s % CW (CW divides
                               // AT_STAGES): mbarrier parity only tells adjacent phases apart, so every
                               // waiter must consume its stage's uses in order.

// debug timeline (RP_ATTN_TIMELINE): per CTA, %globaltimer marks of its first
// unit -- [0] start, [1] producer past the dependency wait, [2] first page
// ready (consumer warp 0), [3] last page consumed, [4] output / partial
// written, [5] split merge done, [6] end
__device__ long long* g_attn_tl = nullptr;
__device__ __forceinline__ long long attn_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ATL(k) do { if (g_attn_tl) g_attn_tl[blockIdx.x * 8 + (k)] = attn_gtimer(); } while (0)

template <int HD, int CW, int NQT>
struct AttnCfg {
  static constexpr int HALVES = HD / 64;             // 128-byte column halves (TMA boxes) per row
  static constexpr int TILE_BYTES = kPage * HD * 2;  // K (or V) block of one page
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int MR = 8 * NQT;                 // query rows per work unit (<= 8: decode, <= 16: prefill)
  static constexpr int MERGE_FLOATS = CW * MR * (HD + 2);
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int SMEM = AT_STAGES * STAGE_BYTES + MERGE_FLOATS * 4 + 1024 + 256;   // bars: full, empty, kvready
  static_assert(AT_STAGES % CW == 0, "stage ownership");
};

// S^T = K Q^T: the key tokens are the MMA rows (m16) and the <= 8 query rows
// of a work unit are the n8 columns, so no MMA lane is padding; P^T reaches
// the PV MMA through movmatrix.trans; O^T = V^T P^T keeps head_dim on the rows.
template <int HD, int CW, int NQT>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
attn_kernel(const __grid_constant__ CUtensorMap kv_map, const act_t* __restrict__ q, const act_t* __restrict__ q_lo,
            const int* __restrict__ page_table, int maxp, const AttnItem* __restrict__ items, const int* n_items_dev,
            int n_items_host, act_t* __restrict__ out, act_t* __restrict__ out_lo, float* __restrict__ partial,
            int* __restrict__ tickets, ModelDims m, int layer, QkvFuse fz) {
  using C = AttnCfg<HD, CW, NQT>;
  constexpr int MR = C::MR;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  float* mrg = (float*)(sm + AT_STAGES * C::STAGE_BYTES);
  uint64_t* bars = (uint64_t*)(mrg + C::MERGE_FLOATS);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(bars);
  const uint32_t empty0 = full0 + 8 * AT_STAGES;
  // fused QKV reduction (decode): the consumers append the current token's
  // k / v to its page, then release the producer's load of that page
  const uint32_t kvready = full0 + 16 * AT_STAGES;
  const bool fused = NQT == 1 && fz.part != nullptr;
  const bool skip_mma = fz.dbg & 1;
  if (fz.dbg & 2) q_lo = nullptr;

  // Decode (NQT == 1): the work list, page tables and every KV page except
  // the one holding a row's current position come from kernels that finished
  // before the QKV GEMM started (the round control of the previous step,
  // earlier steps' KV appends), so the producer streams pages before the
  // programmatic-dependency wait and waits only at the first page the QKV
  // GEMM still writes (its fused KV append); consumers wait before reading Q.
  // Prefill (rope_append wrote every prompt page) waits up front.
  constexpr bool kEarly = NQT == 1;
  if (threadIdx.x == 0) ATL(0);
  if (!kEarly) pdl_wait();
  pdl_launch_dependents();
  const int n_items = n_items_dev ? *n_items_dev : n_items_host;
  const int n_units = n_items * m.KV;            // flat (item, KV head) work units
  const int g = m.H / m.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < AT_STAGES; ++i) { bar_init(full0 + 8 * i, 1); bar_init(empty0 + 8 * i, 1); }
    bar_init(kvready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    // ===================== producer warp =====================
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&kv_map) : "memory");
    bool waited = !kEarly;
    long long gpage = 0;
    int kvn = 0;                                      // fused: KV-append units so far (kvready parity)
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int it = u / m.KV, kvh = u % m.KV;
      const AttnItem I = items[it];
      const int p_lo = I.kv_lo / kPage, npg = (I.kv_hi + kPage - 1) / kPage - p_lo;
      const int* ptab = page_table + (size_t)I.pt_row * maxp + p_lo;
      const bool kvu = fused && I.kv_hi == I.pos0 + 1;   // this unit holds the current token
      for (int j0 = 0; j0 < npg; j0 += 32) {
        const int mine = j0 + lane < npg ? ptab[j0 + lane] : 0;   // coalesced page-id batch
        const int cnt = min(32, npg - j0);
        for (int jj = 0; jj < cnt; ++jj) {
          const int page = __shfl_sync(0xffffffffu, mine, jj);
          if (lane == 0) {
            if (fused) {
              if (kvu && (p_lo + j0 + jj) == I.pos0 / kPage) {   // wait for the consumers' append
                mbar_wait_wd(kvready, (uint32_t)(kvn & 1), 300, it, I.pos0);
                ++kvn;
              }
            } else if (!waited && (p_lo + j0 + jj + 1) * kPage > I.pos0) {
              pdl_wait();
              waited = true;
              if (u == (int)blockIdx.x) ATL(1);
            }
            const long long gp = gpage + j0 + jj;
            const int st = (int)(gp % AT_STAGES);
            const uint32_t ph = (uint32_t)((gp / AT_STAGES) & 1);
            mbar_wait_wd(empty0 + 8 * st, ph ^ 1, 100 + st, gp, (long long)it * 1000 + npg);
            const uint32_t fb = full0 + 8 * st;
            bar_expect_tx(fb, C::STAGE_BYTES);
            const int row_k = (int)(kv_block_elems(layer, page, kvh, 0, m.n_pages, m.KV, HD) / HD);
            const uint32_t dst = sbase + st * C::STAGE_BYTES;
#pragma unroll
            for (int h = 0; h < C::HALVES; ++h) {
              tma2d(dst + h * 8192, &kv_map, fb, h * 64, row_k);
              tma2d(dst + C::TILE_BYTES + h * 8192, &kv_map, fb, h * 64, row_k + kPage);
            }
          }
        }
      }
      gpage += npg;
    }
    return;
  }

  // ===================== consumer warps =====================
  if (kEarly) pdl_wait();                         // Q and the current KV row come from the QKV GEMM
  const float scale = 1.4426950408889634f * rsqrtf((float)HD);
  const int tq = lane >> 2, tr = lane & 3;      // fragment row / column-pair coordinates
  long long gpage = 0;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int it = u / m.KV, kvh = u % m.KV;
    const AttnItem I = items[it];
    const int nrows = I.n_qtok * g;
    const int p_lo = I.kv_lo / kPage, npg = (I.kv_hi + kPage - 1) / kPage - p_lo;
    // ---- Q^T B fragments: qb[nq][kk] = {Q[row][kk*16 + 2tr..], Q[row][kk*16 + 8 + 2tr..]}, row = nq*8 + tq;
    // ql: the same fragments of q's fp16 rounding residual (split precision: S = K q_hi + K q_lo)
    uint32_t qb[NQT][HD / 16][2], ql[NQT][HD / 16][2];
    if (fused) {
      // the QKV GEMM's split partials of this row, summed in split order,
      // times the folded-RMSNorm scale, + bias, rotate-half RoPE at pos0
      float* xs = mrg;                            // [g + 2][HD] pre-RoPE q heads, k, v
      float* xr = mrg + (size_t)(g + 2) * HD;     // [g + 1][HD] rotated q heads, k
      __shared__ float s_rsc;
      const bool kvu = I.kv_hi == I.pos0 + 1;
      const int nrow = I.q_row0;
      const int bnx = (fz.gemm_lo && *fz.n_rows <= 128) ? 128 : 256;
      const int chunk = nrow / bnx, col = nrow % bnx;
      if (threadIdx.x == 0) {
        float sc = 1.f;
        if (fz.ssq) {
          const float* sp = fz.ssq + (size_t)nrow * fz.ssq_stride;
          float ss = 0.f;
          for (int pp = 0; pp < fz.ssq_parts; ++pp) ss += __ldcg(sp + pp);
          sc = 1.0f / sqrtf(ss * fz.inv_d + fz.eps);
        }
        s_rsc = sc;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
      const float sc = s_rsc;
      const int ne = (g + (kvu ? 2 : 0)) * HD;
      for (int e = threadIdx.x; e < ne; e += CW * 32) {
        const int which = e / HD, d = e % HD;
        const int mrow = which < g ? (kvh * g + which) * HD + d
                                   : (which == g ? (m.H + kvh) * HD + d : (m.H + m.KV + kvh) * HD + d);
        const float* pp = fz.part + ((size_t)((chunk * fz.m_tiles + (mrow >> 7)) * fz.splits) * 256 + col) * 128 +
                          (mrow & 127);
        float v = 0.f;
        for (int sp = 0; sp < fz.splits; ++sp) v += __ldcg(pp + (size_t)sp * 256 * 128);
        xs[e] = v * sc + fz.bias[mrow];
      }
      asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
      const int half = HD / 2;
      const float2* csp = fz.cs + (size_t)I.pos0 * half;
      for (int e = threadIdx.x; e < (g + (kvu ? 1 : 0)) * HD; e += CW * 32) {
        const int base = e - e % HD, d = e % HD;
        const float2 cs = csp[d % half];
        xr[e] = d < half ? xs[e] * cs.x - xs[base + d + half] * cs.y : xs[e] * cs.x + xs[base + d - half] * cs.y;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
      if (kvu) {
        // append k (rotated) and v to the current token's page slot; the
        // producer loads that page only after this (kvready)
        const int page = page_table[(size_t)I.pt_row * maxp + I.pos0 / kPage];
        act_t* kd = (act_t*)fz.kv_pool + kv_block_elems(layer, page, kvh, 0, m.n_pages, m.KV, HD) +
                    (size_t)(I.pos0 % kPage) * HD;
        act_t* vd = (act_t*)fz.kv_pool + kv_block_elems(layer, page, kvh, 1, m.n_pages, m.KV, HD) +
                    (size_t)(I.pos0 % kPage) * HD;
        for (int d = threadIdx.x; d < HD; d += CW * 32) {
          kd[d] = to_act(xr[g * HD + d]);
          vd[d] = to_act(xs[(g + 1) * HD + d]);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence_block();
        asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
        if (threadIdx.x == 0) bar_arrive(kvready);
      }
      const float* qr = tq < nrows ? xr + (size_t)tq * HD : nullptr;   // decode: row tq = head tq of this KV head
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        float2 a0 = qr ? make_float2(qr[kk * 16 + 2 * tr], qr[kk * 16 + 2 * tr + 1]) : make_float2(0.f, 0.f);
        float2 a1 = qr ? make_float2(qr[kk * 16 + 8 + 2 * tr], qr[kk * 16 + 9 + 2 * tr]) : make_float2(0.f, 0.f);
        const act2_t h0 = to_act2(a0.x, a0.y), h1 = to_act2(a1.x, a1.y);
        qb[0][kk][0] = *(const uint32_t*)&h0;
        qb[0][kk][1] = *(const uint32_t*)&h1;
        const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
        const act2_t l0 = to_act2(a0.x - f0.x, a0.y - f0.y), l1 = to_act2(a1.x - f1.x, a1.y - f1.y);
        ql[0][kk][0] = q_lo ? *(const uint32_t*)&l0 : 0u;
        ql[0][kk][1] = q_lo ? *(const uint32_t*)&l1 : 0u;
      }
    } else {
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq) {
        const int r = nq * 8 + tq;
        const size_t qo = ((size_t)(I.q_row0 + r / g) * m.H + kvh * g + r % g) * HD;
        const act_t* qr = r < nrows ? q + qo : nullptr;
        const act_t* qlr = r < nrows && q_lo ? q_lo + qo : nullptr;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          qb[nq][kk][0] = qr ? *(const uint32_t*)(qr + kk * 16 + 2 * tr) : 0u;
          qb[nq][kk][1] = qr ? *(const uint32_t*)(qr + kk * 16 + 8 + 2 * tr) : 0u;
          ql[nq][kk][0] = qlr ? *(const uint32_t*)(qlr + kk * 16 + 2 * tr) : 0u;
          ql[nq][kk][1] = qlr ? *(const uint32_t*)(qlr + kk * 16 + 8 + 2 * tr) : 0u;
        }
      }
    }
    // this thread's two query columns per n-tile: rows nq*8 + 2tr + e
    int lim[NQT][2];
#pragma unroll
    for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = nq * 8 + 2 * tr + e;
        lim[nq][e] = r < nrows ? I.pos0 + r / g + 1 : 0;   // keys j < lim visible
      }
    const int kv_hi = I.kv_hi;
    float o[HD / 16][NQT][4];                    // O^T: rows = head dim, cols = query rows
#pragma unroll
    for (int i = 0; i < HD / 16; ++i)
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq) o[i][nq][0] = o[i][nq][1] = o[i][nq][2] = o[i][nq][3] = 0.f;
    float mrun[NQT][2], lrun[NQT][2];
#pragma unroll
    for (int nq = 0; nq < NQT; ++nq) { mrun[nq][0] = mrun[nq][1] = -INFINITY; lrun[nq][0] = lrun[nq][1] = 0.f; }

    for (int j = (int)((warp - gpage % CW + CW) % CW); j < npg; j += CW) {
      const long long gp = gpage + j;   // gp % CW == warp
      const int st = (int)(gp % AT_STAGES);
      mbar_wait_wd(full0 + 8 * st, (uint32_t)((gp / AT_STAGES) & 1), 200 + st, gp, (long long)it * 1000 + npg);
      if (threadIdx.x == 0 && j == 0 && u == (int)blockIdx.x) ATL(2);
      if (skip_mma) {
        __syncwarp();
        if (lane == 0) bar_arrive(empty0 + 8 * st);
        continue;
      }
      const uint32_t kt = sbase + st * C::STAGE_BYTES, vt = kt + C::TILE_BYTES;
      const int tok0 = (p_lo + j) * kPage;
      // ---- S^T = K Q^T (64 tokens x query rows): 4 token tiles of 16
      float s[4][NQT][4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq) s[mt][nq][0] = s[mt][nq][1] = s[mt][nq][2] = s[mt][nq][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int row = mt * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int ch = 2 * kk + (lane >> 4);
          uint32_t a[4];
          ldsm_x4(kt + swz(row, ch), a[0], a[1], a[2], a[3]);
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) {
            mma16816(s[mt][nq], a, qb[nq][kk][0], qb[nq][kk][1]);
            if (q_lo) mma16816(s[mt][nq], a, ql[nq][kk][0], ql[nq][kk][1]);
          }
        }
      }
      // ---- mask + online softmax per query column (log2 domain)
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq) {
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jtok = tok0 + mt * 16 + tq + 8 * h;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool v = jtok < kv_hi && jtok < lim[nq][e];
              float& x = s[mt][nq][2 * h + e];
              x = v ? x * scale : -INFINITY;
              mx[e] = fmaxf(mx[e], x);
            }
          }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 4));
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 8));
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 16));
          const float mn = fmaxf(mrun[nq][e], mx[e]);
          const float base = mn == -INFINITY ? 0.f : mn;
          const float al = exp2f(mrun[nq][e] - base);
          mrun[nq][e] = mn;
          float ps = 0.f;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float& x = s[mt][nq][2 * h + e];
              x = exp2f(x - base);
              ps += x;
            }
          lrun[nq][e] = lrun[nq][e] * al + ps;
#pragma unroll
          for (int i = 0; i < HD / 16; ++i) { o[i][nq][e] *= al; o[i][nq][2 + e] *= al; }
        }
      }
      // ---- O^T += V^T P^T: 4 k-steps of 16 tokens
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t pb[NQT][2];
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq) {
          pb[nq][0] = movtrans(pack_act(s[ks][nq][0], s[ks][nq][1]));   // tokens 0-7 of the k-step
          pb[nq][1] = movtrans(pack_act(s[ks][nq][2], s[ks][nq][3]));   // tokens 8-15
        }
        const int row = ks * 16 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
        for (int mh = 0; mh < HD / 16; ++mh) {
          uint32_t a[4];
          ldsm_x4_t(vt + swz(row, 2 * mh + ((lane >> 3) & 1)), a[0], a[1], a[2], a[3]);
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) mma16816(o[mh][nq], a, pb[nq][0], pb[nq][1]);
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(empty0 + 8 * st);   // stage free for the producer
    }
    gpage += npg;
    if (threadIdx.x == 0 && u == (int)blockIdx.x) ATL(3);
    // ---- merge the consumer warps' (m, l, O) in shared memory: [MR] m, [MR] l, [MR][HD] O
#pragma unroll
    for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        lrun[nq][e] += __shfl_xor_sync(0xffffffffu, lrun[nq][e], 4);
        lrun[nq][e] += __shfl_xor_sync(0xffffffffu, lrun[nq][e], 8);
        lrun[nq][e] += __shfl_xor_sync(0xffffffffu, lrun[nq][e], 16);
      }
    float* wm = mrg + warp * MR * (HD + 2);
    if (tq == 0) {
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          wm[nq * 8 + 2 * tr + e] = mrun[nq][e];
          wm[MR + nq * 8 + 2 * tr + e] = lrun[nq][e];
        }
    }
#pragma unroll
    for (int mh = 0; mh < HD / 16; ++mh)
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = nq * 8 + 2 * tr + e;
          wm[2 * MR + r * HD + mh * 16 + tq] = o[mh][nq][e];
          wm[2 * MR + r * HD + mh * 16 + tq + 8] = o[mh][nq][2 + e];
        }
    asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
    for (int e = threadIdx.x; e < nrows * HD; e += CW * 32) {
      const int r = e / HD, c = e % HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < CW; ++w) M = fmaxf(M, mrg[w * MR * (HD + 2) + r]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < CW; ++w) {
        const float* ww = mrg + w * MR * (HD + 2);
        const float f = exp2f(ww[r] - Mb);
        L += ww[MR + r] * f;
        O += ww[2 * MR + r * HD + c] * f;
      }
      const int tok = I.q_row0 + r / g, head = kvh * g + r % g;
      if (I.nsplit == 1) {
        const float v = L > 0.f ? O / L : 0.f;
        const act_t hv = to_act(v);
        out[((size_t)tok * m.H + head) * HD + c] = hv;
        if (out_lo) out_lo[((size_t)tok * m.H + head) * HD + c] = to_act(v - __half2float(hv));
      } else {
        float* pp = partial + ((size_t)it * m.KV + kvh) * (16 * (HD + 2));
        pp[32 + r * HD + c] = O;
        if (c == 0) { pp[r] = M; pp[16 + r] = L; }
      }
    }
    if (threadIdx.x == 0 && u == (int)blockIdx.x) ATL(4);
    if (I.nsplit > 1) {
      // the last split of this query block to finish merges all splits, in
      // split order (deterministic); the ticket resets itself
      __shared__ int s_last;
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
      if (threadIdx.x == 0) {
        int* tk = tickets + (size_t)I.item0 * m.KV + kvh;
        const int old = atomicAdd(tk, 1);
        s_last = old == I.nsplit - 1;
        if (s_last) *tk = 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
      if (s_last) {
        __threadfence();
        const float* __restrict__ p0 = partial + ((size_t)I.item0 * m.KV + kvh) * (16 * (HD + 2));
        const size_t sstride = (size_t)m.KV * 16 * (HD + 2);
        float* wsm = mrg;                                  // [16][nsplit] split weights
        const int ns = I.nsplit;
        if (threadIdx.x < nrows) {
          const int r = threadIdx.x;
          float M = -INFINITY;
          for (int sp = 0; sp < ns; ++sp) M = fmaxf(M, __ldcg(p0 + sp * sstride + r));
          const float Mb = M == -INFINITY ? 0.f : M;
          float L = 0.f;
          for (int sp = 0; sp < ns; ++sp) {
            const float f = exp2f(__ldcg(p0 + sp * sstride + r) - Mb);
            wsm[r * ns + sp] = f;
            L += __ldcg(p0 + sp * sstride + 16 + r) * f;
          }
          const float inv = L > 0.f ? 1.f / L : 0.f;
          for (int sp = 0; sp < ns; ++sp) wsm[r * ns + sp] *= inv;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
        for (int e = threadIdx.x; e < nrows * (HD / 4); e += CW * 32) {
          const int r = e / (HD / 4), c4 = (e % (HD / 4)) * 4;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int s0 = 0; s0 < ns; s0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u8 = 0; u8 < 8; ++u8)
              v[u8] = s0 + u8 < ns ? __ldcg((const float4*)(p0 + (s0 + u8) * sstride + 32 + r * HD + c4))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u8 = 0; u8 < 8; ++u8) {
              if (s0 + u8 >= ns) break;
              const float w = wsm[r * ns + s0 + u8];
              acc.x += w * v[u8].x; acc.y += w * v[u8].y; acc.z += w * v[u8].z; acc.w += w * v[u8].w;
            }
          }
          const int tok = I.q_row0 + r / g, head = kvh * g + r % g;
          const size_t oo = ((size_t)tok * m.H + head) * HD + c4;
          store_act4(out + oo, out_lo ? out_lo + oo : nullptr, acc);
        }
      }
    }
    if (threadIdx.x == 0 && u == (int)blockIdx.x) ATL(5);
    asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
  }
  if (threadIdx.x == 0) ATL(6);
}

// decode: <= 8 query rows per unit (1 token x g heads): 6 consumer warps;
// prefill: <= 16 rows (floor(16/g) tokens x g heads): 3 consumer warps (the
// 16-row merge buffer leaves room for fewer).
using AttnDec128 = AttnCfg<128, 6, 1>;
using AttnPre128 = AttnCfg<128, 3, 2>;
using AttnDec64 = AttnCfg<64, 6, 1>;
using AttnPre64 = AttnCfg<64, 3, 2>;

void attn_set_timeline(long long* p) { cudaMemcpyToSymbol(g_attn_tl, &p, sizeof p); }

int attn_smem_bytes(int hd) { return hd == 128 ? AttnDec128::SMEM : AttnDec64::SMEM; }

int attn_init_attrs() {
  cudaError_t e[4] = {
      cudaFuncSetAttribute(attn_kernel<128, 6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnDec128::SMEM),
      cudaFuncSetAttribute(attn_kernel<128, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnPre128::SMEM),
      cudaFuncSetAttribute(attn_kernel<64, 6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnDec64::SMEM),
      cudaFuncSetAttribute(attn_kernel<64, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnPre64::SMEM)};
  for (auto x : e)
    if (x != cudaSuccess) return -1;
  return 0;
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The pool as [n_pages * L * KV * 2 * 64 rows, hd] fp16 with 64 x 64 boxes.
int make_kv_map(CUtensorMap* map, const void* pool, size_t n_pages, const ModelDims& m) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return -1;
  PFN_encodeTiled_t enc = (PFN_encodeTiled_t)p;
  const unsigned long long rows = (unsigned long long)n_pages * m.L * m.KV * 2 * kPage;
  if (rows >= (1ull << 31)) return -3;
  cuuint64_t dims[2] = {(cuuint64_t)m.hd, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)m.hd * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kPage};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(pool), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

void launch_attention(const CUtensorMap& kv_map, const void* q, const int* page_table, int maxp,
                      const AttnItem* items, const int* n_items_dev, int n_items_host, void* out, float* partial,
                      int* tickets, const ModelDims& m, int layer, bool decode, cudaStream_t st, const void* q_lo,
                      void* out_lo, const QkvFuse* fuse) {
  const dim3 grid(148);   // one wave, persistent over the flat (item, KV head) units
  QkvFuse fz{};
  if (fuse && decode) fz = *fuse;
  if (fuse) fz.dbg = fuse->dbg;
  const auto* qq = (const act_t*)q;
  const auto* ql = (const act_t*)q_lo;
  auto* oo = (act_t*)out;
  auto* ol = (act_t*)out_lo;
  if (m.hd == 128) {
    if (decode)
      launch_pdl(attn_kernel<128, 6, 1>, grid, dim3(AttnDec128::THREADS), AttnDec128::SMEM, st, kv_map, qq, ql,
                 page_table, maxp, items, n_items_dev, n_items_host, oo, ol, partial, tickets, m, layer, fz);
    else
      launch_pdl(attn_kernel<128, 3, 2>, grid, dim3(AttnPre128::THREADS), AttnPre128::SMEM, st, kv_map, qq, ql,
                 page_table, maxp, items, n_items_dev, n_items_host, oo, ol, partial, tickets, m, layer, fz);
  } else {
    if (decode)
      launch_pdl(attn_kernel<64, 6, 1>, grid, dim3(AttnDec64::THREADS), AttnDec64::SMEM, st, kv_map, qq, ql,
                 page_table, maxp, items, n_items_dev, n_items_host, oo, ol, partial, tickets, m, layer, fz);
    else
      launch_pdl(attn_kernel<64, 3, 2>, grid, dim3(AttnPre64::THREADS), AttnPre64::SMEM, st, kv_map, qq, ql,
                 page_table, maxp, items, n_items_dev, n_items_host, oo, ol, partial, tickets, m, layer, fz);
  }
}

}  // namespace rp
