// Decode attention over sibling groups (K4'): the G responses
// of a prompt share its full prompt pages (reading Z17), so one
// work unit = (group of <= 8 live siblings, KV head, page split) reads every
// shared page ONCE from L2/HBM into shared memory and every member's query
// columns consume it there; the members' private pages (the forked partial
// prompt page and the response tokens) follow, one fill per member.  The
// per-row kernel (k_attn.cu) re-streamed the shared pages once per sibling
// (8x the L2->SM bytes at G = 8): without any MMA it already takes 80 us per
// layer at 256 rows x 1 K context (this kernel: 36 us), profiles/r02_attn_group_ab.txt.
//
// CTA = 1 producer warp + 8 consumer warps.  Consumer warp w holds the g <= 8
// query heads of one member as the n8 columns of m16n8k16 MMAs; small groups
// replicate a member over rep = 8 / n_mem (rounded down to a power of two)
// warps that split its pages, merged in shared memory.  Every consumer warp
// waits for and releases EVERY stage use in order (the empty barrier counts
// 8 arrivals) and computes only the uses it owns: each warp's mbarrier phase
// stays in step with the ring whatever the mix of shared and private pages.
// Split units write (m, l, O) partials per member; when every unit of the
// launch is resident at once (units <= grid, and not in a single-GPU local
// group whose other members' kernels may hold SMs) the splits of a group
// merge cooperatively -- each waits for all and merges its 1/nsplit share of
// the member rows -- else the last split to finish (ticket) merges them all;
// both in split order.
#include <cuda.h>
#include "common.cuh"
#include "kernels.h"
#include "attn_mma.cuh"

namespace rp {

constexpr int AG_STAGES = 6;   // 64-token pages (K + V) in flight per SM
constexpr int AG_CW = 8;       // consumer warps

template <int HD>
struct AgCfg {
  static constexpr int HALVES = HD / 64;
  static constexpr int TILE_BYTES = kPage * HD * 2;
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int OST = HD + 4;                       // O row stride in the warp state (bank spread)
  static constexpr int WST = 16 + 8 * OST;                 // per warp: [8] m, [8] l, [8][OST] O
  static constexpr int MB = 16 + 8 * HD;                   // partial floats per member: [8] m, [8] l, [8][HD] O
  static constexpr int SMEM = AG_STAGES * STAGE_BYTES + AG_CW * WST * 4 + 1024 + 128;
  static constexpr int THREADS = (AG_CW + 1) * 32;
};
static_assert(AgCfg<128>::SMEM + 64 <= 232448, "group attention smem");
static_assert(AG_CW * AgCfg<64>::WST >= 2 * 64 * 32, "split-merge weights fit the warp states");

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// S^T = K Q^T and O^T += V^T P^T for one member's n-tile on one staged page
// (the fragment layouts of attn_kernel: key tokens on the MMA rows).
template <int HD>
__device__ __forceinline__ void ag_page(uint32_t kt, uint32_t vt, int tok0, bool has_lo, int lane,
                                        const uint32_t (&qb)[HD / 16][2], const uint32_t (&ql)[HD / 16][2],
                                        const int (&lim)[2], float scale, float (&o)[HD / 16][4], float (&mrun)[2],
                                        float (&lrun)[2]) {
  const int tq = lane >> 2;
  float s[4][4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) s[mt][0] = s[mt][1] = s[mt][2] = s[mt][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int row = mt * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
      uint32_t a[4];
      ldsm_x4(kt + swz(row, 2 * kk + (lane >> 4)), a[0], a[1], a[2], a[3]);
      mma16816(s[mt], a, qb[kk][0], qb[kk][1]);
      if (has_lo) mma16816(s[mt], a, ql[kk][0], ql[kk][1]);
    }
  }
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jtok = tok0 + mt * 16 + tq + 8 * h;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float& x = s[mt][2 * h + e];
        x = jtok < lim[e] ? x * scale : -INFINITY;
        mx[e] = fmaxf(mx[e], x);
      }
    }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 4));
    mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 8));
    mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 16));
    const float mn = fmaxf(mrun[e], mx[e]);
    const float base = mn == -INFINITY ? 0.f : mn;
    const float al = exp2f(mrun[e] - base);
    mrun[e] = mn;
    float ps = 0.f;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float& x = s[mt][2 * h + e];
        x = exp2f(x - base);
        ps += x;
      }
    lrun[e] = lrun[e] * al + ps;
#pragma unroll
    for (int i = 0; i < HD / 16; ++i) { o[i][e] *= al; o[i][2 + e] *= al; }
  }
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const uint32_t pb0 = movtrans(pack_act(s[ks][0], s[ks][1]));
    const uint32_t pb1 = movtrans(pack_act(s[ks][2], s[ks][3]));
    const int row = ks * 16 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
    for (int mh = 0; mh < HD / 16; ++mh) {
      uint32_t a[4];
      ldsm_x4_t(vt + swz(row, 2 * mh + ((lane >> 3) & 1)), a[0], a[1], a[2], a[3]);
      mma16816(o[mh], a, pb0, pb1);
    }
  }
}

// Split merge of member rows [r0, r1) (row = x * g + r) of one (group,
// KV head): out = sum_s w_s O_s with w_s = 2^(m_s - M) / L, in split order.
// m and l of every (row, split) are loaded at once (independent loads).
template <int HD>
__device__ __forceinline__ void ag_merge_rows(const float* __restrict__ p0, size_t sstride, int ns, int r0, int r1,
                                              int g, const AttnGroupItem* I, int kvh, const ModelDims& m,
                                              act_t* __restrict__ out, act_t* __restrict__ out_lo, float* smem) {
  using C = AgCfg<HD>;
  const int nr = r1 - r0;
  float* wsm = smem;                 // [64][ns]
  float* lsm = smem + 64 * 32;       // [64][ns]
  for (int e = threadIdx.x; e < nr * ns; e += AG_CW * 32) {
    const int xr = r0 + e / ns, sp = e % ns;
    const float* px = p0 + (size_t)(xr / g) * C::MB + sp * sstride;
    wsm[e] = __ldcg(px + xr % g);
    lsm[e] = __ldcg(px + 8 + xr % g);
  }
  asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
  for (int j = threadIdx.x; j < nr; j += AG_CW * 32) {
    float M = -INFINITY;
    for (int sp = 0; sp < ns; ++sp) M = fmaxf(M, wsm[j * ns + sp]);
    const float Mb = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    for (int sp = 0; sp < ns; ++sp) {
      const float f = exp2f(wsm[j * ns + sp] - Mb);
      wsm[j * ns + sp] = f;
      L += lsm[j * ns + sp] * f;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    for (int sp = 0; sp < ns; ++sp) wsm[j * ns + sp] *= inv;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
  for (int e = threadIdx.x; e < nr * (HD / 4); e += AG_CW * 32) {
    const int j = e / (HD / 4), d4 = (e % (HD / 4)) * 4, xr = r0 + j, x = xr / g, r = xr % g;
    const float* px = p0 + (size_t)x * C::MB + 16 + r * HD + d4;
    const float* wr = wsm + j * ns;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < ns; s0 += 8) {
      float4 vv[8];
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8)
        vv[u8] = s0 + u8 < ns ? __ldcg((const float4*)(px + (s0 + u8) * sstride)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8) {
        if (s0 + u8 >= ns) break;
        const float w = wr[s0 + u8];
        acc.x += w * vv[u8].x; acc.y += w * vv[u8].y; acc.z += w * vv[u8].z; acc.w += w * vv[u8].w;
      }
    }
    const size_t oo = ((size_t)I->q_row[x] * m.H + kvh * g + r) * HD + d4;
    store_act4(out + oo, out_lo ? out_lo + oo : nullptr, acc);
  }
}

template <int HD>
__global__ void __launch_bounds__((AG_CW + 1) * 32, 1)
attn_group_kernel(const __grid_constant__ CUtensorMap kv_map, const act_t* __restrict__ q,
                  const act_t* __restrict__ q_lo, const int* __restrict__ page_table, int maxp,
                  const AttnGroupItem* __restrict__ items, const int* __restrict__ n_items_dev,
                  act_t* __restrict__ out, act_t* __restrict__ out_lo, float* __restrict__ partial,
                  int* __restrict__ tickets, ModelDims m, int layer, int dbg, int may_spin,
                  float* __restrict__ rowpart, int* __restrict__ rtickets) {
  using C = AgCfg<HD>;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  float* wst = (float*)(sm + AG_STAGES * C::STAGE_BYTES);     // [AG_CW][WST]
  uint64_t* bars = (uint64_t*)(wst + AG_CW * C::WST);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(bars);
  const uint32_t empty0 = full0 + 8 * AG_STAGES;

  // The work list, the page tables and every page but the one holding a
  // member's current position were written before this step's QKV GEMM
  // started: the producer streams them before the dependency wait (as in
  // attn_kernel); consumers wait before reading Q.
  pdl_launch_dependents();
  const int n_units = *n_items_dev * m.KV;
  const bool coop = may_spin && n_units <= (int)gridDim.x;
  const int g = m.H / m.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < AG_STAGES; ++i) { bar_init(full0 + 8 * i, 1); bar_init(empty0 + 8 * i, AG_CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == AG_CW) {
    // ===================== producer warp =====================
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&kv_map) : "memory");
    bool waited = false;
    long long gp = 0;
    auto fill = [&](int page, int kvh) {   // lane 0
      const int st = (int)(gp % AG_STAGES);
      mbar_wait_wd(empty0 + 8 * st, (uint32_t)(((gp / AG_STAGES) & 1) ^ 1), 400 + st, gp, page);
      const uint32_t fb = full0 + 8 * st;
      bar_expect_tx(fb, C::STAGE_BYTES);
      const int row_k = (int)(kv_block_elems(layer, page, kvh, 0, m.n_pages, m.KV, HD) / HD);
      const uint32_t dst = sbase + st * C::STAGE_BYTES;
#pragma unroll
      for (int h = 0; h < C::HALVES; ++h) {
        tma2d(dst + h * 8192, &kv_map, fb, h * 64, row_k);
        tma2d(dst + C::TILE_BYTES + h * 8192, &kv_map, fb, h * 64, row_k + kPage);
      }
    };
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int it = u / m.KV, kvh = u % m.KV;
      const int v = ((const int*)(items + it))[lane];
      const int n_mem = __shfl_sync(0xffffffffu, v, 0), snp = __shfl_sync(0xffffffffu, v, 1);
      const int pg_lo = __shfl_sync(0xffffffffu, v, 2), pg_hi = __shfl_sync(0xffffffffu, v, 3);
      const int my_pt = __shfl_sync(0xffffffffu, v, 16 + (lane & 7));
      const int my_pos = __shfl_sync(0xffffffffu, v, 24 + (lane & 7));
      const int pt0 = __shfl_sync(0xffffffffu, v, 16);
      const int s_hi = min(pg_hi, snp);
      // shared prompt pages: complete before the round's first decode step
      for (int j0 = pg_lo; j0 < s_hi; j0 += 32) {
        const int mine = j0 + lane < s_hi ? page_table[(size_t)pt0 * maxp + j0 + lane] : 0;
        const int cnt = min(32, s_hi - j0);
        for (int jj = 0; jj < cnt; ++jj) {
          const int page = __shfl_sync(0xffffffffu, mine, jj);
          if (lane == 0) fill(page, kvh);
          ++gp;
        }
      }
      // private pages, member by member at each page index
      for (int p = max(pg_lo, snp); p < pg_hi; ++p) {
        const bool has = lane < n_mem && p * kPage <= my_pos;
        const int mine = has ? page_table[(size_t)my_pt * maxp + p] : -1;
        for (int x = 0; x < n_mem; ++x) {
          const int page = __shfl_sync(0xffffffffu, mine, x);
          const int px = __shfl_sync(0xffffffffu, v, 24 + x);
          if (page < 0) continue;
          if (lane == 0) {
            if (!waited && (p + 1) * kPage > px) {   // the page the QKV GEMM appends to this step
              pdl_wait();
              waited = true;
            }
            fill(page, kvh);
          }
          ++gp;
        }
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  pdl_wait();
  const float scale = 1.4426950408889634f * rsqrtf((float)HD);
  const int tq = lane >> 2, tr = lane & 3;
  const bool has_lo = q_lo != nullptr && !(dbg & 2);   // dbg (RP_AG_DBG, measurement only): 1 no MMAs, 2 no q_lo MMAs
  float* ws = wst + warp * C::WST;
  long long gp = 0;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int it = u / m.KV, kvh = u % m.KV;
    const int v = ((const int*)(items + it))[lane];
    const int n_mem = __shfl_sync(0xffffffffu, v, 0), snp = __shfl_sync(0xffffffffu, v, 1);
    const int pg_lo = __shfl_sync(0xffffffffu, v, 2), pg_hi = __shfl_sync(0xffffffffu, v, 3);
    const int nsplit = __shfl_sync(0xffffffffu, v, 4), item0 = __shfl_sync(0xffffffffu, v, 5);
    const int rep = __shfl_sync(0xffffffffu, v, 6);
    const int x = warp / rep, sub = warp % rep;        // this warp's member and replica
    const bool valid = x < n_mem;
    uint32_t qb[HD / 16][2], ql[HD / 16][2];
    int lim[2];
    {
      const int row = __shfl_sync(0xffffffffu, v, 8 + (x & 7));
      const int pos = __shfl_sync(0xffffffffu, v, 24 + (x & 7));
      const size_t qo = ((size_t)row * m.H + kvh * g + tq) * HD;
      const act_t* qr = valid && tq < g ? q + qo : nullptr;
      const act_t* qlr = valid && tq < g && has_lo ? q_lo + qo : nullptr;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qb[kk][0] = qr ? *(const uint32_t*)(qr + kk * 16 + 2 * tr) : 0u;
        qb[kk][1] = qr ? *(const uint32_t*)(qr + kk * 16 + 8 + 2 * tr) : 0u;
        ql[kk][0] = qlr ? *(const uint32_t*)(qlr + kk * 16 + 2 * tr) : 0u;
        ql[kk][1] = qlr ? *(const uint32_t*)(qlr + kk * 16 + 8 + 2 * tr) : 0u;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) lim[e] = valid && 2 * tr + e < g ? pos + 1 : 0;
    }
    float o[HD / 16][4];
#pragma unroll
    for (int i = 0; i < HD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrun[2] = {-INFINITY, -INFINITY}, lrun[2] = {0.f, 0.f};

    int i = 0;   // stage uses of this unit so far
    auto use = [&](int tok0, bool own) {
      const int st = (int)(gp % AG_STAGES);
      mbar_wait_wd(full0 + 8 * st, (uint32_t)((gp / AG_STAGES) & 1), 500 + st, gp, (long long)it * 1000 + i);
      if (own && !(dbg & 1)) {
        const uint32_t kt = sbase + st * C::STAGE_BYTES;
        ag_page<HD>(kt, kt + C::TILE_BYTES, tok0, has_lo, lane, qb, ql, lim, scale, o, mrun, lrun);
      }
      __syncwarp();
      if (lane == 0) bar_arrive(empty0 + 8 * st);
      ++gp;
      ++i;
    };
    const int s_hi = min(pg_hi, snp);
    for (int p = pg_lo; p < s_hi; ++p) use(p * kPage, valid && i % rep == sub);
    for (int p = max(pg_lo, snp); p < pg_hi; ++p)
      for (int y = 0; y < n_mem; ++y) {
        const int py = __shfl_sync(0xffffffffu, v, 24 + y);
        if (p * kPage > py) continue;
        use(p * kPage, y == x && i % rep == sub);
      }

    // ---- this warp's (m, l, O) per head column into shared memory
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      lrun[e] += __shfl_xor_sync(0xffffffffu, lrun[e], 4);
      lrun[e] += __shfl_xor_sync(0xffffffffu, lrun[e], 8);
      lrun[e] += __shfl_xor_sync(0xffffffffu, lrun[e], 16);
    }
    if (tq == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e) { ws[2 * tr + e] = mrun[e]; ws[8 + 2 * tr + e] = lrun[e]; }
    }
#pragma unroll
    for (int mh = 0; mh < HD / 16; ++mh)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float* orow = ws + 16 + (2 * tr + e) * C::OST + mh * 16 + tq;
        orow[0] = o[mh][e];
        orow[8] = o[mh][2 + e];
      }
    asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");

    // ---- combine each member's rep warps; output or split partial
    const AttnGroupItem* I = items + it;
    const int nel = n_mem * g * (HD / 4);
    for (int e = threadIdx.x; e < nel; e += AG_CW * 32) {
      const int xe = e / (g * (HD / 4)), r = (e / (HD / 4)) % g, d4 = (e % (HD / 4)) * 4;
      const int w0 = xe * rep;
      float M = -INFINITY;
      for (int k = 0; k < rep; ++k) M = fmaxf(M, wst[(w0 + k) * C::WST + r]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k = 0; k < rep; ++k) {
        const float* wk = wst + (w0 + k) * C::WST;
        const float f = exp2f(wk[r] - Mb);
        L += wk[8 + r] * f;
        const float* orow = wk + 16 + r * C::OST + d4;
        acc.x += orow[0] * f; acc.y += orow[1] * f; acc.z += orow[2] * f; acc.w += orow[3] * f;
      }
      if (I->rowmerge) {
        if (I->nspl[xe] == 1) {
          const float inv = L > 0.f ? 1.f / L : 0.f;
          acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
          const size_t oo = ((size_t)I->q_row[xe] * m.H + kvh * g + r) * HD + d4;
          store_act4(out + oo, out_lo ? out_lo + oo : nullptr, acc);
        } else {
          float* pm = rowpart + (((size_t)I->q_row[xe] * m.KV + kvh) * kRowSplits + I->sidx[xe]) * C::MB;
          if (d4 == 0) { pm[r] = M; pm[8 + r] = L; }
          *(float4*)(pm + 16 + r * HD + d4) = acc;
        }
      } else if (nsplit == 1) {
        const float inv = L > 0.f ? 1.f / L : 0.f;
        acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
        const size_t oo = ((size_t)I->q_row[xe] * m.H + kvh * g + r) * HD + d4;
        store_act4(out + oo, out_lo ? out_lo + oo : nullptr, acc);
      } else {
        float* pm = partial + ((size_t)it * m.KV + kvh) * 8 * C::MB + (size_t)xe * C::MB;
        if (d4 == 0) { pm[r] = M; pm[8 + r] = L; }
        *(float4*)(pm + 16 + r * HD + d4) = acc;
      }
    }
    if (I->rowmerge) {
      // per member row: the last of its units to finish merges its partials
      // (split order; the row's ticket resets itself)
      __shared__ int s_lastr[8];
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
      if (threadIdx.x < n_mem) {
        const int x = threadIdx.x, ns = I->nspl[x];
        int last = 0;
        if (ns > 1) {
          int* tk = rtickets + (size_t)I->q_row[x] * m.KV + kvh;
          last = atomicAdd(tk, 1) == ns - 1;
          if (last) *tk = 0;
        }
        s_lastr[x] = last;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
      for (int x = 0; x < n_mem; ++x) {
        if (!s_lastr[x]) continue;
        __threadfence();
        const float* rb = rowpart + ((size_t)I->q_row[x] * m.KV + kvh) * kRowSplits * C::MB;
        ag_merge_rows<HD>(rb - (size_t)x * C::MB, C::MB, I->nspl[x], x * g, (x + 1) * g, g, I, kvh, m, out, out_lo,
                          wst);
        asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
      }
    } else if (nsplit > 1) {
      __shared__ int s_last;
      const float* __restrict__ p0 = partial + (size_t)item0 * m.KV * 8 * C::MB + (size_t)kvh * 8 * C::MB;
      const size_t sstride = (size_t)m.KV * 8 * C::MB;
      int* arrive = tickets + (size_t)item0 * m.KV + kvh;
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
      if (coop) {
        // every split of the group is resident: wait for all partials, then
        // merge this split's share of the member rows
        int* depart = tickets + (size_t)(item0 + 1) * m.KV + kvh;   // item0 + 1 is this group's (nsplit > 1)
        if (threadIdx.x == 0) {
          atomicAdd(arrive, 1);
          uint32_t spins = 0;
          while (ld_acquire_i32(arrive) < nsplit) {
            __nanosleep(64);
            if (++spins == (1u << 26)) {
              printf("rollpacker watchdog: group attention merge stuck (item %d, kvh %d)\n", item0, kvh);
              __trap();
            }
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
        const int sp = it - item0, R = n_mem * g;
        ag_merge_rows<HD>(p0, sstride, nsplit, sp * R / nsplit, (sp + 1) * R / nsplit, g, I, kvh, m, out, out_lo, wst);
        asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
        if (threadIdx.x == 0 && atomicAdd(depart, 1) == nsplit - 1) {   // the last to leave resets both
          *arrive = 0;
          *depart = 0;
        }
      } else {
        // the last split to finish merges all splits (the ticket resets itself)
        if (threadIdx.x == 0) {
          const int old = atomicAdd(arrive, 1);
          s_last = old == nsplit - 1;
          if (s_last) *arrive = 0;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");
        if (s_last) {
          __threadfence();
          ag_merge_rows<HD>(p0, sstride, nsplit, 0, n_mem * g, g, I, kvh, m, out, out_lo, wst);
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(AG_CW * 32) : "memory");   // warp states reused by the next unit
  }
}

int attn_group_init_attrs() {
  cudaError_t e[2] = {
      cudaFuncSetAttribute(attn_group_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, AgCfg<128>::SMEM),
      cudaFuncSetAttribute(attn_group_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, AgCfg<64>::SMEM)};
  for (auto x : e)
    if (x != cudaSuccess) return -1;
  return 0;
}

size_t attn_group_partial_floats(int hd) { return (size_t)8 * (16 + 8 * hd); }

void launch_attention_group(const CUtensorMap& kv_map, const void* q, const void* q_lo, const int* page_table,
                            int maxp, const AttnGroupItem* items, const int* n_items_dev, void* out, void* out_lo,
                            float* partial, int* tickets, const ModelDims& m, int layer, cudaStream_t st,
                            int dbg, int may_spin, float* rowpart, int* rtickets) {
  const dim3 grid(148);   // one wave, persistent over the flat (group item, KV head) units
  const auto* qq = (const act_t*)q;
  const auto* ql = (const act_t*)q_lo;
  auto* oo = (act_t*)out;
  auto* ol = (act_t*)out_lo;
  if (m.hd == 128)
    launch_pdl(attn_group_kernel<128>, grid, dim3(AgCfg<128>::THREADS), AgCfg<128>::SMEM, st, kv_map, qq, ql,
               page_table, maxp, items, n_items_dev, oo, ol, partial, tickets, m, layer, dbg, may_spin, rowpart, rtickets);
  else
    launch_pdl(attn_group_kernel<64>, grid, dim3(AgCfg<64>::THREADS), AgCfg<64>::SMEM, st, kv_map, qq, ql,
               page_table, maxp, items, n_items_dev, oo, ol, partial, tickets, m, layer, dbg, may_spin, rowpart, rtickets);
}

}  // namespace rp
