// Paged-KV GQA attention for decode and prefill (K4/K5).
//
// The KV pool is addressed by TMA as a 2-D tensor of token rows x head_dim
// (bf16): page p, layer l, KV head h, K|V is the 64-row block starting at row
// (((p*L + l)*KV + h)*2 + kv)*64.  One CTA = 1 producer warp + 3 consumer
// warps.  The producer streams whole pages (K and V, SWIZZLE_128B boxes of 64
// columns) into a 6-stage mbarrier ring; consumer warp w (of 3) owns the
// pages with global index = w mod 3 and therefore always the same 2 stages.  Work item = (query block, KV head, key
// split): the 16 MMA rows are the (query token, query head) pairs served by
// one KV head -- decode: 1 token x g heads (g = H/KV <= 8); prefill:
// floor(16/g) tokens x g heads with per-row causal limits.  S = Q K^T and
// O += P V run on mma.sync m16n8k16 (bf16, fp32 accumulate; a 16-row MMA is
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

namespace rp {

constexpr int AT_CWARPS = 3;                  // consumer warps
constexpr int AT_THREADS = (AT_CWARPS + 1) * 32;
constexpr int AT_STAGES = 6;                  // multiple of AT_CWARPS: stage s is always consumed by
                                              // warp s % AT_CWARPS, so every warp waits on each of its
                                              // stages' uses in order (mbarrier parity only tells
                                              // adjacent phases apart)
static_assert(AT_STAGES % AT_CWARPS == 0, "stage ownership");

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(uint32_t*)&v;
}
__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

template <int HD>
struct AttnCfg {
  static constexpr int HALVES = HD / 64;             // 128-byte column halves (TMA boxes) per row
  static constexpr int TILE_BYTES = kPage * HD * 2;  // K (or V) block of one page
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int MERGE_FLOATS = AT_CWARPS * 16 * (HD + 2);
  static constexpr int SMEM = AT_STAGES * STAGE_BYTES + MERGE_FLOATS * 4 + 1024 + 256;
};

// byte offset of (row, 16-byte chunk) in a [64][HD] tile stored as HD/64
// SWIZZLE_128B boxes of [64][64]
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)((chunk >> 3) * 8192 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(AT_THREADS, 1)
attn_kernel(const __grid_constant__ CUtensorMap kv_map, const __nv_bfloat16* __restrict__ q,
            const int* __restrict__ page_table, int maxp, const AttnItem* __restrict__ items, const int* n_items_dev,
            int n_items_host, __nv_bfloat16* __restrict__ out, float* __restrict__ partial, int* __restrict__ tickets,
            ModelDims m, int layer) {
  using C = AttnCfg<HD>;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  float* mrg = (float*)(sm + AT_STAGES * C::STAGE_BYTES);
  uint64_t* bars = (uint64_t*)(mrg + C::MERGE_FLOATS);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(bars);
  const uint32_t empty0 = full0 + 8 * AT_STAGES;

  pdl_wait();
  pdl_launch_dependents();
  const int n_items = n_items_dev ? *n_items_dev : n_items_host;
  const int n_units = n_items * m.KV;            // flat (item, KV head) work units
  const int g = m.H / m.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < AT_STAGES; ++i) { bar_init(full0 + 8 * i, 1); bar_init(empty0 + 8 * i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int row_stride_blk = kPage;   // rows per K|V block

  if (warp == AT_CWARPS) {
    // ===================== producer warp =====================
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&kv_map) : "memory");
    long long gpage = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int it = u / m.KV, kvh = u % m.KV;
      const AttnItem I = items[it];
      const int p_lo = I.kv_lo / kPage, npg = (I.kv_hi + kPage - 1) / kPage - p_lo;
      const int* ptab = page_table + (size_t)I.pt_row * maxp + p_lo;
      for (int j0 = 0; j0 < npg; j0 += 32) {
        const int mine = j0 + lane < npg ? ptab[j0 + lane] : 0;   // coalesced page-id batch
        const int cnt = min(32, npg - j0);
        for (int jj = 0; jj < cnt; ++jj) {
          const int page = __shfl_sync(0xffffffffu, mine, jj);
          if (lane == 0) {
            const long long gp = gpage + j0 + jj;
            const int st = (int)(gp % AT_STAGES);
            const uint32_t ph = (uint32_t)((gp / AT_STAGES) & 1);
            mbar_wait_wd(empty0 + 8 * st, ph ^ 1, 100 + st, gp, (long long)it * 1000 + npg);
            const uint32_t fb = full0 + 8 * st;
            bar_expect_tx(fb, C::STAGE_BYTES);
            const int row_k = (((page * m.L + layer) * m.KV + kvh) * 2 + 0) * row_stride_blk;
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
  const float scale = 1.4426950408889634f * rsqrtf((float)HD);
  const int ra = lane >> 2, rb = ra + 8;
  long long gpage = 0;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int it = u / m.KV, kvh = u % m.KV;
    const AttnItem I = items[it];
    const int nrows = I.n_qtok * g;
    const int p_lo = I.kv_lo / kPage, npg = (I.kv_hi + kPage - 1) / kPage - p_lo;
    // ---- Q fragments (A operand 16 x HD), rows r = tok*g + head
    uint32_t qa[HD / 16][4];
    {
      const int c = 2 * (lane & 3);
      const __nv_bfloat16* q0 = ra < nrows ? q + ((size_t)(I.q_row0 + ra / g) * m.H + kvh * g + ra % g) * HD : nullptr;
      const __nv_bfloat16* q1 = rb < nrows ? q + ((size_t)(I.q_row0 + rb / g) * m.H + kvh * g + rb % g) * HD : nullptr;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qa[kk][0] = q0 ? *(const uint32_t*)(q0 + kk * 16 + c) : 0u;
        qa[kk][1] = q1 ? *(const uint32_t*)(q1 + kk * 16 + c) : 0u;
        qa[kk][2] = q0 ? *(const uint32_t*)(q0 + kk * 16 + 8 + c) : 0u;
        qa[kk][3] = q1 ? *(const uint32_t*)(q1 + kk * 16 + 8 + c) : 0u;
      }
    }
    const int lim_a = ra < nrows ? I.pos0 + ra / g + 1 : 0;   // keys j < lim visible
    const int lim_b = rb < nrows ? I.pos0 + rb / g + 1 : 0;
    const int kv_hi = I.kv_hi;
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;

    for (int j = (int)((warp - gpage % AT_CWARPS + AT_CWARPS) % AT_CWARPS); j < npg; j += AT_CWARPS) {
      const long long gp = gpage + j;   // gp % AT_CWARPS == warp
      const int st = (int)(gp % AT_STAGES);
      mbar_wait_wd(full0 + 8 * st, (uint32_t)((gp / AT_STAGES) & 1), 200 + st, gp, (long long)it * 1000 + npg);
      const uint32_t kt = sbase + st * C::STAGE_BYTES, vt = kt + C::TILE_BYTES;
      const int tok0 = (p_lo + j) * kPage;
      // ---- S = Q K^T (16 x 64)
      float s[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
          const int row = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = 2 * kk + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kt + swz(row, ch), b0, b1, b2, b3);
          mma16816(s[2 * n2], qa[kk], b0, b1);
          mma16816(s[2 * n2 + 1], qa[kk], b2, b3);
        }
      }
      // ---- mask + online softmax (log2 domain)
      float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jj = tok0 + nt * 8 + 2 * (lane & 3) + e;
          const bool va = jj < kv_hi && jj < lim_a, vb = jj < kv_hi && jj < lim_b;
          s[nt][e] = va ? s[nt][e] * scale : -INFINITY;
          s[nt][2 + e] = vb ? s[nt][2 + e] * scale : -INFINITY;
          mx_a = fmaxf(mx_a, s[nt][e]);
          mx_b = fmaxf(mx_b, s[nt][2 + e]);
        }
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
      const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
      const float base_a = mn_a == -INFINITY ? 0.f : mn_a, base_b = mn_b == -INFINITY ? 0.f : mn_b;
      const float al_a = exp2f(m_a - base_a), al_b = exp2f(m_b - base_b);
      m_a = mn_a; m_b = mn_b;
      float ps_a = 0.f, ps_b = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        s[nt][0] = exp2f(s[nt][0] - base_a); s[nt][1] = exp2f(s[nt][1] - base_a);
        s[nt][2] = exp2f(s[nt][2] - base_b); s[nt][3] = exp2f(s[nt][3] - base_b);
        ps_a += s[nt][0] + s[nt][1];
        ps_b += s[nt][2] + s[nt][3];
      }
      l_a = l_a * al_a + ps_a;
      l_b = l_b * al_b + ps_b;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) { o[i][0] *= al_a; o[i][1] *= al_a; o[i][2] *= al_b; o[i][3] *= al_b; }
      // ---- O += P V: 4 k-steps of 16 tokens
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t pa[4];
        pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
        pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
        pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
        pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
        const int row = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
        for (int dt = 0; dt < HD / 8; dt += 2) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vt + swz(row, dt + (lane >> 4)), b0, b1, b2, b3);
          mma16816(o[dt], pa, b0, b1);
          mma16816(o[dt + 1], pa, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(empty0 + 8 * st);   // stage free for the producer
    }
    gpage += npg;
    // ---- merge the consumer warps' (m, l, O) in shared memory
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    float* wm = mrg + warp * 16 * (HD + 2);          // [16] m, [16] l, [16][HD] O
    if ((lane & 3) == 0) { wm[ra] = m_a; wm[16 + ra] = l_a; wm[rb] = m_b; wm[16 + rb] = l_b; }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int c = i * 8 + 2 * (lane & 3);
      *(float2*)(wm + 32 + ra * HD + c) = make_float2(o[i][0], o[i][1]);
      *(float2*)(wm + 32 + rb * HD + c) = make_float2(o[i][2], o[i][3]);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(AT_CWARPS * 32) : "memory");
    for (int e = threadIdx.x; e < nrows * HD; e += AT_CWARPS * 32) {
      const int r = e / HD, c = e % HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < AT_CWARPS; ++w) M = fmaxf(M, mrg[w * 16 * (HD + 2) + r]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < AT_CWARPS; ++w) {
        const float* ww = mrg + w * 16 * (HD + 2);
        const float f = exp2f(ww[r] - Mb);
        L += ww[16 + r] * f;
        O += ww[32 + r * HD + c] * f;
      }
      const int tok = I.q_row0 + r / g, head = kvh * g + r % g;
      if (I.nsplit == 1) {
        out[((size_t)tok * m.H + head) * HD + c] = __float2bfloat16(L > 0.f ? O / L : 0.f);
      } else {
        float* pp = partial + ((size_t)it * m.KV + kvh) * (16 * (HD + 2));
        pp[32 + r * HD + c] = O;
        if (c == 0) { pp[r] = M; pp[16 + r] = L; }
      }
    }
    if (I.nsplit > 1) {
      // the last split of this query block to finish merges all splits, in
      // split order (deterministic); the ticket resets itself
      __shared__ int s_last;
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(AT_CWARPS * 32) : "memory");
      if (threadIdx.x == 0) {
        int* tk = tickets + (size_t)I.item0 * m.KV + kvh;
        const int old = atomicAdd(tk, 1);
        s_last = old == I.nsplit - 1;
        if (s_last) *tk = 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(AT_CWARPS * 32) : "memory");
      if (s_last) {
        __threadfence();
        // per-row split weights w[r][s] = 2^(m_s - M) / L into smem (reuses the
        // merge buffer), then O = sum_s w[r][s] * O_s with float4 loads of all
        // splits in flight; fixed split order -> deterministic
        const float* __restrict__ p0 = partial + ((size_t)I.item0 * m.KV + kvh) * (16 * (HD + 2));
        const size_t sstride = (size_t)m.KV * 16 * (HD + 2);
        float* wsm = mrg;                                  // [16][nsplit]
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
        asm volatile("bar.sync 1, %0;" ::"r"(AT_CWARPS * 32) : "memory");
        for (int e = threadIdx.x; e < nrows * (HD / 4); e += AT_CWARPS * 32) {
          const int r = e / (HD / 4), c4 = (e % (HD / 4)) * 4;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int s0 = 0; s0 < ns; s0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              v[u] = s0 + u < ns ? __ldcg((const float4*)(p0 + (s0 + u) * sstride + 32 + r * HD + c4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (s0 + u >= ns) break;
              const float w = wsm[r * ns + s0 + u];
              acc.x += w * v[u].x; acc.y += w * v[u].y; acc.z += w * v[u].z; acc.w += w * v[u].w;
            }
          }
          const int tok = I.q_row0 + r / g, head = kvh * g + r % g;
          __nv_bfloat162* o2 = (__nv_bfloat162*)(out + ((size_t)tok * m.H + head) * HD + c4);
          o2[0] = __floats2bfloat162_rn(acc.x, acc.y);
          o2[1] = __floats2bfloat162_rn(acc.z, acc.w);
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(AT_CWARPS * 32) : "memory");
  }
}

int attn_smem_bytes(int hd) { return hd == 128 ? AttnCfg<128>::SMEM : AttnCfg<64>::SMEM; }

int attn_init_attrs() {
  cudaError_t e1 = cudaFuncSetAttribute(attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        AttnCfg<128>::SMEM);
  cudaError_t e2 = cudaFuncSetAttribute(attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        AttnCfg<64>::SMEM);
  return (e1 == cudaSuccess && e2 == cudaSuccess) ? 0 : -1;
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The pool as [n_pages * L * KV * 2 * 64 rows, hd] bf16 with 64 x 64 boxes.
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
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

void launch_attention(const CUtensorMap& kv_map, const void* q, const int* page_table, int maxp,
                      const AttnItem* items, const int* n_items_dev, int n_items_host, void* out, float* partial,
                      int* tickets, const ModelDims& m, int layer, cudaStream_t st) {
  const int grid = 148;   // one wave, persistent over the flat (item, KV head) units
  if (m.hd == 128)
    launch_pdl(attn_kernel<128>, dim3(grid), dim3(AT_THREADS), AttnCfg<128>::SMEM, st, kv_map,
               (const __nv_bfloat16*)q, page_table, maxp, items, n_items_dev, n_items_host, (__nv_bfloat16*)out,
               partial, tickets, m, layer);
  else
    launch_pdl(attn_kernel<64>, dim3(grid), dim3(AT_THREADS), AttnCfg<64>::SMEM, st, kv_map,
               (const __nv_bfloat16*)q, page_table, maxp, items, n_items_dev, n_items_host, (__nv_bfloat16*)out,
               partial, tickets, m, layer);
}

}  // namespace rp
