// Paged-KV GQA attention for decode and prefill (K4/K5).
//
// One CTA = one (query block, KV head, key split).  The MMA rows are the
// (query token, query head) pairs served by one KV head: decode has 1 token
// x g heads (g = H/KV <= 8, padded to 16); prefill packs floor(16/g) tokens.
// The key range is streamed page by page (64 tokens) through a 3-stage
// cp.async ring with an XOR-swizzled layout (conflict-free ldmatrix); each of
// the 4 warps owns 16 tokens of a page: S = Q K^T and O += P V run on
// mma.sync m16n8k16 (bf16 in, fp32 accumulate) with an online softmax in the
// log2 domain.  The 4 warp states merge in shared memory; multi-split blocks
// write (m, l, O) partials that attn_merge combines in split order.
// Decode attention moves g FLOP per KV byte, far below the B200 ridge point,
// so the bound is HBM: the design goal is bytes in flight, not FLOPs.
#include "common.cuh"
#include "kernels.h"

namespace rp {

constexpr int AT_WARPS = 4, AT_STAGES = 3;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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

template <int HD>
struct AttnCfg {
  static constexpr int CH = HD / 8;                    // 16-byte chunks per row
  static constexpr int TILE_BYTES = kPage * HD * 2;    // one K (or V) page block
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int SMEM = AT_STAGES * STAGE_BYTES;
};

// swizzled byte offset of (row, chunk) inside a [64][HD] bf16 tile
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * HD * 2 + ((chunk ^ (row & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(AT_WARPS * 32)
attn_kernel(const __nv_bfloat16* __restrict__ q, const uint8_t* __restrict__ pool, const int* __restrict__ page_table,
            int maxp, const AttnItem* __restrict__ items, const int* n_items_dev, int n_items_host,
            __nv_bfloat16* __restrict__ out, float* __restrict__ partial, ModelDims m, int layer) {
  using C = AttnCfg<HD>;
  extern __shared__ __align__(128) uint8_t sm[];
  const int n_items = n_items_dev ? *n_items_dev : n_items_host;
  const int kvh = blockIdx.y;
  const int g = m.H / m.KV;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float scale = 1.4426950408889634f * rsqrtf((float)HD);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);

  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const AttnItem I = items[it];
    const int tpb = 16 / g;
    const int nrows = I.n_qtok * g;
    // ---- Q fragments (A operand, 16 x HD), rows r = tok*g + head
    uint32_t qa[HD / 16][4];
    {
      const int r0 = lane >> 2, r1 = r0 + 8, c = 2 * (lane & 3);
      const __nv_bfloat16* q0 = nullptr;
      const __nv_bfloat16* q1 = nullptr;
      if (r0 < nrows) q0 = q + ((size_t)(I.q_row0 + r0 / g) * m.H + kvh * g + r0 % g) * HD;
      if (r1 < nrows) q1 = q + ((size_t)(I.q_row0 + r1 / g) * m.H + kvh * g + r1 % g) * HD;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qa[kk][0] = q0 ? *(const uint32_t*)(q0 + kk * 16 + c) : 0u;
        qa[kk][1] = q1 ? *(const uint32_t*)(q1 + kk * 16 + c) : 0u;
        qa[kk][2] = q0 ? *(const uint32_t*)(q0 + kk * 16 + 8 + c) : 0u;
        qa[kk][3] = q1 ? *(const uint32_t*)(q1 + kk * 16 + 8 + c) : 0u;
      }
    }
    (void)tpb;
    // causal limits of this thread's two rows (keys j < lim allowed)
    const int ra = lane >> 2, rb = ra + 8;
    const int lim_a = ra < nrows ? I.pos0 + ra / g + 1 : 0;
    const int lim_b = rb < nrows ? I.pos0 + rb / g + 1 : 0;
    const int kv_hi = I.kv_hi;

    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;

    const int p_lo = I.kv_lo / kPage, p_hi = (kv_hi + kPage - 1) / kPage;
    const int npg = p_hi - p_lo;
    const int* ptab = page_table + (size_t)I.pt_row * maxp;
    const size_t blk_k = (size_t)((layer * m.KV + kvh) * 2 + 0) * C::TILE_BYTES;

    auto issue = [&](int pi) {
      if (pi < npg) {
        const int p = p_lo + pi;
        const uint8_t* kb = pool + (size_t)ptab[p] * m.page_bytes + blk_k;
        const uint32_t st = sbase + (pi % AT_STAGES) * C::STAGE_BYTES;
        const int tok0 = p * kPage;
        for (int e = tid; e < 2 * kPage * C::CH; e += AT_WARPS * 32) {
          const int kv = e / (kPage * C::CH), rem = e % (kPage * C::CH);
          const int row = rem / C::CH, ch = rem % C::CH;
          const bool ok = tok0 + row < kv_hi;
          const uint8_t* src = kb + kv * C::TILE_BYTES + row * HD * 2 + ch * 16;
          cp_async16(st + kv * C::TILE_BYTES + swz<HD>(row, ch), ok ? (const void*)src : (const void*)kb, ok ? 16 : 0);
        }
      }
      cp_commit();
    };

#pragma unroll
    for (int s = 0; s < AT_STAGES - 1; ++s) issue(s);

    for (int pi = 0; pi < npg; ++pi) {
      cp_wait<AT_STAGES - 2>();
      __syncthreads();
      issue(pi + AT_STAGES - 1);
      const uint32_t kt = sbase + (pi % AT_STAGES) * C::STAGE_BYTES;
      const uint32_t vt = kt + C::TILE_BYTES;
      const int tok_base = (p_lo + pi) * kPage + 16 * warp;
      if (tok_base < kv_hi) {
        // ---- S = Q K^T over this warp's 16 tokens (two n8 tiles)
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const int row = 16 * warp + (lane & 7) + ((lane >> 4) << 3);
          const int ch = 2 * kk + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma16816(s[0], qa[kk], b0, b1);
          mma16816(s[1], qa[kk], b2, b3);
        }
        // ---- mask + online softmax (log2 domain)
        float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = tok_base + nt * 8 + 2 * (lane & 3) + e;
            const bool va = j < kv_hi && j < lim_a, vb = j < kv_hi && j < lim_b;
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
        float p[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          p[nt][0] = exp2f(s[nt][0] - base_a); p[nt][1] = exp2f(s[nt][1] - base_a);
          p[nt][2] = exp2f(s[nt][2] - base_b); p[nt][3] = exp2f(s[nt][3] - base_b);
        }
        l_a = l_a * al_a + p[0][0] + p[0][1] + p[1][0] + p[1][1];
        l_b = l_b * al_b + p[0][2] + p[0][3] + p[1][2] + p[1][3];
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) { o[i][0] *= al_a; o[i][1] *= al_a; o[i][2] *= al_b; o[i][3] *= al_b; }
        uint32_t pa[4];
        pa[0] = pack_bf16(p[0][0], p[0][1]);
        pa[1] = pack_bf16(p[0][2], p[0][3]);
        pa[2] = pack_bf16(p[1][0], p[1][1]);
        pa[3] = pack_bf16(p[1][2], p[1][3]);
        // ---- O += P V  (V rows = tokens: ldmatrix.trans)
#pragma unroll
        for (int dt = 0; dt < HD / 8; dt += 2) {
          const int row = 16 * warp + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int ch = dt + (lane >> 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vt + swz<HD>(row, ch), b0, b1, b2, b3);
          mma16816(o[dt], pa, b0, b1);
          mma16816(o[dt + 1], pa, b2, b3);
        }
      }
    }
    cp_wait<0>();
    __syncthreads();
    // ---- merge the 4 warps: smem [4][16] m, l and [4][16][HD] O (fp32)
    float* sm_m = (float*)sm;
    float* sm_l = sm_m + AT_WARPS * 16;
    float* sm_o = sm_l + AT_WARPS * 16;
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    if ((lane & 3) == 0) {
      sm_m[warp * 16 + ra] = m_a; sm_l[warp * 16 + ra] = l_a;
      sm_m[warp * 16 + rb] = m_b; sm_l[warp * 16 + rb] = l_b;
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int c = i * 8 + 2 * (lane & 3);
      sm_o[(warp * 16 + ra) * HD + c] = o[i][0];
      sm_o[(warp * 16 + ra) * HD + c + 1] = o[i][1];
      sm_o[(warp * 16 + rb) * HD + c] = o[i][2];
      sm_o[(warp * 16 + rb) * HD + c + 1] = o[i][3];
    }
    __syncthreads();
    for (int e = tid; e < nrows * HD; e += AT_WARPS * 32) {
      const int r = e / HD, c = e % HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < AT_WARPS; ++w) M = fmaxf(M, sm_m[w * 16 + r]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < AT_WARPS; ++w) {
        const float f = exp2f(sm_m[w * 16 + r] - Mb);
        L += sm_l[w * 16 + r] * f;
        O += sm_o[(w * 16 + r) * HD + c] * f;
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
    __syncthreads();
  }
}

// Combine the splits of multi-split query blocks in split order.
template <int HD>
__global__ void attn_merge_kernel(const AttnItem* __restrict__ items, const int* n_items_dev, int n_items_host,
                                  const float* __restrict__ partial, __nv_bfloat16* __restrict__ out, ModelDims m) {
  const int n_items = n_items_dev ? *n_items_dev : n_items_host;
  const int g = m.H / m.KV;
  const int kvh = blockIdx.y;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const AttnItem I = items[it];
    if (I.nsplit == 1 || it != I.item0) continue;
    const int nrows = I.n_qtok * g;
    const float* __restrict__ p0 = partial + ((size_t)I.item0 * m.KV + kvh) * (16 * (HD + 2));
    const size_t sstride = (size_t)m.KV * 16 * (HD + 2);
    for (int e = threadIdx.x; e < nrows * HD; e += blockDim.x) {
      const int r = e / HD, c = e % HD;
      float M = -INFINITY;
      for (int s = 0; s < I.nsplit; ++s) M = fmaxf(M, p0[s * sstride + r]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f, O = 0.f;
      for (int s = 0; s < I.nsplit; ++s) {
        const float* pp = p0 + s * sstride;
        const float f = exp2f(pp[r] - Mb);
        L += pp[16 + r] * f;
        O += pp[32 + r * HD + c] * f;
      }
      const int tok = I.q_row0 + r / g, head = kvh * g + r % g;
      out[((size_t)tok * m.H + head) * HD + c] = __float2bfloat16(L > 0.f ? O / L : 0.f);
    }
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

void launch_attention(const void* q, const void* kv_pool, const int* page_table, int maxp, const AttnItem* items,
                      const int* n_items_dev, int n_items_host, void* out, float* partial, const ModelDims& m,
                      int layer, cudaStream_t st) {
  const int gx = (2 * 148 + m.KV - 1) / m.KV;
  dim3 grid(gx < 1 ? 1 : gx, m.KV);
  if (m.hd == 128)
    attn_kernel<128><<<grid, AT_WARPS * 32, AttnCfg<128>::SMEM, st>>>(
        (const __nv_bfloat16*)q, (const uint8_t*)kv_pool, page_table, maxp, items, n_items_dev, n_items_host,
        (__nv_bfloat16*)out, partial, m, layer);
  else
    attn_kernel<64><<<grid, AT_WARPS * 32, AttnCfg<64>::SMEM, st>>>(
        (const __nv_bfloat16*)q, (const uint8_t*)kv_pool, page_table, maxp, items, n_items_dev, n_items_host,
        (__nv_bfloat16*)out, partial, m, layer);
}

void launch_attn_merge(const AttnItem* items, const int* n_items_dev, int n_items_host, const float* partial,
                       void* out, const ModelDims& m, cudaStream_t st) {
  dim3 grid((4 * 148 + m.KV - 1) / m.KV, m.KV);
  if (m.hd == 128)
    attn_merge_kernel<128><<<grid, 128, 0, st>>>(items, n_items_dev, n_items_host, partial, (__nv_bfloat16*)out, m);
  else
    attn_merge_kernel<64><<<grid, 128, 0, st>>>(items, n_items_dev, n_items_host, partial, (__nv_bfloat16*)out, m);
}

}  // namespace rp
