// Model-side elementwise kernels: weight formula (Z12), embedding
// gather, RMSNorm, RoPE + paged-KV append, prompt-page fork (K6-K8).
#include <algorithm>
#include "common.cuh"
#include "kernels.h"
#include "gemm.h"

namespace rp {

// ------------------------------------------------------------- weight formula
// Generates the [rows, cols] block whose element (r, c) is element
// (r0 + r, c0 + c) of the logical [*, in_full] tensor `tid` (TP shards are
// blocks of the full tensor), into rows dst_row0 + r of the destination
// matrix (`cols` columns).  mode 0: 16-bit values; mode 1: fp32 (biases,
// exact widening of the bf16 value); mode 2: gate/up rows interleaved in
// 64-row blocks of a [2*rows, cols] tensor (`up` selects the second half of
// each 128-row block).  The value is the bf16 of the formula; `f16` stores it
// as fp16 (GEMM operands, reading Z20), else as bf16.  tiled != 0 stores the
// destination in 128 x 64 blocks, block (R / 128, C / 64) at ((R / 128) *
// cols / 64 + C / 64) * 8192 elements, row-major inside (weight_tiled_index):
// every TMA box of the GEMM is then one contiguous 16 KB read.
__host__ __device__ __forceinline__ long long weight_tiled_index(long long R, long long C, long long cols) {
  return ((R >> 7) * (cols >> 6) + (C >> 6)) * 8192 + (R & 127) * 64 + (C & 63);
}

__global__ void init_weights_kernel(void* out, long long rows, int cols, long long r0, int c0, int in_full,
                                    uint32_t tid, uint32_t k0, uint32_t k1, int mode, int up, int f16,
                                    long long dst_row0, int tiled) {
  const float a = 0.034641016151377546f;   // fl32(0.02 * sqrt(3))
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols, c = e % cols;
    const long long i = (r0 + r) * in_full + (c0 + c);          // logical index
    const U4 x = philox((uint32_t)(i >> 2), tid, 0u, 0x57454947u, k0, k1);
    const float u2m1 =
        __fsub_rn(__fmul_rn(__fadd_rn(__uint2float_rn(u4_word(x, (int)(i & 3)) >> 9), 0.5f), 2.384185791015625e-07f),
                  1.0f);
    const __nv_bfloat16 v = __float2bfloat16_rn(__fmul_rn(a, u2m1));
    if (mode == 1) {
      ((float*)out)[e] = __bfloat162float(v);
      continue;
    }
    const long long R = dst_row0 + (mode == 2 ? (r / 64) * 128 + (r % 64) + (up ? 64 : 0) : r);
    const long long o = tiled ? weight_tiled_index(R, c, cols) : R * cols + c;
    if (f16) ((__half*)out)[o] = __float2half_rn(__bfloat162float(v));
    else ((__nv_bfloat16*)out)[o] = v;
  }
}

void launch_init_weights(void* out, long long rows, int cols, long long r0, int c0, int in_full, uint32_t tid,
                         uint64_t seed, int mode, int up, cudaStream_t st, int f16, long long dst_row0, int tiled) {
  const long long n = rows * cols;
  long long blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
  init_weights_kernel<<<grid, 256, 0, st>>>(out, rows, cols, r0, c0, in_full, tid, (uint32_t)seed,
                                            (uint32_t)(seed >> 32), mode, up, f16, dst_row0, tiled);
}

// Row kernels: one wave of 148 CTAs for device-side (decode) row counts; up
// to 8 CTAs per SM for large host-known (prefill) row counts.
static inline int row_grid(const int* n_dev, int n_host) {
  if (n_dev) return 148;
  return n_host < 148 ? (n_host > 0 ? n_host : 1) : (n_host < 148 * 8 ? n_host : 148 * 8);
}

// ------------------------------------------------------------------ embedding
__global__ void embed_kernel(const int* tok, const int* n_dev, int n_host, const __nv_bfloat16* emb, float* x,
                             int d) {
  pdl_wait();
  pdl_launch_dependents();
  const int n = n_dev ? *n_dev : n_host;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const __nv_bfloat162* e = (const __nv_bfloat162*)(emb + (size_t)tok[r] * d);
    float2* o = (float2*)(x + (size_t)r * d);
    for (int c = threadIdx.x; c < d / 2; c += blockDim.x) o[c] = __bfloat1622float2(e[c]);
  }
}

void launch_embed(const int* tok, const int* n_dev, int n_host, const void* emb, float* x, int d, cudaStream_t st) {
  launch_pdl(embed_kernel, dim3(row_grid(n_dev, n_host)), dim3(256), 0, st, tok, n_dev, n_host,
             (const __nv_bfloat16*)emb, x, d);
}

// -------------------------------------------------------------------- RMSNorm
// h[r] = fp16( x[src] / sqrt(mean(x[src]^2) + eps) * gamma ),  src = gather ? gather[r] : r
// (gamma == nullptr: unit gain -- the engine folds the gains into the weights
// of the consuming GEMM at init)
// One CTA (256 threads) per row.  With `delta` (tensor parallelism):
// x[r] += delta[r] first (the all-reduced partial of a row-parallel GEMM) and
// the updated row is written back.
__global__ void rmsnorm_kernel(float* x, const float* delta, const int* gather, const int* n_dev, int n_host,
                               const float* gamma, act_t* h, act_t* h_lo, int d, float eps) {
  __shared__ float red[32];
  pdl_wait();
  pdl_launch_dependents();
  const int n = n_dev ? *n_dev : n_host;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const int src = gather ? gather[r] : r;
    float4* xr = (float4*)(x + (size_t)src * d);
    float ss = 0.f;
    if (delta) {
      const float4* dr = (const float4*)(delta + (size_t)src * d);
      for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
        float4 v = xr[c];
        const float4 a = dr[c];
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
        xr[c] = v;
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    } else {
      for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
        float4 v = xr[c];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      v = warp_sum(v);
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
    __syncthreads();
    act_t* hr = h + (size_t)r * d;
    act_t* hl = h_lo ? h_lo + (size_t)r * d : nullptr;
    const float4* g4 = (const float4*)gamma;
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
      const float4 v = xr[c], g = g4 ? g4[c] : make_float4(1.f, 1.f, 1.f, 1.f);
      store_act4(hr + 4 * c, hl ? hl + 4 * c : nullptr,
                 make_float4(v.x * inv * g.x, v.y * inv * g.y, v.z * inv * g.z, v.w * inv * g.w));
    }
  }
}

void launch_rmsnorm(float* x, const float* delta, const int* gather, const int* n_dev, int n_host,
                    const float* gamma, void* h, int d, float eps, cudaStream_t st, void* h_lo) {
  launch_pdl(rmsnorm_kernel, dim3(row_grid(n_dev, n_host)), dim3(256), 0, st, x, delta, gather, n_dev, n_host, gamma,
             (act_t*)h, (act_t*)h_lo, d, eps);
}

// --------------------------------------------------- TP add + RMSNorm (peer)
// Tensor-parallel decode: the row-parallel GEMM of every rank pushed its fp32
// partial into recv[src] of this rank (NVLink stores, gemm_tcgen05 push) and
// counted its finished output units in flags[src].  Wait until every source
// delivered this use's units, then x[r] += sum_src recv[src][r] in rank order
// (identical bits on every rank), write x back and h = fp16(x / rms * gamma).
// gen = output units of this slot consumed so far on this rank (cumulative:
// the units per use depend on the live count); the last CTA advances it.
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void tp_norm_kernel(float* x, const float* recv, int tp, size_t src_stride,
                               const unsigned long long* flags, unsigned long long* gen, int* done, int m_tiles,
                               int splits, int coop_min, const int* n_dev, const float* gamma, act_t* h,
                               act_t* h_lo, int d, float eps) {
  __shared__ float red[32];
  __shared__ unsigned long long s_units;
  pdl_wait();
  pdl_launch_dependents();
  const int n = *n_dev;
  if (n <= 0) return;
  if (threadIdx.x == 0) {
    // output units the producer GEMM signals per use (its cooperative
    // split-K reduction finishes one column slice per split)
    const int n_chunks = (n + 255) / 256;
    const bool coop = splits > 1 && m_tiles * n_chunks * splits <= 148 && min(256, n) >= coop_min;
    const unsigned long long units = (unsigned long long)m_tiles * n_chunks * (coop ? splits : 1);
    const unsigned long long target = *(volatile unsigned long long*)gen + units;
    s_units = units;
    for (int q = 0; q < tp; ++q) {
      uint32_t spins = 0;
      while (ld_acquire_sys_u64(flags + q) < target) {
        if (++spins == (1u << 28)) {
          printf("rollpacker watchdog: TP peer partial stuck (rank slot %d, %llu < %llu)\n", q,
                 ld_acquire_sys_u64(flags + q), target);
          __trap();
        }
      }
    }
  }
  __syncthreads();
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    float4* xr = (float4*)(x + (size_t)r * d);
    float ss = 0.f;
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
      float4 s = __ldcg((const float4*)(recv + (size_t)r * d) + c);
      for (int q = 1; q < tp; ++q) {
        const float4 a = __ldcg((const float4*)(recv + q * src_stride + (size_t)r * d) + c);
        s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
      }
      float4 v = xr[c];
      v.x += s.x; v.y += s.y; v.z += s.z; v.w += s.w;
      xr[c] = v;
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      v = warp_sum(v);
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
    __syncthreads();
    act_t* hr = h + (size_t)r * d;
    act_t* hl = h_lo ? h_lo + (size_t)r * d : nullptr;
    const float4* g4 = (const float4*)gamma;
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
      const float4 v = xr[c], g = g4 ? g4[c] : make_float4(1.f, 1.f, 1.f, 1.f);
      store_act4(hr + 4 * c, hl ? hl + 4 * c : nullptr,
                 make_float4(v.x * inv * g.x, v.y * inv * g.y, v.z * inv * g.z, v.w * inv * g.w));
    }
  }
  // this use of the slot is consumed once every CTA is past its reads
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      *done = 0;
      *gen += s_units;
    }
  }
}

void launch_tp_norm(float* x, const float* recv, int tp, size_t src_stride, const unsigned long long* flags,
                    unsigned long long* gen, int* done, int m_tiles, int splits, int coop_min, int max_grid,
                    const int* n_dev, int n_rows_grid, const float* gamma, void* h, int d, float eps,
                    cudaStream_t st, void* h_lo) {
  // max_grid bounds the CTAs that spin on the peers' flags (single-GPU local
  // groups: the peers' GEMMs must find free SMs)
  const int grid = std::min(row_grid(n_dev, n_rows_grid), max_grid > 0 ? max_grid : 1 << 30);
  launch_pdl(tp_norm_kernel, dim3(grid), dim3(256), 0, st, x, recv, tp, src_stride, flags, gen, done, m_tiles, splits,
             coop_min, n_dev, gamma, (act_t*)h, (act_t*)h_lo, d, eps);
}

// ------------------------------------------------------ folded norm gains
__global__ void scale_cols_kernel(__half* w, long long rows, int cols, const float* __restrict__ gamma, int tiled) {
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    // column of element e (tiled: block e / 8192 is column block (e / 8192) % (cols / 64))
    const int c = tiled ? (int)(((e >> 13) % (cols >> 6)) * 64 + (e & 63)) : (int)(e % cols);
    w[e] = __float2half_rn(__half2float(w[e]) * gamma[c]);
  }
}

void launch_scale_cols(void* w, long long rows, int cols, const float* gamma, cudaStream_t st, int tiled) {
  const long long n = rows * cols;
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 64);
  scale_cols_kernel<<<grid, 256, 0, st>>>((__half*)w, rows, cols, gamma, tiled);
}

// -------------------------------------------------------- RoPE + KV append
// qkv row r (fp32, bias already added): [q heads | k heads | v heads] x hd.
// Rotate-half RoPE at position row_pos[r] (angle in fp64, then fp32 sincos
// of the reduced angle), q -> q_out[r][H][hd] fp16, k/v -> KV page (fp16).
__global__ void rope_append_kernel(const float* qkv, const int* n_dev, int n_host, const int* row_pos,
                                   const int* row_pt, const int* page_table, int maxp, act_t* q_out, act_t* q_lo,
                                   uint8_t* kv_pool, ModelDims m, int layer, const double* inv_freq) {
  extern __shared__ float cs[];   // [hd/2] cos, [hd/2] sin
  pdl_wait();
  pdl_launch_dependents();
  const int n = n_dev ? *n_dev : n_host;
  const int half = m.hd / 2, W = (m.H + 2 * m.KV) * m.hd;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const int pos = row_pos[r];
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
      double ang = (double)pos * inv_freq[i];
      ang = ang - 6.283185307179586 * floor(ang / 6.283185307179586);
      float s, c;
      sincosf((float)ang, &s, &c);
      cs[i] = c; cs[half + i] = s;
    }
    __syncthreads();
    const float* row = qkv + (size_t)r * W;
    const int page = page_table[(size_t)row_pt[r] * maxp + pos / kPage];
    const int prow = pos % kPage;
    act_t* kbase = (act_t*)kv_pool + (size_t)prow * m.hd;
    // q and k: rotated pairs
    for (int e = threadIdx.x; e < (m.H + m.KV) * half; e += blockDim.x) {
      const int head = e / half, i = e % half;
      const float* src = row + head * m.hd;
      const float x1 = src[i], x2 = src[i + half], c = cs[i], s = cs[half + i];
      const float o1 = x1 * c - x2 * s, o2 = x2 * c + x1 * s;
      if (head < m.H) {
        const size_t qo = ((size_t)r * m.H + head) * m.hd;
        const act_t h1 = to_act(o1), h2 = to_act(o2);
        q_out[qo + i] = h1; q_out[qo + i + half] = h2;
        if (q_lo) {                      // rounding residual (split precision)
          q_lo[qo + i] = to_act(o1 - __half2float(h1));
          q_lo[qo + i + half] = to_act(o2 - __half2float(h2));
        }
      } else {
        const int kh = head - m.H;
        act_t* dst = kbase + kv_block_elems(layer, page, kh, 0, m.n_pages, m.KV, m.hd);
        dst[i] = to_act(o1); dst[i + half] = to_act(o2);
      }
    }
    for (int e = threadIdx.x; e < m.KV * m.hd; e += blockDim.x) {
      const int kh = e / m.hd, i = e % m.hd;
      act_t* dst = kbase + kv_block_elems(layer, page, kh, 1, m.n_pages, m.KV, m.hd);
      dst[i] = to_act(row[(m.H + m.KV) * m.hd + e]);
    }
    __syncthreads();
  }
}

void launch_rope_append(const float* qkv, const int* n_dev, int n_host, const int* row_pos, const int* row_pt,
                        const int* page_table, int maxp, void* q_out, void* kv_pool, const ModelDims& m, int layer,
                        const double* inv_freq, cudaStream_t st, void* q_lo) {
  launch_pdl(rope_append_kernel, dim3(row_grid(n_dev, n_host)), dim3(256), m.hd * sizeof(float), st, qkv, n_dev,
             n_host, row_pos, row_pt, page_table, maxp, (act_t*)q_out, (act_t*)q_lo, (uint8_t*)kv_pool, m, layer,
             inv_freq);
}

// ------------------------------------------------------------- prompt fork
// Copy the first `rows` tokens of every (layer, kv head, K|V) block of page
// src into page dst (the G siblings' private copy of a partial prompt page).
__global__ void kv_fork_kernel(const int* jobs, int n, uint8_t* pool, ModelDims m) {
  const int blocks = m.L * m.KV * 2;
  for (int j = blockIdx.x; j < n * blocks; j += gridDim.x) {
    const int job = j / blocks, blk = j % blocks;
    const int src = jobs[3 * job], dst = jobs[3 * job + 1], rows = jobs[3 * job + 2];
    const int layer = blk / (m.KV * 2), kvh = (blk / 2) % m.KV, kv = blk % 2;
    const int4* s = (const int4*)((const act_t*)pool + kv_block_elems(layer, src, kvh, kv, m.n_pages, m.KV, m.hd));
    int4* d = (int4*)((act_t*)pool + kv_block_elems(layer, dst, kvh, kv, m.n_pages, m.KV, m.hd));
    const int n16 = rows * m.hd * 2 / 16;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
  }
}

void launch_kv_fork(const int* jobs, int n, void* kv_pool, const ModelDims& m, cudaStream_t st) {
  if (n <= 0) return;
  kv_fork_kernel<<<148 * 4, 256, 0, st>>>(jobs, n, (uint8_t*)kv_pool, m);
}

}  // namespace rp
