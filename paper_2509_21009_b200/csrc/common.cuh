// Shared device helpers of the CUDA path (sm_100a).  Shares nothing with
// oracle/: the Philox round, the weight formula and the Gumbel mapping are
// re-implemented here from DESIGN.md §3 (Z10, Z12).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdio>

namespace rp {

// Activation / KV-cache / GEMM-operand element type (reading Z20):
// fp16.  Its 11-bit significand keeps the teacher-forced logits of the
// 28-layer 7B decoder within the north-star 2e-2 of the fp64 oracle, which
// bf16 activations (8 bits) miss by ~7x; the weights are the bf16 values of
// the Z12 formula re-encoded exactly in fp16 (magnitudes below 6.1e-5 round to
// the fp16 subnormal grid, <= 3e-8).
using act_t = __half;
using act2_t = __half2;
__device__ __forceinline__ act_t to_act(float a) { return __float2half_rn(a); }
__device__ __forceinline__ act2_t to_act2(float a, float b) { return __floats2half2_rn(a, b); }
// fp16 of 4 consecutive values (8-byte aligned) and, when lo != nullptr, their
// rounding residuals fp16(v - float(fp16(v))): split-precision activations
// (reading Z22) carry hi + lo ~ 22 significant bits into the next GEMM
__device__ __forceinline__ void store_act4(act_t* hi, act_t* lo, float4 v) {
  const act2_t h01 = to_act2(v.x, v.y), h23 = to_act2(v.z, v.w);
  ((act2_t*)hi)[0] = h01;
  ((act2_t*)hi)[1] = h23;
  if (lo) {
    const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
    ((act2_t*)lo)[0] = to_act2(v.x - f01.x, v.y - f01.y);
    ((act2_t*)lo)[1] = to_act2(v.z - f23.x, v.w - f23.y);
  }
}


constexpr int kPage = 64;          // tokens per KV page (DESIGN.md §5 D1)
// KV pool layout: [L][n_pages][KV][K|V][kPage][hd] fp16, layer-major, so the pages one
// layer's attention reads lie in one contiguous [n_pages][KV][2][kPage][hd] slab (16 pages of the 7B
// shape per 2 MB TLB entry instead of one): element offset of the (layer, page, kv head, K|V) block.
__host__ __device__ __forceinline__ size_t kv_block_elems(int layer, int page, int kvh, int kv, int n_pages, int KV,
                                                          int hd) {
  return (((((size_t)layer * n_pages + page) * KV + kvh) * 2 + kv) * kPage) * hd;
}
constexpr int kAttnChunk = 512;    // tokens per decode-attention split
constexpr int kAttnFillUnits = 2 * 148;  // (row, kv head) units that fill the GPU without splits

// ---------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = mulhi32(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = mulhi32(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

__host__ __device__ __forceinline__ uint32_t u4_word(const U4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// u = ((x >> 9) + 0.5) * 2^-23, exact in fp32, strictly inside (0, 1).
__device__ __forceinline__ float u01(uint32_t x) {
  return (__uint2float_rn(x >> 9) + 0.5f) * 1.1920928955078125e-07f;
}

// Orderable encoding of a float for packed (value, index) argmax with
// atomicMax on uint64: larger value wins, then lower index.
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ unsigned long long pack_arg(float v, uint32_t idx) {
  return ((unsigned long long)f2ord(v) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}
__host__ __device__ __forceinline__ uint32_t unpack_idx(unsigned long long p) {
  return 0xFFFFFFFFu - (uint32_t)(p & 0xFFFFFFFFull);
}

// mbarrier wait with a watchdog: a wait that polls ~2^28 times (seconds) is
// a deadlock -- report it and trap instead of hanging the GPU.  (try_wait
// suspends the thread for a bounded time per poll, so 2^22 polls >> any
// legitimate wait in these kernels.)
__device__ __forceinline__ void mbar_wait_wd(uint32_t bar, uint32_t phase, int tag, long long d0 = 0, long long d1 = 0) {
  uint32_t ok = 0;
  uint32_t spins = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    if (!ok && ++spins == (1u << 23)) __trap();
    if (!ok && spins == (1u << 22)) {
      printf("rollpacker watchdog: mbarrier wait stuck (tag %d, block %d,%d, thread %d, phase %u, %lld %lld)\n",
             tag, blockIdx.x, blockIdx.y, threadIdx.x, phase, d0, d1);
    }
  } while (!ok);
}

// Programmatic dependent launch (PDL).  Every kernel of the step is launched
// with programmatic stream serialization: it may start while its predecessor
// finishes.  Each kernel first waits for the predecessor (griddepcontrol.wait)
// before touching its outputs, then lets its own successor launch.  Because
// the trigger comes after the wait, a kernel's pre-wait code can rely on all
// kernels before its predecessor having completed.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024).
// Returns the exclusive prefix; *total receives the block sum.
__device__ __forceinline__ int block_exscan(int v, int* total, int* smem /*>=33 ints*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) smem[lane] = w;      // inclusive per-warp totals
  }
  __syncthreads();
  int base = wid ? smem[wid - 1] : 0;
  int tot = smem[nw - 1];
  __syncthreads();
  *total = tot;
  return base + x - v;
}

// Programmatic dependent launch is switched off on the calling thread while
// a context of a single-GPU local group (rp_local_group_create) issues work:
// several contexts then share one GPU, and a PDL-launched kernel parked in
// griddepcontrol.wait would hold SMs another context's producer needs.
extern thread_local bool g_no_pdl;

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace rp
