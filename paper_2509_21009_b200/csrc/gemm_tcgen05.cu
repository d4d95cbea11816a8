// Swap-AB decode/prefill GEMM on the 5th-generation tensor cores (sm_100a).
//
//   D[m, n] = sum_k W[m, k] * X[n, k]      (W: weights [M, K] fp16, K-major;
//                                           X: activations [N, K] fp16, K-major)
//
// Weights fill the UMMA M=128 tile; the live batch (or prompt tokens) is the
// UMMA N dimension, read at run time from device memory so the same launch is
// valid for every live count inside a captured CUDA graph.  Operands are
// staged by TMA (SWIZZLE_128B, 64-element K blocks) into a 4-stage
// shared-memory ring; one elected thread issues tcgen05.mma into a
// double-buffered TMEM accumulator (2 x 256 fp32 columns); four epilogue warps
// read TMEM with tcgen05.ld and apply the fused epilogue.
//
// Work = m_tiles x n_chunks(256) x splits.  Split-K (fixed per weight shape,
// independent of N, so results are batch invariant) writes fp32 partials that
// are summed in split order (deterministic): by the tile's last CTA (ticket),
// by a designated reducer split, or cooperatively by all split CTAs of the
// tile (one column slice each) -- the same sums bit for bit.
//
// Epilogues (DESIGN.md §5 K1/K2): F32 (+bias) for QKV and logits, RESID
// (fp32 residual +=) for O/down, SWIGLU (tile rows 0-63 gate, 64-127 up of the
// same 64 features, weights interleaved at init) for gate||up, BF16 store.
#include <cuda.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"
#include "gemm.h"

namespace rp {

constexpr int BM = 128, BK = 64, BN = 256;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB
constexpr int B_BYTES = BN * BK * 2;         // 32 KB (widest activation tile)
// 200 KB of stages: everything the 227 KB opt-in leaves beside the epilogue
// buffers.  Bytes in flight per SM set the weight-streaming rate at small N
// (Little's law: ~6 us of loaded HBM latency), so the ring takes the rest.
constexpr int RING_BYTES = 200 * 1024;
constexpr int MAX_STAGES = 12;               // ring depth at small N (18 KB stages)
constexpr int XCH_BYTES = 64 * 33 * 4;       // swiglu exchange
constexpr int TS = BM + 4;                   // fp32 row stride of the epilogue staging tile
constexpr int STG_BYTES = 32 * TS * 4;       // [32 columns][128 rows] fp32 staging for 16-byte stores
constexpr int RSC_BYTES = BN * 4;             // per-column RMSNorm scales of the current item
constexpr int GEMM_SMEM = RING_BYTES + XCH_BYTES + STG_BYTES + RSC_BYTES + 1024 /*align*/ + 8 * (2 * MAX_STAGES + 4) + 16;
static_assert(GEMM_SMEM <= 232448, "GEMM shared memory above the sm_100 opt-in limit");
constexpr int GEMM_THREADS = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) { mbar_wait_wd(bar, phase, 1); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups of
// 128 B rows -> stride byte offset 1024; version 1 (sm_100); layout type 2.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO
  d |= (uint64_t)1 << 46;                    // version
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A and B fp16
// (bits 7-9, 10-12 = 0; bf16 would be 1), both K-major, N >> 3, M >> 4.
__device__ __forceinline__ uint32_t make_idesc(int n, int m = BM) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
// CTA-pair (cta_group::2) forms: the leader issues the M=256 MMA over both
// CTAs' shared memory (each holds its 128 weight rows and half of the
// activation rows) into both CTAs' TMEM; commits multicast to both CTAs.
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
      : "memory");
}
// shared::cluster address of the same shared-memory offset in cluster CTA 0
__device__ __forceinline__ uint32_t leader_addr(uint32_t a) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// generic address of the same shared-memory object in cluster CTA `rank`
__device__ __forceinline__ const float* dsm_peer(const float* p, uint32_t rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return (const float*)r;
}
__device__ __forceinline__ uint32_t dsm_peer_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
  uint32_t ok = 0, spins = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    if (!ok && ++spins == (1u << 24)) {
      printf("rollpacker watchdog: split-K cluster exchange stuck (block %d)\n", blockIdx.x);
      __trap();
    }
  } while (!ok);
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define TMEM_LD32(taddr, r)                                                                                   \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"        \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),      \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),             \
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),           \
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),           \
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                                  \
      : "r"(taddr));                                                                                          \
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// debug timeline: [0] CTA start, [1] setup done, [2+2i] item i first stage ready,
// [3+2i] item i last MMA issued (i < 3), [8+i] item i epilogue done (i < 3)
#define TL(k) do { if (a.timeline) a.timeline[blockIdx.x * 16 + (k)] = gtimer(); } while (0)

struct Item { int tile, chunk, split; };
// split fastest, then tile, then chunk; with `chunks_inner` (split-precision
// GEMMs, 128-column chunks) the chunks of a tile are adjacent items, so the
// CTAs that read the same weight tile run together and share it through L2
__device__ __forceinline__ Item decode_item(int it, int m_tiles, int splits, int n_chunks = 1, bool chunks_inner = false) {
  Item r;
  r.split = it % splits;
  int q = it / splits;
  if (chunks_inner) {
    r.chunk = q % n_chunks;
    r.tile = q / n_chunks;
  } else {
    r.tile = q % m_tiles;
    r.chunk = q / m_tiles;
  }
  return r;
}

// ---- split-K reduction helpers: rows r4..r4+3 of columns cb + 4u (u < RU)
constexpr int RU = 4;
template <int S>
__device__ __forceinline__ void reduce_splits(float4 (&acc)[RU], const float* __restrict__ pb, int cb, int col_hi,
                                              int r4) {
  float4 t[S][RU];
#pragma unroll
  for (int sp = 0; sp < S; ++sp)
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int col = cb + 4 * u;
      t[sp][u] = col < col_hi ? __ldcg((const float4*)(pb + (size_t)sp * BN * BM + (size_t)col * BM + r4))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
  for (int u = 0; u < RU; ++u) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp = 0; sp < S; ++sp) { v.x += t[sp][u].x; v.y += t[sp][u].y; v.z += t[sp][u].z; v.w += t[sp][u].w; }
    acc[u] = v;
  }
}
__device__ __forceinline__ void reduce_splits_loop(float4 (&acc)[RU], const float* __restrict__ pb, int cb, int col_hi,
                                                   int r4, int S) {
#pragma unroll
  for (int u = 0; u < RU; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int sp = 0; sp < S; ++sp) {
    float4 t[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int col = cb + 4 * u;
      t[u] = col < col_hi ? __ldcg((const float4*)(pb + (size_t)sp * BN * BM + (size_t)col * BM + r4))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) { acc[u].x += t[u].x; acc[u].y += t[u].y; acc[u].z += t[u].z; acc[u].w += t[u].w; }
  }
}

// the same sums from the split CTAs' shared memory (cluster DSMEM), split order
template <int S>
__device__ __forceinline__ void reduce_splits_dsm(float4 (&acc)[RU], const float* const (&pp)[8], int cb, int col_hi,
                                                  int r4) {
  float4 t[S][RU];
#pragma unroll
  for (int sp = 0; sp < S; ++sp)
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int col = cb + 4 * u;
      t[sp][u] = col < col_hi ? *(const float4*)(pp[sp] + (size_t)col * BM + r4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
  for (int u = 0; u < RU; ++u) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp = 0; sp < S; ++sp) { v.x += t[sp][u].x; v.y += t[sp][u].y; v.z += t[sp][u].z; v.w += t[sp][u].w; }
    acc[u] = v;
  }
}

// Tensor-parallel push: this output unit's stores (local and NVLink peer) are
// released at system scope, then every destination's counter is bumped.
__device__ __forceinline__ void push_signal(const GemmArgs& a, int et) {
  if (!a.push_n) return;
  __threadfence_system();
  named_bar(1, 128);
  if (et == 0)
    for (int q = 0; q < a.push_n; ++q)
      asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(a.push_flag[q]) : "memory");
}

// CG = 1: one CTA per 128-row weight tile.  CG = 2 (no split-K, launched as
// clusters of 2): a CTA pair per 256-row tile -- each CTA loads its 128
// weight rows and half of the activation rows, the leader issues
// tcgen05.mma.cta_group::2 (M = 256) and each CTA's TMEM holds its 128 output
// rows, so a stage carries half the activation bytes per SM and the ring runs
// deeper (the wide-batch regime is bound by ring bytes per FLOP).
// LO = 1: split-precision activations (GemmArgs::lo) -- a separate
// instantiation, because runtime lo branches in the producer and MMA loops
// cost ~25% of the weight-streaming rate at small N even when off (measured:
// profiles/r02_gemm_lo_bisect.txt).
template <int CG, int LO>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB16,
                    const __grid_constant__ CUtensorMap tmB64, const __grid_constant__ CUtensorMap tmB256,
                    const __grid_constant__ CUtensorMap tmL16, const __grid_constant__ CUtensorMap tmL64,
                    const __grid_constant__ CUtensorMap tmL256, GemmArgs a) {
  const int N = a.n_dev ? *a.n_dev : a.n_host;
  if (N <= 0) return;
  if (threadIdx.x == 0) TL(0);
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const int cta_id = CG == 2 ? (int)blockIdx.x / 2 : (int)blockIdx.x;   // work-unit owner (the pair)
  const int n_ctas = CG == 2 ? (int)gridDim.x / 2 : (int)gridDim.x;
  const bool leader = crank == 0;
  const int m_tiles = a.M / (BM * CG);
  // LO, N <= 128 (narrow): one chunk whose hi rows and then lo rows form the
  // MMA's N, so a row's hi and lo products come out of one MMA (the weight
  // tile is read from shared memory once per K step).  LO, N > 128 (wide):
  // 256-column chunks, the hi rows and the lo rows multiplied by two MMAs into
  // two TMEM accumulators (columns [0, 256) and [256, 512): no double
  // buffering) -- per element the same two fp32 sums as the narrow form, so
  // the result does not depend on the batch size.
  const bool wide = LO && N > 128;
  const int BNX = (LO && !wide) ? 128 : BN;
  const int n_chunks = (N + BNX - 1) / BNX;
  const int n_items = m_tiles * n_chunks * a.splits;
  if (cta_id >= n_items) return;                   // both CTAs of a pair leave together
  const int kb_total = a.K / BK;
  // cooperative split-K reduction: grid fits one wave and the chunk is wide
  // enough that a single CTA reducing the whole tile would be the bottleneck
  const bool coop = !a.dsm && a.splits > 1 && n_items <= n_ctas && min(BNX, N) >= a.coop_min;
  if (a.dsm && n_items != n_ctas) {                // the host sized the cluster grid for one chunk
    if (threadIdx.x == 0) printf("rollpacker: dsm split-K grid %d != items %d\n", n_ctas, n_items);
    __trap();
  }

  // Ring geometry from the widest activation chunk: 16/64/256-row boxes; at
  // small N the stages shrink and the ring deepens (more weight bytes in
  // flight per SM for the HBM-bound small-batch regime).
  // (pair: each CTA holds half of the 16-padded chunk, at most 128 rows)
  // (pair, narrow LO: CTA 0 holds the chunk's hi rows and CTA 1 its lo rows,
  // so the pair MMA's N is [hi | lo] and each CTA stages as many bytes as
  // without split precision)
  const bool pair_narrow = CG == 2 && LO && !wide;
  const int wmax = (CG == 2 && !pair_narrow) ? ((min(BNX, N) + 15) & ~15) / 2 : min(BNX, N);
  const int brow_max = wmax > 192 ? 256 : wmax > 48 ? 64 : 16;
  const int b_rows = ((wmax + brow_max - 1) / brow_max) * brow_max;
  // split-precision activations (LO): the stage's activation tile is the
  // chunk's fp16 rows (hi, padded to whole boxes) followed by their fp16
  // rounding residuals (lo) -- except a narrow pair, where each CTA holds one
  const int NLO = (LO && !pair_narrow) ? 2 : 1;
  const int STAGE_BYTES = A_BYTES + ((NLO * b_rows * BK * 2 + 1023) & ~1023);
  const int STAGES = min(MAX_STAGES, RING_BYTES / STAGE_BYTES);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* xch = (float*)(smem + RING_BYTES);
  float* stg = (float*)(smem + RING_BYTES + XCH_BYTES);
  float* rsc = (float*)(smem + RING_BYTES + XCH_BYTES + STG_BYTES);
  uint64_t* bars = (uint64_t*)(smem + RING_BYTES + XCH_BYTES + STG_BYTES + RSC_BYTES);
  // bars: full[MAX_STAGES], empty[MAX_STAGES], tfull[2], tempty[2]; then tmem slot, ticket
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * MAX_STAGES + 4);
  int* ticket = (int*)(tmem_slot + 1);
  // dsm: every split CTA of the cluster arrives once when its partial is in
  // its shared memory (the ring, free after the item's last MMA)
  const uint32_t dsm_bar = smem_u32(bars + 2 * MAX_STAGES + 5);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + MAX_STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * MAX_STAGES), tempty0 = smem_u32(bars + 2 * MAX_STAGES + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(full0 + 8 * i, 1); mbar_init(empty0 + 8 * i, 1); }
    // tempty: 128 epilogue threads (single CTA) or one elected arrival per CTA (pair, leader's barrier)
    for (int i = 0; i < 2; ++i) { mbar_init(tfull0 + 8 * i, 1); mbar_init(tempty0 + 8 * i, CG == 2 ? 2 : 128); }
    if (a.dsm) mbar_init(dsm_bar, a.splits);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB16) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB64) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB256) : "memory");
    if (LO) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmL16) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmL64) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmL256) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2 || a.dsm) cluster_sync_all();        // the peers' barriers exist before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TL(1);
  if (!(warp == 0 && lane == 0)) pdl_wait();   // the producer waits after its weight prefetch
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      int stage = 0; uint32_t phase = 0;
      bool first = true;
      for (int it = cta_id; it < n_items; it += n_ctas) {
        Item I = decode_item(it, m_tiles, a.splits, n_chunks, LO && !wide);
        const int kb0 = (int)((long)I.split * kb_total / a.splits), kb1 = (int)((long)(I.split + 1) * kb_total / a.splits);
        const int wrow = (I.tile * CG + (int)crank) * BM;   // this CTA's 128 weight rows
        // A box coordinates of k-block kb: (kb * 64, wrow) row-major, or the
        // start row of tile (wrow / 128, kb) in the tiled layout (16 KB contiguous)
        const int kbt = a.K / BK;
#define A_C0(kb) (a.a_tiled ? 0 : (kb) * BK)
#define A_C1(kb) (a.a_tiled ? ((wrow / BM) * kbt + (kb)) * BM : wrow)
        int n0 = I.chunk * BNX, nc = min(BNX, N - n0);
        if (CG == 2 && !pair_narrow) {        // this CTA's half of the 16-padded chunk
          const int half = ((nc + 15) & ~15) / 2;
          n0 += (int)crank * half;
          nc = half;
        }
        // X boxes: one 256-row box for wide chunks, else a few 64- or 16-row boxes
        const CUtensorMap* tb = nc > 192 ? &tmB256 : nc > 48 ? &tmB64 : &tmB16;
        const CUtensorMap* tl = nc > 192 ? &tmL256 : nc > 48 ? &tmL64 : &tmL16;
        if (pair_narrow && crank == 1) tb = tl;   // CTA 1 of a narrow pair stages the lo rows
        const int brow = nc > 192 ? 256 : nc > 48 ? 64 : 16;
        const int nbox = (nc + brow - 1) / brow;
        const int lo_off = nbox * brow * BK * 2;           // LO: residual rows follow the hi rows
        // pair: the leader arms its full barrier with both CTAs' bytes; every
        // TMA of the pair completes on the leader's barrier
        const uint32_t stage_tx = (uint32_t)CG * (A_BYTES + NLO * nbox * brow * BK * 2);
        const int cnt = kb1 - kb0;
        // rotate the K order per tile so the CTAs do not all request the same
        // activation tile at the same time (an L2 hot spot).  The rotation
        // depends on the weight tile only, so a row's accumulation order is
        // the same in every 256-row chunk: results are batch invariant
        // (identical for any live count, position in the batch or DP split)
        const int rot = (I.tile * 7) % cnt;
        int j0 = 0;
        if (first) {
          // Programmatic dependent launch: the weights do not depend on the
          // previous kernel, so the first ring's worth of weight tiles is
          // requested before waiting for it; activations only after.
          first = false;
          const int npre = min(cnt, STAGES);
          for (int j = 0; j < npre; ++j) {
            const int kb = kb0 + (j + rot) % cnt;
            const uint32_t fb = full0 + 8 * j;
            if (leader) mbar_expect_tx(fb, stage_tx);
            if (CG == 2) tma_load_2d_pair(smem_u32(smem + j * STAGE_BYTES), &tmA, leader_addr(fb), A_C0(kb), A_C1(kb), pol_w);
            else tma_load_2d(smem_u32(smem + j * STAGE_BYTES), &tmA, fb, A_C0(kb), A_C1(kb), pol_w);
          }
          pdl_wait();
          for (int j = 0; j < npre; ++j) {
            const int kb = kb0 + (j + rot) % cnt;
            const uint32_t fb = full0 + 8 * j;
            const uint32_t sa = smem_u32(smem + j * STAGE_BYTES);
            for (int b = 0; b < nbox; ++b) {
              if (CG == 2) tma_load_2d_pair(sa + A_BYTES + b * brow * BK * 2, tb, leader_addr(fb), kb * BK, n0 + brow * b, pol_x);
              else tma_load_2d(sa + A_BYTES + b * brow * BK * 2, tb, fb, kb * BK, n0 + brow * b, pol_x);
              if (LO && NLO == 2) {
                if (CG == 2) tma_load_2d_pair(sa + A_BYTES + lo_off + b * brow * BK * 2, tl, leader_addr(fb), kb * BK, n0 + brow * b, pol_x);
                else tma_load_2d(sa + A_BYTES + lo_off + b * brow * BK * 2, tl, fb, kb * BK, n0 + brow * b, pol_x);
              }
            }
          }
          j0 = npre;
          stage = npre % STAGES;
          phase = npre == STAGES ? 1u : 0u;
        }
        for (int j = j0; j < cnt; ++j) {
          const int kb = kb0 + (j + rot) % cnt;
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          if (leader) mbar_expect_tx(fb, stage_tx);
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          if (CG == 2) {
            const uint32_t lb = leader_addr(fb);
            tma_load_2d_pair(sa, &tmA, lb, A_C0(kb), A_C1(kb), pol_w);
            for (int b = 0; b < nbox; ++b) {
              tma_load_2d_pair(sa + A_BYTES + b * brow * BK * 2, tb, lb, kb * BK, n0 + brow * b, pol_x);
              if (LO && NLO == 2) tma_load_2d_pair(sa + A_BYTES + lo_off + b * brow * BK * 2, tl, lb, kb * BK, n0 + brow * b, pol_x);
            }
          } else {
            tma_load_2d(sa, &tmA, fb, A_C0(kb), A_C1(kb), pol_w);
            for (int b = 0; b < nbox; ++b) {
              tma_load_2d(sa + A_BYTES + b * brow * BK * 2, tb, fb, kb * BK, n0 + brow * b, pol_x);
              if (LO) tma_load_2d(sa + A_BYTES + lo_off + b * brow * BK * 2, tl, fb, kb * BK, n0 + brow * b, pol_x);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ===== MMA issuer (single thread; the pair's leader for CG = 2) =====
      int stage = 0; uint32_t phase = 0; int local = 0;
      for (int it = cta_id; it < n_items; it += n_ctas, ++local) {
        Item I = decode_item(it, m_tiles, a.splits, n_chunks, LO && !wide);
        const int kb0 = (int)((long)I.split * kb_total / a.splits), kb1 = (int)((long)(I.split + 1) * kb_total / a.splits);
        const int nc = min(BNX, N - I.chunk * BNX);
        // narrow LO: N = the hi rows (whole boxes) + the 16-padded lo rows
        const int hi_rows = nc > 192 ? 256 : nc > 48 ? ((nc + 63) & ~63) : ((nc + 15) & ~15);
        const int nmma = pair_narrow ? 2 * hi_rows : (LO && !wide) ? hi_rows + ((nc + 15) & ~15) : (nc + 15) & ~15;
        const uint32_t idesc = make_idesc(nmma, BM * CG);
        // wide LO: one accumulator pair (all 512 columns), phases alternate per item
        const int acc = wide ? 0 : (local & 1);
        const uint32_t acc_phase = wide ? (local & 1) : ((local >> 1) & 1);
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        if (!wide) {
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full0 + 8 * stage, phase);
            if (kb == kb0 && local < 3) TL(2 + 2 * local);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint64_t da = make_sdesc(sa), db = make_sdesc(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {  // +32 B along K per UMMA_K=16 step
              if (CG == 2) umma_f16_pair(tmem_d, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              else umma_f16(tmem_d, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            if (CG == 2) umma_commit_pair(empty0 + 8 * stage);
            else umma_commit(empty0 + 8 * stage);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        } else {
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full0 + 8 * stage, phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            // the lo rows follow this CTA's hi rows (the pair: each CTA's half)
            const int cta_rows = CG == 2 ? ((((nc + 15) & ~15) / 2 > 48) ? ((((nc + 15) & ~15) / 2 + 63) & ~63)
                                                                          : ((((nc + 15) & ~15) / 2 + 15) & ~15))
                                         : hi_rows;
            const uint64_t da = make_sdesc(sa), db = make_sdesc(sa + A_BYTES),
                           dl = make_sdesc(sa + A_BYTES + cta_rows * BK * 2);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
              if (CG == 2) {
                umma_f16_pair(tmem_d, da + 2 * k, db + 2 * k, idesc, accum);
                umma_f16_pair(tmem_d + BN, da + 2 * k, dl + 2 * k, idesc, accum);
              } else {
                umma_f16(tmem_d, da + 2 * k, db + 2 * k, idesc, accum);          // W . x_hi
                umma_f16(tmem_d + BN, da + 2 * k, dl + 2 * k, idesc, accum);     // W . x_lo
              }
            }
            if (CG == 2) umma_commit_pair(empty0 + 8 * stage);
            else umma_commit(empty0 + 8 * stage);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
        if (CG == 2) umma_commit_pair(tfull0 + 8 * acc);
        else umma_commit(tfull0 + 8 * acc);
        if (local < 3) TL(3 + 2 * local);
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue warpgroup =====
    const int q = warp - 4;                 // TMEM lane quarter
    const int et = threadIdx.x - 128;       // 0..127
    int local = 0;
    int rsc_chunk = -1;                     // chunk whose RMSNorm scales are in rsc
    for (int it = cta_id; it < n_items; it += n_ctas, ++local) {
      Item I = decode_item(it, m_tiles, a.splits, n_chunks, LO && !wide);
      if (CG == 2) I.tile = I.tile * 2 + (int)crank;   // this CTA's 128-row tile (the pair has no split-K)
      const int n0 = I.chunk * BNX, nc = min(BNX, N - n0);
      // LO: the lo columns start after the hi rows (narrow) or at column 256 (wide)
      const int hi_rows = wide ? BN : nc > 48 ? ((nc + 63) & ~63) : ((nc + 15) & ~15);
      const int acc = wide ? 0 : (local & 1);
      const uint32_t acc_phase = wide ? (local & 1) : ((local >> 1) & 1);
      if (a.ssq_in && I.chunk != rsc_chunk) {
        // folded RMSNorm: column scales of this chunk (once per chunk; every
        // decode item shares chunk 0), computed while the item's MMAs run.
        // Parts are loaded 8 at a time and summed in part order (deterministic).
        rsc_chunk = I.chunk;
        named_bar(3, 128);
        for (int cc = et; cc < nc; cc += 128) {
          const float* sp = a.ssq_in + (size_t)(n0 + cc) * a.ssq_stride;
          float ss = 0.f;
          int p = 0;
          for (; p + 8 <= a.ssq_parts; p += 8) {
            float t[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) t[k] = __ldcg(sp + p + k);
#pragma unroll
            for (int k = 0; k < 8; ++k) ss += t[k];
          }
          for (; p < a.ssq_parts; ++p) ss += __ldcg(sp + p);
          rsc[cc] = 1.0f / sqrtf(ss * a.norm_inv_d + a.norm_eps);
        }
        named_bar(3, 128);
      }
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      const int row = 32 * q + lane;        // row within the tile
      const int m = I.tile * BM + row;
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(32 * q) << 16);
      const bool split = a.splits > 1;
      if (split) {
        // fp32 partials: part[((tile*n_chunks+chunk)*splits+split)][col][row],
        // staged through shared memory so every thread writes float4s
        float* part = a.dsm ? (float*)smem
                            : a.partial + ((size_t)((I.chunk * m_tiles + I.tile) * a.splits + I.split)) * BN * BM;
        for (int c0 = 0; c0 < nc; c0 += 32) {
          uint32_t r[32];
          TMEM_LD32(tbase + c0, r);
          if (LO) {                            // + W . x_lo (the residual columns)
            uint32_t rl[32];
            TMEM_LD32(tbase + hi_rows + c0, rl);
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(rl[j]));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[j * TS + row] = __uint_as_float(r[j]);
          named_bar(2, 128);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int idx = et + 128 * i, n = idx >> 5, m4 = (idx & 31) * 4;
            if (c0 + n < nc) {
              if (a.dsm) *(float4*)(part + (size_t)(c0 + n) * BM + m4) = *(const float4*)(stg + n * TS + m4);
              else __stcg((float4*)(part + (size_t)(c0 + n) * BM + m4), *(const float4*)(stg + n * TS + m4));
            }
          }
          named_bar(2, 128);
        }
      }
      bool last = true;
      int col_lo = 0, col_hi = nc;
      if (split && et == 0 && local == 0) TL(11);   // partials written
      if (split && a.epi == EPI_PARTIAL) {
        // the consumer kernel reduces the splits (decode attention sums the
        // QKV partials of its rows): no ticket, no wait, no epilogue here
        tc_fence_before();
        mbar_arrive(tempty0 + 8 * acc);
        continue;
      }
      if (split) {
        tc_fence_before();
        mbar_arrive(tempty0 + 8 * acc);     // TMEM stage free for the next item
        int* ctr = a.counters + I.chunk * m_tiles + I.tile;
        if (a.dsm) {
          // cluster exchange: release this CTA's partial to the cluster, one
          // arrival on every split CTA's barrier, wait for all splits; then
          // each CTA reduces its 1/splits of the columns from their shared
          // memory (split order: the same sums as the global paths)
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          named_bar(1, 128);
          if (et == 0)
            for (int r = 0; r < a.splits; ++r) mbar_arrive_remote(dsm_peer_u32(dsm_bar, (uint32_t)r));
          mbar_wait_cluster(dsm_bar, 0);
          const int per = ((nc + a.splits - 1) / a.splits + 3) & ~3;
          col_lo = min(nc, I.split * per);
          col_hi = min(nc, col_lo + per);
        } else if (coop) {
          __threadfence();
          named_bar(1, 128);
          // One wave (every CTA of the grid is resident, so waiting on the
          // other splits cannot deadlock): all split CTAs of the tile wait for
          // its partials, then each reduces its own 1/splits of the columns
          // (in split order: deterministic).  The last to finish resets.
          if (et == 0) {
            atomicAdd(ctr, 1);
            uint32_t spins = 0;
            while (atomicAdd(ctr, 0) < a.splits) {
              __nanosleep(64);
              if (++spins == (1u << 24)) {
                printf("rollpacker watchdog: split-K wait stuck (block %d)\n", blockIdx.x);
                __trap();
              }
            }
          }
          named_bar(1, 128);
          __threadfence();
          const int per = ((nc + a.splits - 1) / a.splits + 3) & ~3;
          col_lo = min(nc, I.split * per);
          col_hi = min(nc, col_lo + per);
        } else if (n_items <= (int)gridDim.x && !a.no_spin) {
          // One wave: split S-1 is the tile's designated reducer.  The other
          // splits publish their partials with a fire-and-forget release add
          // and leave at once (their SM goes to the next kernel's prefetch);
          // the reducer acquires the count, resets it and reduces in split
          // order (the same sums as the ticket path, bit for bit).
          named_bar(1, 128);
          if (I.split != a.splits - 1) {
            if (et == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
            last = false;
          } else {
            if (et == 0) {
              uint32_t spins = 0;
              int v;
              do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (++spins == (1u << 26)) {
                  printf("rollpacker watchdog: split-K reducer stuck (block %d)\n", blockIdx.x);
                  __trap();
                }
              } while (v < a.splits - 1);
              *ctr = 0;
            }
            named_bar(1, 128);
            last = true;
          }
        } else {
          __threadfence();
          named_bar(1, 128);
          if (et == 0) {
            int old = atomicAdd(ctr, 1);
            *ticket = (old == a.splits - 1);
            if (old == a.splits - 1) *ctr = 0;
          }
          named_bar(1, 128);
          last = *ticket != 0;
          __threadfence();
        }
        if (et == 0 && local == 0) TL(12);        // ticket taken
      }
      if (!last) continue;
      if (split && a.epi != EPI_SWIGLU) {
        // ---- in-order split-K reduction by the last CTA of the tile.  Threads
        // are remapped to 4 consecutive rows (float4) x columns so every load
        // is 16 B and 8 independent loads per split are in flight per thread;
        // the fixed split order keeps the sum deterministic.
        const float* __restrict__ pb = a.partial + ((size_t)((I.chunk * m_tiles + I.tile) * a.splits)) * BN * BM;
        const int r4 = (et & 31) * 4;              // rows r4..r4+3 of the tile
        const int m4 = I.tile * BM + r4;
        for (int cb = col_lo + (et >> 5); cb < col_hi; cb += 4 * RU) {
          float4 acc[RU];
          // every split's partials requested at once (one L2 round trip),
          // summed in split order (deterministic, bit-identical to a loop)
          if (a.dsm) {
            const float* pp[8];
#pragma unroll
            for (int sp = 0; sp < 8; ++sp) pp[sp] = dsm_peer((const float*)smem, (uint32_t)min(sp, a.splits - 1));
            switch (a.splits) {
              case 2: reduce_splits_dsm<2>(acc, pp, cb, col_hi, r4); break;
              case 3: reduce_splits_dsm<3>(acc, pp, cb, col_hi, r4); break;
              case 4: reduce_splits_dsm<4>(acc, pp, cb, col_hi, r4); break;
              case 5: reduce_splits_dsm<5>(acc, pp, cb, col_hi, r4); break;
              case 6: reduce_splits_dsm<6>(acc, pp, cb, col_hi, r4); break;
              case 7: reduce_splits_dsm<7>(acc, pp, cb, col_hi, r4); break;
              default: reduce_splits_dsm<8>(acc, pp, cb, col_hi, r4); break;
            }
          } else switch (a.splits) {
            case 2: reduce_splits<2>(acc, pb, cb, col_hi, r4); break;
            case 3: reduce_splits<3>(acc, pb, cb, col_hi, r4); break;
            case 4: reduce_splits<4>(acc, pb, cb, col_hi, r4); break;
            case 5: reduce_splits<5>(acc, pb, cb, col_hi, r4); break;
            case 6: reduce_splits<6>(acc, pb, cb, col_hi, r4); break;
            default: reduce_splits_loop(acc, pb, cb, col_hi, r4, a.splits); break;
          }
          if (a.timeline && et == 0 && local == 0 && cb == col_lo) {   // debug: the partials have arrived
            asm volatile("" ::"f"(acc[0].x), "f"(acc[RU - 1].w));
            TL(14);
          }
          if (a.ssq_in) {
#pragma unroll
            for (int u = 0; u < RU; ++u) {
              const int col = cb + 4 * u;
              const float sc = col < col_hi ? rsc[col] : 0.f;
              acc[u].x *= sc; acc[u].y *= sc; acc[u].z *= sc; acc[u].w *= sc;
            }
          }
          if (a.epi == EPI_QKV_ROPE) {
            // rows r4..r4+3 of head-dim index i0 = (m4 % hd); the rotate-half
            // partner rows (i +- hd/2) live in lane ^ (hd/8) of this warp
            const RopeArgs& R = a.rope;
            const int hd = R.hd, half = hd >> 1;
            const int head = m4 / hd, i0 = m4 % hd;
            const bool is_q = head < R.H, is_v = head >= R.H + R.KV;
            const bool lo = i0 < half;
            const float4 bb = a.bias ? *(const float4*)(a.bias + m4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < RU; ++u) {
              float4 v = acc[u];
              v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
              float4 p;
              p.x = __shfl_xor_sync(0xffffffffu, v.x, hd >> 3);
              p.y = __shfl_xor_sync(0xffffffffu, v.y, hd >> 3);
              p.z = __shfl_xor_sync(0xffffffffu, v.z, hd >> 3);
              p.w = __shfl_xor_sync(0xffffffffu, v.w, hd >> 3);
              const int col = cb + 4 * u;
              if (col >= col_hi) continue;
              const int n = n0 + col;
              const int pos = R.row_pos[n];
              float4 o = v;
              if (!is_v) {
                const float2* cs = R.cs + (size_t)pos * half + (lo ? i0 : i0 - half);
                const float4 c01 = *(const float4*)cs, c23 = *(const float4*)(cs + 2);   // (c,s) x 4
                const float sg = lo ? -1.f : 1.f;    // lo: x c - x' s ; hi: x c + x' s
                o.x = v.x * c01.x + sg * p.x * c01.y;
                o.y = v.y * c01.z + sg * p.y * c01.w;
                o.z = v.z * c23.x + sg * p.z * c23.y;
                o.w = v.w * c23.z + sg * p.w * c23.w;
              }
              act2_t o01 = to_act2(o.x, o.y), o23 = to_act2(o.z, o.w);
              uint2 packed;
              packed.x = *(uint32_t*)&o01;
              packed.y = *(uint32_t*)&o23;
              act_t* dst;
              if (is_q) {
                dst = R.q_out + ((size_t)n * R.H + head) * hd + i0;
                if (R.q_lo) {                  // q's rounding residual (split precision)
                  const float2 f01 = __half22float2(o01), f23 = __half22float2(o23);
                  act2_t l01 = to_act2(o.x - f01.x, o.y - f01.y), l23 = to_act2(o.z - f23.x, o.w - f23.y);
                  uint2 pl;
                  pl.x = *(uint32_t*)&l01;
                  pl.y = *(uint32_t*)&l23;
                  *(uint2*)(R.q_lo + ((size_t)n * R.H + head) * hd + i0) = pl;
                }
              } else {
                const int kh = is_v ? head - R.H - R.KV : head - R.H;
                const int page = R.page_table[(size_t)R.row_pt[n] * R.maxp + pos / kPage];
                dst = (act_t*)R.kv_pool + kv_block_elems(R.layer, page, kh, is_v ? 1 : 0, R.n_pages, R.KV, hd) +
                      (size_t)(pos % kPage) * hd + i0;
              }
              *(uint2*)dst = packed;
            }
            continue;
          }
          float4 old[RU];
          if (a.epi == EPI_RESID) {
#pragma unroll
            for (int u = 0; u < RU; ++u) {
              const int col = cb + 4 * u;
              if (col < col_hi) old[u] = *(const float4*)((float*)a.out + (size_t)(n0 + col) * a.ldo + m4);
            }
          }
          float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
          if (a.bias) bb = *(const float4*)(a.bias + m4);
#pragma unroll
          for (int u = 0; u < RU; ++u) {
            const int col = cb + 4 * u;
            if (col >= col_hi) continue;
            const size_t o = (size_t)(n0 + col) * a.ldo + m4;
            float4 v = acc[u];
            if (a.epi == EPI_RESID) {
              v.x += old[u].x; v.y += old[u].y; v.z += old[u].z; v.w += old[u].w;
              *(float4*)((float*)a.out + o) = v;
              if (a.ssq_out) {
                // fp16(x) for the next GEMM and this tile's sum of squares of
                // column n (the warp covers the tile's 128 rows: lanes x 4)
                const size_t xo = (size_t)(n0 + col) * a.ldxb + m4;
                store_act4(a.xb_out + xo, a.xb_lo ? a.xb_lo + xo : nullptr, v);
                float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
                if (lane == 0) a.ssq_out[(size_t)(n0 + col) * a.ssq_stride + I.tile] = ss;
              }
            } else if (a.epi == EPI_F32) {
              v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
              if (a.push_n) {
                for (int q = 0; q < a.push_n; ++q) *(float4*)(a.push_dst[q] + o) = v;
              } else {
                *(float4*)((float*)a.out + o) = v;
              }
            } else {
              act2_t* ob = (act2_t*)((act_t*)a.out + o);
              ob[0] = to_act2(v.x + bb.x, v.y + bb.y);
              ob[1] = to_act2(v.z + bb.z, v.w + bb.w);
            }
          }
        }
        if (et == 0 && local == 0) TL(13);        // reduction + epilogue done
        push_signal(a, et);
        if (coop) {
          // second counter: the last split CTA of the tile to finish resets both
          __threadfence();
          named_bar(1, 128);
          if (et == 0) {
            int* ctr = a.counters + I.chunk * m_tiles + I.tile;
            int* done = a.counters + 32768 + I.chunk * m_tiles + I.tile;
            if (atomicAdd(done, 1) == a.splits - 1) { *done = 0; atomicExch(ctr, 0); }
          }
        }
        continue;
      }
      // ---- epilogue proper over columns of this chunk.  All global loads of
      // a 32-column chunk are issued before any store (memory-level
      // parallelism; the compiler cannot hoist loads across stores to `out`).
      const float bias = a.bias ? a.bias[m] : 0.f;
      const float* __restrict__ part0 =
          a.partial + ((size_t)((I.chunk * m_tiles + I.tile) * a.splits)) * BN * BM;
      for (int c0 = 0; c0 < nc; c0 += 32) {
        float v[32];
        if (split) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
          for (int s = 0; s < a.splits; ++s) {
            const float* __restrict__ p = part0 + (size_t)s * BN * BM + (size_t)c0 * BM + row;
            float u[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) u[j] = (c0 + j < nc) ? __ldcg(p + j * BM) : 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += u[j];
          }
        } else {
          uint32_t r[32];
          TMEM_LD32(tbase + c0, r);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (LO) {                            // + W . x_lo (the residual columns)
            TMEM_LD32(tbase + hi_rows + c0, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r[j]);
          }
        }
        if (a.ssq_in) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= (c0 + j < nc) ? rsc[c0 + j] : 0.f;
        }
        // Output goes through a shared-memory transpose so each thread writes
        // 16-byte vectors of consecutive features (a row-owning thread would
        // otherwise issue 32 scalar stores per chunk).
        if (a.epi == EPI_SWIGLU) {
          // rows 64..127 (quarters 2,3) hold `up`, rows 0..63 hold `gate`
          act_t* st2 = (act_t*)stg;                   // [32 columns][72] fp16
          act_t* st2l = st2 + 32 * 72;                // its rounding residuals (split precision)
          named_bar(2, 128);
          if (q >= 2) {
#pragma unroll
            for (int j = 0; j < 32; ++j) xch[(row - 64) * 33 + j] = v[j];
          }
          named_bar(2, 128);
          if (q < 2) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float f = silu_f(v[j]) * xch[row * 33 + j];
              const act_t h = to_act(f);
              st2[j * 72 + row] = h;
              if (a.out_lo) st2l[j * 72 + row] = to_act(f - __half2float(h));
            }
          }
          named_bar(2, 128);
          const int f0 = I.tile * 64;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int idx = et + 128 * i, n = idx >> 3, f8 = (idx & 7) * 8;
            if (c0 + n < nc) {
              const size_t oo = (size_t)(n0 + c0 + n) * a.ldo + f0 + f8;
              *(uint4*)((act_t*)a.out + oo) = *(const uint4*)(st2 + n * 72 + f8);
              if (a.out_lo) *(uint4*)(a.out_lo + oo) = *(const uint4*)(st2l + n * 72 + f8);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[j * TS + row] = v[j] + bias;
          named_bar(2, 128);
          const int mt0 = I.tile * BM;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int idx = et + 128 * i, n = idx >> 5, m4 = (idx & 31) * 4;
            if (c0 + n >= nc) continue;
            float4 val = *(const float4*)(stg + n * TS + m4);
            const size_t o = (size_t)(n0 + c0 + n) * a.ldo + mt0 + m4;
            if (a.epi == EPI_RESID) {
              const float4 old = *(const float4*)((float*)a.out + o);
              val.x += old.x; val.y += old.y; val.z += old.z; val.w += old.w;
              *(float4*)((float*)a.out + o) = val;
              if (a.ssq_out) {   // warp = one column n, lanes = the tile's 128 rows x 4
                const size_t xo = (size_t)(n0 + c0 + n) * a.ldxb + mt0 + m4;
                store_act4(a.xb_out + xo, a.xb_lo ? a.xb_lo + xo : nullptr, val);
                float ss = val.x * val.x + val.y * val.y + val.z * val.z + val.w * val.w;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
                if (lane == 0) a.ssq_out[(size_t)(n0 + c0 + n) * a.ssq_stride + I.tile] = ss;
              }
            } else if (a.epi == EPI_F32) {
              if (a.push_n) {
                for (int q = 0; q < a.push_n; ++q) *(float4*)(a.push_dst[q] + o) = val;
              } else {
                *(float4*)((float*)a.out + o) = val;
              }
            } else {
              act2_t* ob = (act2_t*)((act_t*)a.out + o);
              ob[0] = to_act2(val.x, val.y);
              ob[1] = to_act2(val.z, val.w);
            }
          }
        }
        named_bar(2, 128);                   // staging reused by the next chunk
      }
      if (!split) {
        tc_fence_before();
        if (CG == 2) {                       // one arrival per CTA on the leader's barrier
          named_bar(1, 128);
          if (et == 0) mbar_arrive_remote(leader_addr(tempty0 + 8 * acc));
        } else {
          mbar_arrive(tempty0 + 8 * acc);   // all TMEM reads of this item done
        }
      }
      push_signal(a, et);
      if (et == 0 && local < 3) TL(8 + local);
    }
  }
  tc_fence_before();
  __syncthreads();
  // pair: the leader's MMAs into this CTA's TMEM are done; dsm: no CTA leaves
  // while a peer may still read its partial
  if (CG == 2 || a.dsm) cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

int make_tmap_act(CUtensorMap* map, const void* base, int rows, int cols, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int gemm_smem_bytes() { return GEMM_SMEM; }

// Split-K through distributed shared memory (RP_GEMM_DSM=1):
// the splits of a tile run as one thread-block cluster, so the whole grid
// must be resident at once -- g_cluster_cap[s] = CTAs of cluster size s the
// device holds concurrently (cudaOccupancyMaxActiveClusters; 4-CTA clusters
// strand SMs of the 16/18/20-SM GPCs), which bounds the split count.
static int g_cluster_cap[9] = {0};
// Off by default: parity-green, but the capacity-bounded split counts (qkv 3,
// o 4, down 4 instead of 4 / 5 / 5) cost more than the exchange saves
// (7B decode step 4.17 vs 4.04 ms at 16 rows, 10.60 vs 10.41 at 256,
// profiles/r02_gemm_dsm_ab.txt).
bool gemm_dsm_enabled() {
  static const bool v = getenv("RP_GEMM_DSM") && atoi(getenv("RP_GEMM_DSM")) != 0;
  return v;
}
int gemm_cluster_cap(int s) { return s >= 2 && s <= 8 ? g_cluster_cap[s] : 0; }

int gemm_init_attrs() {
  const bool ok =
      cudaFuncSetAttribute(gemm_tcgen05_kernel<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM) ==
          cudaSuccess &&
      cudaFuncSetAttribute(gemm_tcgen05_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM) ==
          cudaSuccess &&
      cudaFuncSetAttribute(gemm_tcgen05_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM) ==
          cudaSuccess &&
      cudaFuncSetAttribute(gemm_tcgen05_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM) ==
          cudaSuccess;
  if (ok && !g_cluster_cap[2]) {
    for (int cs = 2; cs <= 8; ++cs) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(GEMM_THREADS);
      cfg.dynamicSmemBytes = GEMM_SMEM;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, gemm_tcgen05_kernel<1, 1>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      g_cluster_cap[cs] = n * cs;
    }
  }
  return ok ? 0 : -1;
}

static int pick_splits(int M, int K, int n_sms, bool dsm);
int gemm_pick_splits(int M, int K, int n_sms) { return pick_splits(M, K, n_sms, gemm_dsm_enabled()); }
// the split count of a GEMM reduced through DSMEM (bounded by the resident
// cluster capacity; the plain rule until gemm_init_attrs measured it)
int gemm_pick_splits_dsm(int M, int K, int n_sms) { return pick_splits(M, K, n_sms, true); }

static int pick_splits(int M, int K, int n_sms, bool dsm) {
  // Fill the SMs for a single 256-column chunk: minimise the critical path
  // ceil(items / n_sms) * ceil(kb / splits) (+ a small per-split cost).
  const int tiles = M / BM, kb = K / BK;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 16 && s <= kb; ++s) {
    const int items = tiles * s;
    // split-K only within one wave: a multi-wave split (ticket reduction,
    // partial traffic, uneven waves) measured slower than no split, e.g.
    // 13824 x 5120 at N=136: 4 splits 58.6 us vs none 45.0 us
    if (s > 1 && items > n_sms) break;
    // with DSMEM split-K (once the cluster capacities are known) every split
    // count must fit its cluster size's resident capacity
    if (s > 1 && dsm && g_cluster_cap[2] && (s > 8 || items > g_cluster_cap[s])) continue;
    const double waves = (double)((items + n_sms - 1) / n_sms);
    const double cost = waves * ((kb + s - 1) / s + 4) + (s > 1 ? 2.0 : 0.0);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = s; }
  }
  return best;
}

// Cooperative split-K from 16-wide chunks up: on the 7B decode step 9-11%
// faster at 56-100 live rows than the earlier 96, 5.5% at 40-48 rows, 3% at
// 32 rows, 2% at 20-24 rows, neutral at 128 and at 12-16; never cooperative
// is 16% slower at ~114 rows; 8 is 1% slower at 12 rows
// (profiles/r01_coop_min_ab.txt).
int gemm_coop_min() {
  static const int v = getenv("RP_COOP_MIN") ? atoi(getenv("RP_COOP_MIN")) : 16;
  return v;
}

// With RP_GEMM_PAIR=1, unsplit GEMMs whose weight rows pair up run as CTA
// pairs (clusters of 2, one per TPC).  Off by default: parity-green, but on
// the 7B decode step it is ~1% faster above 128 live rows and 2.5-6% slower
// at 16-64 rows, where the rollout spends most steps
// (profiles/r01_gemm_chain_experiment.txt).
void gemm_launch(const GemmPlan& p, const GemmArgs& a0, int grid, cudaStream_t st) {
  static const bool pair = getenv("RP_GEMM_PAIR") != nullptr;
  GemmArgs a = a0;
  a.a_tiled = p.a_tiled;
  a.lo = a0.lo && p.has_lo;
  // DSMEM split-K: one item per CTA (the caller guarantees one chunk: <= 256
  // rows), the tile's splits one cluster, the grid resident at once
  const int dsm_items = (a.M / BM) * a.splits;
  const bool dsm = a.dsm && a.splits >= 2 && a.splits <= 8 && a.epi != EPI_SWIGLU && a.epi != EPI_PARTIAL &&
                   !a.timeline && dsm_items <= gemm_cluster_cap(a.splits);
  a.dsm = 0;
  // no_spin (single-GPU local groups): every split-K tile is reduced by its
  // last CTA (ticket), never by CTAs waiting for each other, because other
  // contexts' kernels may hold the SMs the waited-for splits need
  a.coop_min = a0.no_spin ? 0x7FFFFFFF : gemm_coop_min();
  // CTA pairs: with RP_GEMM_PAIR=1, and always for split-precision GEMMs
  // without split-K (gate/up: the pair stages the hi and the lo rows in
  // different CTAs, so the ring keeps the depth of the plain GEMM)
  if ((pair || a.lo) && a.splits == 1 && a.M % (2 * BM) == 0 && !a.timeline && grid % 2 == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_no_pdl ? 1 : 2;
    cudaLaunchKernelEx(&cfg, a.lo ? gemm_tcgen05_kernel<2, 1> : gemm_tcgen05_kernel<2, 0>, p.tmA, p.tmB16, p.tmB64,
                       p.tmB256, p.tmL16, p.tmL64, p.tmL256, a);
    return;
  }
  if (dsm) {
    a.dsm = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(dsm_items);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.splits; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_no_pdl ? 1 : 2;
    cudaLaunchKernelEx(&cfg, a.lo ? gemm_tcgen05_kernel<1, 1> : gemm_tcgen05_kernel<1, 0>, p.tmA, p.tmB16, p.tmB64,
                       p.tmB256, p.tmL16, p.tmL64, p.tmL256, a);
    return;
  }
  launch_pdl(a.lo ? gemm_tcgen05_kernel<1, 1> : gemm_tcgen05_kernel<1, 0>, dim3(grid), dim3(GEMM_THREADS), GEMM_SMEM,
             st, p.tmA, p.tmB16, p.tmB64, p.tmB256, p.tmL16, p.tmL64, p.tmL256, a);
}

int make_plan(GemmPlan* p, const void* W, int M, int K, const void* X, int rows_cap, int w_tiled, const void* X_lo) {
  p->a_tiled = w_tiled;
  // tiled: the weights are M*K/64 rows of 64 elements, 128 consecutive rows per tile
  if (w_tiled ? make_tmap_act(&p->tmA, W, (int)((long long)M * K / BK), BK, 128) : make_tmap_act(&p->tmA, W, M, K, 128))
    return -1;
  if (make_tmap_act(&p->tmB16, X, rows_cap, K, 16)) return -1;
  if (make_tmap_act(&p->tmB64, X, rows_cap, K, 64)) return -1;
  if (make_tmap_act(&p->tmB256, X, rows_cap, K, 256)) return -1;
  // the split-precision residual of the activations (same layout), or X again when absent
  p->has_lo = X_lo != nullptr;
  const void* L = X_lo ? X_lo : X;
  if (make_tmap_act(&p->tmL16, L, rows_cap, K, 16)) return -1;
  if (make_tmap_act(&p->tmL64, L, rows_cap, K, 64)) return -1;
  if (make_tmap_act(&p->tmL256, L, rows_cap, K, 256)) return -1;
  return 0;
}

}  // namespace rp
