// Host interface of the tcgen05 GEMM (gemm_tcgen05.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace rp {

// EPI_PARTIAL (split-K only): write the fp32 split partials and stop -- the
// decode QKV GEMM, whose splits the attention kernel sums (k_attn.cu QkvFuse).
enum GemmEpi { EPI_F32 = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_ACT = 3, EPI_QKV_ROPE = 4, EPI_PARTIAL = 5 };

// Fused QKV epilogue (decode, split-K path): bias, rotate-half RoPE from a
// per-position cos/sin table, q -> q_out fp16 [n][H][hd], k/v -> KV page
// (fp16, reading Z20).
struct RopeArgs {
  __half* q_out;
  __half* q_lo;           // fp16 residual of q (split precision), or nullptr
  uint8_t* kv_pool;
  const int* page_table;
  const int* row_pos;
  const int* row_pt;
  const float2* cs;       // [pos][hd/2] (cos, sin)
  size_t page_bytes;
  int maxp, layer, H, KV, hd;
  int n_pages;            // KV pool pages (layout: kv_block_elems)
};

struct GemmArgs {
  int M, K;               // weight rows (multiple of 128), reduction dim (multiple of 64)
  const int* n_dev;       // live N read on device (nullptr -> n_host)
  int n_host;
  int splits;             // split-K factor (1 = direct epilogue)
  int coop_min;           // cooperative split-K reduction from this chunk width up (set by gemm_launch)
  int no_spin;            // 1: no inter-CTA waits (ticket reduction only; single-GPU local groups)
  int dsm;                // 1: the splits of a tile form a thread-block cluster and reduce through
                          // distributed shared memory (one item per CTA; set by gemm_launch)
  int a_tiled;            // weights stored in 128 x 64 tiles (set by gemm_launch from the plan)
  // Split-precision activations (reading Z22): D = W . x_hi + W . x_lo with
  // x_lo = fp16(x - x_hi), two MMAs per K step, fp32 accumulation -- the
  // activation operand carries ~22 significant bits.  The weights are exact
  // fp16 (the bf16 formula values), so only the activation rounding matters.
  int lo;
  __half* xb_lo;          // FOLD producer: fp16 residual of x next to xb_out
  __half* out_lo;         // SWIGLU: fp16 residual of the output next to `out`
  int epi;                // GemmEpi
  void* out;              // out[n * ldo + m] (SWIGLU: out[n * ldo + feature])
  int ldo;
  const float* bias;      // [M] or nullptr (EPI_F32 / EPI_ACT)
  float* partial;         // split-K partials (splits > 1)
  int* counters;          // split-K tickets, zero-initialised, self-resetting
  long long* timeline;    // debug: per-CTA %globaltimer stamps [grid][16] (nullptr = off)
  RopeArgs rope;          // EPI_QKV_ROPE only
  // Folded RMSNorm (the gains are folded into the consuming weights at init):
  // a RESID producer also writes
  // fp16(x) to xb_out[n * ldxb + m] and the sum of squares of its 128-feature
  // tile to ssq_out[n * ssq_stride + tile]; a consumer (ssq_in != nullptr)
  // multiplies output column n by rsqrt(sum_p ssq_in[n * ssq_stride + p] *
  // norm_inv_d + norm_eps), p < ssq_parts, before bias / SwiGLU / RoPE.
  __half* xb_out;
  int ldxb;
  float* ssq_out;
  const float* ssq_in;
  int ssq_parts, ssq_stride;
  float norm_inv_d, norm_eps;
  // Tensor-parallel push (decode, row-parallel O/down): an F32 output tile is
  // written to push_dst[q] (rank q's receive slot for this rank, row stride
  // ldo; q = 0..push_n-1, local or NVLink peer memory) instead of `out`, then
  // each finished output unit adds 1 to push_flag[q] (system-scope release).
  float* push_dst[8];
  unsigned long long* push_flag[8];
  int push_n;
};

struct GemmPlan {
  CUtensorMap tmA;        // weights [M, K] fp16, box 64 x 128; tiled: [M*K/64, 64] (128 x 64 tiles, each contiguous)
  int a_tiled;
  CUtensorMap tmB16, tmB64, tmB256;   // activations [rows_cap, K], boxes of 16 / 64 / 256 rows
  CUtensorMap tmL16, tmL64, tmL256;   // their fp16 rounding residuals (split precision), same boxes
  int has_lo;
};

int make_tmap_act(CUtensorMap* map, const void* base, int rows, int cols, int box_rows);
int gemm_init_attrs();
// chunk width from which a one-wave split-K GEMM reduces cooperatively (RP_COOP_MIN overrides;
// tp_norm must use the same value to count the producer's signals)
int gemm_coop_min();
int gemm_smem_bytes();
int gemm_pick_splits(int M, int K, int n_sms);
bool gemm_dsm_enabled();        // DSMEM split-K reduction (RP_GEMM_DSM=1; off by default)
int gemm_cluster_cap(int s);    // CTAs of cluster size s resident at once (0 before gemm_init_attrs)
int gemm_pick_splits_dsm(int M, int K, int n_sms);
void gemm_launch(const GemmPlan& p, const GemmArgs& a, int grid, cudaStream_t st);
int make_plan(GemmPlan* p, const void* W, int M, int K, const void* X, int rows_cap, int w_tiled,
              const void* X_lo = nullptr);

}  // namespace rp
