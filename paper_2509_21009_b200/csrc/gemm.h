// Host interface of the tcgen05 GEMM (gemm_tcgen05.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace rp {

enum GemmEpi { EPI_F32 = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_BF16 = 3 };

struct GemmArgs {
  int M, K;               // weight rows (multiple of 128), reduction dim (multiple of 64)
  const int* n_dev;       // live N read on device (nullptr -> n_host)
  int n_host;
  int splits;             // split-K factor (1 = direct epilogue)
  int epi;                // GemmEpi
  void* out;              // out[n * ldo + m] (SWIGLU: out[n * ldo + feature])
  int ldo;
  const float* bias;      // [M] or nullptr (EPI_F32 / EPI_BF16)
  float* partial;         // split-K partials (splits > 1)
  int* counters;          // split-K tickets, zero-initialised, self-resetting
  long long* timeline;    // debug: per-CTA %globaltimer stamps [grid][16] (nullptr = off)
};

struct GemmPlan {
  CUtensorMap tmA;        // weights [M, K], box 64 x 128
  CUtensorMap tmB16, tmB64, tmB256;   // activations [rows_cap, K], boxes of 16 / 64 / 256 rows
};

int make_tmap_bf16(CUtensorMap* map, const void* base, int rows, int cols, int box_rows);
int gemm_init_attrs();
int gemm_smem_bytes();
int gemm_pick_splits(int M, int K, int n_sms);
void gemm_launch(const GemmPlan& p, const GemmArgs& a, int grid, cudaStream_t st);
int make_plan(GemmPlan* p, const void* W, int M, int K, const void* X, int rows_cap);

}  // namespace rp
