/* Oracle-side weight generator (TEST INFRASTRUCTURE ONLY, see
 * oracle/__init__.py): the formula of DESIGN.md reading Z12 written out in
 * plain C for large tensors (the 7B-shaped CPU baseline).  Shares no code
 * with the CUDA path; pinned element-for-element against oracle/weights.py
 * (itself pinned by the Random123 KATs) in tests/test_oracle_weights.py.
 * Output: float32 holding the bf16-rounded value. */
#include <stdint.h>
#include <string.h>

static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0; c[1] = (uint32_t)p1; c[2] = n2; c[3] = (uint32_t)p0;
  }
}

static float bf16_rne(float x) {
  uint32_t b; memcpy(&b, &x, 4);
  b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  float y; memcpy(&y, &b, 4);
  return y;
}

/* out[i] for i in [i0, i0 + n) of tensor `tid`. */
void oracle_weights(float* out, int64_t i0, int64_t n, uint32_t tid, uint64_t seed) {
  const float a = 0.034641016151377546f;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    const int64_t i = i0 + j;
    uint32_t c[4] = {(uint32_t)(i >> 2), tid, 0u, 0x57454947u};
    philox10(c, k0, k1);
    const uint32_t x = c[i & 3];
    volatile float u = ((float)(x >> 9) + 0.5f) * 2.384185791015625e-07f;  /* exact */
    volatile float u2 = u - 1.0f;                                           /* exact */
    volatile float w = a * u2;                                              /* one rounding */
    out[j] = bf16_rne(w);
  }
}
