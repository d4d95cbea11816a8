// Device-memory collectives of a single-GPU local group (SURVEY.md §4 item 4:
// several logical ranks in one process on one device, exchanging through
// device memory instead of NCCL).  They carry exactly the messages the NCCL
// path carries -- the per-step cutoff counts of the DP exchange (a11), the
// round membership (a13), the TP all-reduces of prefill partials and of the
// packed argmax (a7, a9) -- so the multi-rank logic runs under `pytest -m gpu`
// on one GPU.  Not a performance path.
//
// Protocol per (group, collective call), every member in the same order:
//   publish: e = state[0] + 1; copy my bytes to slots[e & 1][me]; the last
//            CTA releases gen[me] = e and stores state[0] = e;
//   reduce:  e = state[0]; acquire gen[q] >= e for every member q; combine
//            slots[e & 1][q] in rank order (bit-identical on every member).
// A member overwrites parity (e & 1) at epoch e + 2 only after its reduce of
// e + 1, which needed every member's publish of e + 1, which each member
// issued after finishing its reduce of e: the slots are never reused early.
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace rp {

thread_local bool g_no_pdl = false;

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void local_publish_kernel(const int4* __restrict__ src, size_t n16, uint8_t* slots, size_t slot_bytes,
                                     int size, int me, unsigned long long* gen, int* state) {
  const int e = state[0] + 1;
  int4* dst = (int4*)(slots + ((size_t)(e & 1) * size + me) * slot_bytes);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    __stcg(dst + i, src[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(state + 1, 1) == (int)gridDim.x - 1) {
      state[1] = 0;
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(gen + me), "l"((unsigned long long)e) : "memory");
      state[0] = e;
    }
  }
}

__global__ void local_reduce_kernel(int op, void* dst, size_t bytes, const uint8_t* slots, size_t slot_bytes, int size,
                                    const unsigned long long* gen, const int* state) {
  const int e = state[0];
  if (threadIdx.x == 0) {
    for (int q = 0; q < size; ++q) {
      uint32_t spins = 0;
      while (ld_acquire_gpu_u64(gen + q) < (unsigned long long)e) {
        __nanosleep(128);
        if (++spins == (1u << 26)) {
          printf("rollpacker watchdog: local-group collective stuck (member %d, epoch %d)\n", q, e);
          __trap();
        }
      }
    }
  }
  __syncthreads();
  const uint8_t* base = slots + (size_t)(e & 1) * size * slot_bytes;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  if (op == LOP_GATHER) {
    const size_t n4 = bytes / 4;
    for (int q = 0; q < size; ++q)
      for (size_t i = tid; i < n4; i += nth)
        ((int*)dst)[(size_t)q * n4 + i] = __ldcg((const int*)(base + (size_t)q * slot_bytes) + i);
  } else if (op == LOP_SUM_F32) {
    const size_t n = bytes / 4;
    for (size_t i = tid; i < n; i += nth) {
      float s = __ldcg((const float*)base + i);
      for (int q = 1; q < size; ++q) s += __ldcg((const float*)(base + (size_t)q * slot_bytes) + i);
      ((float*)dst)[i] = s;
    }
  } else {
    const size_t n = bytes / 8;
    for (size_t i = tid; i < n; i += nth) {
      unsigned long long m = __ldcg((const unsigned long long*)base + i);
      for (int q = 1; q < size; ++q) {
        const unsigned long long v = __ldcg((const unsigned long long*)(base + (size_t)q * slot_bytes) + i);
        m = v > m ? v : m;
      }
      ((unsigned long long*)dst)[i] = m;
    }
  }
}

void launch_local_publish(const void* src, size_t bytes, uint8_t* slots, size_t slot_bytes, int size, int me,
                          unsigned long long* gen, int* state, cudaStream_t st) {
  const size_t n16 = (bytes + 15) / 16;
  const int grid = (int)std::min<size_t>(std::max<size_t>(1, (n16 + 255) / 256), 64);
  local_publish_kernel<<<grid, 256, 0, st>>>((const int4*)src, n16, slots, slot_bytes, size, me, gen, state);
}

void launch_local_reduce(int op, void* dst, size_t bytes, const uint8_t* slots, size_t slot_bytes, int size,
                         const unsigned long long* gen, const int* state, cudaStream_t st) {
  // at most 8 CTAs spin per member, so the other members' kernels find SMs
  const int grid = (int)std::min<size_t>(std::max<size_t>(1, bytes / 4 / (256 * 16)), 8);
  local_reduce_kernel<<<grid, 256, 0, st>>>(op, dst, bytes, slots, slot_bytes, size, gen, state);
}

__global__ void host_gate_kernel(const volatile int* flag) {
  uint32_t spins = 0;
  while (*flag == 0) {
    __nanosleep(1000);
    if (++spins == (1u << 24)) {
      printf("rollpacker watchdog: profiling gate never released\n");
      __trap();
    }
  }
}

void launch_host_gate(const int* flag, cudaStream_t st) { host_gate_kernel<<<1, 1, 0, st>>>(flag); }

}  // namespace rp
