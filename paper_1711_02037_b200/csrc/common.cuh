// common.cuh — shared device helpers for the rnmf-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace rnmf_gpu {

constexpr int kWarp = 32;

// Error raised by any CUDA runtime failure; mapped to RNMF_CUDA_ERROR at the C ABI.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RNMF_CUDA(expr)                                                                    \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::rnmf_gpu::CudaError(std::string("CUDA error ") + cudaGetErrorName(_e) + " (" + \
                                  cudaGetErrorString(_e) + ") at " __FILE__ ":" +          \
                                  std::to_string(__LINE__) + ": " #expr);                  \
  } while (0)

#define RNMF_CUDA_LAUNCH() RNMF_CUDA(cudaGetLastError())

// ---- warp reductions ------------------------------------------------------------------------
// Butterfly (xor) reductions: every lane ends with the bitwise-identical total, because each
// level combines the same two operands (a+b == b+a in IEEE arithmetic).
template <typename V>
__device__ __forceinline__ V warp_allreduce_sum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

// ---- memory-model helpers for cross-CTA traffic ---------------------------------------------
// Data written by other CTAs during the same launch is read with ld.global.cg (L2, never a
// possibly-stale L1 line).
template <typename V>
__device__ __forceinline__ V ld_cg(const V* p) {
  return __ldcg(p);
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier for a cooperatively launched grid.  `counter` is zeroed before the launch;
// `epoch` is a per-CTA count of barriers passed so far (identical on every CTA).  After the
// E-th barrier the counter equals E * gridDim.x.
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    // bar.sync orders the CTA's writes before this release (cumulativity); the acquire load
    // orders every later read of the CTA (after the bar.sync below) after all arrivals.
    const unsigned target = epoch * gridDim.x;
    red_release_gpu_add(counter, 1u);
    while (ld_acquire_gpu(counter) < target) {
    }
  }
  __syncthreads();
}

// ---- misc -------------------------------------------------------------------------------------
template <typename T>
struct vec2_of;
template <>
struct vec2_of<float> {
  using type = float2;
};
template <>
struct vec2_of<double> {
  using type = double2;
};

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace rnmf_gpu
