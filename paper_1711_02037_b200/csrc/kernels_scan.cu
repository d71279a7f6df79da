// kernels_scan.cu — one HBM pass over X computing everything the reference derives from X
// outside the GEMMs:
//   * first non-finite / first negative entry (check_nonnegative_finite, p/src/hals.cpp:17-34,
//     and allFinite, p/src/sketch.cpp:54)
//   * sum(X)   -> mean(X) for random_init's scale (p/src/hals.cpp:119)
//   * sum(X^2) -> ||X||_F for rel_err (p/src/rhals.cpp:131)
// The reference makes up to 7 separate passes for these; here it is one
// vectorised streaming read at HBM bandwidth.  Sums are fp64 with a fixed reduction order, so
// the result is bitwise reproducible.
#include "common.cuh"
#include "kernels.h"

namespace rnmf_gpu {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanBlocksPerSm = 4;
constexpr int kScanSms = 148;

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int n = 2;
};

template <typename T>
__device__ __forceinline__ void scan_one(T v, unsigned long long idx, double& s, double& s2,
                                         unsigned long long& bad_nf, unsigned long long& bad_neg) {
  const double d = static_cast<double>(v);
  if (!isfinite(d)) {
    bad_nf = min(bad_nf, idx);
  } else {
    if (d < 0.0) bad_neg = min(bad_neg, idx);
    s += d;
    s2 += d * d;
  }
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const T* __restrict__ x, int64_t count,
                                                            unsigned long long* bad,
                                                            double* part) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  double s = 0.0, s2 = 0.0;
  unsigned long long bad_nf = ~0ull, bad_neg = ~0ull;
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % sizeof(V)) == 0;
  int64_t vec_end = 0;
  if (aligned) {
    const int64_t nvec = count / VN;
    vec_end = nvec * VN;
    const V* xv = reinterpret_cast<const V*>(x);
    int64_t i = tid;
    // 4 independent 16-byte loads in flight per thread
    for (; i + 3 * nthreads < nvec; i += 4 * nthreads) {
      V v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + i + u * nthreads);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const T* e = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
        for (int q = 0; q < VN; ++q)
          scan_one(e[q], (unsigned long long)((i + u * nthreads) * VN + q), s, s2, bad_nf, bad_neg);
      }
    }
    for (; i < nvec; i += nthreads) {
      V v = __ldcs(xv + i);
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int q = 0; q < VN; ++q) scan_one(e[q], (unsigned long long)(i * VN + q), s, s2, bad_nf, bad_neg);
    }
  }
  for (int64_t i = vec_end + tid; i < count; i += nthreads) scan_one(x[i], (unsigned long long)i, s, s2, bad_nf, bad_neg);

  // block reduction (fixed order)
  __shared__ double red_s[kScanThreads / 32], red_s2[kScanThreads / 32];
  s = warp_allreduce_sum(s);
  s2 = warp_allreduce_sum(s2);
  if (lane_id() == 0) {
    red_s[warp_id()] = s;
    red_s2[warp_id()] = s2;
  }
  if (bad_nf != ~0ull) atomicMin(&bad[0], bad_nf);
  if (bad_neg != ~0ull) atomicMin(&bad[1], bad_neg);
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kScanThreads / 32; ++w) {
      a += red_s[w];
      b += red_s2[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void scan_finalize_kernel(const double* part, int nparts, double* out) {
  // one warp per output, lanes stride the partials, butterfly reduce
  const int which = threadIdx.x >> 5;  // 0: sum, 1: sumsq
  if (which > 1) return;
  double v = 0.0;
  for (int i = lane_id(); i < nparts; i += 32) v += part[2 * i + which];
  v = warp_allreduce_sum(v);
  if (lane_id() == 0) out[which] = v;
}

}  // namespace

int scan_grid() { return kScanSms * kScanBlocksPerSm; }

template <typename T>
int launch_scan(const T* x, int64_t count, unsigned long long* bad, double* part, double* out,
                cudaStream_t stream) {
  RNMF_CUDA(cudaMemsetAsync(bad, 0xff, 2 * sizeof(unsigned long long), stream));
  scan_kernel<T><<<scan_grid(), kScanThreads, 0, stream>>>(x, count, bad, part);
  RNMF_CUDA_LAUNCH();
  scan_finalize_kernel<<<1, 64, 0, stream>>>(part, scan_grid(), out);
  RNMF_CUDA_LAUNCH();
  return 2;
}

template int launch_scan<float>(const float*, int64_t, unsigned long long*, double*, double*, cudaStream_t);
template int launch_scan<double>(const double*, int64_t, unsigned long long*, double*, double*, cudaStream_t);

}  // namespace rnmf_gpu
