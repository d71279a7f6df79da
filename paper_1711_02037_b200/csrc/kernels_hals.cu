// kernels_hals.cu — the full-space factor updates of the deterministic HALS solver (rnmf::hals_fit,
// p/src/hals.cpp:268-323), the speed-up baseline the reference's `bench` command times rHALS against.
//
// hals_w_phase (p/src/hals.cpp:172-178) applies clamped_col_update (:67-73) to the columns of W in
// order; column j's update reads W * HH^T(:,j), i.e. row i only needs its own (partly updated)
// row.  hals_h_phase (:182-193) is the same with the roles of rows and columns exchanged for H
// (clamped_row_update, :75-81): column c of H only needs itself.  So both phases are one kernel:
// thread per row r of A (W, or H^T through strides), the row's k entries in fp64 registers, the k
// sequential updates
//     A(r,j) <- [A(r,j) + (P(r,j) - A(r,:) G(:,j) - alpha A(r,j) - beta) / max(G(j,j) + alpha, floor)]_+
// with P = X H^T, G = H H^T (W phase) or P = X^T W, G = W^T W (H phase), G broadcast from shared
// memory.  The X-streaming products come from the sketch GEMM kernels (X passes, HBM-bound).
#include "common.cuh"
#include "kernels.h"

namespace rnmf_gpu {

namespace {

constexpr double kHalsFloor = 1e-12;  // p/include/rnmf/hals.hpp:67 (kDivisionFloor)
constexpr int kHalsThreads = 128;

template <typename T, typename P, int KH>
__global__ void __launch_bounds__(kHalsThreads) hals_rows_kernel(T* __restrict__ a, int64_t rows, int k, int64_t sr,
                                                                 int64_t sj, const P* __restrict__ p, int64_t pr,
                                                                 int64_t pj, const double* __restrict__ gram,
                                                                 double alpha, double beta) {
  extern __shared__ double g_s[];  // k x k Gram, then 1 / denominators
  double* rden = g_s + k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) g_s[e] = gram[e];
  for (int j = threadIdx.x; j < k; j += blockDim.x) rden[j] = 1.0 / fmax(gram[j * k + j] + alpha, kHalsFloor);
  __syncthreads();
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    double v[KH];
#pragma unroll
    for (int c = 0; c < KH; ++c) v[c] = c < k ? double(a[r * sr + c * sj]) : 0.0;
    for (int j = 0; j < k; ++j) {
      // (A(r,:) G(:,j)) with the current row, and A(r,j) itself (register array, static indices)
      double s0 = 0.0, s1 = 0.0, vj = v[0];
#pragma unroll
      for (int c = 0; c < KH; c += 2) {
        if (c < k) s0 = fma(v[c], g_s[c * k + j], s0);
        if (c + 1 < k) s1 = fma(v[c + 1], g_s[(c + 1) * k + j], s1);
        if (c == j) vj = v[c];
        if (c + 1 == j) vj = v[c + 1];
      }
      double num = double(p[r * pr + j * pj]) - (s0 + s1) - alpha * vj;
      if (beta != 0.0) num -= beta;
      const double nv = fmax(vj + num * rden[j], 0.0);
#pragma unroll
      for (int c = 0; c < KH; ++c)
        if (c == j) v[c] = nv;
    }
#pragma unroll
    for (int c = 0; c < KH; ++c)
      if (c < k) a[r * sr + c * sj] = T(v[c]);
  }
}

template <typename T, typename P>
int launch_rows(T* a, int64_t rows, int k, int64_t sr, int64_t sj, const P* p, int64_t pr, int64_t pj,
                const double* gram, double alpha, double beta, cudaStream_t st) {
  if (rows <= 0 || k <= 0) return 0;
  const int blocks = int(std::min<int64_t>(ceil_div(rows, kHalsThreads), 148 * 16));
  const size_t smem = sizeof(double) * size_t(k) * (k + 1);
  if (k <= 16)
    hals_rows_kernel<T, P, 16><<<blocks, kHalsThreads, smem, st>>>(a, rows, k, sr, sj, p, pr, pj, gram, alpha, beta);
  else if (k <= 32)
    hals_rows_kernel<T, P, 32><<<blocks, kHalsThreads, smem, st>>>(a, rows, k, sr, sj, p, pr, pj, gram, alpha, beta);
  else if (k <= 64)
    hals_rows_kernel<T, P, 64><<<blocks, kHalsThreads, smem, st>>>(a, rows, k, sr, sj, p, pr, pj, gram, alpha, beta);
  else
    throw CudaError("hals: rank above 64");
  RNMF_CUDA_LAUNCH();
  return 1;
}

}  // namespace

template <typename T>
int launch_hals_w_update(T* w, int64_t m, int k, const T* xht, const double* hht, double alpha, double beta,
                         cudaStream_t st) {
  return launch_rows<T, T>(w, m, k, k, 1, xht, k, 1, hht, alpha, beta, st);
}

template <typename T>
int launch_hals_h_update(T* h, int64_t n, int k, const T* xtw, const double* wtw, double alpha, double beta,
                         cudaStream_t st) {
  // column c of H (k x n, row-major) is "row" c with stride n between its entries; X^T W is n x k
  return launch_rows<T, T>(h, n, k, 1, n, xtw, k, 1, wtw, alpha, beta, st);
}

template int launch_hals_w_update<float>(float*, int64_t, int, const float*, const double*, double, double, cudaStream_t);
template int launch_hals_w_update<double>(double*, int64_t, int, const double*, const double*, double, double,
                                          cudaStream_t);
template int launch_hals_h_update<float>(float*, int64_t, int, const float*, const double*, double, double, cudaStream_t);
template int launch_hals_h_update<double>(double*, int64_t, int, const double*, const double*, double, double,
                                          cudaStream_t);

}  // namespace rnmf_gpu
