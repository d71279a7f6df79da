// kernels_tsqr.cu — Householder TSQR: the thin QR of the sketch (economic_qr, p/src/core.cpp:7-16,
// called at p/src/sketch.cpp:62,63,68 on Y (m x l) and X^T Q (n x l)).
//
// rHALS depends only on range(Q) (SURVEY §0 finding 4), so any stable orthonormal basis is a
// valid replacement for Eigen's Householder Q.  TSQR is used because it is unconditionally
// stable: it survives the exactly rank-deficient sketches of config 1 where CholeskyQR fails.
//
// Level structure (all in fp64):
//   level 0: the rows of A are split into nb0 = max(1, rows/BR) contiguous blocks (each has
//            between BR and 2BR-1 rows, >= l); every CTA factors its block in shared memory with
//            Householder reflectors (Eigen/LAPACK sign convention), writes its R (l x l) into the
//            next level's input and its explicit block Q (dorg2r in place) into a level buffer.
//   level i: the stacked R's (nb_{i-1} l x l) are factored the same way, until one block remains.
//   combine: top-down, G_L = Q_L; G_i[block b] = Q_i[block b] * G_{i+1}[rows b*l .. b*l+l);
//            G_0 is the thin Q of A.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <vector>

namespace rnmf_gpu {

namespace {

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;

inline int lp_of(int l) { return l + 1; }  // odd fp64 row stride -> conflict-free column walks

// Rows per block target for a given sketch width: blocks hold up to 2*BR-1 rows in smem.
inline int64_t block_rows_target(int l, int max_smem) {
  const int64_t per_row = int64_t(lp_of(l)) * sizeof(double);
  const int64_t reserve = 4096;  // tau, w, reduction scratch
  return (int64_t(max_smem) - reserve) / (2 * per_row);
}

inline int64_t nblocks_for(int64_t rows, int l, int max_smem) {
  const int64_t br = block_rows_target(l, max_smem);
  return std::max<int64_t>(1, rows / std::max<int64_t>(br, 1));
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_allreduce_sum(v);
  __syncthreads();
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kQrWarps; ++w) s += red[w];
  return s;
}

// Factor one block per CTA.  in: rows x l (ld l) of TIn; rout: (nb*l) x l fp64 (this block's R at
// rows b*l..); qout: rows x l fp64 explicit block Q.
template <typename TIn>
__global__ void __launch_bounds__(kQrThreads, 1) tsqr_factor_kernel(const TIn* __restrict__ in, int64_t rows, int l,
                                                                    int64_t nb, double* __restrict__ rout,
                                                                    double* __restrict__ qout) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lp = l + 1;
  const int64_t b = blockIdx.x;
  const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
  const int R = int(r1 - r0);
  double* A = reinterpret_cast<double*>(smem);  // [R][lp]
  double* tau = A + size_t(R) * lp;             // [l]
  double* w = tau + l;                          // [l]
  double* red = w + l;                          // [kQrWarps]
  __shared__ double sh_beta, sh_tau, sh_inv;

  for (int64_t e = threadIdx.x; e < int64_t(R) * l; e += kQrThreads) {
    const int r = int(e / l), c = int(e % l);
    A[r * lp + c] = double(in[(r0 + r) * l + c]);
  }
  __syncthreads();

  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
  for (int j = 0; j < l; ++j) {
    // ||A[j+1:, j]||^2
    double part = 0.0;
    for (int i = j + 1 + tid; i < R; i += kQrThreads) part += A[i * lp + j] * A[i * lp + j];
    const double tail = block_sum(part, red);
    if (tid == 0) {
      const double c0 = A[j * lp + j];
      if (tail <= 2.2250738585072014e-308) {  // Eigen: tailSqNorm <= (numeric_limits::min)()
        sh_tau = 0.0;
        sh_beta = c0;
        sh_inv = 0.0;
      } else {
        double beta = sqrt(c0 * c0 + tail);
        if (c0 >= 0.0) beta = -beta;
        sh_beta = beta;
        sh_inv = 1.0 / (c0 - beta);
        sh_tau = (beta - c0) / beta;
      }
    }
    __syncthreads();
    const double t = sh_tau, inv = sh_inv;
    for (int i = j + 1 + tid; i < R; i += kQrThreads) A[i * lp + j] *= inv;  // zero tail -> 0 * 0
    if (tid == 0) {
      A[j * lp + j] = sh_beta;
      tau[j] = t;
    }
    __syncthreads();
    if (t != 0.0 && j + 1 < l) {
      // w[c] = A[j][c] + sum_{i>j} v_i A[i][c]; warp per column, lanes over rows
      for (int c = j + 1 + wid; c < l; c += kQrWarps) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < R; i += 32) s += A[i * lp + j] * A[i * lp + c];
        s = warp_allreduce_sum(s);
        if (lane == 0) w[c] = (A[j * lp + c] + s) * t;
      }
      __syncthreads();
      const int nc = l - j - 1;
      for (int64_t e = tid; e < int64_t(R - j) * nc; e += kQrThreads) {
        const int i = j + int(e / nc), c = j + 1 + int(e % nc);
        const double vi = (i == j) ? 1.0 : A[i * lp + j];
        A[i * lp + c] -= w[c] * vi;
      }
      __syncthreads();
    }
  }
  // R (upper triangle of the top l rows)
  for (int e = tid; e < l * l; e += kQrThreads) {
    const int i = e / l, c = e % l;
    rout[(b * l + i) * l + c] = c >= i ? A[i * lp + c] : 0.0;
  }
  __syncthreads();
  // explicit Q in place (LAPACK dorg2r): i = l-1 .. 0
  for (int i = l - 1; i >= 0; --i) {
    const double t = tau[i];
    if (i < l - 1 && t != 0.0) {
      for (int c = i + 1 + wid; c < l; c += kQrWarps) {
        double s = 0.0;
        for (int r = i + 1 + lane; r < R; r += 32) s += A[r * lp + i] * A[r * lp + c];
        s = warp_allreduce_sum(s);
        if (lane == 0) w[c] = (A[i * lp + c] + s) * t;  // row i of column c (v_i = 1)
      }
      __syncthreads();
      const int nc = l - i - 1;
      for (int64_t e = tid; e < int64_t(R - i) * nc; e += kQrThreads) {
        const int r = i + int(e / nc), c = i + 1 + int(e % nc);
        const double vr = (r == i) ? 1.0 : A[r * lp + i];
        A[r * lp + c] -= w[c] * vr;
      }
      __syncthreads();
    }
    for (int r = tid; r < R; r += kQrThreads) {
      if (r > i)
        A[r * lp + i] *= -t;
      else if (r == i)
        A[r * lp + i] = 1.0 - t;
      else
        A[r * lp + i] = 0.0;
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < int64_t(R) * l; e += kQrThreads) {
    const int r = int(e / l), c = int(e % l);
    qout[(r0 + r) * l + c] = A[r * lp + c];
  }
}

// G_i[rows of block b] = Q_i[rows of block b] * G_{i+1}[b*l .. b*l+l)  (one CTA per block).
template <typename TOut>
__global__ void __launch_bounds__(kQrThreads) tsqr_combine_kernel(const double* __restrict__ qlev, int64_t rows, int l,
                                                                  int64_t nb, const double* __restrict__ gup,
                                                                  TOut* __restrict__ gout) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* M = reinterpret_cast<double*>(smem);  // [l][l]
  const int64_t b = blockIdx.x;
  const int64_t r0 = rows * b / nb, r1 = rows * (b + 1) / nb;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) M[e] = gup[b * l * l + e];
  __syncthreads();
  const int64_t total = (r1 - r0) * l;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t r = r0 + e / l;
    const int c = int(e % l);
    const double* qr = qlev + r * l;
    double s = 0.0;
    for (int t = 0; t < l; ++t) s += qr[t] * M[t * l + c];
    gout[r * l + c] = TOut(s);
  }
}

template <typename TOut>
__global__ void copy_cast_kernel(const double* __restrict__ in, int64_t count, TOut* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = TOut(in[i]);
}

struct Level {
  int64_t rows, nb;
  double* qbuf;  // rows x l
};

}  // namespace

int tsqr_max_l(int max_smem) {
  int l = 1;
  while (l < 256 && block_rows_target(l + 1, max_smem) >= l + 1) ++l;
  return l;
}

// Workspace: for each level, a fp64 Q buffer (rows_i x l) and an R buffer (nb_i*l x l), plus two
// combine buffers of the largest upper-level size.
int64_t tsqr_workspace_doubles(int64_t rows, int l, int max_smem) {
  int64_t total = 0, r = rows, maxup = 0;
  bool first = true;
  while (true) {
    const int64_t nb = nblocks_for(r, l, max_smem);
    total += r * l + nb * l * l;
    if (!first) maxup = std::max(maxup, r * l);
    first = false;
    if (nb == 1) break;
    r = nb * l;
  }
  return total + 2 * maxup + 64;
}

template <typename T>
int launch_tsqr(const T* a, int64_t rows, int l, T* q_out, double* ws, int max_smem, cudaStream_t stream) {
  if (rows < l) throw CudaError("tsqr: rows < cols");
  if (block_rows_target(l, max_smem) < l)
    throw CudaError("tsqr: sketch width " + std::to_string(l) + " exceeds the shared-memory TSQR limit " +
                    std::to_string(tsqr_max_l(max_smem)));
  int launches = 0;
  std::vector<Level> levels;
  double* p = ws;
  int64_t r = rows;
  const void* in = a;
  bool in_is_double = false;
  int64_t maxup = 0;
  while (true) {
    const int64_t nb = nblocks_for(r, l, max_smem);
    Level lev{r, nb, p};
    p += r * l;
    double* rbuf = p;
    p += nb * l * l;
    const int64_t maxR = ceil_div(r, nb);  // largest block
    const size_t sm = size_t(maxR) * lp_of(l) * sizeof(double) + size_t(2 * l + kQrWarps) * sizeof(double);
    if (sm > size_t(max_smem)) throw CudaError("tsqr: block does not fit shared memory");
    if (in_is_double) {
      auto f = tsqr_factor_kernel<double>;
      RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      f<<<unsigned(nb), kQrThreads, sm, stream>>>(static_cast<const double*>(in), r, l, nb, rbuf, lev.qbuf);
    } else {
      auto f = tsqr_factor_kernel<T>;
      RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      f<<<unsigned(nb), kQrThreads, sm, stream>>>(static_cast<const T*>(in), r, l, nb, rbuf, lev.qbuf);
    }
    RNMF_CUDA_LAUNCH();
    ++launches;
    if (!levels.empty()) maxup = std::max(maxup, r * l);
    levels.push_back(lev);
    if (nb == 1) break;
    in = rbuf;
    in_is_double = true;
    r = nb * l;
  }
  double* g0 = p;
  double* g1 = p + maxup;
  const size_t msm = size_t(l) * l * sizeof(double);
  if (levels.size() == 1) {
    copy_cast_kernel<T><<<unsigned(std::min<int64_t>(ceil_div(rows * l, 256), 1184)), 256, 0, stream>>>(
        levels[0].qbuf, rows * l, q_out);
    RNMF_CUDA_LAUNCH();
    return launches + 1;
  }
  // top level's Q is G_L
  const double* gup = levels.back().qbuf;
  for (int i = int(levels.size()) - 2; i >= 0; --i) {
    const Level& lev = levels[size_t(i)];
    if (i == 0) {
      tsqr_combine_kernel<T><<<unsigned(lev.nb), kQrThreads, msm, stream>>>(lev.qbuf, lev.rows, l, lev.nb, gup, q_out);
    } else {
      double* gout = (gup == g0) ? g1 : g0;
      tsqr_combine_kernel<double><<<unsigned(lev.nb), kQrThreads, msm, stream>>>(lev.qbuf, lev.rows, l, lev.nb, gup, gout);
      gup = gout;
    }
    RNMF_CUDA_LAUNCH();
    ++launches;
  }
  return launches;
}

template int launch_tsqr<float>(const float*, int64_t, int, float*, double*, int, cudaStream_t);
template int launch_tsqr<double>(const double*, int64_t, int, double*, double*, int, cudaStream_t);

}  // namespace rnmf_gpu
