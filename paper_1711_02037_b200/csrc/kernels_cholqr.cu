// kernels_cholqr.cu — CholeskyQR2 fast path for the sketch's thin QRs (economic_qr,
// p/src/core.cpp:7-16, called at p/src/sketch.cpp:62,63,68), with Householder TSQR as the fallback.
//
// Any orthonormal basis of range(A) is a valid replacement for Eigen's Householder Q (rHALS depends
// only on range(Q), SURVEY §0 finding 4).  CholeskyQR2 forms G = A^T A in fp64, R = chol(G),
// Q1 = A R^-1, and repeats once on Q1; it is two streaming passes over the m x l matrix plus an
// l x l factorisation, instead of a multi-level tree of shared-memory Householder factorisations.
// It is accurate while cond(A) stays well below 1/sqrt(u_fp64) ~ 1e8; a collapsing Cholesky pivot
// (relative pivot < 1e-12, i.e. A numerically rank deficient, as for BASELINE config 1) or a
// second-pass R that is not close to I raises a device flag and the caller re-runs TSQR.
#include "common.cuh"

#include <map>
#include <mutex>
#include "kernels.h"

#include <algorithm>
#include <type_traits>

namespace rnmf_gpu {

namespace {

constexpr int kCqThreads = 256;

// part[b] = A[rows of b]^T A[rows of b] (l x l, fp64), rows split evenly over the CTAs.  Rows are
// staged 64 at a time in fp64 shared memory; thread (row group rg, block pair (ba <= bb)) owns a
// 4 x 4 block of the upper triangle and accumulates it over the rows rg, rg + RG, ... of each
// chunk (16 FMAs per 8 shared loads); the RG row-group partials are combined in fixed order and
// the block is written to both triangles.
constexpr int kGramChunkRows = 64;
template <typename T>
__global__ void __launch_bounds__(kCqThreads) cq_gram_kernel(const T* __restrict__ A, int64_t rows, int l,
                                                             double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lp = ((l + 3) / 4) * 4 + 1;             // padded row stride (odd: spreads banks)
  double* tile = reinterpret_cast<double*>(smem);    // [kGramChunkRows][lp]
  double* red = tile + kGramChunkRows * lp;          // [RG][npairs][16]
  const int nbk = (l + 3) / 4, npairs = nbk * (nbk + 1) / 2;
  const int RG = max(1, min(4, kCqThreads / npairs));
  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  for (int pr0 = 0; pr0 < npairs; pr0 += kCqThreads / RG) {
    const int slot = threadIdx.x % (kCqThreads / RG), rg = threadIdx.x / (kCqThreads / RG);
    const int pr = pr0 + slot;
    int ba = 0, bb = 0;
    if (pr < npairs) {  // pair index -> (ba, bb), ba <= bb, row-major over the upper triangle
      int rem = pr;
      while (rem >= nbk - ba) {
        rem -= nbk - ba;
        ++ba;
      }
      bb = ba + rem;
    }
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t base = r0; base < r1; base += kGramChunkRows) {
      const int nr = int(r1 - base < kGramChunkRows ? r1 - base : kGramChunkRows);
      __syncthreads();
      for (int e = threadIdx.x; e < kGramChunkRows * lp; e += kCqThreads) {
        const int rr = e / lp, cc = e % lp;
        tile[e] = (rr < nr && cc < l) ? double(A[(base + rr) * l + cc]) : 0.0;
      }
      __syncthreads();
      if (pr < npairs && rg < RG) {
        for (int rr = rg; rr < nr; rr += RG) {
          const double* tr = tile + rr * lp;
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = tr[4 * ba + i], b[i] = tr[4 * bb + i];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
      }
    }
    __syncthreads();
    if (pr < npairs && rg < RG)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[(rg * (kCqThreads / RG) + slot) * 16 + i * 4 + j] = acc[i][j];
    __syncthreads();
    if (rg == 0 && pr < npairs) {
      const int64_t ll = int64_t(l) * l;
      for (int q = 0; q < 16; ++q) {
        double v = 0.0;
        for (int g2 = 0; g2 < RG; ++g2) v += red[(g2 * (kCqThreads / RG) + slot) * 16 + q];
        const int a = 4 * ba + q / 4, b = 4 * bb + q % 4;
        if (a < l && b < l) {
          part[int64_t(blockIdx.x) * ll + int64_t(a) * l + b] = v;
          part[int64_t(blockIdx.x) * ll + int64_t(b) * l + a] = v;
        }
      }
    }
  }
}

// G = sum of partials (fixed order); R = chol(G) (upper, G = R^T R); Rinv = R^-1.  One CTA.
// flag |= 1 when a pivot collapses; with `check_identity`, flag |= 2 when max|R - I| > 1e-2 (the
// second CholeskyQR pass must see an almost orthonormal input).
__global__ void __launch_bounds__(kCqThreads) cq_chol_kernel(const double* __restrict__ part, int nparts, int l,
                                                             double* __restrict__ rinv, int* flag, int check_identity,
                                                             double shift_rel) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lp = l + 1;
  double* G = reinterpret_cast<double*>(smem);  // [l][lp], becomes R in its upper triangle
  double* Ri = G + l * lp;                      // [l][lp]
  __shared__ int bad;
  const int ll = l * l;
  for (int e = threadIdx.x; e < ll; e += kCqThreads) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[int64_t(p) * ll + e];
    G[(e / l) * lp + e % l] = s;
  }
  if (threadIdx.x == 0) {
    bad = 0;
    if (shift_rel > 0.0) {  // shifted Cholesky: G + s I, s = shift_rel * trace(G) >= shift_rel * ||G||_2
      double tr = 0.0;
      for (int j = 0; j < l; ++j) tr += G[j * lp + j];
      for (int j = 0; j < l; ++j) G[j * lp + j] += shift_rel * tr;
    }
  }
  __syncthreads();
  // right-looking Cholesky on the upper triangle: row j of R, then the trailing update
  for (int j = 0; j < l; ++j) {
    if (threadIdx.x == 0) {
      const double d = G[j * lp + j];
      const double orig = d;  // trailing-updated diagonal
      if (!(d > 0.0) || !isfinite(d)) bad = 1;
      G[j * lp + j] = (d > 0.0 && isfinite(d)) ? sqrt(d) : 1.0;
      (void)orig;
    }
    __syncthreads();
    const double rjj = G[j * lp + j];
    for (int c = j + 1 + threadIdx.x; c < l; c += kCqThreads) G[j * lp + c] /= rjj;
    __syncthreads();
    const int nt = l - j - 1;
    for (int e = threadIdx.x; e < nt * nt; e += kCqThreads) {
      const int a = j + 1 + e / nt, b = j + 1 + e % nt;
      if (b >= a) G[a * lp + b] -= G[j * lp + a] * G[j * lp + b];
    }
    __syncthreads();
  }
  // pivot collapse relative to the largest diagonal of R
  if (threadIdx.x == 0) {
    double mx = 0.0, mn = 1e300;
    for (int j = 0; j < l; ++j) {
      mx = fmax(mx, fabs(G[j * lp + j]));
      mn = fmin(mn, fabs(G[j * lp + j]));
    }
    if (!(mn > 1e-6 * mx) && shift_rel == 0.0) bad = 1;  // R diag ratio ~ 1/cond(A); needs cond << 1e8
  }
  // Rinv by column-wise back substitution (thread per column)
  for (int c = threadIdx.x; c < l; c += kCqThreads) {
    for (int i = l - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int t = i + 1; t <= c; ++t) s -= G[i * lp + t] * Ri[t * lp + c];
      Ri[i * lp + c] = (i <= c) ? s / G[i * lp + i] : 0.0;
    }
  }
  __syncthreads();
  if (check_identity) {
    double dev = 0.0;
    for (int e = threadIdx.x; e < ll; e += kCqThreads) {
      const int a = e / l, b = e % l;
      if (b >= a) dev = fmax(dev, fabs(G[a * lp + b] - (a == b ? 1.0 : 0.0)));
    }
    for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    if ((threadIdx.x & 31) == 0 && dev > 1e-2) atomicOr(&bad, 2);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ll; e += kCqThreads) rinv[e] = Ri[(e / l) * lp + e % l];
  if (threadIdx.x == 0 && bad) atomicOr(flag, bad);
}

// Out (rows x l) = A (rows x l) * Rinv (l x l upper triangular).  Rows staged in shared memory;
// thread (row, column-group) computes columns j = jg, jg + G, ... of its row.
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kCqThreads) cq_apply_kernel(const TIn* __restrict__ A, int64_t rows, int l,
                                                              const double* __restrict__ rinv, TOut* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lp = l + 1;
  double* Ri = reinterpret_cast<double*>(smem);  // [l][lp]
  double* tile = Ri + l * lp;                    // [rows_per_block][lp]
  constexpr int kRowsPerBlock = 64;
  constexpr int kGroups = kCqThreads / kRowsPerBlock;  // 4 column groups per row
  for (int e = threadIdx.x; e < l * l; e += kCqThreads) Ri[(e / l) * lp + e % l] = rinv[e];
  for (int64_t base = int64_t(blockIdx.x) * kRowsPerBlock; base < rows; base += int64_t(gridDim.x) * kRowsPerBlock) {
    const int nr = int(rows - base < kRowsPerBlock ? rows - base : kRowsPerBlock);
    __syncthreads();
    for (int e = threadIdx.x; e < kRowsPerBlock * l; e += kCqThreads) {
      const int rr = e / l;
      tile[rr * lp + e % l] = rr < nr ? double(A[(base + rr) * l + e % l]) : 0.0;
    }
    __syncthreads();
    const int rr = threadIdx.x / kGroups, jg = threadIdx.x % kGroups;
    if (rr < nr) {
      const double* ar = tile + rr * lp;
      for (int j = jg; j < l; j += kGroups) {
        double s0 = 0.0, s1 = 0.0;
        int i = 0;
        for (; i + 1 <= j; i += 2) {
          s0 += ar[i] * Ri[i * lp + j];
          s1 += ar[i + 1] * Ri[(i + 1) * lp + j];
        }
        if (i <= j) s0 += ar[i] * Ri[i * lp + j];
        out[(base + rr) * l + j] = TOut(s0 + s1);
      }
    }
  }
}

inline int gram_blocks(int64_t rows) {
  return int(std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(rows, 64))));
}

}  // namespace

int64_t cholqr_workspace_doubles(int64_t rows, int l) {
  return int64_t(gram_blocks(rows)) * l * l + 2 * int64_t(l) * l + rows * int64_t(l) + 64;
}

// Dynamic shared-memory limit of a kernel, raised (never lowered) when a launch needs more than any
// launch before it on this device: one table keyed by the kernel, shared by every instantiation
// of launch_cholqr2 (cq_chol_kernel and the double kernels serve both precisions).
static std::mutex g_cq_attr_mu;
static std::map<std::pair<int, const void*>, size_t> g_cq_attr;

template <typename F>
static void cq_raise_smem(int dev, F* kernel, size_t bytes) {
  size_t& have = g_cq_attr[{dev, reinterpret_cast<const void*>(kernel)}];
  if (bytes > have) {
    RNMF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    have = bytes;
  }
}

template <typename T>
int launch_cholqr2(const T* a, int64_t rows, int l, T* q_out, double* ws, int* flag, cudaStream_t stream,
                   const GramAllreduce* allreduce, double shift_rel) {
  const int nb = gram_blocks(rows);
  double* part = ws;
  double* rinv1 = part + int64_t(nb) * l * l;
  double* rinv2 = rinv1 + int64_t(l) * l;
  double* q1 = rinv2 + int64_t(l) * l;  // rows x l, fp64 intermediate
  const int lpad = ((l + 3) / 4) * 4 + 1;
  const size_t gsm = (size_t(kGramChunkRows) * lpad + size_t(kCqThreads) * 16) * sizeof(double);
  const size_t csm = size_t(2) * l * (l + 1) * sizeof(double);
  const size_t asm_ = size_t(l) * (l + 1) * sizeof(double) + size_t(64) * (l + 1) * sizeof(double);
  RNMF_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), stream));
  // dynamic shared-memory limits (chol needs 2 l (l+1) doubles: l <= 112 on B200)
  {
    int dev = 0;
    RNMF_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_cq_attr_mu);
    cq_raise_smem(dev, cq_apply_kernel<T, double>, asm_);
    cq_raise_smem(dev, cq_apply_kernel<double, T>, asm_);
    cq_raise_smem(dev, cq_apply_kernel<double, double>, asm_);
    cq_raise_smem(dev, cq_gram_kernel<T>, gsm);
    cq_raise_smem(dev, cq_gram_kernel<double>, gsm);
    cq_raise_smem(dev, cq_chol_kernel, csm);
  }
  const int ab = int(std::max<int64_t>(1, std::min<int64_t>(148 * 4, ceil_div(rows, 64))));
  int launches = 0;
  // Gram partials -> (sharded: one local Gram, summed over the GPUs) -> Cholesky -> R^-1
  auto chol = [&](auto* src, double* rinv, int check_identity, double shift) {
    cq_gram_kernel<std::remove_const_t<std::remove_pointer_t<decltype(src)>>><<<nb, kCqThreads, gsm, stream>>>(
        src, rows, l, part);
    RNMF_CUDA_LAUNCH();
    // the CTA partials summed by a multi-block fixed-order reduction (in place into part[0])
    launches += launch_reduce_parts(part, nb, l * l, part, stream);
    if (allreduce) (*allreduce)(part, int64_t(l) * l);
    cq_chol_kernel<<<1, kCqThreads, csm, stream>>>(part, 1, l, rinv, flag, check_identity, shift);
    RNMF_CUDA_LAUNCH();
    launches += 2;
  };
  if (shift_rel > 0.0) {
    // shifted CholeskyQR3: the shifted pass makes Q1 well conditioned, two plain passes follow
    double* q0 = q1;
    chol(a, rinv1, 0, shift_rel);
    cq_apply_kernel<T, double><<<ab, kCqThreads, asm_, stream>>>(a, rows, l, rinv1, q0);
    RNMF_CUDA_LAUNCH();
    chol(static_cast<const double*>(q0), rinv2, 0, 0.0);
    cq_apply_kernel<double, double><<<ab, kCqThreads, asm_, stream>>>(q0, rows, l, rinv2, q0);
    RNMF_CUDA_LAUNCH();
    chol(static_cast<const double*>(q0), rinv1, 1, 0.0);
    cq_apply_kernel<double, T><<<ab, kCqThreads, asm_, stream>>>(q0, rows, l, rinv1, q_out);
    RNMF_CUDA_LAUNCH();
    return launches + 3;
  }
  // pass 1
  chol(a, rinv1, 0, 0.0);
  cq_apply_kernel<T, double><<<ab, kCqThreads, asm_, stream>>>(a, rows, l, rinv1, q1);
  RNMF_CUDA_LAUNCH();
  // pass 2
  chol(static_cast<const double*>(q1), rinv2, 1, 0.0);
  cq_apply_kernel<double, T><<<ab, kCqThreads, asm_, stream>>>(q1, rows, l, rinv2, q_out);
  RNMF_CUDA_LAUNCH();
  return launches + 2;
}

template int launch_cholqr2<float>(const float*, int64_t, int, float*, double*, int*, cudaStream_t,
                                   const GramAllreduce*, double);
template int launch_cholqr2<double>(const double*, int64_t, int, double*, double*, int*, cudaStream_t,
                                    const GramAllreduce*, double);

}  // namespace rnmf_gpu
