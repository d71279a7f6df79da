// kernels_nndsvd.cu — InitScheme::Svd, the NNDSVD split of a randomized rank-k SVD
// (nndsvd_init, p/src/hals.cpp:126-170), after the second rqb (on the GPU, kernels_xgemm/cholqr):
//
//   B (l x n) = U S V^T      from the eigen-decomposition of the l x l Gram B B^T (cyclic Jacobi in
//                            one CTA, fp64; only the leading k pairs are used, which are well above
//                            the rounding floor of the squared spectrum)
//   u_j = Q U(:,j) (m),  v_j = B^T U(:,j) / s_j (n)      (the reference's Q * svd.matrixU(), V)
//   column / row j of W / H = coefficients x the positive or the negative part of u_j / v_j,
//   zeros replaced by mean(X)/100
// The split does not depend on the sign convention of the singular pairs (flipping u_j and v_j
// together swaps the two sections and leaves the chosen one unchanged), so any SVD matches.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kNThreads = 256;

// Eigen-decomposition of the symmetric l x l matrix G (l <= 64): parallel cyclic Jacobi with the
// round-robin pairing (l/2 disjoint rotations per step, l - 1 steps per sweep).  Outputs the
// eigenvalues in descending order and the matching unit eigenvectors (columns of vec, l x l).
__global__ void __launch_bounds__(kNThreads) jacobi_eig_kernel(const double* __restrict__ g, int l,
                                                               double* __restrict__ eval,
                                                               double* __restrict__ evec) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int np = l + (l & 1);  // even player count (a dummy index l when l is odd)
  const int lp = np + 1;
  double* A = reinterpret_cast<double*>(smem);  // [np][lp]
  double* V = A + np * lp;                      // [np][lp]
  double* cs = V + np * lp;                     // [np/2][2]
  int* pr = reinterpret_cast<int*>(cs + np);    // [np] pairing: pr[2t], pr[2t+1]
  __shared__ double off;
  __shared__ int perm[64];
  const int tid = threadIdx.x;
  for (int e = tid; e < np * np; e += kNThreads) {
    const int a = e / np, b = e % np;
    A[a * lp + b] = (a < l && b < l) ? g[a * l + b] : 0.0;
    V[a * lp + b] = a == b ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = np / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) {
      double s = 0.0, d = 0.0;
      for (int a = 0; a < l; ++a)
        for (int b = 0; b < l; ++b) {
          const double v = A[a * lp + b] * A[a * lp + b];
          if (a == b) d += v; else s += v;
        }
      off = (s <= 1e-30 * d) ? -1.0 : s;
    }
    __syncthreads();
    if (off < 0.0) break;
    for (int step = 0; step < np - 1; ++step) {
      // round robin: player 0 fixed, the others rotate
      if (tid < half) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + step) % (np - 1); };
        int p = player(tid), q = player(np - 1 - tid);
        if (p > q) { const int t = p; p = q; q = t; }
        pr[2 * tid] = p;
        pr[2 * tid + 1] = q;
        double c = 1.0, sn = 0.0;
        if (q < l) {
          const double apq = A[p * lp + q];
          if (apq != 0.0) {
            const double theta = (A[q * lp + q] - A[p * lp + p]) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = t * c;
          }
        }
        cs[2 * tid] = c;
        cs[2 * tid + 1] = sn;
      }
      __syncthreads();
      // rows: A <- J^T A (pairs are disjoint, all rotations at once)
      for (int e = tid; e < half * np; e += kNThreads) {
        const int t = e / np, col = e % np;
        const int p = pr[2 * t], q = pr[2 * t + 1];
        const double c = cs[2 * t], sn = cs[2 * t + 1];
        const double ap = A[p * lp + col], aq = A[q * lp + col];
        A[p * lp + col] = c * ap - sn * aq;
        A[q * lp + col] = sn * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int e = tid; e < half * np; e += kNThreads) {
        const int t = e / np, row = e % np;
        const int p = pr[2 * t], q = pr[2 * t + 1];
        const double c = cs[2 * t], sn = cs[2 * t + 1];
        const double ap = A[row * lp + p], aq = A[row * lp + q];
        A[row * lp + p] = c * ap - sn * aq;
        A[row * lp + q] = sn * ap + c * aq;
        const double vp = V[row * lp + p], vq = V[row * lp + q];
        V[row * lp + p] = c * vp - sn * vq;
        V[row * lp + q] = sn * vp + c * vq;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {  // descending order of the eigenvalues (stable selection)
    for (int a = 0; a < l; ++a) perm[a] = a;
    for (int a = 0; a < l; ++a) {
      int best = a;
      for (int b = a + 1; b < l; ++b)
        if (A[perm[b] * lp + perm[b]] > A[perm[best] * lp + perm[best]]) best = b;
      const int t = perm[a];
      perm[a] = perm[best];
      perm[best] = t;
    }
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += kNThreads) {
    const int r = e / l, c = e % l;
    evec[r * l + c] = V[r * lp + perm[c]];
  }
  for (int a = tid; a < l; a += kNThreads) eval[a] = A[perm[a] * lp + perm[a]];
}

// Thread (row slot, j): u(r, j) = (S U(:, :k) diag(scale))(r, j) for rows r = slot, slot + slots, ...
// (slots = 256 / k per CTA, grid-strided).  `transpose`: S is stored l x rows (B), element (r, i) =
// S[i * rows + r].
template <typename T>
__device__ __forceinline__ double nndsvd_u(const T* __restrict__ S, int64_t rows, int l, bool transpose,
                                           const double* Us, int k, int64_t r, int j) {
  double u0 = 0.0, u1 = 0.0;
  int i = 0;
  for (; i + 1 < l; i += 2) {
    const double s0 = double(transpose ? S[int64_t(i) * rows + r] : S[r * l + i]);
    const double s1 = double(transpose ? S[int64_t(i + 1) * rows + r] : S[r * l + i + 1]);
    u0 += s0 * Us[i * k + j];
    u1 += s1 * Us[(i + 1) * k + j];
  }
  if (i < l) u0 += double(transpose ? S[int64_t(i) * rows + r] : S[r * l + i]) * Us[i * k + j];
  return u0 + u1;
}

// per-CTA partial sums of squares of the positive / negative parts of each column of u:
// part[b][j][2]
template <typename T>
__global__ void __launch_bounds__(kNThreads) nndsvd_norms_kernel(const T* __restrict__ S, int64_t rows, int l,
                                                                 bool transpose, const double* __restrict__ U, int k,
                                                                 const double* __restrict__ colscale,
                                                                 double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* Us = reinterpret_cast<double*>(smem);  // [l][k]
  double* red = Us + l * k;                      // [kNThreads][2]
  for (int e = threadIdx.x; e < l * k; e += kNThreads) Us[e] = U[(e / k) * l + e % k] * colscale[e % k];
  __syncthreads();
  const int slots = kNThreads / k, j = threadIdx.x % k, slot = threadIdx.x / k;
  double ap = 0.0, an = 0.0;
  if (slot < slots)
    for (int64_t r = int64_t(blockIdx.x) * slots + slot; r < rows; r += int64_t(gridDim.x) * slots) {
      const double u = nndsvd_u(S, rows, l, transpose, Us, k, r, j);
      const double pos = fmax(u, 0.0), neg = fmax(-u, 0.0);
      ap += pos * pos;
      an += neg * neg;
    }
  red[2 * threadIdx.x] = ap;
  red[2 * threadIdx.x + 1] = an;
  __syncthreads();
  if (threadIdx.x < k) {  // fixed-order sum over the slots of column j = threadIdx.x
    double sp = 0.0, sn = 0.0;
    for (int q = 0; q < slots; ++q) {
      sp += red[2 * (q * k + threadIdx.x)];
      sn += red[2 * (q * k + threadIdx.x) + 1];
    }
    part[(int64_t(blockIdx.x) * k + threadIdx.x) * 2] = sp;
    part[(int64_t(blockIdx.x) * k + threadIdx.x) * 2 + 1] = sn;
  }
}

// out(r, j) = cpos_j * max(u, 0) + cneg_j * max(-u, 0), zeros replaced by `fill`; out is rows x k
// row-major (W) or, with `out_transposed`, k x rows (H).
template <typename T>
__global__ void __launch_bounds__(kNThreads) nndsvd_apply_kernel(const T* __restrict__ S, int64_t rows, int l,
                                                                 bool transpose, const double* __restrict__ U, int k,
                                                                 const double* __restrict__ colscale,
                                                                 const double* __restrict__ coef, double fill,
                                                                 T* __restrict__ out, bool out_transposed) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* Us = reinterpret_cast<double*>(smem);
  for (int e = threadIdx.x; e < l * k; e += kNThreads) Us[e] = U[(e / k) * l + e % k] * colscale[e % k];
  __syncthreads();
  const int slots = kNThreads / k, j = threadIdx.x % k, slot = threadIdx.x / k;
  if (slot >= slots) return;
  const double cp = coef[2 * j], cn = coef[2 * j + 1];
  for (int64_t r = int64_t(blockIdx.x) * slots + slot; r < rows; r += int64_t(gridDim.x) * slots) {
    const double u = nndsvd_u(S, rows, l, transpose, Us, k, r, j);
    const double v = cp * fmax(u, 0.0) + cn * fmax(-u, 0.0);
    const T o = T(v > 0.0 ? v : fill);
    if (out_transposed)
      out[int64_t(j) * rows + r] = o;
    else
      out[r * k + j] = o;
  }
}

inline int nblocks(int64_t rows) { return int(std::max<int64_t>(1, std::min<int64_t>(592, ceil_div(rows, 16)))); }

}  // namespace

int launch_jacobi_eig(const double* g, int l, double* eval, double* evec, cudaStream_t stream) {
  if (l > 64) throw CudaError("NNDSVD: sketch width above 64");
  const int np = l + (l & 1);
  const size_t sm = (size_t(2) * np * (np + 1) + np) * sizeof(double) + np * sizeof(int) + 16;
  RNMF_CUDA(cudaFuncSetAttribute(jacobi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  jacobi_eig_kernel<<<1, kNThreads, sm, stream>>>(g, l, eval, evec);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int nndsvd_norm_blocks(int64_t rows) { return nblocks(rows); }

template <typename T>
int launch_nndsvd_norms(const T* s, int64_t rows, int l, bool transpose, const double* u, int k,
                        const double* colscale, double* part, cudaStream_t stream) {
  if (k > 64) throw CudaError("NNDSVD: rank above 64");
  const size_t sm = (size_t(l) * k + size_t(kNThreads) * 2) * sizeof(double);
  RNMF_CUDA(cudaFuncSetAttribute(nndsvd_norms_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  nndsvd_norms_kernel<T><<<nblocks(rows), kNThreads, sm, stream>>>(s, rows, l, transpose, u, k, colscale, part);
  RNMF_CUDA_LAUNCH();
  return 1;
}

template <typename T>
int launch_nndsvd_apply(const T* s, int64_t rows, int l, bool transpose, const double* u, int k,
                        const double* colscale, const double* coef, double fill, T* out, bool out_transposed,
                        cudaStream_t stream) {
  const size_t sm = size_t(l) * k * sizeof(double);
  RNMF_CUDA(cudaFuncSetAttribute(nndsvd_apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  nndsvd_apply_kernel<T><<<nblocks(rows), kNThreads, sm, stream>>>(s, rows, l, transpose, u, k, colscale, coef, fill,
                                                                   out, out_transposed);
  RNMF_CUDA_LAUNCH();
  return 1;
}

#define RNMF_NINST(T)                                                                                          \
  template int launch_nndsvd_norms<T>(const T*, int64_t, int, bool, const double*, int, const double*, double*, \
                                      cudaStream_t);                                                          \
  template int launch_nndsvd_apply<T>(const T*, int64_t, int, bool, const double*, int, const double*,         \
                                      const double*, double, T*, bool, cudaStream_t);
RNMF_NINST(float)
RNMF_NINST(double)

}  // namespace rnmf_gpu
