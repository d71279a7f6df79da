// kernels_xgemm.cu — X-streaming "tall-times-skinny" GEMMs of the sketch and of the full-space
// metrics, plus the small dense helpers around them.
//
//   xw  : Y = X * S          (m x n) * (n x c)    Y = X Omega, Y = X Z   (p/src/sketch.cpp:60,64)
//   xtw : P = X^T * S        (n x m) * (m x c)    X^T Q, B = Q^T X        (p/src/sketch.cpp:63,69)
//   xw_metrics  : one X pass computing ||X - W H||^2 and the projected ||grad_W||^2
//   xtw_metrics : one X pass computing the projected ||grad_H||^2
//                 (full_space_metrics, p/src/rhals.cpp:140-148)
//
// These are the FMA ("exact") kernels: fp32 FFMA for fp32 X, DFMA for fp64 X.  X is streamed
// once per call with 16-byte vector loads, double-buffered through shared memory with a
// register prefetch of the next tile; the small operand S stays L2/SMEM resident.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kBM = 128;  // X rows per CTA (xw) / X columns per CTA (xtw)

template <typename T>
struct Tile;
template <>
struct Tile<float> {
  static constexpr int BK = 32;
  static constexpr int VN = 4;
  using V = float4;
};
template <>
struct Tile<double> {
  static constexpr int BK = 16;
  static constexpr int VN = 2;
  using V = double2;
};

template <typename T, int CPAD>
struct XwSmem {
  static constexpr int BK = Tile<T>::BK;
  static constexpr int XS = kBM + 4;  // row stride of the [BK][BM] X tile (keeps 16B alignment)
  static constexpr int SP = CPAD + 1; // row stride of the [BK][CPAD] S tile (bank-conflict pad)
  static constexpr size_t x_bytes = size_t(2) * BK * XS * sizeof(T);
  static constexpr size_t s_bytes = size_t(2) * BK * SP * sizeof(T);
  static constexpr size_t s_off = x_bytes;
  static constexpr size_t base = ((x_bytes + s_bytes + 15) / 16) * 16;
  // metrics extras: W^T tile [CPAD][BM+4] (T) and H H^T [CPAD*CPAD] (double)
  static constexpr size_t wt_off = base;
  static constexpr size_t wt_bytes = size_t(CPAD) * XS * sizeof(T);
  static constexpr size_t hh_off = ((wt_off + wt_bytes + 15) / 16) * 16;
  static constexpr size_t hh_bytes = size_t(CPAD) * CPAD * sizeof(double);
  static constexpr size_t metrics_total = hh_off + hh_bytes;
};

template <typename T>
__device__ __forceinline__ void load8(const T* p, T (&a)[8]) {
  if constexpr (sizeof(T) == 4) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    const float4 v = *reinterpret_cast<const float4*>(p + 4);
    a[0] = u.x, a[1] = u.y, a[2] = u.z, a[3] = u.w, a[4] = v.x, a[5] = v.y, a[6] = v.z, a[7] = v.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 u = *reinterpret_cast<const double2*>(p + 2 * q);
      a[2 * q] = u.x, a[2 * q + 1] = u.y;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// xw: Y = X S.  One CTA owns 128 rows of X and all c output columns; it walks K = n in BK chunks.
// Thread (ty, tx) accumulates rows ty*8..ty*8+7 x columns tx + 16 t.
template <typename T, int CPAD, bool VECX, bool METRICS>
__global__ void __launch_bounds__(kThreads) xw_kernel(const T* __restrict__ X, int64_t m, int64_t n, int64_t ldx,
                                                      const T* __restrict__ S, int c, T* __restrict__ Y,
                                                      const T* __restrict__ W, int k,
                                                      const double* __restrict__ hht,
                                                      double* part_obj, double* part_pgw) {
  using L = XwSmem<T, CPAD>;
  constexpr int BK = Tile<T>::BK, VN = Tile<T>::VN, TC = CPAD / 16, XS = L::XS, SP = L::SP;
  using V = typename Tile<T>::V;
  extern __shared__ __align__(16) unsigned char smem[];
  T* Xs = reinterpret_cast<T*>(smem);                 // [2][BK][XS]
  T* Ss = reinterpret_cast<T*>(smem + L::s_off);      // [2][BK][SP]

  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t row0 = int64_t(blockIdx.x) * kBM;

  // X tile loader: VECX -> 4 vectors of VN per thread; else BM*BK/256 scalars per thread.
  constexpr int XV = kBM * BK / VN / kThreads;  // = 4
  constexpr int XE = kBM * BK / kThreads;       // 16 (f32) / 8 (f64)
  constexpr int SE = BK * CPAD / kThreads;
  V xr[VECX ? XV : 1];
  T xsr[VECX ? 1 : XE];
  T sr[SE];

  auto gload = [&](int64_t k0) {
    if constexpr (VECX) {
#pragma unroll
      for (int u = 0; u < XV; ++u) {
        const int v = tid + kThreads * u;
        const int r = v / (BK / VN), kv = v % (BK / VN);
        const int64_t gr = row0 + r, gk = k0 + int64_t(kv) * VN;
        if (gr < m && gk < n)
          xr[u] = __ldcs(reinterpret_cast<const V*>(X + gr * ldx + gk));
        else
          xr[u] = V{};
      }
    } else {
#pragma unroll
      for (int u = 0; u < XE; ++u) {
        const int e = tid + kThreads * u;
        const int r = e / BK, kk = e % BK;
        const int64_t gr = row0 + r, gk = k0 + kk;
        xsr[u] = (gr < m && gk < n) ? __ldcs(X + gr * ldx + gk) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < SE; ++u) {
      const int e = tid + kThreads * u;
      const int kk = e / CPAD, j = e % CPAD;
      const int64_t gk = k0 + kk;
      sr[u] = (gk < n && j < c) ? S[gk * c + j] : T(0);
    }
  };
  auto sstore = [&](int buf) {
    T* xs = Xs + buf * BK * XS;
    if constexpr (VECX) {
#pragma unroll
      for (int u = 0; u < XV; ++u) {
        const int v = tid + kThreads * u;
        const int r = v / (BK / VN), kv = v % (BK / VN);
        const T* e = reinterpret_cast<const T*>(&xr[u]);
#pragma unroll
        for (int q = 0; q < VN; ++q) xs[(kv * VN + q) * XS + r] = e[q];
      }
    } else {
#pragma unroll
      for (int u = 0; u < XE; ++u) {
        const int e = tid + kThreads * u;
        xs[(e % BK) * XS + e / BK] = xsr[u];
      }
    }
    T* ss = Ss + buf * BK * SP;
#pragma unroll
    for (int u = 0; u < SE; ++u) {
      const int e = tid + kThreads * u;
      ss[(e / CPAD) * SP + e % CPAD] = sr[u];
    }
  };

  T* WsT = nullptr;
  double* HH = nullptr;
  if constexpr (METRICS) {
    WsT = reinterpret_cast<T*>(smem + L::wt_off);  // [CPAD][XS]
    HH = reinterpret_cast<double*>(smem + L::hh_off);
    for (int e = tid; e < CPAD * kBM; e += kThreads) {
      const int j = e / kBM, r = e % kBM;
      const int64_t gr = row0 + r;
      WsT[j * XS + r] = (j < k && gr < m) ? W[gr * k + j] : T(0);
    }
    for (int e = tid; e < k * k; e += kThreads) HH[e] = hht[e];
  }

  T acc[8][TC];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int t = 0; t < TC; ++t) acc[i][t] = T(0);
  double rss = 0.0;

  const int64_t nk = ceil_div(n, BK);
  gload(0);
  sstore(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) gload((kt + 1) * BK);
    const T* xs = Xs + buf * BK * XS;
    const T* ss = Ss + buf * BK * SP;
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      T a[8];
      load8(xs + kk * XS + ty * 8, a);
      T b[TC];
#pragma unroll
      for (int t = 0; t < TC; ++t) b[t] = ss[kk * SP + tx + 16 * t];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int t = 0; t < TC; ++t) acc[i][t] = fma(a[i], b[t], acc[i][t]);
    }
    if constexpr (METRICS) {
      // residual (X - W H) on this tile: rows ty*8.., K-columns tx + 16 q
      const int64_t k0 = kt * BK;
      T tile_ss = T(0);
#pragma unroll
      for (int q = 0; q < BK / 16; ++q) {
        const int kk = tx + 16 * q;
        if (k0 + kk < n) {
          T dot[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) dot[i] = T(0);
          for (int j = 0; j < k; ++j) {
            const T sv = ss[kk * SP + j];
            T wv[8];
            load8(WsT + j * XS + ty * 8, wv);
#pragma unroll
            for (int i = 0; i < 8; ++i) dot[i] = fma(wv[i], sv, dot[i]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (row0 + ty * 8 + i < m) {
              const T r = xs[kk * XS + ty * 8 + i] - dot[i];
              tile_ss = fma(r, r, tile_ss);
            }
          }
        }
      }
      rss += double(tile_ss);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }

  if constexpr (!METRICS) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t r = row0 + ty * 8 + i;
      if (r >= m) continue;
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        const int j = tx + 16 * t;
        if (j < c) Y[r * c + j] = acc[i][t];
      }
    }
  } else {
    double pgw = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rl = ty * 8 + i;
      if (row0 + rl >= m) continue;
#pragma unroll
      for (int t = 0; t < TC; ++t) {
        const int j = tx + 16 * t;
        if (j >= k) continue;
        double wv = 0.0;
        for (int q = 0; q < k; ++q) wv += double(WsT[q * XS + rl]) * HH[q * k + j];
        const double g = -2.0 * (double(acc[i][t]) - wv);
        const double gp = WsT[j * XS + rl] > T(0) ? g : fmin(g, 0.0);
        pgw += gp * gp;
      }
    }
    __shared__ double red[2][kThreads / 32];
    rss = warp_allreduce_sum(rss);
    pgw = warp_allreduce_sum(pgw);
    if (lane_id() == 0) {
      red[0][warp_id()] = rss;
      red[1][warp_id()] = pgw;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) a += red[0][w], b += red[1][w];
      part_obj[blockIdx.x] = a;
      part_pgw[blockIdx.x] = b;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// xtw: part[s] = X[rows_s]^T S[rows_s].  CTA (bx, s) owns 128 columns of X (= output rows) and
// row slice s of X; it walks the rows in BK chunks.  X tiles are [BK][128] row-major slices, read
// with 16-byte vectors along the contiguous column dimension.
template <typename T, int CPAD, bool VECX>
__global__ void __launch_bounds__(kThreads) xtw_kernel(const T* __restrict__ X, int64_t m, int64_t n, int64_t ldx,
                                                       const T* __restrict__ S, int c, T* __restrict__ part,
                                                       int splits) {
  using L = XwSmem<T, CPAD>;
  constexpr int BK = Tile<T>::BK, VN = Tile<T>::VN, TC = CPAD / 16, XS = L::XS, SP = L::SP;
  using V = typename Tile<T>::V;
  extern __shared__ __align__(16) unsigned char smem[];
  T* Xs = reinterpret_cast<T*>(smem);
  T* Ss = reinterpret_cast<T*>(smem + L::s_off);

  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t n0 = int64_t(blockIdx.x) * kBM;
  const int s = blockIdx.y;
  const int64_t rbeg = m * s / splits, rend = m * (s + 1) / splits;

  constexpr int XV = kBM * BK / VN / kThreads;
  constexpr int XE = kBM * BK / kThreads;
  constexpr int SE = BK * CPAD / kThreads;
  V xr[VECX ? XV : 1];
  T xsr[VECX ? 1 : XE];
  T sr[SE];

  auto gload = [&](int64_t r0) {
    if constexpr (VECX) {
#pragma unroll
      for (int u = 0; u < XV; ++u) {
        const int v = tid + kThreads * u;
        const int kk = v / (kBM / VN), nv = v % (kBM / VN);
        const int64_t gr = r0 + kk, gn = n0 + int64_t(nv) * VN;
        if (gr < rend && gn < n)
          xr[u] = __ldcs(reinterpret_cast<const V*>(X + gr * ldx + gn));
        else
          xr[u] = V{};
      }
    } else {
#pragma unroll
      for (int u = 0; u < XE; ++u) {
        const int e = tid + kThreads * u;
        const int kk = e / kBM, nl = e % kBM;
        const int64_t gr = r0 + kk, gn = n0 + nl;
        xsr[u] = (gr < rend && gn < n) ? __ldcs(X + gr * ldx + gn) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < SE; ++u) {
      const int e = tid + kThreads * u;
      const int kk = e / CPAD, j = e % CPAD;
      const int64_t gr = r0 + kk;
      sr[u] = (gr < rend && j < c) ? S[gr * c + j] : T(0);
    }
  };
  auto sstore = [&](int buf) {
    T* xs = Xs + buf * BK * XS;
    if constexpr (VECX) {
#pragma unroll
      for (int u = 0; u < XV; ++u) {
        const int v = tid + kThreads * u;
        const int kk = v / (kBM / VN), nv = v % (kBM / VN);
        *reinterpret_cast<V*>(xs + kk * XS + nv * VN) = xr[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < XE; ++u) {
        const int e = tid + kThreads * u;
        xs[(e / kBM) * XS + e % kBM] = xsr[u];
      }
    }
    T* ss = Ss + buf * BK * SP;
#pragma unroll
    for (int u = 0; u < SE; ++u) {
      const int e = tid + kThreads * u;
      ss[(e / CPAD) * SP + e % CPAD] = sr[u];
    }
  };

  T acc[8][TC];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int t = 0; t < TC; ++t) acc[i][t] = T(0);

  const int64_t nk = ceil_div(rend - rbeg, BK);
  if (nk > 0) {
    gload(rbeg);
    sstore(0);
  }
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) gload(rbeg + (kt + 1) * BK);
    const T* xs = Xs + buf * BK * XS;
    const T* ss = Ss + buf * BK * SP;
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      T a[8];
      load8(xs + kk * XS + ty * 8, a);
      T b[TC];
#pragma unroll
      for (int t = 0; t < TC; ++t) b[t] = ss[kk * SP + tx + 16 * t];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int t = 0; t < TC; ++t) acc[i][t] = fma(a[i], b[t], acc[i][t]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
  T* out = part + int64_t(s) * n * c;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gn = n0 + ty * 8 + i;
    if (gn >= n) continue;
#pragma unroll
    for (int t = 0; t < TC; ++t) {
      const int j = tx + 16 * t;
      if (j < c) out[gn * c + j] = acc[i][t];
    }
  }
}

// Fixed-order reduction of the split partials: out[n][c] (or out[c][n]) = sum_s part[s][n][c].
template <typename T>
__global__ void splitk_reduce_kernel(const T* __restrict__ part, int splits, int64_t n, int c,
                                     T* __restrict__ out, bool transpose_out) {
  const int64_t total = n * c;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < splits; ++s) acc += double(part[int64_t(s) * total + e]);
    const int64_t ni = e / c;
    const int j = int(e % c);
    if (transpose_out)
      out[int64_t(j) * n + ni] = T(acc);
    else
      out[e] = T(acc);
  }
}

// Metrics grad_H epilogue: for each (X column col, j), sum the split partials of (W^T X)(j, col) in
// fixed order, form grad_H(j, col) = -2 ((W^T X)(j, col) - ((W^T W) H)(j, col)), project by
// H(j, col), square; one partial sum per CTA.
// grad_H = -2 (sum_s part[s] - (W^T W) H), projected: a block covers 64 (col, j) entries with 4
// split groups each (group g sums s = g, g + 4, ... with 4 independent accumulators, all loads of
// an unrolled step in flight); the groups are combined in fixed order (deterministic).
constexpr int kGhEntries = 64, kGhGroups = kThreads / kGhEntries;
template <typename T>
__global__ void __launch_bounds__(kThreads) xtw_metrics_reduce_kernel(const T* __restrict__ part, int splits,
                                                                      int64_t n, int k,
                                                                      const T* __restrict__ H,
                                                                      const double* __restrict__ wtw,
                                                                      double* part_pgh) {
  __shared__ double gsum[kGhGroups][kGhEntries];
  __shared__ double bsum[kGhGroups][kGhEntries];
  __shared__ double red[kThreads / 32];
  const int ei = threadIdx.x % kGhEntries, gi = threadIdx.x / kGhEntries;
  const int64_t e = int64_t(blockIdx.x) * kGhEntries + ei;  // e = col * k + j
  const int64_t total = n * k;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  if (e < total) {
    int s = gi;
    for (; s + 3 * kGhGroups < splits; s += 4 * kGhGroups) {
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = part[int64_t(s + u * kGhGroups) * total + e];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] += double(v[u]);
    }
    for (; s < splits; s += kGhGroups) a[0] += double(part[int64_t(s) * total + e]);
  }
  gsum[gi][ei] = (a[0] + a[1]) + (a[2] + a[3]);
  // ((W^T W) H)(j, col): the k-long dot product split over the 4 groups as well (t = gi, gi + 4, ..)
  const int64_t col = e < total ? e / k : 0;
  const int j = e < total ? int(e - col * k) : 0;
  double bp = 0.0;
  if (e < total)
    for (int t = gi; t < k; t += kGhGroups) bp += wtw[j * k + t] * double(H[int64_t(t) * n + col]);
  bsum[gi][ei] = bp;
  __syncthreads();
  double acc = 0.0;
  if (gi == 0 && e < total) {
    double wx = 0.0, b = 0.0;
#pragma unroll
    for (int g = 0; g < kGhGroups; ++g) wx += gsum[g][ei];
#pragma unroll
    for (int g = 0; g < kGhGroups; ++g) b += bsum[g][ei];
    const double g = -2.0 * (wx - b);
    const double hv = double(H[int64_t(j) * n + col]);
    const double gp = hv > 0.0 ? g : fmin(g, 0.0);
    acc = gp * gp;
  }
  acc = warp_allreduce_sum(acc);
  if (lane_id() == 0) red[warp_id()] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    part_pgh[blockIdx.x] = t;
  }
}

// ---- small helpers ---------------------------------------------------------------------------
constexpr int kGramChunk = 64;
constexpr int kGramAcc = 16;  // entries per thread -> c <= 64

// part[b] = A[rows of b]^T A[rows of b] (c x c), rows split evenly over gridDim.x CTAs.
// Register-blocked: thread (block bi, bj; row group grp) keeps a 4 x 4 block of the Gram in fp64
// registers and walks the rows grp, grp + G, .. of each 64-row chunk (two 16-byte loads per operand
// for 16 DFMAs; the one-entry-per-thread version was shared-memory-load bound, 170 us at C4 size);
// the G row groups are summed in a fixed order at the end.
template <typename T>
__global__ void __launch_bounds__(kThreads) gram_rows_kernel(const T* __restrict__ A, int64_t rows, int c,
                                                             double* part) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* tile = reinterpret_cast<double*>(smem);  // [kGramChunk][cp], reused as red[G][cp * cp]
  const int cp = (c + 3) & ~3;
  const int nb = cp / 4, nblk = nb * nb;
  const int G = kThreads / nblk;  // >= 1 for c <= 64
  const int tid = threadIdx.x;
  const int blk = tid % nblk, grp = tid / nblk;
  const bool active = grp < G;
  const int bi = blk / nb, bj = blk % nb;
  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int cc = c * c;
  double acc[4][4] = {};
  for (int e = tid; e < kGramChunk * cp; e += kThreads) tile[e] = 0.0;  // the pad columns stay zero
  for (int64_t base = r0; base < r1; base += kGramChunk) {
    const int nr = int(r1 - base < kGramChunk ? r1 - base : kGramChunk);
    __syncthreads();
    const T* src = A + base * c;  // nr rows, contiguous
    for (int e = tid; e < nr * c; e += kThreads) {
      const int r = e / c;
      tile[r * cp + (e - r * c)] = double(src[e]);
    }
    __syncthreads();
    if (active) {
      for (int r = grp; r < nr; r += G) {
        const double2* ta = reinterpret_cast<const double2*>(tile + r * cp + 4 * bi);
        const double2* tb = reinterpret_cast<const double2*>(tile + r * cp + 4 * bj);
        const double2 a0 = ta[0], a1 = ta[1], b0 = tb[0], b1 = tb[1];
        const double av[4] = {a0.x, a0.y, a1.x, a1.y}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] += av[x] * bv[y];
      }
    }
  }
  __syncthreads();
  double* red = tile;
  if (active) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) red[grp * cp * cp + (4 * bi + x) * cp + 4 * bj + y] = acc[x][y];
  }
  __syncthreads();
  for (int e = tid; e < cc; e += kThreads) {
    const int i = e / c, j = e - i * c;
    double sum = 0.0;
    for (int g2 = 0; g2 < G; ++g2) sum += red[g2 * cp * cp + i * cp + j];
    part[int64_t(blockIdx.x) * cc + e] = sum;
  }
}

// part[b] = A[:, cols of b] A[:, cols of b]^T (c x c) for A (c x cols) row-major.
template <typename T>
__global__ void __launch_bounds__(kThreads) gram_cols_kernel(const T* __restrict__ A, int c, int64_t cols,
                                                             double* part) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* tile = reinterpret_cast<double*>(smem);  // [c][kGramChunk]
  const int64_t c0 = cols * blockIdx.x / gridDim.x, c1 = cols * (blockIdx.x + 1) / gridDim.x;
  const int cc = c * c;
  double acc[kGramAcc] = {};
  for (int64_t base = c0; base < c1; base += kGramChunk) {
    const int nc = int(c1 - base < kGramChunk ? c1 - base : kGramChunk);
    __syncthreads();
    for (int e = threadIdx.x; e < c * kGramChunk; e += kThreads) {
      const int a = e / kGramChunk, q = e % kGramChunk;
      tile[e] = q < nc ? double(A[int64_t(a) * cols + base + q]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kGramAcc; ++u) {
      const int e = threadIdx.x + kThreads * u;
      if (e < cc) {
        const int a = e / c, b = e % c;
        double s = acc[u];
        for (int q = 0; q < nc; ++q) s += tile[a * kGramChunk + q] * tile[b * kGramChunk + q];
        acc[u] = s;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kGramAcc; ++u) {
    const int e = threadIdx.x + kThreads * u;
    if (e < cc) part[int64_t(blockIdx.x) * cc + e] = acc[u];
  }
}

// out[e] = sum_p part[p][e]: a block covers 64 entries x 4 part groups (4 independent loads in
// flight per thread), groups combined in fixed order (deterministic)
// (called in place, out == part, by the CholeskyQR Gram reduction: no __restrict__; each entry is
// read by its own block before that block writes it)
__global__ void __launch_bounds__(256) reduce_parts_kernel(const double* part, int nparts, int len, double* out) {
  // 32 entries x 8 part-slices per block; each slice keeps 8 independent loads in flight, the
  // slices are combined in fixed order (deterministic)
  __shared__ double gs[8][33];
  const int ei = threadIdx.x % 32, gi = threadIdx.x / 32;
  const int e = blockIdx.x * 32 + ei;
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (e < len) {
    int p = gi;
    for (; p + 56 < nparts; p += 64) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[int64_t(p + 8 * u) * len + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += v[u];
    }
    for (; p < nparts; p += 8) a[0] += part[int64_t(p) * len + e];
  }
  gs[gi][ei] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  if (gi == 0 && e < len) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += gs[q][ei];
    out[e] = t;
  }
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t rows, int64_t cols, T* __restrict__ out) {
  __shared__ T tile[32][33];
  const int64_t bx = int64_t(blockIdx.x) * 32, by = int64_t(blockIdx.y) * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = by + j, cidx = bx + threadIdx.x;
    if (r < rows && cidx < cols) tile[j][threadIdx.x] = in[r * cols + cidx];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = bx + j, cidx = by + threadIdx.x;  // out is cols x rows
    if (r < cols && cidx < rows) out[r * rows + cidx] = tile[threadIdx.x][j];
  }
}

template <typename T>
__global__ void scale_cast_kernel(const double* __restrict__ in, int64_t count, double scale, T* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = T(in[i] * scale);
}

template <typename T>
__global__ void widen_kernel(const T* __restrict__ in, int64_t count, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = double(in[i]);
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int count, double* out) {
  double v = 0.0;
  for (int i = lane_id(); i < count; i += 32) v += part[i];
  v = warp_allreduce_sum(v);
  if (threadIdx.x == 0) out[0] = v;
}

// res[0] = sum(pobj), res[1] = sum(ppgw) + sum(ppgh): the three partial sums of the metrics in one
// warp each (fixed order), one launch
__global__ void metrics_finalize_kernel(const double* __restrict__ pobj, int nobj, const double* __restrict__ ppgw,
                                        int npgw, const double* __restrict__ ppgh, int npgh, double* res) {
  __shared__ double v3[3];
  const int w = threadIdx.x / 32;
  const double* p = w == 0 ? pobj : w == 1 ? ppgw : ppgh;
  const int cnt = w == 0 ? nobj : w == 1 ? npgw : npgh;
  double v = 0.0;
  for (int i = lane_id(); i < cnt; i += 32) v += p[i];
  v = warp_allreduce_sum(v);
  if (lane_id() == 0) v3[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    res[0] = v3[0];
    res[1] = v3[1] + v3[2];
  }
}

__global__ void timestamp_kernel(unsigned long long* out) { *out = globaltimer_ns(); }

template <typename F>
void set_smem(F* f, size_t bytes) {
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

inline bool x_vec_ok(const void* x, int64_t n, int64_t ldx, int vn, size_t esz) {
  return (reinterpret_cast<uintptr_t>(x) % (vn * esz)) == 0 && (n % vn) == 0 && (ldx % vn) == 0;
}

template <typename T, int CPAD>
void xw_dispatch_vec(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, cudaStream_t st) {
  using L = XwSmem<T, CPAD>;
  const size_t sm = L::base;
  const dim3 grid(unsigned(ceil_div(m, kBM)));
  if (x_vec_ok(x, n, ldx, Tile<T>::VN, sizeof(T))) {
    auto f = xw_kernel<T, CPAD, true, false>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, s, c, y, nullptr, 0, nullptr, nullptr, nullptr);
  } else {
    auto f = xw_kernel<T, CPAD, false, false>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, s, c, y, nullptr, 0, nullptr, nullptr, nullptr);
  }
  RNMF_CUDA_LAUNCH();
}

template <typename T, int CPAD>
void xw_metrics_dispatch(const T* x, int64_t m, int64_t n, int64_t ldx, const T* ht, const T* w, int k,
                         const double* hht, double* po, double* pw, cudaStream_t st) {
  using L = XwSmem<T, CPAD>;
  const size_t sm = L::metrics_total;
  const dim3 grid(unsigned(ceil_div(m, kBM)));
  if (x_vec_ok(x, n, ldx, Tile<T>::VN, sizeof(T))) {
    auto f = xw_kernel<T, CPAD, true, true>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, ht, k, nullptr, w, k, hht, po, pw);
  } else {
    auto f = xw_kernel<T, CPAD, false, true>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, ht, k, nullptr, w, k, hht, po, pw);
  }
  RNMF_CUDA_LAUNCH();
}

template <typename T, int CPAD>
void xtw_dispatch(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits, cudaStream_t st) {
  using L = XwSmem<T, CPAD>;
  const size_t sm = L::base;
  const dim3 grid(unsigned(ceil_div(n, kBM)), unsigned(splits));
  if (x_vec_ok(x, n, ldx, Tile<T>::VN, sizeof(T))) {
    auto f = xtw_kernel<T, CPAD, true>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, s, c, part, splits);
  } else {
    auto f = xtw_kernel<T, CPAD, false>;
    set_smem(f, sm);
    f<<<grid, kThreads, sm, st>>>(x, m, n, ldx, s, c, part, splits);
  }
  RNMF_CUDA_LAUNCH();
}

#define RNMF_CPAD_SWITCH(c, CALL)                                                   \
  do {                                                                              \
    if ((c) <= 16) { constexpr int CP = 16; CALL; }                                 \
    else if ((c) <= 32) { constexpr int CP = 32; CALL; }                            \
    else if ((c) <= 48) { constexpr int CP = 48; CALL; }                            \
    else if ((c) <= 64) { constexpr int CP = 64; CALL; }                            \
    else if ((c) <= 96) { constexpr int CP = 96; CALL; }                            \
    else if ((c) <= 128) { constexpr int CP = 128; CALL; }                          \
    else throw CudaError("X-streaming GEMM: column count " + std::to_string(c) +    \
                         " exceeds 128");                                           \
  } while (0)

}  // namespace

// ================================================================================================
template <typename T>
int launch_xw(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, cudaStream_t stream) {
  RNMF_CPAD_SWITCH(c, (xw_dispatch_vec<T, CP>(x, m, n, ldx, s, c, y, stream)));
  return 1;
}

int xw_metrics_blocks(int64_t m) { return int(ceil_div(m, kBM)); }

template <typename T>
int launch_xw_metrics(const T* x, int64_t m, int64_t n, int64_t ldx, const T* ht, const T* w, int k,
                      const double* hht, double* part_obj, double* part_pgw, int* nblocks,
                      cudaStream_t stream) {
  RNMF_CPAD_SWITCH(k, (xw_metrics_dispatch<T, CP>(x, m, n, ldx, ht, w, k, hht, part_obj, part_pgw, stream)));
  *nblocks = xw_metrics_blocks(m);
  return 1;
}

int xtw_default_splits(int64_t m, int64_t n) {
  const int64_t colblocks = ceil_div(n, kBM);
  const int64_t target = 2 * 148;
  int64_t s = ceil_div(target, colblocks);
  s = std::max<int64_t>(1, std::min<int64_t>(s, ceil_div(m, 64)));
  return int(std::min<int64_t>(s, 1024));
}

template <typename T>
int launch_xtw(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits, T* out,
               bool transpose_out, cudaStream_t stream) {
  if (splits <= 0) splits = xtw_default_splits(m, n);
  RNMF_CPAD_SWITCH(c, (xtw_dispatch<T, CP>(x, m, n, ldx, s, c, part, splits, stream)));
  const int64_t total = n * c;
  const int blocks = int(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  splitk_reduce_kernel<T><<<blocks, 256, 0, stream>>>(part, splits, n, c, out, transpose_out);
  RNMF_CUDA_LAUNCH();
  return 2;
}

template <typename T>
int launch_xtw_metrics(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, int k, const T* h,
                       const double* wtw, T* part, int splits, double* part_pgh, int* nblocks,
                       cudaStream_t stream) {
  if (splits <= 0) splits = xtw_default_splits(m, n);
  RNMF_CPAD_SWITCH(k, (xtw_dispatch<T, CP>(x, m, n, ldx, w, k, part, splits, stream)));
  int b = 0;
  launch_grad_h_reduce<T>(part, splits, n, k, h, wtw, part_pgh, &b, stream);
  *nblocks = b;
  return 2;
}

template <typename T>
int launch_grad_h_reduce(const T* part, int splits, int64_t n, int k, const T* h, const double* wtw, double* part_pgh,
                         int* nblocks, cudaStream_t stream) {
  const int blocks = int(ceil_div(n * k, kGhEntries));
  xtw_metrics_reduce_kernel<T><<<blocks, kThreads, 0, stream>>>(part, splits, n, k, h, wtw, part_pgh);
  RNMF_CUDA_LAUNCH();
  *nblocks = blocks;
  return 1;
}

template <typename T>
int launch_splitk_reduce(const T* part, int splits, int64_t n, int c, T* out, bool transpose_out, cudaStream_t stream) {
  const int64_t total = n * c;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 8)));
  splitk_reduce_kernel<T><<<blocks, 256, 0, stream>>>(part, splits, n, c, out, transpose_out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int64_t grad_h_blocks(int64_t n, int k) { return ceil_div(n * k, kGhEntries); }

int gram_parts(int64_t len) { return int(std::max<int64_t>(1, std::min<int64_t>(296, ceil_div(len, 16)))); }

template <typename T>
int launch_gram_rows(const T* a, int64_t rows, int c, double* part, double* g, cudaStream_t stream) {
  if (c > 64) throw CudaError("gram: column count above 64 not supported");
  const int np = gram_parts(rows);
  const int cp = (c + 3) & ~3, groups = kThreads / ((cp / 4) * (cp / 4));
  const size_t sm = size_t(std::max(kGramChunk * cp, groups * cp * cp)) * sizeof(double);
  gram_rows_kernel<T><<<np, kThreads, sm, stream>>>(a, rows, c, part);
  RNMF_CUDA_LAUNCH();
  reduce_parts_kernel<<<unsigned(ceil_div(c * c, 32)), 256, 0, stream>>>(part, np, c * c, g);
  RNMF_CUDA_LAUNCH();
  return 2;
}

template <typename T>
int launch_gram_cols(const T* a, int c, int64_t cols, double* part, double* g, cudaStream_t stream) {
  if (c > 64) throw CudaError("gram: row count above 64 not supported");
  const int np = gram_parts(cols);
  const size_t sm = size_t(kGramChunk) * c * sizeof(double);
  gram_cols_kernel<T><<<np, kThreads, sm, stream>>>(a, c, cols, part);
  RNMF_CUDA_LAUNCH();
  reduce_parts_kernel<<<unsigned(ceil_div(c * c, 32)), 256, 0, stream>>>(part, np, c * c, g);
  RNMF_CUDA_LAUNCH();
  return 2;
}

template <typename T>
int launch_transpose(const T* in, int64_t rows, int64_t cols, T* out, cudaStream_t stream) {
  const dim3 grid(unsigned(ceil_div(cols, 32)), unsigned(ceil_div(rows, 32)));
  transpose_kernel<T><<<grid, dim3(32, 8), 0, stream>>>(in, rows, cols, out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

template <typename T>
int launch_scale_cast(const double* in, int64_t count, double scale, T* out, cudaStream_t stream) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 148 * 8)));
  scale_cast_kernel<T><<<blocks, 256, 0, stream>>>(in, count, scale, out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

template <typename T>
int launch_widen(const T* in, int64_t count, double* out, cudaStream_t stream) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), 148 * 8)));
  widen_kernel<T><<<blocks, 256, 0, stream>>>(in, count, out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int launch_reduce_parts(const double* part, int nparts, int len, double* out, cudaStream_t stream) {
  reduce_parts_kernel<<<unsigned(ceil_div(len, 32)), 256, 0, stream>>>(part, nparts, len, out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int launch_metrics_finalize(const double* pobj, int nobj, const double* ppgw, int npgw, const double* ppgh, int npgh,
                            double* res, cudaStream_t stream) {
  metrics_finalize_kernel<<<1, 96, 0, stream>>>(pobj, nobj, ppgw, npgw, ppgh, npgh, res);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int launch_sum_parts(const double* part, int count, double* out, cudaStream_t stream) {
  sum_parts_kernel<<<1, 32, 0, stream>>>(part, count, out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int launch_timestamp(unsigned long long* out, cudaStream_t stream) {
  timestamp_kernel<<<1, 1, 0, stream>>>(out);
  RNMF_CUDA_LAUNCH();
  return 1;
}

#define RNMF_INST(T)                                                                                          \
  template int launch_xw<T>(const T*, int64_t, int64_t, int64_t, const T*, int, T*, cudaStream_t);           \
  template int launch_xw_metrics<T>(const T*, int64_t, int64_t, int64_t, const T*, const T*, int, const double*, \
                                    double*, double*, int*, cudaStream_t);                                    \
  template int launch_xtw<T>(const T*, int64_t, int64_t, int64_t, const T*, int, T*, int, T*, bool, cudaStream_t); \
  template int launch_xtw_metrics<T>(const T*, int64_t, int64_t, int64_t, const T*, int, const T*, const double*, T*, \
                                     int, double*, int*, cudaStream_t);                                       \
  template int launch_splitk_reduce<T>(const T*, int, int64_t, int, T*, bool, cudaStream_t);                 \
  template int launch_grad_h_reduce<T>(const T*, int, int64_t, int, const T*, const double*, double*, int*,   \
                                       cudaStream_t);                                                         \
  template int launch_gram_rows<T>(const T*, int64_t, int, double*, double*, cudaStream_t);                  \
  template int launch_gram_cols<T>(const T*, int, int64_t, double*, double*, cudaStream_t);                  \
  template int launch_transpose<T>(const T*, int64_t, int64_t, T*, cudaStream_t);                            \
  template int launch_scale_cast<T>(const double*, int64_t, double, T*, cudaStream_t);                       \
  template int launch_widen<T>(const T*, int64_t, double*, cudaStream_t);

RNMF_INST(float)
RNMF_INST(double)

}  // namespace rnmf_gpu
