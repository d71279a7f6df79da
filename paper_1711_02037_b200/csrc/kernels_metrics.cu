// kernels_metrics.cu — full-space metrics in ONE pass over X (full_space_metrics,
// p/src/rhals.cpp:140-148): objective ||X - W H||^2 from the explicit residual (as the reference
// computes it), grad_W = -2 (X H^T - W (H H^T)) projected by W, and the per-row-tile partials of
// W^T X (one slot per persistent CTA) that the grad_H reduction (xtw_metrics_reduce) finishes.  FMA arithmetic in the working
// precision (the EXACT / verification math mode).
//
// CTA = 128 rows of X, walking the columns in 32-wide chunks; the next chunk is prefetched into
// registers (16-byte loads) while the current one is consumed from shared memory.  2 CTAs / SM.  Per chunk each thread computes (register blocked):
//   WH     rows 8ty..8ty+7  x cols 2tx, 2tx+1       (16 outputs, k FMAs each)  -> residual^2
//   X H^T  rows 8ty..8ty+7  x j = tx + 16 u         (accumulated over all chunks)
//   W^T X  j 4jq..4jq+3     x cols 4cq..4cq+3 over a 128/RQ row slice, combined through smem
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kMThreads = 256;
constexpr int kMBM = 128;  // rows per tile
constexpr int kMBN = 32;   // columns per chunk

template <typename T, int KP>
struct MetCfg {
  static constexpr int kXR = kMBN + 4;          // Xr[r][c] row stride (keeps 16 B alignment)
  static constexpr int kWS = kMBM + 4;          // WsT[j][r]
  static constexpr int kWR = KP + 4;            // Wr[r][j]
  static constexpr int kHS = kMBN + 4;          // Hs[j][c]
  static constexpr int RQ = kMThreads / (2 * KP);  // row slices for W^T X
  static constexpr size_t xr = 0;
  static constexpr size_t ws = xr + sizeof(T) * size_t(kMBM) * kXR;
  static constexpr size_t wr = ws + sizeof(T) * size_t(KP) * kWS;
  static constexpr size_t hs = wr + sizeof(T) * size_t(kMBM) * kWR;
  static constexpr size_t wx = hs + sizeof(T) * size_t(KP) * kHS;   // [RQ][KP][32] partials
  static constexpr size_t hh = wx + sizeof(T) * size_t(RQ) * KP * kMBN;
  static constexpr size_t total = hh + sizeof(double) * size_t(KP) * KP + 64;
};

template <typename T>
struct V4;
template <>
struct V4<float> {
  using type = float4;
};
template <>
struct V4<double> {
  using type = double2;
};

template <typename T, int KP>
__global__ void __launch_bounds__(kMThreads, 2) metrics_kernel(const T* __restrict__ X, int64_t m, int64_t n,
                                                               int64_t ldx, const T* __restrict__ W,
                                                               const T* __restrict__ H, int k,
                                                               const double* __restrict__ hht,
                                                               T* __restrict__ wtx_part, double* part_obj,
                                                               double* part_pgw) {
  const bool do_wtx = wtx_part != nullptr;
  using C = MetCfg<T, KP>;
  constexpr int RQ = C::RQ;
  constexpr int ROWS_Q = kMBM / RQ;  // rows per W^T X slice
  extern __shared__ __align__(16) unsigned char smem[];
  T* Xr = reinterpret_cast<T*>(smem + C::xr);
  T* WsT = reinterpret_cast<T*>(smem + C::ws);
  T* Wr = reinterpret_cast<T*>(smem + C::wr);
  T* Hs = reinterpret_cast<T*>(smem + C::hs);
  T* WX = reinterpret_cast<T*>(smem + C::wx);
  double* HH = reinterpret_cast<double*>(smem + C::hh);

  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  // W^T X decomposition: block (jq, cq) of 4 x 4 outputs, row slice rq
  const int blk = tid % (2 * KP), rq = tid / (2 * KP);
  const int jq = blk / 8, cq = blk % 8;

  for (int e = tid; e < k * k; e += kMThreads) HH[e] = hht[e];
  const int64_t ntiles = ceil_div(m, kMBM);
  const int64_t nchunks = ceil_div(n, kMBN);
  double obj = 0.0, pgw = 0.0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kMBM;
    __syncthreads();
    // W rows of the tile, both layouts (zero-padded to KP columns / past m)
    for (int e = tid; e < kMBM * KP; e += kMThreads) {
      const int r = e / KP, j = e % KP;
      const T v = (j < k && row0 + r < m) ? W[(row0 + r) * k + j] : T(0);
      WsT[j * C::kWS + r] = v;
      Wr[r * C::kWR + j] = v;
    }
    T xht[8][KP / 16];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int u = 0; u < KP / 16; ++u) xht[i][u] = T(0);

    // register prefetch of chunk 0: X as 16-byte vectors (the pitch ldx is a multiple of the
    // vector width and the pad columns are zero), H scalars
    using Vec = typename V4<T>::type;                  // 16-byte vector
    constexpr int EPV = 16 / sizeof(T);                // elements per vector
    constexpr int kXV = kMBM * kMBN / EPV / kMThreads; // vectors per thread
    constexpr int kHE = 64 * kMBN / kMThreads;        // H elements per thread (<= 8, KP <= 64)
    Vec xr[kXV];
    T hr[kHE];
    auto gload = [&](int64_t c0) {
#pragma unroll
      for (int u = 0; u < kXV; ++u) {
        const int v = tid + kMThreads * u;
        const int r = v / (kMBN / EPV), c4 = v % (kMBN / EPV);
        const int64_t gc = c0 + EPV * c4;
        if (row0 + r < m && gc < ldx)
          xr[u] = __ldcs(reinterpret_cast<const Vec*>(X + (row0 + r) * ldx + gc));
        else
          xr[u] = Vec{};
      }
#pragma unroll
      for (int u = 0; u < kHE; ++u) {
        const int e = tid + kMThreads * u;
        const int j = e / kMBN, c = e % kMBN;
        hr[u] = (e < KP * kMBN && j < k && c0 + c < n) ? H[int64_t(j) * n + c0 + c] : T(0);
      }
    };
    gload(0);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t c0 = ch * kMBN;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kXV; ++u) {
        const int v = tid + kMThreads * u;
        const int r = v / (kMBN / EPV), c4 = v % (kMBN / EPV);
        *reinterpret_cast<Vec*>(Xr + r * C::kXR + EPV * c4) = xr[u];
      }
#pragma unroll
      for (int u = 0; u < kHE; ++u) {
        const int e = tid + kMThreads * u;
        if (e < KP * kMBN) Hs[(e / kMBN) * C::kHS + e % kMBN] = hr[u];
      }
      __syncthreads();
      if (ch + 1 < nchunks) gload(c0 + kMBN);
      // ---- WH (rows 8ty.., cols 2tx, 2tx+1) and the residual
      {
        T wh[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) wh[i][0] = wh[i][1] = T(0);
        for (int j = 0; j < k; ++j) {
          const T* wp = WsT + j * C::kWS + ty * 8;
          const T h0 = Hs[j * C::kHS + 2 * tx], h1 = Hs[j * C::kHS + 2 * tx + 1];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const T wv = wp[i];
            wh[i][0] = fma(wv, h0, wh[i][0]);
            wh[i][1] = fma(wv, h1, wh[i][1]);
          }
        }
        T tss = T(0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = ty * 8 + i;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = 2 * tx + q;
            if (row0 + r < m && c0 + c < n) {
              const T rs = Xr[r * C::kXR + c] - wh[i][q];
              tss = fma(rs, rs, tss);
            }
          }
        }
        obj += double(tss);
      }
      // ---- X H^T accumulation (rows 8ty.., j = tx + 16 u)
#pragma unroll 4
      for (int c = 0; c < kMBN; ++c) {
        const T* xp = Xr + (ty * 8) * C::kXR + c;
        T xv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = xp[i * C::kXR];
#pragma unroll
        for (int u = 0; u < KP / 16; ++u) {
          const T hv = Hs[(tx + 16 * u) * C::kHS + c];
#pragma unroll
          for (int i = 0; i < 8; ++i) xht[i][u] = fma(xv[i], hv, xht[i][u]);
        }
      }
      // ---- W^T X over this tile's rows: block (jq, cq), slice rq
      if (do_wtx) {
        T acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
        for (int rr = 0; rr < ROWS_Q; ++rr) {
          const int r = rq * ROWS_Q + rr;
          const T* wp = Wr + r * C::kWR + jq * 4;
          const T* xp = Xr + r * C::kXR + cq * 4;
          T wv[4], xv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) wv[a] = wp[a], xv[a] = xp[a];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(wv[a], xv[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) WX[(rq * KP + jq * 4 + a) * kMBN + cq * 4 + b] = acc[a][b];
      }
      __syncthreads();
      // combine the RQ slices in fixed order and add this tile's contribution to the CTA's partial
      // of W^T X (slot blockIdx.x): the same thread owns the same (c, j) in every tile, so the
      // read-modify-write needs no synchronisation
      const bool first_tile = tile == blockIdx.x;
      for (int e = tid; e < (do_wtx ? k * kMBN : 0); e += kMThreads) {
        const int j = e / kMBN, c = e % kMBN;
        if (c0 + c < n) {
          T v = T(0);
#pragma unroll
          for (int q = 0; q < RQ; ++q) v += WX[(q * KP + j) * kMBN + c];
          T* dst = wtx_part + (int64_t(blockIdx.x) * n + c0 + c) * k + j;
          *dst = first_tile ? v : *dst + v;
        }
      }
    }
    // ---- projected grad_W for the tile's rows
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = ty * 8 + i;
      if (row0 + r >= m) continue;
#pragma unroll
      for (int u = 0; u < KP / 16; ++u) {
        const int j = tx + 16 * u;
        if (j >= k) continue;
        double wv = 0.0;
        for (int q = 0; q < k; ++q) wv += double(Wr[r * C::kWR + q]) * HH[q * k + j];
        const double g = -2.0 * (double(xht[i][u]) - wv);
        const double gp = Wr[r * C::kWR + j] > T(0) ? g : fmin(g, 0.0);
        pgw += gp * gp;
      }
    }
  }
  __shared__ double red[2][kMThreads / 32];
  obj = warp_allreduce_sum(obj);
  pgw = warp_allreduce_sum(pgw);
  if (lane_id() == 0) {
    red[0][warp_id()] = obj;
    red[1][warp_id()] = pgw;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kMThreads / 32; ++w) a += red[0][w], b += red[1][w];
    part_obj[blockIdx.x] = a;
    part_pgw[blockIdx.x] = b;
  }
}

template <typename T, int KP>
void metrics_dispatch(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, const T* h, int k, const double* hht,
                      T* wtx_part, double* po, double* pw, int grid, cudaStream_t st) {
  using C = MetCfg<T, KP>;
  auto f = metrics_kernel<T, KP>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::total)));
  f<<<grid, kMThreads, C::total, st>>>(x, m, n, ldx, w, h, k, hht, wtx_part, po, pw);
  RNMF_CUDA_LAUNCH();
}

}  // namespace

int metrics_tiles(int64_t m) { return int(ceil_div(m, kMBM)); }
// persistent: 2 resident CTAs per SM (__launch_bounds__(256, 2)), a CTA walks tiles blockIdx.x + i*grid
int metrics_grid(int64_t m, int sm_count) { return int(std::min<int64_t>(ceil_div(m, kMBM), 2 * int64_t(sm_count))); }

template <typename T>
int launch_metrics_fused(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, const T* h, int k,
                         const double* hht, T* wtx_part, double* part_obj, double* part_pgw, int sm_count,
                         cudaStream_t stream) {
  const int grid = metrics_grid(m, sm_count);
  if (sizeof(T) == 8 && k > 32) throw CudaError("metrics: fp64 rank above 32 (use the two-pass path)");
  if (k <= 16)
    metrics_dispatch<T, 16>(x, m, n, ldx, w, h, k, hht, wtx_part, part_obj, part_pgw, grid, stream);
  else if (k <= 32)
    metrics_dispatch<T, 32>(x, m, n, ldx, w, h, k, hht, wtx_part, part_obj, part_pgw, grid, stream);
  else if (k <= 64) {
    if constexpr (sizeof(T) == 4) metrics_dispatch<T, 64>(x, m, n, ldx, w, h, k, hht, wtx_part, part_obj, part_pgw, grid, stream);
  }
  else
    throw CudaError("metrics: rank above 64");
  return 1;
}

template int launch_metrics_fused<float>(const float*, int64_t, int64_t, int64_t, const float*, const float*, int,
                                         const double*, float*, double*, double*, int, cudaStream_t);
template int launch_metrics_fused<double>(const double*, int64_t, int64_t, int64_t, const double*, const double*, int,
                                          const double*, double*, double*, double*, int, cudaStream_t);

}  // namespace rnmf_gpu
