// kernels_metrics.cu — full-space metrics in ONE pass over X (full_space_metrics,
// p/src/rhals.cpp:140-148): objective ||X - W H||^2 from the explicit residual (as the reference
// computes it), grad_W = -2 (X H^T - W (H H^T)) projected by W, and per-CTA partials of W^T X
// that the grad_H reduction (launch_grad_h_reduce) finishes.  FMA arithmetic in the working
// precision (the EXACT / verification math mode).
//
// Persistent CTAs (2 per SM for fp32) walk 128-row tiles of X; within a tile the 32-column
// chunks of X and of a zero-padded copy of H arrive by TMA into an S-stage shared-memory ring
// (one thread issues, mbarrier completion), so no thread spends registers or issue slots on the
// X stream.  Out-of-range rows / columns arrive as zeros (TMA fill; W rows past m and H columns
// past n are zero too), which makes every product below exactly zero there: the inner loops
// carry no bounds checks.  Per chunk, register-blocked FMA products from shared memory:
//   WH, X H^T  one pass over j for RT rows x CT cols per thread (RT * CT = 16): the H(j, cols)
//           load feeds both products; X H^T keeps RT x KP accumulators over the whole tile,
//           summed over the column groups with shuffles at the end of the tile (grad_W
//           epilogue); WH gives the residual of the chunk
//   W^T X   4 j x 4 cols over a 128/RQ-row slice per thread, combined in fixed order through
//           shared memory into the CTA's partial (global, read-modify-write)
// Operands are read with 16-byte shared loads arranged so that each is reused at least four
// times (the previous row-major-only version was shared-memory-bandwidth bound).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kMThreads = 256;
constexpr int kMBM = 128;  // rows per tile
constexpr int kMBN = 32;   // columns per chunk

template <typename T, int KP>
struct MetCfg {
  static constexpr int S = (sizeof(T) == 8 || KP == 64) ? 2 : 3;  // TMA stages
  static constexpr int RT = KP >= 32 ? 1 : 32 / KP;               // rows per thread (WH, X H^T)
  static constexpr int CT = 16 / RT;                              // columns per thread (WH, X H^T)
  static constexpr int NCG = kMBN / CT;                           // column groups (adjacent lanes)
  static constexpr int RQ = kMThreads / (2 * KP);                 // W^T X row slices
  static constexpr int kWR = KP + 4;                              // Wr[r][j] row stride
  static constexpr int kWX = kMBN + 1;                            // WX[q][j][c] row stride
  static constexpr size_t xs_bytes = sizeof(T) * size_t(kMBM) * kMBN;
  static constexpr size_t hs_bytes = sizeof(T) * size_t(KP) * kMBN;
  static constexpr size_t xs = 0;                                  // S x [BM][BN]
  static constexpr size_t hs = xs + S * xs_bytes;                  // S x [KP][BN]
  static constexpr size_t ws = hs + S * hs_bytes;                  // WsT[j][r]
  static constexpr size_t wr = ws + sizeof(T) * size_t(KP) * kMBM; // Wr[r][j]
  static constexpr size_t wx = wr + sizeof(T) * size_t(kMBM) * kWR;
  static constexpr size_t hh = (wx + sizeof(T) * size_t(RQ) * KP * kWX + 15) / 16 * 16;
  static constexpr size_t bars = (hh + sizeof(double) * size_t(KP) * KP + 15) / 16 * 16;
  static constexpr size_t total = bars + 8 * S + 128;  // + alignment slack of the base
  static constexpr uint32_t stage_tx = uint32_t(xs_bytes + hs_bytes);
};

// N elements from shared memory with 16-byte loads (p 16-byte aligned)
template <typename T, int N>
__device__ __forceinline__ void ld16(const T* p, T (&v)[N]) {
  if constexpr (sizeof(T) == 4) {
    static_assert(N % 4 == 0, "");
#pragma unroll
    for (int u = 0; u < N / 4; ++u) {
      const float4 f = reinterpret_cast<const float4*>(p)[u];
      v[4 * u] = f.x, v[4 * u + 1] = f.y, v[4 * u + 2] = f.z, v[4 * u + 3] = f.w;
    }
  } else {
    static_assert(N % 2 == 0, "");
#pragma unroll
    for (int u = 0; u < N / 2; ++u) {
      const double2 d = reinterpret_cast<const double2*>(p)[u];
      v[2 * u] = d.x, v[2 * u + 1] = d.y;
    }
  }
}

template <typename T>
__global__ void pad_h_kernel(const T* __restrict__ h, int k, int64_t n, int kp, int64_t npad, T* __restrict__ hp) {
  const int64_t total = int64_t(kp) * npad;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / npad);
    const int64_t c = e % npad;
    hp[e] = (j < k && c < n) ? h[int64_t(j) * n + c] : T(0);
  }
}

template <typename T, int KP>
__global__ void __launch_bounds__(kMThreads, (sizeof(T) == 4 && KP <= 32) ? 2 : 1)
    metrics_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_h, int64_t m,
                   int64_t n, const T* __restrict__ W, int k, const double* __restrict__ hht,
                   T* __restrict__ wtx_part, double* part_obj, double* part_pgw) {
  using C = MetCfg<T, KP>;
  constexpr int S = C::S, RT = C::RT, CT = C::CT, NCG = C::NCG, RQ = C::RQ;
  constexpr int ROWS_Q = kMBM / RQ;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  T* WsT = reinterpret_cast<T*>(smem + C::ws);
  T* Wr = reinterpret_cast<T*>(smem + C::wr);
  T* WX = reinterpret_cast<T*>(smem + C::wx);
  double* HH = reinterpret_cast<double*>(smem + C::hh);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::bars);
  const bool do_wtx = wtx_part != nullptr;

  const int tid = threadIdx.x;
  const int rg = tid / NCG, cg = tid % NCG;             // WH / X H^T mapping
  const int blk = tid % (2 * KP), rq = tid / (2 * KP);  // W^T X mapping
  const int jq = blk / 8, cq = blk % 8;

  const int64_t ntiles = ceil_div(m, kMBM);
  const int64_t nch = ceil_div(n, kMBN);
  const int64_t my_tiles = int64_t(blockIdx.x) < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nch;

  if (tid == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_h);
    for (int s = 0; s < S; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  for (int e = tid; e < k * k; e += kMThreads) HH[(e / k) * KP + e % k] = hht[e];
  __syncthreads();

  auto issue = [&](int64_t q) {  // thread 0: chunk q of this CTA into stage q % S
    const int s = int(q % S);
    const int64_t tile = blockIdx.x + (q / nch) * gridDim.x, ch = q % nch;  // (thread 0 only)
    tc::mbar_arrive_expect_tx(&full[s], C::stage_tx);
    tc::tma_load_2d(smem + C::xs + s * C::xs_bytes, &map_x, &full[s], int(ch * kMBN), int(tile * kMBM));
    tc::tma_load_2d(smem + C::hs + s * C::hs_bytes, &map_h, &full[s], int(ch * kMBN), 0);
  };
  if (tid == 0)
    for (int64_t q = 0; q < (total < S - 1 ? total : S - 1); ++q) issue(q);

  double obj = 0.0, pgw = 0.0;
  T xh[RT][KP];
  // W^T X combine: this thread's fixed (c, j) entries of the 32 x k chunk block (e = tid + 256 u)
  constexpr int kCmb = (32 * KP + kMThreads - 1) / kMThreads;
  int cmb_c[kCmb], cmb_j[kCmb];
#pragma unroll
  for (int u = 0; u < kCmb; ++u) {
    const int e = tid + kMThreads * u;
    cmb_c[u] = e < k * kMBN ? e / k : kMBN;  // kMBN: inactive
    cmb_j[u] = e < k * kMBN ? e % k : 0;
  }
  T* const wtx_cta = do_wtx ? wtx_part + int64_t(blockIdx.x) * n * k : nullptr;
  int64_t tile = blockIdx.x, ch = 0;
  for (int64_t q = 0; q < total; ++q, ++ch) {
    if (ch == nch) ch = 0, tile += gridDim.x;
    const int64_t row0 = tile * kMBM, c0 = ch * kMBN;
    const bool first_tile = q < nch;
    if (ch == 0) {
      // W rows of the tile in both layouts, zero past m and past k
      for (int e = tid; e < kMBM * KP; e += kMThreads) {
        const int r = e / KP, j = e % KP;
        const T v = (j < k && row0 + r < m) ? W[(row0 + r) * k + j] : T(0);
        WsT[j * kMBM + r] = v;
        Wr[r * C::kWR + j] = v;
      }
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int j = 0; j < KP; ++j) xh[i][j] = T(0);
      __syncthreads();
    }
    if (tid == 0 && q + S - 1 < total) issue(q + S - 1);  // refills the stage consumed at q - 1
    const int s = int(q % S);
    tc::mbar_wait(&full[s], uint32_t((q / S) & 1));
    const T* Xs = reinterpret_cast<const T*>(smem + C::xs + s * C::xs_bytes);
    const T* Hs = reinterpret_cast<const T*>(smem + C::hs + s * C::hs_bytes);

    // ---- WH and X H^T for rows RT*rg.., columns CT*cg.. (all j), then the residual: per j one
    // 16-byte H load (8 lanes of a phase cover 128 contiguous bytes), W(rows, j) uniform per phase
    {
      T xv[RT][CT], wh[RT][CT];
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        ld16(Xs + (RT * rg + i) * kMBN + CT * cg, xv[i]);
#pragma unroll
        for (int c = 0; c < CT; ++c) wh[i][c] = T(0);
      }
#pragma unroll
      for (int j = 0; j < KP; ++j) {
        if (j < k) {
          T hv[CT], wv[RT];
          ld16(Hs + j * kMBN + CT * cg, hv);
          if constexpr (RT * sizeof(T) >= 16)
            ld16(WsT + j * kMBM + RT * rg, wv);
          else
#pragma unroll
            for (int i = 0; i < RT; ++i) wv[i] = WsT[j * kMBM + RT * rg + i];
#pragma unroll
          for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int c = 0; c < CT; ++c) {
              wh[i][c] = fma(wv[i], hv[c], wh[i][c]);
              xh[i][j] = fma(xv[i][c], hv[c], xh[i][j]);
            }
        }
      }
      T tss = T(0);
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int c = 0; c < CT; ++c) {
          const T rs = xv[i][c] - wh[i][c];
          tss = fma(rs, rs, tss);
        }
      obj += double(tss);
    }
    // ---- W^T X over this chunk: block (jq, cq), row slice rq
    if (do_wtx) {
      T acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
#pragma unroll 4
      for (int rr = 0; rr < ROWS_Q; ++rr) {
        const int r = rq * ROWS_Q + rr;
        T wv[4], xv[4];
        ld16(Wr + r * C::kWR + jq * 4, wv);
        ld16(Xs + r * kMBN + cq * 4, xv);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(wv[a], xv[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) WX[(rq * KP + jq * 4 + a) * C::kWX + cq * 4 + b] = acc[a][b];
    }
    __syncthreads();  // WX complete; stage s fully consumed
    if (do_wtx) {
      // fixed-order sum of the RQ slices into this CTA's partial of W^T X (slot blockIdx.x, layout
      // [n][k]); the same thread owns the same (c, j) in every tile (no synchronisation needed)
#pragma unroll
      for (int u = 0; u < kCmb; ++u) {
        const int c = cmb_c[u], j = cmb_j[u];
        if (c < kMBN && c0 + c < n) {
          T v = T(0);
#pragma unroll
          for (int qq = 0; qq < RQ; ++qq) v += WX[(qq * KP + j) * C::kWX + c];
          T* dst = wtx_cta + (c0 + c) * k + j;
          *dst = first_tile ? v : *dst + v;
        }
      }
    }
    __syncthreads();  // WX may be overwritten by the next chunk

    if (ch == nch - 1) {
      // ---- end of tile: X H^T summed over the NCG column groups (adjacent lanes, fixed
      // butterfly), then projected grad_W; group member cg takes j = cg, cg + NCG, ...
#pragma unroll
      for (int off = 1; off < NCG; off <<= 1)
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int j = 0; j < KP; ++j) xh[i][j] += __shfl_xor_sync(0xffffffffu, xh[i][j], off);
      // (W HH^T)(r, j) for the RT x KP/NCG owned outputs, independent accumulation chains
      constexpr int JPL = KP / NCG;  // j per lane
      double wv[RT][JPL];
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int t = 0; t < JPL; ++t) wv[i][t] = 0.0;
      for (int qq = 0; qq < k; ++qq) {
        double hq[JPL];
#pragma unroll
        for (int t = 0; t < JPL; ++t) hq[t] = HH[qq * KP + cg + NCG * t];
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const double wq = double(Wr[(RT * rg + i) * C::kWR + qq]);
#pragma unroll
          for (int t = 0; t < JPL; ++t) wv[i][t] = fma(wq, hq[t], wv[i][t]);
        }
      }
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int r = RT * rg + i;
#pragma unroll
        for (int t = 0; t < JPL; ++t) {
          const int j = cg + NCG * t;
          T xhj = T(0);
#pragma unroll
          for (int jj = 0; jj < KP; ++jj)
            if (jj == j) xhj = xh[i][jj];  // (unrolled select: xh stays in registers)
          if (row0 + r < m && j < k) {
            const double g = -2.0 * (double(xhj) - wv[i][t]);
            const double gp = Wr[r * C::kWR + j] > T(0) ? g : fmin(g, 0.0);
            pgw += gp * gp;
          }
        }
      }
      __syncthreads();  // Wr / WsT are rewritten by the next tile
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
                      T* hpad, T* wtx_part, double* po, double* pw, int grid, cudaStream_t st) {
  using C = MetCfg<T, KP>;
  const int64_t npad = ceil_div(n, kMBN) * kMBN;
  const int pgrid = int(std::min<int64_t>(ceil_div(int64_t(KP) * npad, 256), 1024));
  pad_h_kernel<T><<<pgrid, 256, 0, st>>>(h, k, n, KP, npad, hpad);
  RNMF_CUDA_LAUNCH();
  const CUtensorMap mx = make_tma_2d(x, int(sizeof(T)), m, n, ldx, kMBN, kMBM);
  const CUtensorMap mh = make_tma_2d(hpad, int(sizeof(T)), KP, npad, npad, kMBN, KP);
  auto f = metrics_kernel<T, KP>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::total)));
  f<<<grid, kMThreads, C::total, st>>>(mx, mh, m, n, w, k, hht, wtx_part, po, pw);
  RNMF_CUDA_LAUNCH();
}

int metrics_kp(int k) { return k <= 16 ? 16 : k <= 32 ? 32 : 64; }

}  // namespace

// persistent: up to 2 resident CTAs per SM (fp32, k <= 32), a CTA walks tiles blockIdx.x + i*grid
int metrics_grid(int64_t m, int k, int elem_bytes, int sm_count) {
  const int per_sm = (elem_bytes == 4 && k <= 32) ? 2 : 1;
  return int(std::min<int64_t>(ceil_div(m, kMBM), int64_t(per_sm) * sm_count));
}

int64_t metrics_hpad_len(int k, int64_t n) { return int64_t(metrics_kp(k)) * ceil_div(n, kMBN) * kMBN; }

template <typename T>
int launch_metrics_fused(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, const T* h, int k,
                         const double* hht, T* hpad, T* wtx_part, double* part_obj, double* part_pgw, int sm_count,
                         cudaStream_t stream) {
  const int grid = metrics_grid(m, k, int(sizeof(T)), sm_count);
  if (sizeof(T) == 8 && k > 32) throw CudaError("metrics: fp64 rank above 32 (use the two-pass path)");
  if ((ldx * int64_t(sizeof(T))) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    throw CudaError("metrics: X rows must be 16-byte aligned");
  if (k <= 16)
    metrics_dispatch<T, 16>(x, m, n, ldx, w, h, k, hht, hpad, wtx_part, part_obj, part_pgw, grid, stream);
  else if (k <= 32)
    metrics_dispatch<T, 32>(x, m, n, ldx, w, h, k, hht, hpad, wtx_part, part_obj, part_pgw, grid, stream);
  else if (k <= 64) {
    if constexpr (sizeof(T) == 4)
      metrics_dispatch<T, 64>(x, m, n, ldx, w, h, k, hht, hpad, wtx_part, part_obj, part_pgw, grid, stream);
  } else
    throw CudaError("metrics: rank above 64");
  return 2;
}

template int launch_metrics_fused<float>(const float*, int64_t, int64_t, int64_t, const float*, const float*, int,
                                         const double*, float*, float*, double*, double*, int, cudaStream_t);
template int launch_metrics_fused<double>(const double*, int64_t, int64_t, int64_t, const double*, const double*, int,
                                          const double*, double*, double*, double*, double*, int, cudaStream_t);

}  // namespace rnmf_gpu
