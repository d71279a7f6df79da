// kernels_xw.cu — Y = X S, the sketch's X-streaming product (Y = X Omega, Y = X Z;
// p/src/sketch.cpp:60,64), FMA in the working precision (EXACT math mode).
//
// Persistent CTAs (128 threads) walk 128-row tiles of X.  The 128-byte-wide column chunks of X
// (32 fp32 / 16 fp64 columns, SWIZZLE_128B) and the matching rows of S (zero-padded to CPAD
// columns) arrive by TMA into a 3-stage shared-memory ring (one issuing thread, mbarrier
// completion); rows / columns past the matrix arrive as zeros, so the inner loop has no bounds
// checks.  Thread (row group ty, column group tx) accumulates rows ty + 16 i (i < 8) x columns
// tx*CT .. tx*CT + CT - 1 of Y in registers for the whole tile: per k, 8 swizzled X loads (rows
// 16 apart sit in different 16-byte chunks of their 128-byte rows: no bank conflicts) and CT / EPV
// vector loads of S feed 8 * CT FMAs.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <algorithm>

namespace rnmf_gpu {

namespace {

constexpr int kXwThreads = 128;
constexpr int kXwBM = 128;
constexpr int kXwRT = 8;   // rows per thread (ty + 16 i)
constexpr int kXwRG = 16;  // row groups
constexpr int kXwCG = 8;   // column groups

template <typename T, int CPAD>
struct XwCfg2 {
  static constexpr int BK = 128 / int(sizeof(T));  // k per chunk: one 128-byte swizzle row of X
  static constexpr int CT = CPAD / kXwCG;          // output columns per thread
  static constexpr int S = 3;
  static constexpr size_t xs_bytes = size_t(kXwBM) * 128;
  static constexpr size_t ss_bytes = sizeof(T) * size_t(BK) * CPAD;
  static constexpr size_t xs = 0;
  static constexpr size_t ss = xs + S * xs_bytes;
  static constexpr size_t bars = (ss + S * ss_bytes + 15) / 16 * 16;
  static constexpr size_t total = bars + 8 * S + 1024;
  static constexpr uint32_t stage_tx = uint32_t(xs_bytes + ss_bytes);
};

template <typename T>
__global__ void pad_cols_kernel(const T* __restrict__ s, int64_t rows, int c, int cpad, T* __restrict__ out) {
  const int64_t total = rows * cpad;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / cpad;
    const int j = int(e % cpad);
    out[e] = j < c ? s[r * c + j] : T(0);
  }
}

template <typename T, int CPAD>
__global__ void __launch_bounds__(kXwThreads) xw_tma_kernel(const __grid_constant__ CUtensorMap map_x,
                                                            const __grid_constant__ CUtensorMap map_s, int64_t m,
                                                            int64_t n, int c, T* __restrict__ Y) {
  using C = XwCfg2<T, CPAD>;
  constexpr int S = C::S, BK = C::BK, CT = C::CT;
  constexpr int EPV = 16 / int(sizeof(T));
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::bars);
  const int tid = threadIdx.x, ty = tid % kXwRG, tx = tid / kXwRG;

  const int64_t ntiles = ceil_div(m, kXwBM), nch = ceil_div(n, BK);
  const int64_t my_tiles = int64_t(blockIdx.x) < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nch;
  if (tid == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_s);
    for (int s = 0; s < S; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t q) {
    const int s = int(q % S);
    const int64_t tile = blockIdx.x + (q / nch) * gridDim.x, ch = q % nch;
    tc::mbar_arrive_expect_tx(&full[s], C::stage_tx);
    tc::tma_load_2d(smem + C::xs + s * C::xs_bytes, &map_x, &full[s], int(ch * BK), int(tile * kXwBM));
    tc::tma_load_2d(smem + C::ss + s * C::ss_bytes, &map_s, &full[s], 0, int(ch * BK));
  };
  if (tid == 0)
    for (int64_t q = 0; q < (total < S - 1 ? total : S - 1); ++q) issue(q);

  T acc[kXwRT][CT];
  int64_t tile = blockIdx.x, ch = 0;
  for (int64_t q = 0; q < total; ++q, ++ch) {
    if (ch == nch) ch = 0, tile += gridDim.x;
    if (ch == 0) {
#pragma unroll
      for (int i = 0; i < kXwRT; ++i)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[i][j] = T(0);
    }
    if (tid == 0 && q + S - 1 < total) issue(q + S - 1);  // refills the stage consumed at q - 1
    const int s = int(q % S);
    tc::mbar_wait(&full[s], uint32_t((q / S) & 1));
    const unsigned char* Xt = smem + C::xs + s * C::xs_bytes;
    const T* St = reinterpret_cast<const T*>(smem + C::ss + s * C::ss_bytes);
#pragma unroll 2
    for (int kq = 0; kq < BK / EPV; ++kq) {
      T xv[kXwRT][EPV];
#pragma unroll
      for (int i = 0; i < kXwRT; ++i) {
        const int r = ty + kXwRG * i;
        const T* p = reinterpret_cast<const T*>(Xt + r * 128 + ((kq ^ (r & 7)) << 4));
        if constexpr (sizeof(T) == 4) {
          const float4 f = *reinterpret_cast<const float4*>(p);
          xv[i][0] = f.x, xv[i][1] = f.y, xv[i][2] = f.z, xv[i][3] = f.w;
        } else {
          const double2 d = *reinterpret_cast<const double2*>(p);
          xv[i][0] = d.x, xv[i][1] = d.y;
        }
      }
#pragma unroll
      for (int e = 0; e < EPV; ++e) {
        const T* sr = St + (kq * EPV + e) * CPAD + tx * CT;
        T sv[CT];
#pragma unroll
        for (int j = 0; j < CT; ++j) sv[j] = sr[j];
#pragma unroll
        for (int i = 0; i < kXwRT; ++i)
#pragma unroll
          for (int j = 0; j < CT; ++j) acc[i][j] = fma(xv[i][e], sv[j], acc[i][j]);
      }
    }
    __syncthreads();  // stage s consumed by every thread before it is refilled
    if (ch == nch - 1) {
      const int64_t row0 = tile * kXwBM;
#pragma unroll
      for (int i = 0; i < kXwRT; ++i) {
        const int64_t r = row0 + ty + kXwRG * i;
        if (r < m)
#pragma unroll
          for (int j = 0; j < CT; ++j)
            if (tx * CT + j < c) Y[r * c + tx * CT + j] = acc[i][j];
      }
    }
  }
}

template <typename T, int CPAD>
void xw_tma_dispatch(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, T* spad, int sm_count,
                     cudaStream_t st) {
  using C = XwCfg2<T, CPAD>;
  const int pg = int(std::min<int64_t>(ceil_div(n * CPAD, 256), 1024));
  pad_cols_kernel<T><<<pg, 256, 0, st>>>(s, n, c, CPAD, spad);
  RNMF_CUDA_LAUNCH();
  const CUtensorMap mx = make_tma_2d(x, int(sizeof(T)), m, n, ldx, C::BK, kXwBM, true);
  const CUtensorMap ms = make_tma_2d(spad, int(sizeof(T)), n, CPAD, CPAD, CPAD, C::BK);
  auto f = xw_tma_kernel<T, CPAD>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::total)));
  const int per_sm = std::max(1, std::min(4, int((227u * 1024u) / (C::total + 1024))));
  const int grid = int(std::min<int64_t>(ceil_div(m, kXwBM), int64_t(per_sm) * sm_count));
  f<<<grid, kXwThreads, C::total, st>>>(mx, ms, m, n, c, y);
  RNMF_CUDA_LAUNCH();
}

// ------------------------------------------------------------------------------------------------
// P = X^T S (n x c) for S m x c (X^T Q, B = Q^T X; p/src/sketch.cpp:63,69): CTA (column panel of
// 128 X columns, row split) accumulates its panel's 128 x c block over its rows, 32 rows per TMA
// chunk (X panel [32][128] dense: a warp reads 16 consecutive columns of one row, conflict free;
// S [32][CPAD], columns past c zero).  Thread (column group cg, j group jg) owns columns
// cg + 16 i (i < 8) x j = jg*CT ...; partials part[split][n][c] are reduced in fixed order.
constexpr int kXtBN = 128;  // X columns per panel
constexpr int kXtBK = 32;   // rows per chunk

template <typename T, int CPAD>
struct XtwCfg2 {
  static constexpr int CT = CPAD / kXwCG;
  static constexpr int S = 3;
  static constexpr size_t xs_bytes = sizeof(T) * size_t(kXtBK) * kXtBN;
  static constexpr size_t ss_bytes = sizeof(T) * size_t(kXtBK) * CPAD;
  static constexpr size_t xs = 0;
  static constexpr size_t ss = xs + S * xs_bytes;
  static constexpr size_t bars = (ss + S * ss_bytes + 15) / 16 * 16;
  static constexpr size_t total = bars + 8 * S + 1024;
  static constexpr uint32_t stage_tx = uint32_t(xs_bytes + ss_bytes);
};

template <typename T, int CPAD>
__global__ void __launch_bounds__(kXwThreads) xtw_tma_kernel(const __grid_constant__ CUtensorMap map_x,
                                                             const __grid_constant__ CUtensorMap map_s, int64_t m,
                                                             int64_t n, int c, int splits, T* __restrict__ part) {
  using C = XtwCfg2<T, CPAD>;
  constexpr int S = C::S, CT = C::CT;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::bars);
  const int tid = threadIdx.x, cg = tid % kXwRG, jg = tid / kXwRG;
  const int64_t panels = ceil_div(n, kXtBN);
  const int64_t units = panels * splits;
  if (tid == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_s);
    for (int s = 0; s < S; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  int64_t gq = 0;  // chunks consumed by this CTA so far (stage / phase bookkeeping)
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t panel = u % panels, sp = u / panels;
    const int64_t r0 = m * sp / splits, r1 = m * (sp + 1) / splits;
    const int64_t nch = ceil_div(r1 - r0, kXtBK);
    auto issue = [&](int64_t q) {  // chunk q of this unit into stage (gq + q) % S
      const int s = int((gq + q) % S);
      tc::mbar_arrive_expect_tx(&full[s], C::stage_tx);
      tc::tma_load_2d(smem + C::xs + s * C::xs_bytes, &map_x, &full[s], int(panel * kXtBN), int(r0 + q * kXtBK));
      tc::tma_load_2d(smem + C::ss + s * C::ss_bytes, &map_s, &full[s], 0, int(r0 + q * kXtBK));
    };
    if (tid == 0)
      for (int64_t q = 0; q < (nch < S - 1 ? nch : S - 1); ++q) issue(q);
    T acc[kXwRT][CT];
#pragma unroll
    for (int i = 0; i < kXwRT; ++i)
#pragma unroll
      for (int j = 0; j < CT; ++j) acc[i][j] = T(0);
    for (int64_t q = 0; q < nch; ++q) {
      if (tid == 0 && q + S - 1 < nch) issue(q + S - 1);
      const int s = int((gq + q) % S);
      tc::mbar_wait(&full[s], uint32_t(((gq + q) / S) & 1));
      const T* Xt = reinterpret_cast<const T*>(smem + C::xs + s * C::xs_bytes);
      const T* St = reinterpret_cast<const T*>(smem + C::ss + s * C::ss_bytes);
      // rows of the chunk past r1 belong to the next split: masked (the TMA box may cover them)
      const int64_t rem = r1 - (r0 + q * kXtBK);
      const int rows = rem < kXtBK ? int(rem) : kXtBK;
#pragma unroll 4
      for (int rr = 0; rr < rows; ++rr) {
        T xv[kXwRT], sv[CT];
#pragma unroll
        for (int i = 0; i < kXwRT; ++i) xv[i] = Xt[rr * kXtBN + cg + kXwRG * i];
#pragma unroll
        for (int j = 0; j < CT; ++j) sv[j] = St[rr * CPAD + jg * CT + j];
#pragma unroll
        for (int i = 0; i < kXwRT; ++i)
#pragma unroll
          for (int j = 0; j < CT; ++j) acc[i][j] = fma(xv[i], sv[j], acc[i][j]);
      }
      __syncthreads();  // stage consumed before it is refilled
    }
    gq += nch;
    T* dst = part + (sp * n) * c;
#pragma unroll
    for (int i = 0; i < kXwRT; ++i) {
      const int64_t col = panel * kXtBN + cg + kXwRG * i;
      if (col < n)
#pragma unroll
        for (int j = 0; j < CT; ++j)
          if (jg * CT + j < c) dst[col * c + jg * CT + j] = acc[i][j];
    }
  }
}

template <typename T, int CPAD>
void xtw_tma_dispatch(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits,
                      T* spad, int sm_count, cudaStream_t st) {
  using C = XtwCfg2<T, CPAD>;
  const T* sm = s;
  int64_t sp = c;
  if ((int64_t(c) * int64_t(sizeof(T))) % 16 != 0) {  // TMA needs 16-byte row pitches: pad S
    const int pg = int(std::min<int64_t>(ceil_div(m * CPAD, 256), 4096));
    pad_cols_kernel<T><<<pg, 256, 0, st>>>(s, m, c, CPAD, spad);
    RNMF_CUDA_LAUNCH();
    sm = spad;
    sp = CPAD;
  }
  const CUtensorMap mx = make_tma_2d(x, int(sizeof(T)), m, n, ldx, kXtBN, kXtBK);
  const CUtensorMap ms = make_tma_2d(sm, int(sizeof(T)), m, sp, sp, CPAD, kXtBK);  // columns >= c: zero fill
  auto f = xtw_tma_kernel<T, CPAD>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::total)));
  const int per_sm = std::max(1, std::min(4, int((227u * 1024u) / (C::total + 1024))));
  const int64_t units = ceil_div(n, kXtBN) * splits;
  const int grid = int(std::min<int64_t>(units, int64_t(per_sm) * sm_count));
  f<<<grid, kXwThreads, C::total, st>>>(mx, ms, m, n, c, splits, part);
  RNMF_CUDA_LAUNCH();
}

}  // namespace

int64_t xw_tma_spad_len(int64_t n, int c) { return n * (c <= 16 ? 16 : c <= 32 ? 32 : c <= 48 ? 48 : c <= 64 ? 64 : c <= 96 ? 96 : 128); }

template <typename T>
int launch_xw_tma(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, T* spad, int sm_count,
                  cudaStream_t stream) {
  if ((ldx * int64_t(sizeof(T))) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    throw CudaError("xw: X rows must be 16-byte aligned");
  if (c <= 16)
    xw_tma_dispatch<T, 16>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
  else if (c <= 32)
    xw_tma_dispatch<T, 32>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
  else if (c <= 48)
    xw_tma_dispatch<T, 48>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
  else if (c <= 64)
    xw_tma_dispatch<T, 64>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
  else if constexpr (sizeof(T) == 4) {
    if (c <= 96)
      xw_tma_dispatch<T, 96>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
    else if (c <= 128)
      xw_tma_dispatch<T, 128>(x, m, n, ldx, s, c, y, spad, sm_count, stream);
    else
      throw CudaError("xw: width above 128");
  } else {
    return launch_xw<T>(x, m, n, ldx, s, c, y, stream);  // fp64 wider than 64: register budget
  }
  return 2;
}

int xtw_tma_splits(int64_t m, int64_t n, int sm_count) {
  const int64_t panels = ceil_div(n, kXtBN);
  int64_t s = ceil_div(int64_t(2) * sm_count, panels);
  s = std::max<int64_t>(1, std::min<int64_t>(s, ceil_div(m, 4 * kXtBK)));
  return int(std::min<int64_t>(s, 1024));
}

template <typename T>
int launch_xtw_tma(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits, T* out,
                   bool transpose_out, T* spad, int sm_count, cudaStream_t stream) {
  if ((ldx * int64_t(sizeof(T))) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    throw CudaError("xtw: X rows must be 16-byte aligned");
  if (c <= 16)
    xtw_tma_dispatch<T, 16>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
  else if (c <= 32)
    xtw_tma_dispatch<T, 32>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
  else if (c <= 48)
    xtw_tma_dispatch<T, 48>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
  else if (c <= 64)
    xtw_tma_dispatch<T, 64>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
  else if constexpr (sizeof(T) == 4) {
    if (c <= 96)
      xtw_tma_dispatch<T, 96>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
    else if (c <= 128)
      xtw_tma_dispatch<T, 128>(x, m, n, ldx, s, c, part, splits, spad, sm_count, stream);
    else
      throw CudaError("xtw: width above 128");
  } else {
    return launch_xtw<T>(x, m, n, ldx, s, c, part, splits, out, transpose_out, stream);
  }
  return 1 + launch_splitk_reduce<T>(part, splits, n, c, out, transpose_out, stream);
}

template int launch_xtw_tma<float>(const float*, int64_t, int64_t, int64_t, const float*, int, float*, int, float*,
                                   bool, float*, int, cudaStream_t);
template int launch_xtw_tma<double>(const double*, int64_t, int64_t, int64_t, const double*, int, double*, int,
                                    double*, bool, double*, int, cudaStream_t);

template int launch_xw_tma<float>(const float*, int64_t, int64_t, int64_t, const float*, int, float*, float*, int,
                                  cudaStream_t);
template int launch_xw_tma<double>(const double*, int64_t, int64_t, int64_t, const double*, int, double*, double*, int,
                                   cudaStream_t);

}  // namespace rnmf_gpu
