// kernels_tc.cu — tcgen05 (5th-gen tensor core) X-streaming GEMMs for sm_100a.
//
//   tc_xw : Y (m x c) = X (m x n) * S (n x c)        sketch Y = X Omega, Y = X Z (p/src/sketch.cpp:60,64)
//
// Structure (one persistent CTA per SM, 8 warps, warp-specialised):
//   warp 0      TMA producer: X tile (128 rows x 32 cols fp32 = 16 KB, SWIZZLE_128B) and the
//               matching 32-column slab of S^T (N rows x 128 B) into a kStages-deep ring.
//   warp 1      TMEM allocator + single-thread UMMA issue: per stage 4 x tcgen05.mma kind::tf32
//               (M=128, N=NPAD, K=8), accumulator in TMEM, double-buffered across row tiles.
//   warps 2-3   (3xTF32 only) split the X tile in place into tf32 hi and a separate lo tile,
//               so D = X_hi S_hi + X_hi S_lo + X_lo S_hi keeps fp32 accuracy.
//   warps 4-7   epilogue: tcgen05.ld of the 128 x NPAD accumulator, rows written to Y.
// TMA zero-fills out-of-range rows/columns, so ragged m and n need no special cases.  X must have
// a 16-byte aligned row pitch (the caller pads when n % 4 != 0).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <algorithm>
#include <mutex>

namespace rnmf_gpu {

namespace {

constexpr int kTcThreads = 256;
constexpr int kBM = 128;          // rows per tile (UMMA M)
constexpr int kBK = 32;           // fp32 columns per stage = one 128 B swizzle row
constexpr int kXTileBytes = kBM * kBK * 4;

template <int NPAD, bool X3>
struct XwCfg {
  static constexpr int kSBytes = NPAD * kBK * 4;  // one S^T slab (hi or lo)
  static constexpr int kStageBytes = kXTileBytes * (X3 ? 2 : 1) + kSBytes * (X3 ? 2 : 1);
  static constexpr int kStages = std::min(6, (200 * 1024) / kStageBytes);
  static constexpr int kTmemCols = (2 * NPAD <= 32) ? 32 : (2 * NPAD <= 64) ? 64 : (2 * NPAD <= 128) ? 128 : 256;
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct XwParams {
  int64_t m, n;
  int c;
  float* y;
  int64_t ldy;
};

template <int NPAD, bool X3>
__global__ void __launch_bounds__(kTcThreads, 1) tc_xw_kernel(const __grid_constant__ CUtensorMap tmX,
                                                              const __grid_constant__ CUtensorMap tmShi,
                                                              const __grid_constant__ CUtensorMap tmSlo, XwParams p) {
  using C = XwCfg<NPAD, X3>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto xs = [&](int s) { return smem + size_t(s) * C::kStageBytes; };
  auto xlo = [&](int s) { return smem + size_t(s) * C::kStageBytes + kXTileBytes; };
  auto shi = [&](int s) { return smem + size_t(s) * C::kStageBytes + kXTileBytes * (X3 ? 2 : 1); };
  auto slo = [&](int s) { return shi(s) + C::kSBytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(S) * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* split = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = bars + 3 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(p.m, kBM);
  const int nk = int(ceil_div(p.n, kBK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split[s], 64);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmShi);
    if (X3) tc::tma_prefetch(&tmSlo);
  }
  if (warp == 1) tc::tmem_alloc<C::kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (tc::elect_one()) {
      uint32_t it = 0;
      const uint32_t bytes = uint32_t(kXTileBytes + C::kSBytes * (X3 ? 2 : 1));
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], bytes);
          tc::tma_load_2d(xs(s), &tmX, &full[s], kc * kBK, int(t * kBM));
          tc::tma_load_2d(shi(s), &tmShi, &full[s], kc * kBK, 0);
          if (X3) tc::tma_load_2d(slo(s), &tmSlo, &full[s], kc * kBK, 0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer
    constexpr uint32_t idesc = tc::make_idesc_tf32(NPAD, false, false);
    uint32_t it = 0, ti = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      const int acc = int(ti & 1);
      tc::mbar_wait(&tempty[acc], ((ti >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t d = tmem_base + uint32_t(acc * NPAD);
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S);
        tc::mbar_wait(X3 ? &split[s] : &full[s], (it / S) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t xa = tc::smem_u32(xs(s)), ba = tc::smem_u32(shi(s));
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            const uint64_t adesc = tc::make_sdesc(xa + k * 32, 16, 1024);
            const uint64_t bdesc = tc::make_sdesc(ba + k * 32, 16, 1024);
            tc::umma_tf32(d, adesc, bdesc, idesc, (kc | k) != 0);
            if (X3) {
              const uint64_t bl = tc::make_sdesc(tc::smem_u32(slo(s)) + k * 32, 16, 1024);
              const uint64_t al = tc::make_sdesc(tc::smem_u32(xlo(s)) + k * 32, 16, 1024);
              tc::umma_tf32(d, adesc, bl, idesc, 1);
              tc::umma_tf32(d, al, bdesc, idesc, 1);
            }
          }
          tc::umma_commit(&empty[s]);
          if (kc == nk - 1) tc::umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    // ---------------- 3xTF32 split: X -> (hi in place, lo)
    if (X3) {
      const int st = threadIdx.x - 64;  // 0..63
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&full[s], (it / S) & 1);
          float4* x4 = reinterpret_cast<float4*>(xs(s));
          float4* l4 = reinterpret_cast<float4*>(xlo(s));
#pragma unroll 4
          for (int q = st; q < kXTileBytes / 16; q += 64) {
            float4 v = x4[q], lo;
            float h;
            h = tc::tf32_hi(v.x), lo.x = v.x - h, v.x = h;
            h = tc::tf32_hi(v.y), lo.y = v.y - h, v.y = h;
            h = tc::tf32_hi(v.z), lo.z = v.z - h, v.z = h;
            h = tc::tf32_hi(v.w), lo.w = v.w - h, v.w = h;
            x4[q] = v;
            l4[q] = lo;
          }
          tc::fence_proxy_async_smem();
          tc::mbar_arrive(&split[s]);
        }
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> Y
    const int sub = warp & 3;
    uint32_t ti = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      const int acc = int(ti & 1);
      tc::mbar_wait(&tfull[acc], (ti >> 1) & 1);
      tc::tc_fence_after();
      const int64_t row = t * kBM + sub * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(sub * 32) << 16) + uint32_t(acc * NPAD);
#pragma unroll
      for (int cc = 0; cc < NPAD / 16; ++cc) {
        uint32_t r[16];
        tc::tmem_ld_32x32b_x16(taddr + cc * 16, r);
        tc::tmem_ld_wait();
        if (row < p.m) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int col = cc * 16 + q;
            if (col < p.c) p.y[row * p.ldy + col] = __uint_as_float(r[q]);
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------------------------------------
// tc_xtw: part[split] (n x c) = X[rows of split]^T (n x m_s) * S[rows of split] (m_s x c)
//   A = X^T tile: M = 128 X columns (MN-major: four 32-column TMA boxes, LBO = 4 KB),
//       K = 32 X rows per stage (SBO = 1024 B per 8 rows)
//   B = S^T slab (N = NPAD rows of the transposed small operand, K-major)
// One work unit = (128-column tile, row split); units are distributed over persistent CTAs.
template <int NPAD, bool X3 = false>
struct XtwCfg {
  static constexpr int kXBytes = 128 * kBK * 4;  // 32 rows x 128 cols
  static constexpr int kSBytes = NPAD * kBK * 4;
  static constexpr int kStageBytes = (kXBytes + kSBytes) * (X3 ? 2 : 1);
  static constexpr int kStages = std::min(6, (200 * 1024) / kStageBytes);
  static constexpr int kTmemCols = (2 * NPAD <= 32) ? 32 : (2 * NPAD <= 64) ? 64 : (2 * NPAD <= 128) ? 128 : 256;
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 + 256;
};

struct XtwParams {
  int64_t m, n;
  int c;
  int splits;
  float* part;  // splits x n x c
};

template <int NPAD, bool X3>
__global__ void __launch_bounds__(kTcThreads, 1) tc_xtw_kernel(const __grid_constant__ CUtensorMap tmX,
                                                               const __grid_constant__ CUtensorMap tmSt,
                                                               const __grid_constant__ CUtensorMap tmStLo, XtwParams p) {
  using C = XtwCfg<NPAD, X3>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto xs = [&](int s) { return smem + size_t(s) * C::kStageBytes; };
  auto ss = [&](int s) { return smem + size_t(s) * C::kStageBytes + C::kXBytes; };
  auto xl = [&](int s) { return smem + size_t(s) * C::kStageBytes + C::kXBytes + C::kSBytes; };
  auto sl = [&](int s) { return xl(s) + C::kXBytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(S) * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint64_t* split = bars + 2 * S + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ctiles = ceil_div(p.n, 128);
  const int64_t units = ctiles * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&split[s], 64);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmSt);
    if (X3) tc::tma_prefetch(&tmStLo);
  }
  if (warp == 1) tc::tmem_alloc<C::kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // split boundaries on 32-row stage boundaries, so no stage straddles two splits
  const int64_t mstages = ceil_div(p.m, kBK);
  auto unit_rows = [&](int64_t u, int64_t& r0, int64_t& r1) {
    const int64_t sp = u % p.splits;
    r0 = (mstages * sp / p.splits) * kBK;
    r1 = (mstages * (sp + 1) / p.splits) * kBK;
  };

  if (warp == 0) {
    if (tc::elect_one()) {
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t ct = u / p.splits;
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        for (int64_t r = r0; r < r1; r += kBK, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], uint32_t(C::kXBytes + C::kSBytes * (X3 ? 2 : 1)));
#pragma unroll
          for (int b = 0; b < 4; ++b) tc::tma_load_2d(xs(s) + b * 4096, &tmX, &full[s], int(ct * 128 + b * 32), int(r));
          tc::tma_load_2d(ss(s), &tmSt, &full[s], int(r), 0);
          if (X3) tc::tma_load_2d(sl(s), &tmStLo, &full[s], int(r), 0);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::make_idesc_tf32(NPAD, true, false);
    uint32_t it = 0, ti = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ti) {
      int64_t r0, r1;
      unit_rows(u, r0, r1);
      const int acc = int(ti & 1);
      tc::mbar_wait(&tempty[acc], ((ti >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t d = tmem_base + uint32_t(acc * NPAD);
      bool first = true;
      for (int64_t r = r0; r < r1; r += kBK, ++it) {
        const int s = int(it % S);
        tc::mbar_wait(X3 ? &split[s] : &full[s], (it / S) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t xa = tc::smem_u32(xs(s)), ba = tc::smem_u32(ss(s));
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            // MN-major A (SW128_BASE32B): LBO = 4 KB between 32-column boxes, SBO = 512 B per 4 rows
            const uint64_t adesc = tc::make_sdesc(xa + k * 1024, 4096, 512, tc::kLayoutSW128Base32B);
            const uint64_t bdesc = tc::make_sdesc(ba + k * 32, 16, 1024);
            tc::umma_tf32(d, adesc, bdesc, idesc, (first && k == 0) ? 0u : 1u);
            if (X3) {
              const uint64_t al = tc::make_sdesc(tc::smem_u32(xl(s)) + k * 1024, 4096, 512, tc::kLayoutSW128Base32B);
              const uint64_t bl = tc::make_sdesc(tc::smem_u32(sl(s)) + k * 32, 16, 1024);
              tc::umma_tf32(d, adesc, bl, idesc, 1);
              tc::umma_tf32(d, al, bdesc, idesc, 1);
            }
          }
          tc::umma_commit(&empty[s]);
          if (r + kBK >= r1) tc::umma_commit(&tfull[acc]);
        }
        first = false;
        __syncwarp();
      }
      if (r0 >= r1) {  // empty split: still hand an (all-zero) accumulator to the epilogue
        if (tc::elect_one()) tc::mbar_arrive(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    if (X3) {  // 3xTF32 split of the X tile (elementwise, so the swizzled layout is irrelevant)
      const int st = threadIdx.x - 64;
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        for (int64_t r = r0; r < r1; r += kBK, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&full[s], (it / S) & 1);
          float4* x4 = reinterpret_cast<float4*>(xs(s));
          float4* l4 = reinterpret_cast<float4*>(xl(s));
#pragma unroll 4
          for (int q = st; q < C::kXBytes / 16; q += 64) {
            float4 v = x4[q], lo;
            float h;
            h = tc::tf32_hi(v.x), lo.x = v.x - h, v.x = h;
            h = tc::tf32_hi(v.y), lo.y = v.y - h, v.y = h;
            h = tc::tf32_hi(v.z), lo.z = v.z - h, v.z = h;
            h = tc::tf32_hi(v.w), lo.w = v.w - h, v.w = h;
            x4[q] = v;
            l4[q] = lo;
          }
          tc::fence_proxy_async_smem();
          tc::mbar_arrive(&split[s]);
        }
      }
    }
  } else {
    const int sub = warp & 3;
    uint32_t ti = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ti) {
      const int64_t ct = u / p.splits, sp = u % p.splits;
      int64_t r0, r1;
      unit_rows(u, r0, r1);
      const int acc = int(ti & 1);
      tc::mbar_wait(&tfull[acc], (ti >> 1) & 1);
      tc::tc_fence_after();
      const int64_t col = ct * 128 + sub * 32 + lane;  // X column = output row of P
      const uint32_t taddr = tmem_base + (uint32_t(sub * 32) << 16) + uint32_t(acc * NPAD);
      float* out = p.part + (sp * p.n + col) * p.c;
#pragma unroll
      for (int cc = 0; cc < NPAD / 16; ++cc) {
        uint32_t rr[16];
        tc::tmem_ld_32x32b_x16(taddr + cc * 16, rr);
        tc::tmem_ld_wait();
        if (col < p.n) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int j = cc * 16 + q;
            if (j < p.c) out[j] = (r0 < r1) ? __uint_as_float(rr[q]) : 0.f;
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// S (n x c, row-major, ld c) -> S^T hi / lo (npad x ldst, zero rows for j >= c and cols >= n)
__global__ void prep_st_kernel(const float* __restrict__ s, int64_t n, int c, int npad, int64_t ldst,
                               float* __restrict__ st_hi, float* __restrict__ st_lo) {
  const int64_t total = int64_t(npad) * ldst;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / ldst);
    const int64_t kk = e % ldst;
    const float v = (j < c && kk < n) ? s[kk * c + j] : 0.f;
    const float h = tc::tf32_hi(v);
    st_hi[e] = h;
    st_lo[e] = v - h;
  }
}

// ---- host: tensor maps through the driver entry point (no libcuda link dependency) ----------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D fp32 row-major tensor (rows x cols, pitch in elements), box = box_rows x 32 cols, SW128.
CUtensorMap make_map_2d(const float* base, int64_t rows, int64_t cols, int64_t pitch, int box_rows,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(pitch) * sizeof(float)};
  const cuuint32_t box[2] = {cuuint32_t(kBK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

template <int NPAD, bool X3>
void tc_xw_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                  int64_t ldst, int c, float* y, int sm_count, cudaStream_t stream) {
  using C = XwCfg<NPAD, X3>;
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBM);
  const CUtensorMap mh = make_map_2d(st_hi, NPAD, n, ldst, NPAD);
  const CUtensorMap ml = make_map_2d(st_lo, NPAD, n, ldst, NPAD);
  XwParams p{m, n, c, y, c};
  auto f = tc_xw_kernel<NPAD, X3>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  const int64_t ntiles = ceil_div(m, kBM);
  const int grid = int(std::min<int64_t>(ntiles, sm_count));
  f<<<grid, kTcThreads, C::kSmem, stream>>>(mx, mh, ml, p);
  RNMF_CUDA_LAUNCH();
}


template <int NPAD, bool X3>
void tc_xtw_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st, const float* st_lo, int64_t ldst,
                   int c, float* part, int splits, int sm_count, cudaStream_t stream) {
  using C = XtwCfg<NPAD, X3>;
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);  // 32 x 32 boxes
  const CUtensorMap ms = make_map_2d(st, NPAD, m, ldst, NPAD);  // S^T: NPAD rows x m
  const CUtensorMap ml = make_map_2d(X3 ? st_lo : st, NPAD, m, ldst, NPAD);
  XtwParams p{m, n, c, splits, part};
  auto f = tc_xtw_kernel<NPAD, X3>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  const int64_t units = ceil_div(n, 128) * splits;
  const int grid = int(std::min<int64_t>(units, sm_count));
  f<<<grid, kTcThreads, C::kSmem, stream>>>(mx, ms, ml, p);
  RNMF_CUDA_LAUNCH();
}

}  // namespace

CUtensorMap make_tma_2d(const void* base, int elem_bytes, int64_t rows, int64_t cols, int64_t pitch, int box_cols,
                        int box_rows, bool swizzle128) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(pitch) * cuuint64_t(elem_bytes)};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

int tc_xtw_splits(int64_t m, int64_t n, int sm_count) {
  const int64_t ct = ceil_div(n, 128);
  int64_t s = std::max<int64_t>(1, sm_count / ct);
  s = std::min<int64_t>(s, std::max<int64_t>(1, m / (4 * kBK)));
  return int(s);
}

int launch_tc_xtw(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st, const float* st_lo, int c,
                  float* part, int splits, bool x3, int sm_count, cudaStream_t stream) {
  if ((ldx * sizeof(float)) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) % 16) != 0)
    throw CudaError("tc_xtw: X needs a 16-byte aligned base and row pitch");
  const int64_t ldst = tc_st_pitch(m);
  switch (tc_npad(c)) {
    case 16: if (x3) tc_xtw_launch<16, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<16, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 32: if (x3) tc_xtw_launch<32, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<32, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 48: if (x3) tc_xtw_launch<48, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<48, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 64: if (x3) tc_xtw_launch<64, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<64, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 80: if (x3) tc_xtw_launch<80, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<80, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 96: if (x3) tc_xtw_launch<96, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<96, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 112: if (x3) tc_xtw_launch<112, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<112, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    case 128: if (x3) tc_xtw_launch<128, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); else tc_xtw_launch<128, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream); break;
    default: throw CudaError("tc_xtw: column count above 128");
  }
  return 1;
}

namespace {
}  // namespace

int tc_npad(int c) { return int(ceil_div(c, 16) * 16); }

int64_t tc_st_pitch(int64_t n) { return ceil_div(n, 32) * 32; }

int launch_tc_prep_st(const float* s, int64_t n, int c, float* st_hi, float* st_lo, cudaStream_t stream) {
  const int npad = tc_npad(c);
  const int64_t ld = tc_st_pitch(n);
  const int blocks = int(std::min<int64_t>(ceil_div(int64_t(npad) * ld, 256), 148 * 8));
  prep_st_kernel<<<blocks, 256, 0, stream>>>(s, n, c, npad, ld, st_hi, st_lo);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int launch_tc_xw(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo, int c,
                 float* y, bool x3, int sm_count, cudaStream_t stream) {
  if ((ldx * sizeof(float)) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) % 16) != 0)
    throw CudaError("tc_xw: X needs a 16-byte aligned base and row pitch");
  const int64_t ldst = tc_st_pitch(n);
  const int np = tc_npad(c);
#define RNMF_TC_XW(NP)                                                                         \
  case NP:                                                                                     \
    if (x3)                                                                                    \
      tc_xw_launch<NP, true>(x, m, n, ldx, st_hi, st_lo, ldst, c, y, sm_count, stream);        \
    else                                                                                       \
      tc_xw_launch<NP, false>(x, m, n, ldx, st_hi, st_lo, ldst, c, y, sm_count, stream);       \
    break;
  switch (np) {
    RNMF_TC_XW(16)
    RNMF_TC_XW(32)
    RNMF_TC_XW(48)
    RNMF_TC_XW(64)
    RNMF_TC_XW(80)
    RNMF_TC_XW(96)
    RNMF_TC_XW(112)
    RNMF_TC_XW(128)
    default:
      throw CudaError("tc_xw: column count above 128");
  }
#undef RNMF_TC_XW
  return 1;
}

}  // namespace rnmf_gpu
