// kernels_tc.cu — tcgen05 (5th-gen tensor core) X-streaming GEMMs for sm_100a.
//
//   tc_xw : Y (m x c) = X (m x n) * S (n x c)        sketch Y = X Omega, Y = X Z (p/src/sketch.cpp:60,64)
//
//   tc_xtw: part (n x c) = X^T (n x m) * S (m x c)   X^T Q, B^T = X^T Q    (p/src/sketch.cpp:63,69)
//
// Structure (one persistent CTA per SM, warp-specialised):
//   warp 0       TMA producer: X tile (16 KB, 128 B swizzle) and the matching S^T slab(s) into a
//                ring of kStages stages.
//   warp 1       TMEM allocator + single-thread UMMA issue (tcgen05.mma kind::tf32, M = 128).
//   warps 2-3, 8-11 (3xTF32 only) write lo = rna_tf32(X - trunc_tf32(X)) into a 3-slot lo ring;
//                the raw X tile is the hi operand (kind::tf32 truncates), so per K step
//                  D[0:2N)  = X_hi [S_hi; S_lo]^T   (one UMMA, N = 2 NPAD)
//                  D[N:2N) += X_lo S_hi^T
//                so the big term never shares an accumulator with the small ones.
//   warps 4-7    epilogue: every chunk of p.chunk stages lands in a fresh TMEM buffer that the
//                epilogue adds into fp32 registers (round-to-nearest), which bounds the tensor
//                core's truncating accumulation to p.chunk * 32 terms.  Measured on B200
//                (tools/sketch_acc.cu): 3xTF32 with 128-term chunks is more accurate than the FFMA
//                kernels (rms error 3-4e-7 vs 8e-7 - 2e-6 of the result), where whole-K accumulation was
//                2e-5 - 1e-4 with a systematic shrinkage bias.
// TMA zero-fills out-of-range rows/columns, so ragged m and n need no special cases.  X must have
// a 16-byte aligned row pitch (the caller pads when n % 4 != 0).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"
#include "tc_metrics.h"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace rnmf_gpu {

namespace {

constexpr int kTcThreads = 256;
// 3xTF32: six split warps (2-3 and 8-11) produce the lo tile while 0 / 1 / 4-7 keep their roles
constexpr int kTcThreadsX3 = 384;
constexpr int kSplitThreads = 192;
template <bool X3>
constexpr int tc_threads() { return X3 ? kTcThreadsX3 : kTcThreads; }
constexpr int kBM = 128;          // rows per tile (UMMA M)
constexpr int kBK = 32;           // fp32 K elements per stage = one 128 B swizzle row
constexpr int kXTileBytes = kBM * kBK * 4;  // 16 KB: one X stage (either kernel)
#ifndef RNMF_TC_LO_SLOTS
#define RNMF_TC_LO_SLOTS 3
#endif
#ifndef RNMF_TC_SMEM_KB
#define RNMF_TC_SMEM_KB 220
#endif
constexpr int kLoSlots = RNMF_TC_LO_SLOTS;  // 3xTF32 lo-tile ring
constexpr int kSmemBudget = RNMF_TC_SMEM_KB * 1024;
// L2 eviction priorities of the TMA loads (RNMF_TC_NO_L2_HINT: both normal, for comparison)
#ifdef RNMF_TC_NO_L2_HINT
constexpr uint64_t kXPolicy = 0x1000000000000000ull, kSPolicy = 0x1000000000000000ull;
#else
constexpr uint64_t kXPolicy = tc::kL2EvictFirst, kSPolicy = tc::kL2EvictLast;
#endif

// 3xTF32 operand split.  hi = the raw fp32 word: kind::tf32 reads only the top 19 bits, i.e. it
// truncates, so lo = rna_tf32(x - trunc_tf32(x)) is what the tensor core misses.  Only lo is
// written; the X tile in the TMA ring is used unchanged as hi.
__device__ __forceinline__ float tf32_lo(float v) {
  return tc::tf32_hi(v - __uint_as_float(__float_as_uint(v) & 0xffffe000u));
}

__device__ __forceinline__ uint32_t tf32_lo_bits(uint32_t u) {
  // d = x - trunc_tf32(x) (exact), then round d to tf32, nearest with ties away (= cvt.rna.tf32).
  // The low 13 bits are left as they fall: the only reader is kind::tf32, which ignores them (one
  // ALU op less per element; under the 1000 W cap these kernels are power-bound).
  const uint32_t d = __float_as_uint(__uint_as_float(u) - __uint_as_float(u & 0xffffe000u));
  return d + 0x1000u;
}

// lo part of one X stage (N16 float4s) by kSplitThreads threads: explicit shared-space vector
// loads / stores (the tile pointers are generic in C++), all loads of a thread issued first
template <int N16, int NT = kSplitThreads>
__device__ __forceinline__ void split_lo_tile(const float4* __restrict__ x4, float4* __restrict__ l4, int st) {
  constexpr int kIt = (N16 + NT - 1) / NT;
  const uint32_t xs = tc::smem_u32(x4), ls = tc::smem_u32(l4);
  uint32_t v[kIt][4];
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int q = st + i * NT;
    if (q < N16)
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3])
                   : "r"(xs + 16u * uint32_t(q)) : "memory");
  }
#pragma unroll
  for (int i = 0; i < kIt; ++i) {
    const int q = st + i * NT;
    if (q < N16)
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ls + 16u * uint32_t(q)), "r"(tf32_lo_bits(v[i][0])),
                   "r"(tf32_lo_bits(v[i][1])), "r"(tf32_lo_bits(v[i][2])), "r"(tf32_lo_bits(v[i][3]))
                   : "memory");
  }
}

// Shared layout of both kernels.  Ring stage = [X tile 16 KB][S^T hi slab][S^T lo slab (X3)], the
// two slabs adjacent so that X_hi * [S_hi; S_lo]^T is ONE UMMA with N = 2 NPAD.  3xTF32 keeps the
// lo X tiles in a separate 3-slot ring so the TMA ring stays deep.  TMEM accumulator buffer =
// [X_hi S_hi | X_hi S_lo + X_lo S_hi] (2 NPAD columns; NPAD for 1xTF32), double-buffered.
// LT (3xTF32 only): the lo X tile lives in TENSOR MEMORY instead of shared memory -- the split warps
// read their rows of the X stage, write lo with tcgen05.st into 32 TMEM columns per ring stage, and
// the small-term UMMA takes A from TMEM.  That removes the lo tile's shared-memory write and its
// UMMA operand read (ncu: the shared-memory data pipe, LSU + tensor-core wavefronts, was ~100 % busy
// with the lo ring in shared memory), and frees 48 KB for a deeper TMA ring.  The S^T lo slab comes
// by TMA from the prepared global copy.
template <int NPAD, bool X3, bool LT = false>
struct TcCfg {
  static_assert(!LT || X3, "LT is a 3xTF32 layout");
  static constexpr int kSBytes = NPAD * kBK * 4;  // one S^T slab (NPAD rows x 128 B)
  static constexpr int kStageBytes = kXTileBytes + kSBytes * (X3 ? 2 : 1);
  static constexpr int kLoBytes = (X3 && !LT) ? kLoSlots * kXTileBytes : 0;
  static constexpr int kStages = std::min(8, (kSmemBudget - kLoBytes - 2048) / kStageBytes);
  // LT: TMEM lo slot s belongs to ring stage s and is released with it (one commit per stage)
  static constexpr int kLoN = LT ? kStages : kLoSlots;
  static constexpr int kAccCols = X3 ? 2 * NPAD : NPAD;
  static constexpr int kLoCols = LT ? kLoN * kBK : 0;
  static constexpr int kAccBufs = (2 * kAccCols + kLoCols <= 512) ? 2 : 1;
  static constexpr int kLoBase = kAccBufs * kAccCols;  // first TMEM column of the lo ring
  static constexpr int kUsedCols = kAccBufs * kAccCols + kLoCols;
  static constexpr int kTmemCols = kUsedCols <= 32 ? 32 : kUsedCols <= 64 ? 64 : kUsedCols <= 128 ? 128
                                   : kUsedCols <= 256 ? 256 : 512;
  static constexpr int kThreads = LT ? 448 : X3 ? kTcThreadsX3 : kTcThreads;
  static constexpr int kSplit = LT ? 256 : kSplitThreads;  // lo-producing threads
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + kLoBytes + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(kStages >= 2, "ring too shallow");
  static_assert(kUsedCols <= 512, "TMEM");
};

template <int NPAD, bool X3, bool LT = false>
struct TcSmem {
  using C = TcCfg<NPAD, X3, LT>;
  unsigned char* base;
  uint64_t *full, *empty, *lofull, *loempty, *tfull, *tempty;
  uint32_t* tmem_slot;
  __device__ explicit TcSmem(unsigned char* raw) {
    base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + size_t(C::kStages) * C::kStageBytes + C::kLoBytes);
    full = bars;
    empty = full + C::kStages;
    lofull = empty + C::kStages;
    loempty = lofull + C::kLoN;
    tfull = loempty + C::kLoN;
    tempty = tfull + 2;
    tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  }
  __device__ unsigned char* x(int s) const { return base + size_t(s) * C::kStageBytes; }
  __device__ unsigned char* shi(int s) const { return x(s) + kXTileBytes; }
  __device__ unsigned char* slo(int s) const { return shi(s) + C::kSBytes; }
  __device__ unsigned char* lo(int j) const { return base + size_t(C::kStages) * C::kStageBytes + size_t(j) * kXTileBytes; }
  __device__ void init() const {
    for (int s = 0; s < C::kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < C::kLoN; ++j) {
      tc::mbar_init(&lofull[j], LT ? C::kSplit / 32 : C::kSplit);
      tc::mbar_init(&loempty[j], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    tc::fence_mbar_init();
  }
};

#ifdef RNMF_TC_PROF
// (development) cycles CTA 0's roles spend waiting / working in tc_xw_kernel<LT>, read by tools
__device__ long long g_tc_prof[16];
#define TCP_T0() const long long tcp_t0 = clock64()
#define TCP_ADD(slot) do { tcp_acc[slot] += clock64() - tcp_t0; } while (0)
#define TCP_DECL() long long tcp_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}
#define TCP_FLUSH() do { if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64 || threadIdx.x == 128)) for (int i = 0; i < 9; ++i) if (tcp_acc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(&g_tc_prof[i]), (unsigned long long)tcp_acc[i]); } while (0)
#else
#define TCP_T0() do { } while (0)
#define TCP_ADD(slot) do { } while (0)
#define TCP_DECL() do { } while (0)
#define TCP_FLUSH() do { } while (0)
#endif

// LT split warps: 2, 3 and 8..13 -- two warps per TMEM lane quadrant (warp % 4), the first of a
// pair taking K columns 0..15 of the stage and the second 16..31.
__device__ __forceinline__ int lt_half(int warp) { return (warp == 2 || warp == 3 || warp == 8 || warp == 9) ? 0 : 1; }

// lo of 16 K values of one A row -> TMEM (lane = A row, 16 columns from taddr)
__device__ __forceinline__ void lt_store16(uint32_t taddr, const uint32_t (&v)[16]) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = tf32_lo_bits(v[i]);
  tc::tmem_st_32x32b_x16(taddr, r);
  tc::tmem_st_wait();
  tc::tc_fence_before();
}

// One K stage of UMMAs into accumulator buffer d.  a_desc(k, base) builds the A descriptor of
// k-step k (A = X tile hi or lo); B is K-major SW128 in either kernel.
template <int NPAD, bool X3, bool A_MN, bool LT = false, typename ADesc>
__device__ __forceinline__ void issue_stage(uint32_t d, uint32_t xa, uint32_t la, uint32_t ba, bool fresh, ADesc a_desc) {
  constexpr uint32_t idesc1 = tc::make_idesc_tf32(NPAD, A_MN, false);
  constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, A_MN, false);
  constexpr uint32_t idesc_ts = tc::make_idesc_tf32(NPAD, false, false);  // A from TMEM (la = TMEM address)
#pragma unroll
  for (int k = 0; k < kBK / 8; ++k) {
    const uint64_t adesc = a_desc(xa, k);
    const uint64_t bdesc = tc::make_sdesc(ba + k * 32, 16, 1024);
    const uint32_t acc = (fresh && k == 0) ? 0u : 1u;
    if (X3) {
#ifdef RNMF_TC_DBG_NOSLO  // (experiment) hi MMA without the S_lo half
      tc::umma_tf32(d, adesc, bdesc, idesc1, acc);
#else
      tc::umma_tf32(d, adesc, bdesc, idesc2, acc);                                 // X_hi [S_hi; S_lo]
#endif
#ifndef RNMF_TC_DBG_NOLOMMA
      if (LT)
        tc::umma_tf32_ts(d + NPAD, la + uint32_t(k * 8), bdesc, idesc_ts, 1u);     // += X_lo S_hi, A in TMEM
      else
        tc::umma_tf32(d + NPAD, a_desc(la, k), bdesc, idesc1, 1u);                 // += X_lo S_hi (small terms)
#endif
    } else {
      tc::umma_tf32(d, adesc, bdesc, idesc1, acc);
    }
  }
}

// Epilogue: add one accumulator buffer (this warp's 32 lanes) into the fp32 registers a[]:
// a += hihi + small, each add rounded to nearest.
template <int NPAD, bool X3, bool WIDE = true>
__device__ __forceinline__ void drain_acc(uint32_t taddr, float (&a)[NPAD]) {
  if constexpr (X3 && NPAD % 32 == 0 && WIDE) {
    // 32-column loads of both halves, one wait per 32 columns
#pragma unroll
    for (int cc = 0; cc < NPAD / 32; ++cc) {
      uint32_t r0[32], r1[32];
      tc::tmem_ld_32x32b_x32(taddr + cc * 32, r0);
      tc::tmem_ld_32x32b_x32(taddr + NPAD + cc * 32, r1);
      tc::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 32; ++q) a[cc * 32 + q] += __uint_as_float(r0[q]) + __uint_as_float(r1[q]);
    }
  } else {
#pragma unroll
    for (int cc = 0; cc < NPAD / 16; ++cc) {
      uint32_t r0[16];
      tc::tmem_ld_32x32b_x16(taddr + cc * 16, r0);
      if (X3) {
        uint32_t r1[16];
        tc::tmem_ld_32x32b_x16(taddr + NPAD + cc * 16, r1);
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) a[cc * 16 + q] += __uint_as_float(r0[q]) + __uint_as_float(r1[q]);
      } else {
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) a[cc * 16 + q] += __uint_as_float(r0[q]);
      }
    }
  }
}

struct XwParams {
  int64_t m, n;
  int c;
  float* y;
  int64_t ldy;
  int chunk;  // K stages per TMEM accumulation chunk
};

// ------------------------------------------------------------------------------------------------
// tc_xw: Y (m x c) = X (m x n) S (n x c); one 128-row tile per work unit, K = n.
// The K loop is cut into chunks of p.chunk stages; each chunk starts a fresh TMEM accumulator that
// the epilogue adds into fp32 registers, so the tensor core's truncating accumulation never runs
// over more than p.chunk * 32 terms (tools/sketch_acc.cu measures the effect).
template <int NPAD, bool X3, bool LT>
__global__ void __launch_bounds__((TcCfg<NPAD, X3, LT>::kThreads), 1) tc_xw_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                    const __grid_constant__ CUtensorMap tmShi,
                                                                    const __grid_constant__ CUtensorMap tmSlo, XwParams p) {
  using C = TcCfg<NPAD, X3, LT>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const TcSmem<NPAD, X3, LT> sm(smem_raw);
  TCP_DECL();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(p.m, kBM);
  const int nk = int(ceil_div(p.n, kBK));

  if (threadIdx.x == 0) {
    sm.init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmShi);
    if (X3) tc::tma_prefetch(&tmSlo);
  }
  if (warp == 1) tc::tmem_alloc<C::kTmemCols>(sm.tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *sm.tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (tc::elect_one()) {
      uint32_t it = 0;
      // 3xTF32: only the raw S^T slab comes from L2 and the split warps write its lo slab on chip;
      // LT: the split warps only handle X, the lo slab comes by TMA
#ifdef RNMF_TC_XW_SLO_ONCHIP  // (experiment) LT with the S^T lo slab split on chip, as X^T S does
      constexpr bool kSloTma = false;
#else
      constexpr bool kSloTma = LT;
#endif
      const uint32_t bytes = uint32_t(kXTileBytes + C::kSBytes * (kSloTma ? 2 : 1));
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          { TCP_T0(); tc::mbar_wait(&sm.empty[s], ((it / S) & 1) ^ 1); TCP_ADD(0); }
#ifdef RNMF_TC_DBG_NOSLOAD  // (experiment) the S slab only on the first pass over the ring
          if (it >= uint32_t(S)) {
            tc::mbar_arrive_expect_tx(&sm.full[s], uint32_t(kXTileBytes));
            tc::tma_load_2d_hint(sm.x(s), &tmX, &sm.full[s], kc * kBK, int(t * kBM), kXPolicy);
            continue;
          }
#endif
          tc::mbar_arrive_expect_tx(&sm.full[s], bytes);
          tc::tma_load_2d_hint(sm.x(s), &tmX, &sm.full[s], kc * kBK, int(t * kBM), kXPolicy);
          tc::tma_load_2d_hint(sm.shi(s), &tmShi, &sm.full[s], kc * kBK, 0, kSPolicy);
          if (kSloTma) tc::tma_load_2d_hint(sm.slo(s), &tmSlo, &sm.full[s], kc * kBK, 0, kSPolicy);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer
    if constexpr (LT) {
      // descriptors as {lo, hi} words advanced by adds (no make_sdesc per K step), no integer
      // divisions in the loop; the stage's single commit releases the X / S stage and its TMEM lo
      // slot together.  The whole warp runs the loop and one elected lane issues (an `if (lane == 0)`
      // loop makes the compiler wrap every UTCHMMA in an election loop).
      constexpr uint32_t kHi = tc::sdesc_hi(1024, tc::kLayoutSW128);
      constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, false, false);
      constexpr uint32_t idesc_ts = tc::make_idesc_tf32(NPAD, false, false);
      const uint32_t x0 = (tc::smem_u32(sm.x(0)) >> 4) + tc::sdesc_lo_const(16);
      uint32_t ci = 0, s = 0, ph = 0;
      uint32_t d = tmem_base;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int kin = 0;
        for (int kc = 0; kc < nk; ++kc) {
          const bool cend = (kin == p.chunk - 1) || (kc == nk - 1);
          const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
          if (kin == 0) {
            TCP_T0();
            tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
            TCP_ADD(1);
            d = tmem_base + uint32_t(acc * C::kAccCols);
          }
          { TCP_T0(); tc::mbar_wait(&sm.full[s], ph); TCP_ADD(2); }
          { TCP_T0(); tc::mbar_wait(&sm.lofull[s], ph); TCP_ADD(3); }
          tc::tc_fence_after();
          TCP_T0();
          if (tc::elect_one()) {
            const uint32_t xa = x0 + s * uint32_t(C::kStageBytes >> 4), ba = xa + uint32_t(kXTileBytes >> 4);
            const uint32_t la = tmem_base + uint32_t(C::kLoBase) + s * uint32_t(kBK);
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              tc::umma_tf32_w(d, xa + 2 * k, kHi, ba + 2 * k, kHi, idesc2, (kin == 0 && k == 0) ? 0u : 1u);
#ifndef RNMF_TC_DBG_NOLOMMA
              tc::umma_tf32_ts_w(d + NPAD, la + 8 * k, ba + 2 * k, kHi, idesc_ts, 1u);
#endif
            }
            tc::umma_commit(&sm.empty[s]);
            if (cend) tc::umma_commit(&sm.tfull[acc]);
          }
          __syncwarp();
          if (cend) {
            ++ci;
            kin = 0;
          } else {
            ++kin;
          }
          if (++s == uint32_t(S)) s = 0, ph ^= 1;
          TCP_ADD(4);
        }
      }
    } else {
    uint32_t it = 0, ci = 0;
    uint32_t d = tmem_base;
    auto adesc = [](uint32_t base, int k) { return tc::make_sdesc(base + k * 32, 16, 1024); };
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int kin = kc % p.chunk;
        const bool cend = (kin == p.chunk - 1) || (kc == nk - 1);
        const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
        if (kin == 0) {
          tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
          tc::tc_fence_after();
          d = tmem_base + uint32_t(acc * C::kAccCols);
        }
        const int s = int(it % S), j = int(it % kLoSlots);
        tc::mbar_wait(&sm.full[s], (it / S) & 1);
        if (X3) tc::mbar_wait(&sm.lofull[j], (it / kLoSlots) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          issue_stage<NPAD, X3, false>(d, tc::smem_u32(sm.x(s)), tc::smem_u32(sm.lo(j)), tc::smem_u32(sm.shi(s)),
                                       kin == 0, adesc);
          tc::umma_commit(&sm.empty[s]);
          if (X3) tc::umma_commit(&sm.loempty[j]);
          if (cend) tc::umma_commit(&sm.tfull[acc]);
        }
        if (cend) ++ci;
        __syncwarp();
      }
    }
    }
  } else if (warp < 4 || warp >= 8) {
    // ---------------- 3xTF32 split warps
    if constexpr (LT) {
      // lo of this thread's X row (16 of the stage's 32 K values) -> the TMEM lo ring
      const int quad = warp & 3, r = quad * 32 + lane, half = lt_half(warp);
      const uint32_t lane_off = uint32_t(quad * 32) << 16;
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          // full[s] of this pass implies the UMMAs that read TMEM lo slot s a ring ago are done (the
          // producer refilled the stage only after their commit)
          const int s = int(it % S);
          {  // one lane polls the barrier for its warp
            TCP_T0();
            if (lane == 0) tc::mbar_wait(&sm.full[s], (it / S) & 1);
            __syncwarp();
            TCP_ADD(5);
          }
          TCP_T0();
          const uint32_t xrow = tc::smem_u32(sm.x(s)) + uint32_t(r) * 128u;
          uint32_t v[16];
#pragma unroll
          for (int c = 0; c < 4; ++c)  // 16-byte chunk 4 half + c of the row, 128 B swizzle
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[4 * c]), "=r"(v[4 * c + 1]), "=r"(v[4 * c + 2]), "=r"(v[4 * c + 3])
                         : "r"(xrow + uint32_t(((4 * half + c) ^ (r & 7)) * 16)) : "memory");
          tc::tc_fence_after();
#ifndef RNMF_TC_DBG_NOSPLIT
          lt_store16(tmem_base + lane_off + uint32_t(C::kLoBase + s * kBK + half * 16), v);
#ifdef RNMF_TC_XW_SLO_ONCHIP
          split_lo_tile<C::kSBytes / 16, 256>(reinterpret_cast<const float4*>(sm.shi(s)),
                                              reinterpret_cast<float4*>(sm.slo(s)), (quad * 2 + half) * 32 + lane);
          tc::fence_proxy_async_smem();
#endif
#endif
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sm.lofull[s]);
          TCP_ADD(6);
        }
      }
    } else if (X3) {  // lo tiles into their own shared-memory ring
      const int st = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 192;  // 0..191
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S), j = int(it % kLoSlots);
          tc::mbar_wait(&sm.full[s], (it / S) & 1);
          tc::mbar_wait(&sm.loempty[j], ((it / kLoSlots) & 1) ^ 1);
#ifndef RNMF_TC_DBG_NOSPLIT
          split_lo_tile<kXTileBytes / 16>(reinterpret_cast<const float4*>(sm.x(s)), reinterpret_cast<float4*>(sm.lo(j)), st);
          split_lo_tile<C::kSBytes / 16>(reinterpret_cast<const float4*>(sm.shi(s)), reinterpret_cast<float4*>(sm.slo(s)), st);
#endif
          tc::fence_proxy_async_smem();
          tc::mbar_arrive(&sm.lofull[j]);
        }
      }
    }
  } else {
    // ---------------- epilogue: TMEM chunks -> fp32 registers -> Y
    const int sub = warp & 3;
    const int nch = (nk + p.chunk - 1) / p.chunk;
    uint32_t ci = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t row = t * kBM + sub * 32 + lane;
      float a[NPAD];
#pragma unroll
      for (int q = 0; q < NPAD; ++q) a[q] = 0.f;
      for (int ch = 0; ch < nch; ++ch, ++ci) {
        const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
        { TCP_T0(); tc::mbar_wait(&sm.tfull[acc], (C::kAccBufs == 2 ? ci >> 1 : ci) & 1); TCP_ADD(7); }
        TCP_T0();
        tc::tc_fence_after();
        drain_acc<NPAD, X3, !(LT && NPAD > 48)>(tmem_base + (uint32_t(sub * 32) << 16) + uint32_t(acc * C::kAccCols), a);
        tc::tc_fence_before();
        tc::mbar_arrive(&sm.tempty[acc]);
        TCP_ADD(8);
      }
      if (row < p.m) {
#pragma unroll
        for (int q = 0; q < NPAD; ++q)
          if (q < p.c) p.y[row * p.ldy + q] = a[q];
      }
    }
  }
  TCP_FLUSH();
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// Work unit u -> (column tile, row split).  Split-major: the CTAs running at one time take the
// column tiles of ONE row split, so the S^T rows they re-read are one split's (l x m / splits:
// 6 MB at C4 instead of all 51 MB) and neighbouring CTAs read adjacent 512-byte segments of the same
// X rows.  RNMF_TC_XTW_TILE_MAJOR restores the round-1 order (u = tile * splits + split).
#ifdef RNMF_TC_XTW_TILE_MAJOR
#define RNMF_XTW_UNIT_CT(u) ((u) / p.splits)
#define RNMF_XTW_UNIT_SPLIT(u) ((u) % p.splits)
#else
#define RNMF_XTW_UNIT_CT(u) ((u) % ctiles)
#define RNMF_XTW_UNIT_SPLIT(u) ((u) / ctiles)
#endif

// ------------------------------------------------------------------------------------------------
// tc_xtw: part[split] (n x c) = X[rows of split]^T (n x m_s) * S[rows of split] (m_s x c)
//   A = X^T tile: M = 128 X columns (MN-major: four 32-column TMA boxes, LBO = 4 KB),
//       K = 32 X rows per stage (SBO = 512 B per 4 rows, SW128_BASE32B)
//   B = S^T slab (N = NPAD rows of the transposed small operand, K-major)
// One work unit = (128-column tile, row split); units are distributed over persistent CTAs.
struct XtwParams {
  int64_t m, n;
  int c;
  int splits;
  float* part;  // splits x n x c
  int chunk;    // K stages (32 rows each) per TMEM accumulation chunk
};

template <int NPAD, bool X3, bool LT>
__global__ void __launch_bounds__((TcCfg<NPAD, X3, LT>::kThreads), 1) tc_xtw_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                     const __grid_constant__ CUtensorMap tmSt,
                                                                     const __grid_constant__ CUtensorMap tmStLo, XtwParams p) {
  using C = TcCfg<NPAD, X3, LT>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const TcSmem<NPAD, X3, LT> sm(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ctiles = ceil_div(p.n, 128);
  const int64_t units = ctiles * p.splits;

  if (threadIdx.x == 0) {
    sm.init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmSt);
    if (X3) tc::tma_prefetch(&tmStLo);
  }
  if (warp == 1) tc::tmem_alloc<C::kTmemCols>(sm.tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *sm.tmem_slot;

  // split boundaries on 32-row stage boundaries, so no stage straddles two splits
  const int64_t mstages = ceil_div(p.m, kBK);
  auto unit_rows = [&](int64_t u, int64_t& r0, int64_t& r1) {
    const int64_t sp = RNMF_XTW_UNIT_SPLIT(u);
    r0 = (mstages * sp / p.splits) * kBK;
    r1 = (mstages * (sp + 1) / p.splits) * kBK;
  };

  if (warp == 0) {
    if (tc::elect_one()) {
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t ct = RNMF_XTW_UNIT_CT(u);
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        for (int64_t r = r0; r < r1; r += kBK, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&sm.empty[s], ((it / S) & 1) ^ 1);
          // 3xTF32: the raw S^T slab only; its lo slab is written on chip by the split warps
          // the S^T slab raw only: its lo slab is written on chip by the split warps (S^T = Q^T is
          // l x m here, re-read by every column tile; loading a second copy through L2 cost 7 % more
          // DRAM traffic than splitting on chip)
          tc::mbar_arrive_expect_tx(&sm.full[s], uint32_t(kXTileBytes + C::kSBytes));
#pragma unroll
          for (int b = 0; b < 4; ++b)
            tc::tma_load_2d_hint(sm.x(s) + b * 4096, &tmX, &sm.full[s], int(ct * 128 + b * 32), int(r), kXPolicy);
          tc::tma_load_2d_hint(sm.shi(s), &tmSt, &sm.full[s], int(r), 0, kSPolicy);
        }
      }
    }
  } else if (warp == 1) {
    if constexpr (LT) {
      constexpr uint32_t kAHi = tc::sdesc_hi(512, tc::kLayoutSW128Base32B);  // MN-major A: SBO 512 B per 4 rows
      constexpr uint32_t kBHi = tc::sdesc_hi(1024, tc::kLayoutSW128);
      constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, true, false);
      constexpr uint32_t idesc_ts = tc::make_idesc_tf32(NPAD, false, false);
      const uint32_t a0 = (tc::smem_u32(sm.x(0)) >> 4) + tc::sdesc_lo_const(4096);  // LBO 4 KB between boxes
      const uint32_t b0 = (tc::smem_u32(sm.shi(0)) >> 4) + tc::sdesc_lo_const(16);
      uint32_t ci = 0, s = 0, ph = 0;
      uint32_t d = tmem_base;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        if (r0 >= r1) {  // empty split: still hand an (all-zero) chunk to the epilogue
          const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
          tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
          if (tc::elect_one()) tc::mbar_arrive(&sm.tfull[acc]);
          ++ci;
          __syncwarp();
          continue;
        }
        int kin = 0;
        for (int64_t r = r0; r < r1; r += kBK) {
          const bool cend = (kin == p.chunk - 1) || (r + kBK >= r1);
          const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
          if (kin == 0) {
            tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
            d = tmem_base + uint32_t(acc * C::kAccCols);
          }
          tc::mbar_wait(&sm.full[s], ph);
          tc::mbar_wait(&sm.lofull[s], ph);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t xa = a0 + s * uint32_t(C::kStageBytes >> 4), ba = b0 + s * uint32_t(C::kStageBytes >> 4);
            const uint32_t la = tmem_base + uint32_t(C::kLoBase) + s * uint32_t(kBK);
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              tc::umma_tf32_w(d, xa + 64 * k, kAHi, ba + 2 * k, kBHi, idesc2, (kin == 0 && k == 0) ? 0u : 1u);
#ifndef RNMF_TC_DBG_NOLOMMA
              tc::umma_tf32_ts_w(d + NPAD, la + 8 * k, ba + 2 * k, kBHi, idesc_ts, 1u);
#endif
            }
            tc::umma_commit(&sm.empty[s]);
            if (cend) tc::umma_commit(&sm.tfull[acc]);
          }
          __syncwarp();
          if (cend) {
            ++ci;
            kin = 0;
          } else {
            ++kin;
          }
          if (++s == uint32_t(S)) s = 0, ph ^= 1;
        }
      }
    } else {
    uint32_t it = 0, ci = 0;
    uint32_t d = tmem_base;
    // MN-major A (SW128_BASE32B): LBO = 4 KB between 32-column boxes, SBO = 512 B per 4 rows
    auto adesc = [](uint32_t base, int k) { return tc::make_sdesc(base + k * 1024, 4096, 512, tc::kLayoutSW128Base32B); };
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t r0, r1;
      unit_rows(u, r0, r1);
      if (r0 >= r1) {  // empty split: still hand an (all-zero) chunk to the epilogue
        const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
        tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
        if (tc::elect_one()) tc::mbar_arrive(&sm.tfull[acc]);
        ++ci;
        __syncwarp();
        continue;
      }
      int kin = 0;
      for (int64_t r = r0; r < r1; r += kBK, ++it) {
        const bool cend = (kin == p.chunk - 1) || (r + kBK >= r1);
        const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
        if (kin == 0) {
          tc::mbar_wait(&sm.tempty[acc], ((C::kAccBufs == 2 ? ci >> 1 : ci) & 1) ^ 1);
          tc::tc_fence_after();
          d = tmem_base + uint32_t(acc * C::kAccCols);
        }
        const int s = int(it % S), j = int(it % C::kLoN);
        tc::mbar_wait(&sm.full[s], (it / S) & 1);
        if (X3) tc::mbar_wait(&sm.lofull[j], (it / C::kLoN) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          issue_stage<NPAD, X3, true, LT>(d, tc::smem_u32(sm.x(s)),
                                          LT ? tmem_base + uint32_t(C::kLoBase + j * kBK) : tc::smem_u32(sm.lo(j)),
                                          tc::smem_u32(sm.shi(s)), kin == 0, adesc);
          tc::umma_commit(&sm.empty[s]);
          if (X3) tc::umma_commit(&sm.loempty[j]);
          if (cend) tc::umma_commit(&sm.tfull[acc]);
        }
        if (cend) {
          ++ci;
          kin = 0;
        } else {
          ++kin;
        }
        __syncwarp();
      }
    }
    }
  } else if (warp < 4 || warp >= 8) {
    if constexpr (LT) {
      // A row = X column quad * 32 + lane of the tile (box quad); K = 16 of the stage's 32 X rows.
      // SW128_BASE32B: the 32-byte granule of a 128-byte row is XORed with (row & 3).
      const int quad = warp & 3, half = lt_half(warp);
      const uint32_t lane_off = uint32_t(quad * 32) << 16;
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        for (int64_t r = r0; r < r1; r += kBK, ++it) {
          const int s = int(it % S);
          if (lane == 0) tc::mbar_wait(&sm.full[s], (it / S) & 1);
          __syncwarp();
          const uint32_t box = tc::smem_u32(sm.x(s)) + uint32_t(quad) * 4096u + uint32_t(lane & 7) * 4u;
          uint32_t v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int kr = half * 16 + i;
            asm volatile("ld.shared.b32 %0, [%1];"
                         : "=r"(v[i])
                         : "r"(box + uint32_t(kr) * 128u + uint32_t(((lane >> 3) ^ (kr & 3)) << 5)) : "memory");
          }
          tc::tc_fence_after();
#ifndef RNMF_TC_DBG_NOSPLIT
          lt_store16(tmem_base + lane_off + uint32_t(C::kLoBase + s * kBK + half * 16), v);
          split_lo_tile<C::kSBytes / 16, 256>(reinterpret_cast<const float4*>(sm.shi(s)),
                                              reinterpret_cast<float4*>(sm.slo(s)), (quad * 2 + half) * 32 + lane);
          tc::fence_proxy_async_smem();
#endif
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sm.lofull[s]);
        }
      }
    } else if (X3) {  // 3xTF32 lo tiles (elementwise, so the swizzled layout is irrelevant)
      const int st = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 192;
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t r0, r1;
        unit_rows(u, r0, r1);
        for (int64_t r = r0; r < r1; r += kBK, ++it) {
          const int s = int(it % S), j = int(it % kLoSlots);
          tc::mbar_wait(&sm.full[s], (it / S) & 1);
          tc::mbar_wait(&sm.loempty[j], ((it / kLoSlots) & 1) ^ 1);
#ifndef RNMF_TC_DBG_NOSPLIT
          split_lo_tile<kXTileBytes / 16>(reinterpret_cast<const float4*>(sm.x(s)), reinterpret_cast<float4*>(sm.lo(j)), st);
          split_lo_tile<C::kSBytes / 16>(reinterpret_cast<const float4*>(sm.shi(s)), reinterpret_cast<float4*>(sm.slo(s)), st);
#endif
          tc::fence_proxy_async_smem();
          tc::mbar_arrive(&sm.lofull[j]);
        }
      }
    }
  } else {
    const int sub = warp & 3;
    uint32_t ci = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t ct = RNMF_XTW_UNIT_CT(u), sp = RNMF_XTW_UNIT_SPLIT(u);
      int64_t r0, r1;
      unit_rows(u, r0, r1);
      const int64_t nst = (r1 - r0) / kBK;
      const int64_t nch = r0 < r1 ? (nst + p.chunk - 1) / p.chunk : 1;
      const int64_t col = ct * 128 + sub * 32 + lane;  // X column = output row of P
      float a[NPAD];
#pragma unroll
      for (int q = 0; q < NPAD; ++q) a[q] = 0.f;
      for (int64_t ch = 0; ch < nch; ++ch, ++ci) {
        const int acc = C::kAccBufs == 2 ? int(ci & 1) : 0;
        tc::mbar_wait(&sm.tfull[acc], (C::kAccBufs == 2 ? ci >> 1 : ci) & 1);
        tc::tc_fence_after();
        if (r0 < r1) drain_acc<NPAD, X3, !(LT && NPAD > 48)>(tmem_base + (uint32_t(sub * 32) << 16) + uint32_t(acc * C::kAccCols), a);
        tc::tc_fence_before();
        tc::mbar_arrive(&sm.tempty[acc]);
      }
      if (col < p.n) {
        float* out = p.part + (sp * p.n + col) * p.c;
#pragma unroll
        for (int q = 0; q < NPAD; ++q)
          if (q < p.c) out[q] = a[q];
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// S (n x c, row-major, ld c) -> S^T hi / lo (npad x ldst, zero rows for j >= c and cols >= n).
// 3xTF32 (raw): hi = s itself (kind::tf32 truncates it) and lo = rna_tf32(s - trunc_tf32(s)), the
// split the kernels also apply on chip to X and to the S slabs; 1xTF32: hi = rna_tf32(s).
__global__ void prep_st_kernel(const float* __restrict__ s, int64_t n, int c, int npad, int64_t ldst,
                               float* __restrict__ st_hi, float* __restrict__ st_lo, bool raw) {
  const int64_t total = int64_t(npad) * ldst;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / ldst);
    const int64_t kk = e % ldst;
    const float v = (j < c && kk < n) ? s[kk * c + j] : 0.f;
    if (raw) {
      st_hi[e] = v;
      st_lo[e] = tf32_lo(v);
    } else {
      const float h = tc::tf32_hi(v);
      st_hi[e] = h;
      st_lo[e] = tc::tf32_hi(v - h);
    }
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

// K stages (32 columns / rows each) per TMEM accumulation chunk; RNMF_TC_CHUNK overrides.
int g_tc_chunk = 0;
int tc_chunk_stages() {
  if (g_tc_chunk <= 0) {
    const char* e = std::getenv("RNMF_TC_CHUNK");
    const int c = e ? std::atoi(e) : 0;
    g_tc_chunk = c > 0 ? c : 4;
  }
  return g_tc_chunk;
}

// LT (lo X tile in tensor memory) whenever its 448-thread CTA keeps the epilogue's NPAD fp32
// accumulators in registers; RNMF_TC_NO_LT=1 forces the shared-memory lo ring (testing knob)
template <int NPAD, bool X3>
constexpr bool tc_lt_ok() { return X3 && NPAD <= 64; }
inline bool tc_lt_enabled() {
  static const bool off = std::getenv("RNMF_TC_NO_LT") != nullptr;
  return !off;
}

template <int NPAD, bool X3, bool LT>
void tc_xw_launch_lt(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                     int64_t ldst, int c, float* y, int sm_count, cudaStream_t stream) {
  using C = TcCfg<NPAD, X3, LT>;
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBM);
  const CUtensorMap mh = make_map_2d(st_hi, NPAD, n, ldst, NPAD);
  const CUtensorMap ml = make_map_2d(st_lo, NPAD, n, ldst, NPAD);
  XwParams p{m, n, c, y, c, tc_chunk_stages()};
  auto f = tc_xw_kernel<NPAD, X3, LT>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  const int64_t ntiles = ceil_div(m, kBM);
  const int grid = int(std::min<int64_t>(ntiles, sm_count));
  f<<<grid, C::kThreads, C::kSmem, stream>>>(mx, mh, ml, p);
  RNMF_CUDA_LAUNCH();
}

template <int NPAD, bool X3>
void tc_xw_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                  int64_t ldst, int c, float* y, int sm_count, cudaStream_t stream) {
  if constexpr (tc_lt_ok<NPAD, X3>()) {
    if (tc_lt_enabled()) return tc_xw_launch_lt<NPAD, X3, true>(x, m, n, ldx, st_hi, st_lo, ldst, c, y, sm_count, stream);
  }
  tc_xw_launch_lt<NPAD, X3, false>(x, m, n, ldx, st_hi, st_lo, ldst, c, y, sm_count, stream);
}

template <int NPAD, bool X3, bool LT>
void tc_xtw_launch_lt(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st, const float* st_lo, int64_t ldst,
                      int c, float* part, int splits, int sm_count, cudaStream_t stream) {
  using C = TcCfg<NPAD, X3, LT>;
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);  // 32 x 32 boxes
  const CUtensorMap ms = make_map_2d(st, NPAD, m, ldst, NPAD);  // S^T: NPAD rows x m
  const CUtensorMap ml = make_map_2d(X3 ? st_lo : st, NPAD, m, ldst, NPAD);
  XtwParams p{m, n, c, splits, part, tc_chunk_stages()};
  auto f = tc_xtw_kernel<NPAD, X3, LT>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  const int64_t units = ceil_div(n, 128) * splits;
  const int grid = int(std::min<int64_t>(units, sm_count));
  f<<<grid, C::kThreads, C::kSmem, stream>>>(mx, ms, ml, p);
  RNMF_CUDA_LAUNCH();
}

template <int NPAD, bool X3>
void tc_xtw_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st, const float* st_lo, int64_t ldst,
                   int c, float* part, int splits, int sm_count, cudaStream_t stream) {
  if constexpr (tc_lt_ok<NPAD, X3>()) {
    if (tc_lt_enabled())
      return tc_xtw_launch_lt<NPAD, X3, true>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream);
  }
  tc_xtw_launch_lt<NPAD, X3, false>(x, m, n, ldx, st, st_lo, ldst, c, part, splits, sm_count, stream);
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

// Row splits of X^T S: the (column tile, split) units are spread over the persistent CTAs, so pick
// the split count whose unit count fills the last round best (units / (rounds * CTAs)), with at
// least 4 K stages (128 rows) per unit; near-ties go to fewer splits (less partial traffic).
// E.g. C4 (157 column tiles): 8 splits, 94 % of 9 rounds, instead of 1 split and 53 % of 2 rounds.
int tc_xtw_splits(int64_t m, int64_t n, int sm_count) {
  const int64_t ct = ceil_div(n, 128);
  const int64_t G = std::max(sm_count, 1);
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(256, m / (4 * kBK)));
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t units = ct * s;
    const double eff = double(units) / double(ceil_div(units, G) * G);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return int(best);
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

#ifdef RNMF_TC_PROF
void tc_prof_read(long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(long long) * 16);
  if (reset) {
    long long z[16] = {};
    cudaMemcpyToSymbol(g_tc_prof, z, sizeof z);
  }
}
#endif

int tc_npad(int c) { return int(ceil_div(c, 16) * 16); }

void tc_set_chunk(int stages) { g_tc_chunk = stages; }

int64_t tc_st_pitch(int64_t n) { return ceil_div(n, 32) * 32; }

int launch_tc_prep_st(const float* s, int64_t n, int c, float* st_hi, float* st_lo, cudaStream_t stream, bool raw) {
  const int npad = tc_npad(c);
  const int64_t ld = tc_st_pitch(n);
  const int blocks = int(std::min<int64_t>(ceil_div(int64_t(npad) * ld, 256), 148 * 8));
  prep_st_kernel<<<blocks, 256, 0, stream>>>(s, n, c, npad, ld, st_hi, st_lo, raw);
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


// ================================================================================================
// Full-space metrics on the tensor cores (tc_metrics.h).
// ================================================================================================
namespace {

// tc_resid: per 128-row tile t, per 32-column stage: D (128 x 32) = W_t H(:, cols) by 3xTF32
//   UMMAs (A = W tile hi / lo, K-major SW128, resident per tile; B = [H^T hi; H^T lo] slab, 2 x 32
//   rows per 32-wide K atom, so X-free D[0:32) = W_hi H_hi, D[32:64) = W_hi H_lo + W_lo H_hi), then
//   the epilogue reads its row of the X stage from shared memory and accumulates (x - wh)^2.
// Roles: warp 0 TMA producer, warp 1 UMMA issuer, warps 4-7 epilogue (thread = row).
constexpr int kRsThreads = 256;
constexpr int kRsTmemBufs = 4;  // 64-column D buffers

template <int KW>
struct RsCfg {
  static constexpr int kAtoms = KW / 32;
  static constexpr int kWBytes = 2 * kAtoms * kXTileBytes;        // W_hi, W_lo atoms (128 rows each)
  static constexpr int kHtAtomBytes = 2 * 32 * 128;                 // 32 hi rows + 32 lo rows
  static constexpr int kStageBytes = kXTileBytes + kAtoms * kHtAtomBytes;
  static constexpr int kStages = std::min(8, (kSmemBudget - kWBytes - 2048) / kStageBytes);
  static constexpr size_t kSmem = size_t(kWBytes) + size_t(kStages) * kStageBytes + 1024 + 512;
  static_assert(kStages >= 2, "ring too shallow");
};

template <int KW>
__global__ void __launch_bounds__(kRsThreads, 1) tc_resid_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                  const __grid_constant__ CUtensorMap tmWhi,
                                                                  const __grid_constant__ CUtensorMap tmWlo,
                                                                  const __grid_constant__ CUtensorMap tmHhi,
                                                                  const __grid_constant__ CUtensorMap tmHlo, int64_t m,
                                                                  int64_t n, double* __restrict__ part_obj) {
  using C = RsCfg<KW>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* wsm = base;  // [hi atoms][lo atoms], 16 KB each
  auto xst = [&](int s) { return base + C::kWBytes + size_t(s) * C::kStageBytes; };
  auto hst = [&](int s) { return xst(s) + kXTileBytes; };  // atom a: hi rows at a * 8 KB, lo rows +4 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::kWBytes + size_t(S) * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + kRsTmemBufs;
  uint64_t* wfull = tempty + kRsTmemBufs;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  double* red = reinterpret_cast<double*>(wempty + 2);  // 4 doubles

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(m, kBM);
  const int nk = int(ceil_div(n, kBK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + 128);  // UMMA commit (H slab read) + every epilogue thread (X row read)
    }
    for (int b = 0; b < kRsTmemBufs; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 128);
    }
    tc::mbar_init(wfull, 1);
    tc::mbar_init(wempty, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmWhi);
    tc::tma_prefetch(&tmWlo);
    tc::tma_prefetch(&tmHhi);
    tc::tma_prefetch(&tmHlo);
  }
  if (warp == 1) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      uint32_t it = 0, ti = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
        // W tile (hi, lo) once per row tile, after the previous tile's UMMAs are done with it
        tc::mbar_wait(wempty, (ti & 1) ^ 1);
        tc::mbar_arrive_expect_tx(wfull, uint32_t(C::kWBytes));
#pragma unroll
        for (int a = 0; a < C::kAtoms; ++a) {
          tc::tma_load_2d(wsm + a * kXTileBytes, &tmWhi, wfull, a * 32, int(t * kBM));
          tc::tma_load_2d(wsm + (C::kAtoms + a) * kXTileBytes, &tmWlo, wfull, a * 32, int(t * kBM));
        }
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], uint32_t(C::kStageBytes));
          tc::tma_load_2d_hint(xst(s), &tmX, &full[s], kc * kBK, int(t * kBM), kXPolicy);
#pragma unroll
          for (int a = 0; a < C::kAtoms; ++a) {
            tc::tma_load_2d(hst(s) + a * C::kHtAtomBytes, &tmHhi, &full[s], a * 32, kc * kBK);
            tc::tma_load_2d(hst(s) + a * C::kHtAtomBytes + 4096, &tmHlo, &full[s], a * 32, kc * kBK);
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc1 = tc::make_idesc_tf32(32, false, false);
    constexpr uint32_t idesc2 = tc::make_idesc_tf32(64, false, false);
    uint32_t it = 0, ti = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      tc::mbar_wait(wfull, ti & 1);
      tc::tc_fence_after();
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), b = int(it % kRsTmemBufs);
        tc::mbar_wait(&tempty[b], ((it / kRsTmemBufs) & 1) ^ 1);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t d = tmem_base + uint32_t(b * 64);
          const uint32_t wa = tc::smem_u32(wsm), ha = tc::smem_u32(hst(s));
#pragma unroll
          for (int kk = 0; kk < KW / 8; ++kk) {
            const int a = kk / 4, ko = (kk % 4) * 32;
            const uint64_t whi = tc::make_sdesc(wa + a * kXTileBytes + ko, 16, 1024);
            const uint64_t wlo = tc::make_sdesc(wa + (C::kAtoms + a) * kXTileBytes + ko, 16, 1024);
            const uint64_t hb = tc::make_sdesc(ha + a * C::kHtAtomBytes + ko, 16, 1024);  // 64 rows: hi | lo
            tc::umma_tf32(d, whi, hb, idesc2, kk != 0);   // [W_hi H_hi | W_hi H_lo]
            tc::umma_tf32(d + 32, wlo, hb, idesc1, 1u);   // += W_lo H_hi
          }
          tc::umma_commit(&empty[s]);
          tc::umma_commit(&tfull[b]);
          if (kc == nk - 1) tc::umma_commit(wempty);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int sub = warp & 3;
    const int r = sub * 32 + lane;  // row within the tile
    double acc = 0.0;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), b = int(it % kRsTmemBufs);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&tfull[b], (it / kRsTmemBufs) & 1);
        tc::tc_fence_after();
        uint32_t d0[32], d1[32];
        const uint32_t taddr = tmem_base + (uint32_t(sub * 32) << 16) + uint32_t(b * 64);
        tc::tmem_ld_32x32b_x32(taddr, d0);
        tc::tmem_ld_32x32b_x32(taddr + 32, d1);
        // row r of the SW128 X stage: 16-byte chunk c sits at chunk c ^ (r & 7)
        const uint32_t xrow = tc::smem_u32(xst(s)) + uint32_t(r) * 128u;
        float xv[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "r"(xrow + uint32_t((c ^ (r & 7)) * 16)) : "memory");
          xv[4 * c] = __uint_as_float(v0), xv[4 * c + 1] = __uint_as_float(v1);
          xv[4 * c + 2] = __uint_as_float(v2), xv[4 * c + 3] = __uint_as_float(v3);
        }
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&tempty[b]);
        tc::mbar_arrive(&empty[s]);  // every epilogue thread: its X row loads are done
        float ss = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float e = xv[c] - (__uint_as_float(d0[c]) + __uint_as_float(d1[c]));
          ss = fmaf(e, e, ss);
        }
        acc += double(ss);
      }
    }
    // CTA partial: warp sums, fixed order over the 4 epilogue warps
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) red[sub] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) part_obj[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem_base);
  }
}

__global__ void tc_resid_prep_kernel(const float* __restrict__ w, int64_t m, const float* __restrict__ h, int64_t n,
                                     int k, int kw, int64_t npad, float* __restrict__ w_hi, float* __restrict__ w_lo,
                                     float* __restrict__ ht_hi, float* __restrict__ ht_lo) {
  const int64_t tw = m * kw, total = tw + npad * kw;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    float v;
    float *hi, *lo;
    if (e < tw) {
      const int64_t i = e / kw;
      const int j = int(e % kw);
      v = j < k ? w[i * k + j] : 0.f;
      hi = w_hi + e;
      lo = w_lo + e;
    } else {
      const int64_t f = e - tw, c = f / kw;
      const int j = int(f % kw);
      v = (j < k && c < n) ? h[int64_t(j) * n + c] : 0.f;
      hi = ht_hi + f;
      lo = ht_lo + f;
    }
    *hi = v;  // raw hi (truncated by kind::tf32), lo = what the truncation drops
    *lo = tf32_lo(v);
  }
}

__global__ void tc_prep_rows_kernel(const float* __restrict__ src, int c, int64_t n, int npad, int64_t ldst,
                                    float* __restrict__ st_hi, float* __restrict__ st_lo) {
  const int64_t total = int64_t(npad) * ldst;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e / ldst);
    const int64_t kk = e % ldst;
    const float v = (j < c && kk < n) ? src[int64_t(j) * n + kk] : 0.f;
    st_hi[e] = v;  // raw hi (truncated by kind::tf32), lo = what the truncation drops
    st_lo[e] = tf32_lo(v);
  }
}

// projected grad_W partial sums (projected_sq_norm, p/src/hals.cpp:55-65): one row per thread, the
// row's W and X H^T entries in registers (KP >= k), H H^T broadcast from shared memory
constexpr int kPgwThreads = 128;
template <int KP>
__global__ void __launch_bounds__(kPgwThreads) tc_pgw_kernel(const float* __restrict__ xht, const float* __restrict__ w,
                                                             int64_t m, int k, const double* __restrict__ hht,
                                                             double* __restrict__ part) {
  extern __shared__ double sh[];  // hht (k x k), then per-warp sums
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) sh[e] = hht[e];
  __syncthreads();
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    double wv[KP];
#pragma unroll
    for (int p = 0; p < KP; ++p) wv[p] = p < k ? double(w[i * k + p]) : 0.0;
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
      double whh = 0.0;
#pragma unroll
      for (int p = 0; p < KP; ++p)
        if (p < k) whh = fma(wv[p], sh[p * k + j], whh);
      const double g = -2.0 * (double(xht[i * k + j]) - whh);
      const double gi = w[i * k + j] > 0.f ? g : fmin(0.0, g);
      acc = fma(gi, gi, acc);
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  double* ws = sh + k * k;
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < kPgwThreads / 32; ++q) s += ws[q];
    part[blockIdx.x] = s;
  }
}

// All operand splits of one tensor-core metrics evaluation in one launch (regions of a flat index):
//   [0, A)   H rows      -> st_hi / st_lo (npad x ldn): the S^T operand of X H^T
//   [A, B)   W (m x k)   -> w_hi / w_lo (m x kw)      : A operand of the residual's W H
//   [B, C)   H (k x n)   -> ht_hi / ht_lo (ldn x kw)  : B operand of the residual's W H
//   [C, D)   W (m x k)   -> sw_hi / sw_lo (npad x ldm): the S^T operand of X^T W
// hi = rna_tf32(v), lo = rna_tf32(v - hi) everywhere (as the separate prep kernels).
__global__ void tc_metrics_prep_kernel(const float* __restrict__ w, const float* __restrict__ h, int64_t m, int64_t n,
                                       int k, int npad, int kw, int64_t ldn, int64_t ldm, float* __restrict__ st_hi,
                                       float* __restrict__ st_lo, float* __restrict__ w_hi, float* __restrict__ w_lo,
                                       float* __restrict__ ht_hi, float* __restrict__ ht_lo, float* __restrict__ sw_hi,
                                       float* __restrict__ sw_lo) {
  const int64_t A = int64_t(npad) * ldn, B = A + m * kw, Cc = B + ldn * kw, D = Cc + int64_t(npad) * ldm;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < D; e += int64_t(gridDim.x) * blockDim.x) {
    float v;
    float *hi, *lo;
    if (e < A) {
      const int j = int(e / ldn);
      const int64_t c = e % ldn;
      v = (j < k && c < n) ? h[int64_t(j) * n + c] : 0.f;
      hi = st_hi + e;
      lo = st_lo + e;
    } else if (e < B) {
      const int64_t f = e - A, i = f / kw;
      const int j = int(f % kw);
      v = j < k ? w[i * k + j] : 0.f;
      hi = w_hi + f;
      lo = w_lo + f;
    } else if (e < Cc) {
      const int64_t f = e - B, c = f / kw;
      const int j = int(f % kw);
      v = (j < k && c < n) ? h[int64_t(j) * n + c] : 0.f;
      hi = ht_hi + f;
      lo = ht_lo + f;
    } else {
      const int64_t f = e - Cc;
      const int j = int(f / ldm);
      const int64_t i = f % ldm;
      v = (j < k && i < m) ? w[i * k + j] : 0.f;
      hi = sw_hi + f;
      lo = sw_lo + f;
    }
    *hi = v;  // raw hi (truncated by kind::tf32), lo = what the truncation drops
    *lo = tf32_lo(v);
  }
}

template <int KW>
void tc_resid_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* w_hi, const float* w_lo,
                     const float* ht_hi, const float* ht_lo, double* part_obj, int grid, cudaStream_t stream) {
  using C = RsCfg<KW>;
  const int64_t npad = tc_st_pitch(n);
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBM);
  const CUtensorMap mwh = make_map_2d(w_hi, m, KW, KW, kBM);
  const CUtensorMap mwl = make_map_2d(w_lo, m, KW, KW, kBM);
  const CUtensorMap mhh = make_map_2d(ht_hi, npad, KW, KW, 32);
  const CUtensorMap mhl = make_map_2d(ht_lo, npad, KW, KW, 32);
  auto f = tc_resid_kernel<KW>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  f<<<grid, kRsThreads, C::kSmem, stream>>>(mx, mwh, mwl, mhh, mhl, m, n, part_obj);
  RNMF_CUDA_LAUNCH();
}

}  // namespace

int launch_tc_prep_rows(const float* src, int c, int64_t n, float* st_hi, float* st_lo, cudaStream_t stream) {
  const int npad = tc_npad(c);
  const int64_t ld = tc_st_pitch(n);
  const int blocks = int(std::min<int64_t>(ceil_div(int64_t(npad) * ld, 256), 148 * 8));
  tc_prep_rows_kernel<<<blocks, 256, 0, stream>>>(src, c, n, npad, ld, st_hi, st_lo);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int tc_resid_kw(int k) { return k <= 32 ? 32 : 64; }

int launch_tc_metrics_prep(const float* w, int64_t m, const float* h, int64_t n, int k, float* st_hi, float* st_lo,
                           float* w_hi, float* w_lo, float* ht_hi, float* ht_lo, float* sw_hi, float* sw_lo,
                           cudaStream_t stream) {
  const int npad = tc_npad(k), kw = tc_resid_kw(k);
  const int64_t ldn = tc_st_pitch(n), ldm = tc_st_pitch(m);
  const int64_t total = int64_t(npad) * ldn + m * kw + ldn * kw + int64_t(npad) * ldm;
  const int blocks = int(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  tc_metrics_prep_kernel<<<blocks, 256, 0, stream>>>(w, h, m, n, k, npad, kw, ldn, ldm, st_hi, st_lo, w_hi, w_lo,
                                                     ht_hi, ht_lo, sw_hi, sw_lo);
  RNMF_CUDA_LAUNCH();
  return 1;
}


int launch_tc_resid_prep(const float* w, int64_t m, const float* h, int64_t n, int k, float* w_hi, float* w_lo,
                         float* ht_hi, float* ht_lo, cudaStream_t stream) {
  const int kw = tc_resid_kw(k);
  const int64_t npad = tc_st_pitch(n);
  const int64_t total = (m + npad) * kw;
  const int blocks = int(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  tc_resid_prep_kernel<<<blocks, 256, 0, stream>>>(w, m, h, n, k, kw, npad, w_hi, w_lo, ht_hi, ht_lo);
  RNMF_CUDA_LAUNCH();
  return 1;
}

int tc_resid_blocks(int64_t m, int sm_count) { return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, kBM), sm_count))); }

int launch_tc_resid(const float* x, int64_t m, int64_t n, int64_t ldx, const float* w_hi, const float* w_lo,
                    const float* ht_hi, const float* ht_lo, int k, double* part_obj, int* nblocks, int sm_count,
                    cudaStream_t stream) {
  if ((ldx * sizeof(float)) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) % 16) != 0)
    throw CudaError("tc_resid: X needs a 16-byte aligned base and row pitch");
  if (k > 64) throw CudaError("tc_resid: k above 64");
  const int grid = tc_resid_blocks(m, sm_count);
  if (tc_resid_kw(k) == 32)
    tc_resid_launch<32>(x, m, n, ldx, w_hi, w_lo, ht_hi, ht_lo, part_obj, grid, stream);
  else
    tc_resid_launch<64>(x, m, n, ldx, w_hi, w_lo, ht_hi, ht_lo, part_obj, grid, stream);
  *nblocks = grid;
  return 1;
}

int tc_pgw_blocks(int64_t m) { return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, kPgwThreads), 148 * 8))); }

int launch_tc_pgw(const float* xht, const float* w, int64_t m, int k, const double* hht, double* part_pgw,
                  int* nblocks, cudaStream_t stream) {
  const int blocks = tc_pgw_blocks(m);
  const size_t smem = sizeof(double) * (size_t(k) * k + kPgwThreads / 32);
  if (k <= 16)
    tc_pgw_kernel<16><<<blocks, kPgwThreads, smem, stream>>>(xht, w, m, k, hht, part_pgw);
  else if (k <= 32)
    tc_pgw_kernel<32><<<blocks, kPgwThreads, smem, stream>>>(xht, w, m, k, hht, part_pgw);
  else if (k <= 48)
    tc_pgw_kernel<48><<<blocks, kPgwThreads, smem, stream>>>(xht, w, m, k, hht, part_pgw);
  else
    tc_pgw_kernel<64><<<blocks, kPgwThreads, smem, stream>>>(xht, w, m, k, hht, part_pgw);
  RNMF_CUDA_LAUNCH();
  *nblocks = blocks;
  return 1;
}

// ================================================================================================
// Fused metrics pass for k <= 32 (tc_metrics.h launch_tc_xht_resid): ONE read of X gives both
//   X H^T (3xTF32, as tc_xw_kernel with S^T = H)   and   sum (X - W H)^2 (as tc_resid_kernel)
// per 128-row tile.  Ring stage = [X 16 KB][H slab hi | lo (NPAD rows each)][H^T slab hi | lo (32
// rows each)]; the W tile (hi, lo; one 32-wide K atom) is resident per tile; the lo X tiles use
// the split warps' ring.  TMEM: X H^T accumulator chunks (2 x 2 NPAD columns) and a 4-deep ring
// of 64-column W H buffers.  Epilogue warps: per stage the residual of their row (X row from the
// swizzled stage), per chunk the X H^T drain into fp32 registers.
namespace {

template <int NPAD>
struct FzCfg {
  static constexpr int kSBytes = NPAD * kBK * 4;
  static constexpr int kHtBytes = 2 * 32 * 128;                       // H^T hi | lo (32 rows each)
  static constexpr int kWBytes = 2 * kXTileBytes;                     // W hi, lo (128 rows x 32)
  static constexpr int kStageBytes = kXTileBytes + 2 * kSBytes + kHtBytes;
  static constexpr int kLoBytes = kLoSlots * kXTileBytes;
  static constexpr int kStages = std::min(8, (kSmemBudget - kWBytes - kLoBytes - 2048) / kStageBytes);
  static constexpr int kAccCols = 2 * NPAD;
  static constexpr int kRsBase = 2 * kAccCols;                        // W H ring after the X H^T buffers
  static constexpr int kTmemCols = 512;
  static constexpr size_t kSmem = size_t(kWBytes) + size_t(kStages) * kStageBytes + kLoBytes + 1024 + 512;
  static_assert(kStages >= 2, "ring too shallow");
  static_assert(kRsBase + kRsTmemBufs * 64 <= 512, "TMEM");
};

struct FzParams {
  int64_t m, n;
  int c;
  float* y;          // X H^T (m x c)
  int chunk;
  double* part_obj;  // per-CTA residual partials
};

template <int NPAD>
__global__ void __launch_bounds__(kTcThreadsX3, 1) tc_xht_resid_kernel(
    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmShi,
    const __grid_constant__ CUtensorMap tmSlo, const __grid_constant__ CUtensorMap tmWhi,
    const __grid_constant__ CUtensorMap tmWlo, const __grid_constant__ CUtensorMap tmHhi,
    const __grid_constant__ CUtensorMap tmHlo, FzParams p) {
  using C = FzCfg<NPAD>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* wsm = base;
  auto xst = [&](int s) { return base + C::kWBytes + size_t(s) * C::kStageBytes; };
  auto shi = [&](int s) { return xst(s) + kXTileBytes; };
  auto htp = [&](int s) { return shi(s) + 2 * C::kSBytes; };
  auto lo = [&](int j) { return base + C::kWBytes + size_t(S) * C::kStageBytes + size_t(j) * kXTileBytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::kWBytes + size_t(S) * C::kStageBytes + C::kLoBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + S;
  uint64_t* lofull = empty + S;
  uint64_t* loempty = lofull + kLoSlots;
  uint64_t* tfull = loempty + kLoSlots;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + kRsTmemBufs;
  uint64_t* wfull = rempty + kRsTmemBufs;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  double* red = reinterpret_cast<double*>(wempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(p.m, kBM);
  const int nk = int(ceil_div(p.n, kBK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + 128);
    }
    for (int j = 0; j < kLoSlots; ++j) {
      tc::mbar_init(&lofull[j], kSplitThreads);
      tc::mbar_init(&loempty[j], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    for (int b = 0; b < kRsTmemBufs; ++b) {
      tc::mbar_init(&rfull[b], 1);
      tc::mbar_init(&rempty[b], 128);
    }
    tc::mbar_init(wfull, 1);
    tc::mbar_init(wempty, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmShi);
    tc::tma_prefetch(&tmSlo);
    tc::tma_prefetch(&tmWhi);
    tc::tma_prefetch(&tmWlo);
    tc::tma_prefetch(&tmHhi);
    tc::tma_prefetch(&tmHlo);
  }
  if (warp == 1) tc::tmem_alloc<C::kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      uint32_t it = 0, ti = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
        tc::mbar_wait(wempty, (ti & 1) ^ 1);
        tc::mbar_arrive_expect_tx(wfull, uint32_t(C::kWBytes));
        tc::tma_load_2d(wsm, &tmWhi, wfull, 0, int(t * kBM));
        tc::tma_load_2d(wsm + kXTileBytes, &tmWlo, wfull, 0, int(t * kBM));
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          // X and the H / H^T slabs with their lo parts (prepared once per evaluation): the split
          // warps, the busiest role of this kernel, only split X
          tc::mbar_arrive_expect_tx(&full[s], uint32_t(C::kStageBytes));
          tc::tma_load_2d_hint(xst(s), &tmX, &full[s], kc * kBK, int(t * kBM), kXPolicy);
          tc::tma_load_2d(shi(s), &tmShi, &full[s], kc * kBK, 0);
          tc::tma_load_2d(shi(s) + C::kSBytes, &tmSlo, &full[s], kc * kBK, 0);
          tc::tma_load_2d(htp(s), &tmHhi, &full[s], 0, kc * kBK);
          tc::tma_load_2d(htp(s) + 4096, &tmHlo, &full[s], 0, kc * kBK);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc32 = tc::make_idesc_tf32(32, false, false);
    constexpr uint32_t idesc64 = tc::make_idesc_tf32(64, false, false);
    auto adesc = [](uint32_t b, int k) { return tc::make_sdesc(b + k * 32, 16, 1024); };
    uint32_t it = 0, ci = 0, ti = 0;
    uint32_t d = tmem_base;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      tc::mbar_wait(wfull, ti & 1);
      tc::tc_fence_after();
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int kin = kc % p.chunk;
        const bool cend = (kin == p.chunk - 1) || (kc == nk - 1);
        const int acc = int(ci & 1);
        if (kin == 0) {
          tc::mbar_wait(&tempty[acc], ((ci >> 1) & 1) ^ 1);
          d = tmem_base + uint32_t(acc * C::kAccCols);
        }
        const int s = int(it % S), j = int(it % kLoSlots), b = int(it % kRsTmemBufs);
        tc::mbar_wait(&rempty[b], ((it / kRsTmemBufs) & 1) ^ 1);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&lofull[j], (it / kLoSlots) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          // X H^T chunk: X_hi [H_hi; H_lo]^T, += X_lo H_hi^T
          issue_stage<NPAD, true, false>(d, tc::smem_u32(xst(s)), tc::smem_u32(lo(j)), tc::smem_u32(shi(s)), kin == 0,
                                         adesc);
          // W H (this stage's 32 columns): [W_hi H_hi | W_hi H_lo], += W_lo H_hi
          const uint32_t dr = tmem_base + uint32_t(C::kRsBase + b * 64);
          const uint32_t wa = tc::smem_u32(wsm), ha = tc::smem_u32(htp(s));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t whi = tc::make_sdesc(wa + kk * 32, 16, 1024);
            const uint64_t wlo = tc::make_sdesc(wa + kXTileBytes + kk * 32, 16, 1024);
            const uint64_t hb = tc::make_sdesc(ha + kk * 32, 16, 1024);
            tc::umma_tf32(dr, whi, hb, idesc64, kk != 0);
            tc::umma_tf32(dr + 32, wlo, hb, idesc32, 1u);
          }
          tc::umma_commit(&empty[s]);
          tc::umma_commit(&loempty[j]);
          tc::umma_commit(&rfull[b]);
          if (cend) tc::umma_commit(&tfull[acc]);
          if (kc == nk - 1) tc::umma_commit(wempty);
        }
        if (cend) ++ci;
        __syncwarp();
      }
    }
  } else if (warp < 4 || warp >= 8) {
    const int st = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 192;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), j = int(it % kLoSlots);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&loempty[j], ((it / kLoSlots) & 1) ^ 1);
        split_lo_tile<kXTileBytes / 16>(reinterpret_cast<const float4*>(xst(s)), reinterpret_cast<float4*>(lo(j)), st);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&lofull[j]);
      }
    }
  } else {
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t lane_off = uint32_t(sub * 32) << 16;
    double racc = 0.0;
    uint32_t it = 0, ci = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t row = t * kBM + r;
      float a[NPAD];
#pragma unroll
      for (int q = 0; q < NPAD; ++q) a[q] = 0.f;
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), b = int(it % kRsTmemBufs);
        // residual of this stage's 32 columns
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&rfull[b], (it / kRsTmemBufs) & 1);
        tc::tc_fence_after();
        uint32_t d0[32], d1[32];
        const uint32_t taddr = tmem_base + lane_off + uint32_t(C::kRsBase + b * 64);
        tc::tmem_ld_32x32b_x32(taddr, d0);
        tc::tmem_ld_32x32b_x32(taddr + 32, d1);
        const uint32_t xrow = tc::smem_u32(xst(s)) + uint32_t(r) * 128u;
        float xv[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "r"(xrow + uint32_t((c ^ (r & 7)) * 16)) : "memory");
          xv[4 * c] = __uint_as_float(v0), xv[4 * c + 1] = __uint_as_float(v1);
          xv[4 * c + 2] = __uint_as_float(v2), xv[4 * c + 3] = __uint_as_float(v3);
        }
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&rempty[b]);
        tc::mbar_arrive(&empty[s]);  // every epilogue thread: its X row loads are done
        float ss = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float e = xv[c] - (__uint_as_float(d0[c]) + __uint_as_float(d1[c]));
          ss = fmaf(e, e, ss);
        }
        racc += double(ss);
        // X H^T chunk drain
        const bool cend = (kc % p.chunk == p.chunk - 1) || (kc == nk - 1);
        if (cend) {
          const int acc = int(ci & 1);
          tc::mbar_wait(&tfull[acc], (ci >> 1) & 1);
          tc::tc_fence_after();
          drain_acc<NPAD, true>(tmem_base + lane_off + uint32_t(acc * C::kAccCols), a);
          tc::tc_fence_before();
          tc::mbar_arrive(&tempty[acc]);
          ++ci;
        }
      }
      if (row < p.m) {
#pragma unroll
        for (int q = 0; q < NPAD; ++q)
          if (q < p.c) p.y[row * p.c + q] = a[q];
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, off);
    if (lane == 0) red[sub] = racc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) p.part_obj[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int NPAD>
void tc_xht_resid_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                         const float* w_hi, const float* w_lo, const float* ht_hi, const float* ht_lo, int k,
                         float* xht, double* part_obj, int grid, cudaStream_t stream) {
  using C = FzCfg<NPAD>;
  const int64_t ldst = tc_st_pitch(n);
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBM);
  const CUtensorMap mh = make_map_2d(st_hi, NPAD, n, ldst, NPAD);
  const CUtensorMap ml = make_map_2d(st_lo, NPAD, n, ldst, NPAD);
  const CUtensorMap mwh = make_map_2d(w_hi, m, 32, 32, kBM);
  const CUtensorMap mwl = make_map_2d(w_lo, m, 32, 32, kBM);
  const CUtensorMap mhh = make_map_2d(ht_hi, ldst, 32, 32, 32);
  const CUtensorMap mhl = make_map_2d(ht_lo, ldst, 32, 32, 32);
  FzParams p{m, n, k, xht, tc_chunk_stages(), part_obj};
  auto f = tc_xht_resid_kernel<NPAD>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  f<<<grid, kTcThreadsX3, C::kSmem, stream>>>(mx, mh, ml, mwh, mwl, mhh, mhl, p);
  RNMF_CUDA_LAUNCH();
}

// ------------------------------------------------------------------------------------------------
// Fused metrics pass for 32 < k <= 64: as tc_xht_resid_kernel (X H^T by 3xTF32 into TMEM chunks
// drained to fp32 registers, and sum (X - W H)^2 per stage), but the W tile (hi, lo; K = 8 ks
// columns each) is the A operand from TENSOR MEMORY: the epilogue threads store their row of W_hi /
// W_lo with tcgen05.st at the start of each row tile, which keeps shared memory for a deep X ring.
// TMEM columns: [0, 4 NPAD) X H^T chunk buffers | kRb x 64 W H ring | W_hi (64) | W_lo (64).
// Shared: ring stage = [X 16 KB][H slab hi | lo (NPAD rows each)][H^T slab, two 32-wide K atoms of
// (32 hi rows | 32 lo rows)]; kLoW lo-X slots.
template <int NPAD>
struct FwCfg {
  static constexpr int kSBytes = NPAD * kBK * 4;
  static constexpr int kHtBytes = 2 * (2 * 32 * 128);  // 2 K atoms x (hi | lo)
  static constexpr int kStageBytes = kXTileBytes + 2 * kSBytes + kHtBytes;
  static constexpr int kLoW = 2;
  // kLT (k <= 48): the lo X tiles live in tensor memory (kLoW x 32 columns, written by four split
  // warps with tcgen05.st; the small-term UMMA takes A from TMEM) instead of a shared-memory ring,
  // which buys one more TMA stage; the W H ring is then two slots deep.  TMEM is full either way.
  static constexpr bool kLT = NPAD <= 48;
  static constexpr int kLoBytes = kLT ? 0 : kLoW * kXTileBytes;
  static constexpr int kStages = std::min(6, (226 * 1024 - kLoBytes - 2048) / kStageBytes);
  static constexpr int kAccCols = 2 * NPAD;
  static constexpr int kRsBase = 2 * kAccCols;
  static constexpr int kRb = kLT ? 2 : (512 - kRsBase - 128) / 64;  // W H ring depth
  static constexpr int kLoT = kRsBase + kRb * 64;                    // TMEM lo ring (kLT)
  static constexpr int kWBase = kLoT + (kLT ? kLoW * kBK : 0);
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + kLoBytes + 1024 + 512;
  static_assert(kStages >= 3 && kRb >= 2 && kWBase + 128 <= 512, "layout");
};

template <int NPAD>
__global__ void __launch_bounds__(kTcThreadsX3, 1) tc_xht_resid_w_kernel(
    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmShi,
    const __grid_constant__ CUtensorMap tmSlo, const __grid_constant__ CUtensorMap tmHhi,
    const __grid_constant__ CUtensorMap tmHlo, const float* __restrict__ w_hi, const float* __restrict__ w_lo,
    int ks, FzParams p) {
  using C = FwCfg<NPAD>;
  constexpr int S = C::kStages;
  constexpr int LO = C::kLoW;
  constexpr int RB = C::kRb;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto xst = [&](int s) { return base + size_t(s) * C::kStageBytes; };
  auto shi = [&](int s) { return xst(s) + kXTileBytes; };
  auto htp = [&](int s) { return shi(s) + 2 * C::kSBytes; };
  auto lo = [&](int j) { return base + size_t(S) * C::kStageBytes + size_t(j) * kXTileBytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + size_t(S) * C::kStageBytes + C::kLoBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + S;
  uint64_t* lofull = empty + S;
  uint64_t* loempty = lofull + LO;
  uint64_t* tfull = loempty + LO;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + RB;
  uint64_t* wfull = rempty + RB;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  double* red = reinterpret_cast<double*>(wempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(p.m, kBM);
  const int nk = int(ceil_div(p.n, kBK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + 128);
    }
    for (int j = 0; j < LO; ++j) {
      tc::mbar_init(&lofull[j], C::kLT ? 128 : kSplitThreads);
      tc::mbar_init(&loempty[j], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    for (int b = 0; b < RB; ++b) {
      tc::mbar_init(&rfull[b], 1);
      tc::mbar_init(&rempty[b], 128);
    }
    tc::mbar_init(wfull, 128);
    tc::mbar_init(wempty, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmShi);
    tc::tma_prefetch(&tmSlo);
    tc::tma_prefetch(&tmHhi);
    tc::tma_prefetch(&tmHlo);
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (tc::elect_one()) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = int(it % S);
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          // X and the H / H^T slabs with their lo parts: the split warps only split X
          tc::mbar_arrive_expect_tx(&full[s], uint32_t(C::kStageBytes));
          tc::tma_load_2d_hint(xst(s), &tmX, &full[s], kc * kBK, int(t * kBM), kXPolicy);
          tc::tma_load_2d(shi(s), &tmShi, &full[s], kc * kBK, 0);
          tc::tma_load_2d(shi(s) + C::kSBytes, &tmSlo, &full[s], kc * kBK, 0);
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            tc::tma_load_2d(htp(s) + a * 8192, &tmHhi, &full[s], a * 32, kc * kBK);
            tc::tma_load_2d(htp(s) + a * 8192 + 4096, &tmHlo, &full[s], a * 32, kc * kBK);
          }
        }
      }
    }
  } else if (warp == 1) {
    // UMMA issue: shared-memory descriptors as {lo, hi} words advanced by adds, ring indices kept
    // incrementally (no make_sdesc / integer division per stage) -- the issuing thread's time per
    // stage bounds this kernel (18 UMMAs and 3+ commits per 16 KB of X at k = 40)
    constexpr uint32_t idesc32 = tc::make_idesc_tf32(32, false, false);
    constexpr uint32_t idesc64 = tc::make_idesc_tf32(64, false, false);
    constexpr uint32_t idesc1 = tc::make_idesc_tf32(NPAD, false, false);
    constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, false, false);
    constexpr uint32_t kHi = tc::sdesc_hi(1024, tc::kLayoutSW128);
    const uint32_t x0 = (tc::smem_u32(xst(0)) >> 4) + tc::sdesc_lo_const(16);
    const uint32_t l0 = (tc::smem_u32(lo(0)) >> 4) + tc::sdesc_lo_const(16);
    uint32_t ci = 0, ti = 0;
    uint32_t s = 0, sph = 0, j = 0, jph = 0, b = 0, bph = 0;
    uint32_t d = tmem_base;
    const uint32_t wa_hi = tmem_base + uint32_t(C::kWBase), wa_lo = wa_hi + 64u;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      tc::mbar_wait(wfull, ti & 1);  // this tile's W rows are in TMEM
      tc::tc_fence_after();
      int kin = 0;
      for (int kc = 0; kc < nk; ++kc) {
        const bool cend = (kin == p.chunk - 1) || (kc == nk - 1);
        const int acc = int(ci & 1);
        if (kin == 0) {
          tc::mbar_wait(&tempty[acc], ((ci >> 1) & 1) ^ 1);
          d = tmem_base + uint32_t(acc * C::kAccCols);
        }
        tc::mbar_wait(&rempty[b], bph ^ 1);
        tc::mbar_wait(&full[s], sph);
        tc::mbar_wait(&lofull[j], jph);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t xa = x0 + s * uint32_t(C::kStageBytes >> 4), ba = xa + uint32_t(kXTileBytes >> 4);
          const uint32_t la = l0 + j * uint32_t(kXTileBytes >> 4);
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            tc::umma_tf32_w(d, xa + 2 * k, kHi, ba + 2 * k, kHi, idesc2, (kin == 0 && k == 0) ? 0u : 1u);  // X_hi [S_hi; S_lo]
            if (C::kLT)  // += X_lo S_hi, A from tensor memory
              tc::umma_tf32_ts_w(d + NPAD, tmem_base + uint32_t(C::kLoT) + j * uint32_t(kBK) + uint32_t(8 * k), ba + 2 * k,
                                 kHi, idesc1, 1u);
            else
              tc::umma_tf32_w(d + NPAD, la + 2 * k, kHi, ba + 2 * k, kHi, idesc1, 1u);
          }
          const uint32_t dr = tmem_base + uint32_t(C::kRsBase) + b * 64u;
          const uint32_t ha = ba + uint32_t((2 * C::kSBytes) >> 4);  // H^T slab: two 32-wide K atoms of (hi | lo) rows
          for (int kk = 0; kk < ks; ++kk) {
            const uint32_t hb = ha + uint32_t((kk >> 2) * (8192 >> 4) + (kk & 3) * 2);
            tc::umma_tf32_ts_w(dr, wa_hi + uint32_t(kk * 8), hb, kHi, idesc64, kk != 0);  // [W_hi H_hi | W_hi H_lo]
            tc::umma_tf32_ts_w(dr + 32, wa_lo + uint32_t(kk * 8), hb, kHi, idesc32, 1u);  // += W_lo H_hi
          }
          tc::umma_commit(&empty[s]);
          tc::umma_commit(&loempty[j]);
          tc::umma_commit(&rfull[b]);
          if (cend) tc::umma_commit(&tfull[acc]);
          if (kc == nk - 1) tc::umma_commit(wempty);
        }
        __syncwarp();
        if (cend) {
          ++ci;
          kin = 0;
        } else {
          ++kin;
        }
        if (++s == uint32_t(S)) s = 0, sph ^= 1;
        if (++j == uint32_t(LO)) j = 0, jph ^= 1;
        if (++b == uint32_t(RB)) b = 0, bph ^= 1;
      }
    }
  } else if (warp < 4 || warp >= 8) {
    if constexpr (C::kLT) {
      // warps 8..11 (TMEM lane quadrants 0..3): lo of the thread's X row -> the TMEM lo slot
      if (warp >= 8) {
        const int quad = warp & 3, r = quad * 32 + lane;
        const uint32_t lane_off = uint32_t(quad * 32) << 16;
        uint32_t it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
          for (int kc = 0; kc < nk; ++kc, ++it) {
            const int s = int(it % S), j = int(it % LO);
            tc::mbar_wait(&full[s], (it / S) & 1);
            const uint32_t xrow = tc::smem_u32(xst(s)) + uint32_t(r) * 128u;
            uint32_t v0[16], v1[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v0[4 * c]), "=r"(v0[4 * c + 1]), "=r"(v0[4 * c + 2]), "=r"(v0[4 * c + 3])
                           : "r"(xrow + uint32_t((c ^ (r & 7)) * 16)) : "memory");
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v1[4 * c]), "=r"(v1[4 * c + 1]), "=r"(v1[4 * c + 2]), "=r"(v1[4 * c + 3])
                           : "r"(xrow + uint32_t(((4 + c) ^ (r & 7)) * 16)) : "memory");
            }
            tc::mbar_wait(&loempty[j], ((it / LO) & 1) ^ 1);
            tc::tc_fence_after();
            uint32_t r0[16], r1[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) r0[i] = tf32_lo_bits(v0[i]), r1[i] = tf32_lo_bits(v1[i]);
            const uint32_t ta = tmem_base + lane_off + uint32_t(C::kLoT + j * kBK);
            tc::tmem_st_32x32b_x16(ta, r0);
            tc::tmem_st_32x32b_x16(ta + 16, r1);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(&lofull[j]);
          }
        }
      }
    } else {
    const int st = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 192;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), j = int(it % LO);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&loempty[j], ((it / LO) & 1) ^ 1);
        split_lo_tile<kXTileBytes / 16>(reinterpret_cast<const float4*>(xst(s)), reinterpret_cast<float4*>(lo(j)), st);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&lofull[j]);
      }
    }
    }
  } else {
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t lane_off = uint32_t(sub * 32) << 16;
    double racc = 0.0;
    uint32_t it = 0, ci = 0, ti = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
      const int64_t row = t * kBM + r;
      {
        // W row (hi, lo; 64 columns each, zero past k and past m) into TMEM once the previous
        // tile's UMMAs are done with it
        tc::mbar_wait(wempty, (ti & 1) ^ 1);
        tc::tc_fence_after();
#pragma unroll
        for (int part = 0; part < 4; ++part) {
          const float* src = (part < 2 ? w_hi : w_lo) + row * 64 + (part & 1) * 32;
          uint32_t v[32];
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < p.m) f = __ldg(reinterpret_cast<const float4*>(src) + q4);
            v[4 * q4] = __float_as_uint(f.x), v[4 * q4 + 1] = __float_as_uint(f.y);
            v[4 * q4 + 2] = __float_as_uint(f.z), v[4 * q4 + 3] = __float_as_uint(f.w);
          }
          tc::tmem_st_32x32b_x32(tmem_base + lane_off + uint32_t(C::kWBase + part * 32), v);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(wfull);
      }
      float a[NPAD];
#pragma unroll
      for (int q = 0; q < NPAD; ++q) a[q] = 0.f;
      for (int kc = 0; kc < nk; ++kc, ++it) {
        const int s = int(it % S), b = int(it % RB);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::mbar_wait(&rfull[b], (it / RB) & 1);
        tc::tc_fence_after();
        uint32_t d0[32], d1[32];
        const uint32_t taddr = tmem_base + lane_off + uint32_t(C::kRsBase + b * 64);
        tc::tmem_ld_32x32b_x32(taddr, d0);
        tc::tmem_ld_32x32b_x32(taddr + 32, d1);
        const uint32_t xrow = tc::smem_u32(xst(s)) + uint32_t(r) * 128u;
        float xv[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "r"(xrow + uint32_t((c ^ (r & 7)) * 16)) : "memory");
          xv[4 * c] = __uint_as_float(v0), xv[4 * c + 1] = __uint_as_float(v1);
          xv[4 * c + 2] = __uint_as_float(v2), xv[4 * c + 3] = __uint_as_float(v3);
        }
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&rempty[b]);
        tc::mbar_arrive(&empty[s]);  // every epilogue thread: its X row loads are done
        float ss = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float e = xv[c] - (__uint_as_float(d0[c]) + __uint_as_float(d1[c]));
          ss = fmaf(e, e, ss);
        }
        racc += double(ss);
        const bool cend = (kc % p.chunk == p.chunk - 1) || (kc == nk - 1);
        if (cend) {
          const int acc = int(ci & 1);
          tc::mbar_wait(&tfull[acc], (ci >> 1) & 1);
          tc::tc_fence_after();
          drain_acc<NPAD, true>(tmem_base + lane_off + uint32_t(acc * C::kAccCols), a);
          tc::tc_fence_before();
          tc::mbar_arrive(&tempty[acc]);
          ++ci;
        }
      }
      if (row < p.m) {
#pragma unroll
        for (int q = 0; q < NPAD; ++q)
          if (q < p.c) p.y[row * p.c + q] = a[q];
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, off);
    if (lane == 0) red[sub] = racc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) p.part_obj[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

template <int NPAD>
void tc_xht_resid_w_launch(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                           const float* w_hi, const float* w_lo, const float* ht_hi, const float* ht_lo, int k,
                           float* xht, double* part_obj, int grid, cudaStream_t stream) {
  using C = FwCfg<NPAD>;
  const int64_t ldst = tc_st_pitch(n);
  const CUtensorMap mx = make_map_2d(x, m, n, ldx, kBM);
  const CUtensorMap mh = make_map_2d(st_hi, NPAD, n, ldst, NPAD);
  const CUtensorMap ml = make_map_2d(st_lo, NPAD, n, ldst, NPAD);
  const CUtensorMap mhh = make_map_2d(ht_hi, ldst, 64, 64, 32);
  const CUtensorMap mhl = make_map_2d(ht_lo, ldst, 64, 64, 32);
  FzParams p{m, n, k, xht, tc_chunk_stages(), part_obj};
  auto f = tc_xht_resid_w_kernel<NPAD>;
  RNMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem)));
  f<<<grid, kTcThreadsX3, C::kSmem, stream>>>(mx, mh, ml, mhh, mhl, w_hi, w_lo, int(ceil_div(k, 8)), p);
  RNMF_CUDA_LAUNCH();
}

}  // namespace

int launch_tc_xht_resid(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                        const float* w_hi, const float* w_lo, const float* ht_hi, const float* ht_lo, int k, float* xht,
                        double* part_obj, int* nblocks, int sm_count, cudaStream_t stream) {
  if ((ldx * sizeof(float)) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) % 16) != 0)
    throw CudaError("tc_xht_resid: X needs a 16-byte aligned base and row pitch");
  if (k > 64) throw CudaError("tc_xht_resid: k above 64");
  const int grid = tc_resid_blocks(m, sm_count);
  if (k > 32) {  // W from tensor memory (w_hi / w_lo: m x 64, ht_hi / ht_lo: ldst x 64)
    if (tc_npad(k) == 48)
      tc_xht_resid_w_launch<48>(x, m, n, ldx, st_hi, st_lo, w_hi, w_lo, ht_hi, ht_lo, k, xht, part_obj, grid, stream);
    else
      tc_xht_resid_w_launch<64>(x, m, n, ldx, st_hi, st_lo, w_hi, w_lo, ht_hi, ht_lo, k, xht, part_obj, grid, stream);
  } else if (tc_npad(k) == 16)
    tc_xht_resid_launch<16>(x, m, n, ldx, st_hi, st_lo, w_hi, w_lo, ht_hi, ht_lo, k, xht, part_obj, grid, stream);
  else
    tc_xht_resid_launch<32>(x, m, n, ldx, st_hi, st_lo, w_hi, w_lo, ht_hi, ht_lo, k, xht, part_obj, grid, stream);
  *nblocks = grid;
  return 1;
}

}  // namespace rnmf_gpu
