// Rate probe of tcgen05.mma kind::tf32 (M = 128, K = 8), one CTA per SM (development aid): cycles
// per UMMA with A from shared memory (K-major SW128) or tensor memory, N = 16..256, accumulating
// into R rotating accumulators (R = 1: every UMMA depends on the previous one).  The issue loop is
// fully unrolled with precomputed descriptors so the single issuing thread is not the limit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1711_02037_b200/csrc tools/umma_rate.cu -o tools/umma_rate
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace rnmf_gpu;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

// MODE 0: SS; 1: TS; 2: the kernels' pair (SS N=2n into D, SS N=n into D+n); 3: pair (SS 2n, TS n)
template <int MODE, int N, int R>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t xa = tc::smem_u32(base), ba = xa + 16384;
    constexpr uint32_t idk = tc::make_idesc_tf32(uint32_t(N), false, false);
    constexpr uint32_t id2 = tc::make_idesc_tf32(uint32_t(2 * N > 256 ? 256 : 2 * N), false, false);
    uint64_t ad[4], bd[4];
    for (int k = 0; k < 4; ++k) {
      ad[k] = tc::make_sdesc(xa + k * 32, 16, 1024);
      bd[k] = tc::make_sdesc(ba + k * 32, 16, 1024);
    }
    constexpr int W = (MODE >= 2) ? 2 * N : N;  // accumulator width
    const uint32_t abase = tm + 448;           // TS: A operand columns (64 of them)
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t d = tm + uint32_t((u % R) * W);
        const int k = u & 3;
        if (MODE == 0) tc::umma_tf32(d, ad[k], bd[k], idk, 1u);
        if (MODE == 1) tc::umma_tf32_ts(d, abase + k * 8, bd[k], idk, 1u);
        if (MODE == 2) {
          tc::umma_tf32(d, ad[k], bd[k], id2, 1u);
          tc::umma_tf32(d + N, ad[k], bd[k], idk, 1u);
        }
        if (MODE == 3) {
          tc::umma_tf32(d, ad[k], bd[k], id2, 1u);
          tc::umma_tf32_ts(d + N, abase + k * 8, bd[k], idk, 1u);
        }
      }
    }
    tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tm);
  }
}

// The sketch kernels' per-stage issue sequence (8 UMMAs with descriptors rebuilt from the stage /
// slot index, three commits), without any waiting: cycles per stage of the issuing thread + pipe.
template <int NPAD, bool LT, int COMMITS>
__global__ void __launch_bounds__(128, 1) stage_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x < 32) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % 5, j = it % 3;
      const uint32_t xa = tc::smem_u32(base) + s * 32768, la = LT ? tm + 256 + j * 32 : tc::smem_u32(base) + 163840 + j * 16384;
      const uint32_t ba = xa + 16384;
      const uint32_t d = tm + ((it >> 2) & 1) * 128;
      if (tc::elect_one()) {
        constexpr uint32_t idesc1 = tc::make_idesc_tf32(NPAD, false, false);
        constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, false, false);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t adesc = tc::make_sdesc(xa + k * 32, 16, 1024);
          const uint64_t bdesc = tc::make_sdesc(ba + k * 32, 16, 1024);
          tc::umma_tf32(d, adesc, bdesc, idesc2, (it & 3) || k);
          if (LT)
            tc::umma_tf32_ts(d + NPAD, la + k * 8, bdesc, idesc1, 1u);
          else
            tc::umma_tf32(d + NPAD, tc::make_sdesc(la + k * 32, 16, 1024), bdesc, idesc1, 1u);
        }
        if (COMMITS > 0) tc::umma_commit(&bar[1]);
        if (COMMITS > 1) tc::umma_commit(&bar[2]);
        if (COMMITS > 2 && (it & 3) == 3) tc::umma_commit(&bar[3]);
      }
      __syncwarp();
    }
    if (tc::elect_one()) {
      tc::umma_commit(&bar[0]);
      tc::mbar_wait(&bar[0], 0);
    }
    __syncwarp();
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tm);
  }
}

// Optimised issue: descriptors as {lo, hi} words, lo advanced by adds; one commit per stage (+ one per
// 4 stages); ISSUERS = 2: warp 0 issues the hi UMMAs, warp 1 the lo UMMAs (separate accumulators).
__device__ __forceinline__ void umma_lohi(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b64 da, {%1, %2};\n\t"
      "mov.b64 db, {%3, %4};\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t}" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ts_lohi(uint32_t d, uint32_t a_tmem, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %4, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
      : "memory");
}

template <int NPAD, bool LT, int ISSUERS>
__global__ void __launch_bounds__(128, 1) stage2_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  const int warp = threadIdx.x >> 5;
  if (warp < ISSUERS) {
    constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, version 1, SW128
    constexpr uint32_t kLo = (16u >> 4) << 16;                        // LBO 16
    constexpr uint32_t idesc1 = tc::make_idesc_tf32(NPAD, false, false);
    constexpr uint32_t idesc2 = tc::make_idesc_tf32(2 * NPAD, false, false);
    const uint32_t x0 = (tc::smem_u32(base) >> 4) + kLo;
    const bool do_hi = (ISSUERS == 1) || warp == 0, do_lo = (ISSUERS == 1) || warp == 1;
    const long long t0 = clock64();
    uint32_t s = 0;
    for (int it = 0; it < iters; ++it) {
      const uint32_t xa = x0 + s * (32768u >> 4);
      const uint32_t ba = xa + (16384u >> 4);
      const uint32_t d = tm + ((it >> 2) & 1) * (ISSUERS == 2 ? 192 : 128);
      const uint32_t la = tm + 384 + (it & 3) * 32;
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (do_hi) umma_lohi(d, xa + 2 * k, kHi, ba + 2 * k, kHi, idesc2, (it & 3) || k);
          if (do_lo) {
            const uint32_t dl = ISSUERS == 2 ? d + 2 * NPAD : d + NPAD;
            const uint32_t accl = ISSUERS == 2 ? ((it & 3) || k) : 1u;
            if (LT)
              umma_ts_lohi(dl, la + k * 8, ba + 2 * k, kHi, idesc1, accl);
            else
              umma_lohi(dl, xa + 2 * k, kHi, ba + 2 * k, kHi, idesc1, accl);
          }
        }
        tc::umma_commit(&bar[1 + warp * 3]);
        if ((it & 3) == 3) tc::umma_commit(&bar[2 + warp * 3]);
      }
      __syncwarp();
      s = (s == 4) ? 0 : s + 1;
    }
    if (tc::elect_one()) {
      tc::umma_commit(&bar[0 + warp * 3]);
      tc::mbar_wait(&bar[0 + warp * 3], 0);
    }
    __syncwarp();
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tm);
  }
}

template <int NPAD, bool LT, int ISSUERS>
void run_stage2(long long* d) {
  const int smem = 220 * 1024;
  const int iters = 4096;
  CK(cudaFuncSetAttribute(stage2_kernel<NPAD, LT, ISSUERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  stage2_kernel<NPAD, LT, ISSUERS><<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  long long c = 0;
  CK(cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost));
  std::printf("optimised stage issue NPAD=%d %s issuers=%d: %7.1f cycles / stage (8 UMMAs, 1.25 commits)\n", NPAD,
              LT ? "TS-lo" : "SS-lo", ISSUERS, double(c) / iters);
}

template <int NPAD, bool LT, int COMMITS>
void run_stage(long long* d) {
  const int smem = 220 * 1024;
  const int iters = 4096;
  CK(cudaFuncSetAttribute(stage_kernel<NPAD, LT, COMMITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  stage_kernel<NPAD, LT, COMMITS><<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  long long c = 0;
  CK(cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost));
  std::printf("kernel-like stage issue NPAD=%d %s commits=%d: %7.1f cycles / stage (8 UMMAs)\n", NPAD, LT ? "TS-lo" : "SS-lo",
              COMMITS, double(c) / iters);
}

template <int MODE, int N, int R>
void run(long long* d) {
  const int smem = 16384 + 32768 + 1024;
  const int iters = 8192;
  CK(cudaFuncSetAttribute(rate_kernel<MODE, N, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  rate_kernel<MODE, N, R><<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  long long c = 0;
  CK(cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost));
  const char* names[] = {"SS", "TS", "pair SS(2n)+SS(n)", "pair SS(2n)+TS(n)"};
  std::printf("%-18s N=%3d  accumulators=%d  %7.1f cycles / %s\n", names[MODE], N, R, double(c) / iters,
              MODE >= 2 ? "pair" : "UMMA");
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 8));
  run_stage2<64, false, 1>(d); run_stage2<64, true, 1>(d); run_stage2<64, false, 2>(d); run_stage2<64, true, 2>(d); run_stage2<48, true, 1>(d); run_stage2<48, true, 2>(d);
  run_stage<64, false, 0>(d); run_stage<64, false, 2>(d); run_stage<64, false, 3>(d); run_stage<64, true, 3>(d); run_stage<48, false, 3>(d);
  run<0, 16, 1>(d); run<0, 64, 1>(d); run<0, 128, 1>(d); run<0, 256, 1>(d);
  run<0, 16, 2>(d); run<0, 64, 2>(d); run<0, 128, 2>(d);
  run<0, 16, 4>(d); run<0, 64, 4>(d); run<0, 96, 4>(d);
  run<1, 16, 1>(d); run<1, 64, 1>(d); run<1, 128, 1>(d); run<1, 256, 1>(d);
  run<1, 64, 2>(d); run<1, 64, 4>(d); run<1, 96, 4>(d);
  run<2, 48, 1>(d); run<2, 64, 1>(d); run<2, 64, 2>(d); run<2, 48, 4>(d);
  run<3, 48, 1>(d); run<3, 64, 1>(d); run<3, 64, 2>(d); run<3, 48, 4>(d);
  return 0;
}
