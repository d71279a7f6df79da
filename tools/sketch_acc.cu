// Accuracy / speed probe of the X-streaming sketch GEMMs on a B200 (development aid, not a test).
// Y = X S (n x c S) and P = X^T Q (m x c Q) against an fp64 GPU reference, for the FFMA kernels
// (kernels_xw.cu) and the tcgen05 3xTF32 / 1xTF32 kernels (kernels_tc.cu) at several TMEM
// accumulation chunk lengths.  Reports rms(err)/rms(ref), max |err|/sum|terms| and the mean
// signed error relative to rms(ref) (a truncation bias shows up there).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1711_02037_b200/csrc \
//        tools/sketch_acc.cu paper_1711_02037_b200/csrc/{kernels_tc,kernels_xw,kernels_xgemm}.cu -o tools/sketch_acc
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kernels.h"

using namespace rnmf_gpu;
#ifdef RNMF_TC_PROF
namespace rnmf_gpu { void tc_prof_read(long long* out, bool reset); }
#endif

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

// fp64 reference: Y (rows x c) = A (rows x kk, pitch lda, strides sa_r / sa_k) * B (kk x c)
__global__ void ref_kernel(const float* a, int64_t rows, int64_t kk, int64_t sr, int64_t sk, const float* b, int c,
                           double* y, double* mag) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.y + threadIdx.y;
  const int j = threadIdx.x;
  if (r >= rows || j >= c) return;
  double acc = 0, m = 0;
  for (int64_t k = 0; k < kk; ++k) {
    const double t = double(a[r * sr + k * sk]) * double(b[k * c + j]);
    acc += t;
    m += fabs(t);
  }
  y[r * c + j] = acc;
  mag[r * c + j] = m;
}

struct Stats {
  double rms_rel, max_rel, bias_rel;
};

Stats stats(const std::vector<float>& got, const std::vector<double>& ref, const std::vector<double>& mag) {
  double se = 0, sr = 0, sb = 0, mx = 0;
  for (size_t i = 0; i < ref.size(); ++i) {
    const double e = double(got[i]) - ref[i];
    se += e * e;
    sr += ref[i] * ref[i];
    sb += (ref[i] >= 0 ? e : -e);  // signed toward |ref|: negative = shrinkage
    mx = std::max(mx, std::fabs(e) / mag[i]);
  }
  const double rr = std::sqrt(sr / ref.size());
  return {std::sqrt(se / ref.size()) / rr, mx, sb / ref.size() / rr};
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 32256;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 2410;
  const int c = argc > 3 ? atoi(argv[3]) : 36;
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  const int64_t ldx = (n + 31) / 32 * 32;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  std::vector<float> x(size_t(m) * ldx, 0.f), s(size_t(n) * c), q(size_t(m) * c);
  std::mt19937 g(1);
  std::uniform_real_distribution<float> u(0.f, 1.f);
  std::normal_distribution<float> nd(0.f, 1.f);
  // nonnegative, smooth-ish rows (like the faces config: mixtures of a few profiles) plus noise
  std::vector<float> prof(size_t(8) * n);
  for (auto& v : prof) v = u(g);
  for (int64_t i = 0; i < m; ++i) {
    float wv[8];
    for (auto& w : wv) w = u(g);
    for (int64_t j = 0; j < n; ++j) {
      float v = 0.02f * u(g);
      for (int p = 0; p < 8; ++p) v += wv[p] * prof[p * n + j];
      x[size_t(i) * ldx + j] = v / 4.f;
    }
  }
  for (auto& v : s) v = nd(g);
  for (auto& v : q) v = nd(g) / std::sqrt(float(m));
  float *dx, *ds, *dq, *dy, *dp, *dpart, *dh, *dl, *dspad, *dout;
  double *dref, *dmag;
  const int npad = tc_npad(c);
  const int64_t big = std::max(m, n);
  CK(cudaMalloc(&dx, x.size() * 4));
  CK(cudaMalloc(&ds, s.size() * 4));
  CK(cudaMalloc(&dq, q.size() * 4));
  CK(cudaMalloc(&dy, size_t(m) * c * 4));
  CK(cudaMalloc(&dp, size_t(n) * c * 4));
  CK(cudaMalloc(&dpart, size_t(sms) * n * c * 4));
  CK(cudaMalloc(&dh, size_t(npad) * tc_st_pitch(big) * 4));
  CK(cudaMalloc(&dl, size_t(npad) * tc_st_pitch(big) * 4));
  CK(cudaMalloc(&dspad, size_t(std::max(xw_tma_spad_len(n, c), xw_tma_spad_len(m, c))) * 4));
  CK(cudaMalloc(&dout, size_t(n) * c * 4));
  CK(cudaMalloc(&dref, size_t(m) * c * 8));
  CK(cudaMalloc(&dmag, size_t(m) * c * 8));
  CK(cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto&& fn) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
  };
  const double gb = double(m) * n * 4 / 1e9;

  // ---------------- Y = X S
  {
    dim3 blk(c, std::max(1, 256 / c));
    ref_kernel<<<unsigned((m + blk.y - 1) / blk.y), blk>>>(dx, m, n, ldx, 1, ds, c, dref, dmag);
    CK(cudaDeviceSynchronize());
    std::vector<double> ref(size_t(m) * c), mag(size_t(m) * c);
    CK(cudaMemcpy(ref.data(), dref, ref.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mag.data(), dmag, mag.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<float> y(size_t(m) * c);
    auto report = [&](const char* name, float ms) {
      CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
      const Stats st = stats(y, ref, mag);
      std::printf("XW  %-22s rms %.3e  max %.3e  bias %+.3e  %8.4f ms %6.0f GB/s\n", name, st.rms_rel, st.max_rel,
                  st.bias_rel, ms, gb / (ms * 1e-3));
    };
    float ms = timeit([&] { launch_xw_tma<float>(dx, m, n, ldx, ds, c, dy, dspad, sms, 0); });
    report("ffma_tma", ms);
    launch_tc_prep_st(ds, n, c, dh, dl, 0, true);
    for (int x3 = 1; x3 >= 0; --x3)
      for (int ch : {16, 8, 4}) {
        if (!x3 && ch != 2) continue;
        tc_set_chunk(ch);
#ifdef RNMF_TC_PROF
        { long long z[16]; tc_prof_read(z, true); }
#endif
        ms = timeit([&] { launch_tc_xw(dx, m, n, ldx, dh, dl, c, dy, x3, sms, 0); });
#ifdef RNMF_TC_PROF
        {
          long long z[16];
          tc_prof_read(z, true);
          const double stages = double((m + 127) / 128 + sms - 1) / sms * double((n + 31) / 32) * (reps + 1);
          const char* nm2[] = {"producer wait empty", "mma wait tempty", "mma wait full", "mma wait lofull", "mma issue",
                               "split wait full", "split work", "epi wait tfull", "epi drain"};
          for (int i = 0; i < 9; ++i) std::printf("   prof %-20s %9.1f cycles / stage\n", nm2[i], double(z[i]) / stages);
        }
#endif
        char nm[64];
        std::snprintf(nm, sizeof nm, "tc%s chunk=%d", x3 ? "3xtf32" : "1xtf32", ch);
        report(nm, ms);
      }
  }
  // ---------------- P = X^T Q
  {
    dim3 blk(c, std::max(1, 256 / c));
    ref_kernel<<<unsigned((n + blk.y - 1) / blk.y), blk>>>(dx, n, m, 1, ldx, dq, c, dref, dmag);
    CK(cudaDeviceSynchronize());
    std::vector<double> ref(size_t(n) * c), mag(size_t(n) * c);
    CK(cudaMemcpy(ref.data(), dref, ref.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mag.data(), dmag, mag.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<float> p(size_t(n) * c);
    auto report = [&](const char* name, float ms) {
      CK(cudaMemcpy(p.data(), dout, p.size() * 4, cudaMemcpyDeviceToHost));
      const Stats st = stats(p, ref, mag);
      std::printf("XTW %-22s rms %.3e  max %.3e  bias %+.3e  %8.4f ms %6.0f GB/s\n", name, st.rms_rel, st.max_rel,
                  st.bias_rel, ms, gb / (ms * 1e-3));
    };
    const int sp = xtw_tma_splits(m, n, sms);
    float ms = timeit([&] { launch_xtw_tma<float>(dx, m, n, ldx, dq, c, dpart, sp, dout, false, dspad, sms, 0); });
    report("ffma_tma", ms);
    launch_tc_prep_st(dq, m, c, dh, dl, 0, true);
    const int tsp = tc_xtw_splits(m, n, sms);
    for (int x3 = 1; x3 >= 0; --x3)
      for (int ch : {16, 8, 4}) {
        if (!x3 && ch != 2) continue;
        tc_set_chunk(ch);
        ms = timeit([&] {
          launch_tc_xtw(dx, m, n, ldx, dh, dl, c, dpart, tsp, x3, sms, 0);
          launch_splitk_reduce<float>(dpart, tsp, n, c, dout, false, 0);
        });
        char nm[64];
        std::snprintf(nm, sizeof nm, "tc%s chunk=%d", x3 ? "3xtf32" : "1xtf32", ch);
        report(nm, ms);
      }
  }
  return 0;
}
