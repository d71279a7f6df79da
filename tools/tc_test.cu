// Standalone validation / timing of the tcgen05 X-streaming GEMM (kernels_tc.cu) on a B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1711_02037_b200/csrc \
//        tools/tc_test.cu paper_1711_02037_b200/csrc/kernels_tc.cu -o tools/tc_test
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kernels.h"

using namespace rnmf_gpu;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

int xtw_main(int64_t m, int64_t n, int c, int reps);

int main(int argc, char** argv) {
  if (const char* e = std::getenv("TC_XTW")) {
    long long mm = 0, nn = 0;
    int cc = 0, rr = 0;
    std::sscanf(e, "%lld,%lld,%d,%d", &mm, &nn, &cc, &rr);
    return xtw_main(mm, nn, cc, rr);
  }
  const int64_t m = argc > 1 ? atoll(argv[1]) : 1000;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 2410;
  const int c = argc > 3 ? atoi(argv[3]) : 36;
  const int reps = argc > 4 ? atoi(argv[4]) : 5;
  const int64_t ldx = (n + 31) / 32 * 32;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  std::vector<float> x(size_t(m) * ldx, 0.f), s(size_t(n) * c);
  std::mt19937 g(1);
  std::uniform_real_distribution<float> u(0.f, 1.f);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) x[size_t(i) * ldx + j] = u(g);
  for (auto& v : s) v = nd(g);
  float *dx, *ds, *dh, *dl, *dy;
  const int npad = tc_npad(c);
  const int64_t ldst = tc_st_pitch(n);
  CK(cudaMalloc(&dx, x.size() * 4));
  CK(cudaMalloc(&ds, s.size() * 4));
  CK(cudaMalloc(&dh, size_t(npad) * ldst * 4));
  CK(cudaMalloc(&dl, size_t(npad) * ldst * 4));
  CK(cudaMalloc(&dy, size_t(m) * c * 4));
  CK(cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice));
  launch_tc_prep_st(ds, n, c, dh, dl, 0, true);
  // reference on a row sample (fp64)
  std::vector<int64_t> rows;
  for (int64_t i = 0; i < m; i += std::max<int64_t>(1, m / 200)) rows.push_back(i);
  rows.push_back(m - 1);
  for (int x3 = 0; x3 < 2; ++x3) {
    CK(cudaMemset(dy, 0, size_t(m) * c * 4));
    launch_tc_xw(dx, m, n, ldx, dh, dl, c, dy, x3 != 0, prop.multiProcessorCount, 0);
    CK(cudaDeviceSynchronize());
    std::vector<float> y(size_t(m) * c);
    CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxabs = 0;
    for (int64_t i : rows)
      for (int j = 0; j < c; ++j) {
        double ref = 0, mag = 0;
        for (int64_t k = 0; k < n; ++k) {
          ref += double(x[size_t(i) * ldx + k]) * double(s[size_t(k) * c + j]);
          mag += std::fabs(double(x[size_t(i) * ldx + k]) * double(s[size_t(k) * c + j]));
        }
        const double err = std::fabs(double(y[size_t(i) * c + j]) - ref);
        maxabs = std::max(maxabs, err);
        maxrel = std::max(maxrel, err / mag);
      }
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) launch_tc_xw(dx, m, n, ldx, dh, dl, c, dy, x3 != 0, prop.multiProcessorCount, 0);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    const double gbs = double(m) * n * 4 / (ms * 1e-3) / 1e9;
    std::printf("tc_xw m=%lld n=%lld c=%d x3=%d: max |err|/sum|terms| = %.3e (abs %.3e)  %.4f ms  %.0f GB/s\n",
                (long long)m, (long long)n, c, x3, maxrel, maxabs, ms, gbs);
  }
  return 0;
}

// ---- tc_xtw check: P = X^T S, S (m x c), split over rows
int xtw_main(int64_t m, int64_t n, int c, int reps) {
  const int64_t ldx = (n + 31) / 32 * 32;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  std::vector<float> x(size_t(m) * ldx, 0.f), s(size_t(m) * c);
  std::mt19937 g(2);
  std::uniform_real_distribution<float> u(0.f, 1.f);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) x[size_t(i) * ldx + j] = u(g);
  for (auto& v : s) v = nd(g);
  const int npad = tc_npad(c);
  const int64_t ldst = tc_st_pitch(m);
  const int splits = tc_xtw_splits(m, n, prop.multiProcessorCount);
  float *dx, *ds, *dh, *dl, *dp;
  CK(cudaMalloc(&dx, x.size() * 4));
  CK(cudaMalloc(&ds, s.size() * 4));
  CK(cudaMalloc(&dh, size_t(npad) * ldst * 4));
  CK(cudaMalloc(&dl, size_t(npad) * ldst * 4));
  CK(cudaMalloc(&dp, size_t(splits) * n * c * 4));
  CK(cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice));
  launch_tc_prep_st(ds, m, c, dh, dl, 0, true);
  for (int x3 = 0; x3 < 2; ++x3) {
  launch_tc_xtw(dx, m, n, ldx, dh, dl, c, dp, splits, x3, prop.multiProcessorCount, 0);
  CK(cudaDeviceSynchronize());
  std::vector<float> part(size_t(splits) * n * c);
  CK(cudaMemcpy(part.data(), dp, part.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0;
  for (int64_t col = 0; col < n; col += std::max<int64_t>(1, n / 150))
    for (int j = 0; j < c; ++j) {
      double ref = 0, mag = 0, got = 0;
      for (int64_t i = 0; i < m; ++i) {
        const double t = double(x[size_t(i) * ldx + col]) * double(s[size_t(i) * c + j]);
        ref += t;
        mag += std::fabs(t);
      }
      for (int sp = 0; sp < splits; ++sp) got += part[(size_t(sp) * n + col) * c + j];
      maxrel = std::max(maxrel, std::fabs(got - ref) / mag);
    }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) launch_tc_xtw(dx, m, n, ldx, dh, dl, c, dp, splits, x3, prop.multiProcessorCount, 0);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= reps;
  std::printf("tc_xtw m=%lld n=%lld c=%d splits=%d x3=%d: max |err|/sum|terms| = %.3e  %.4f ms  %.0f GB/s\n",
              (long long)m, (long long)n, c, splits, x3, maxrel, ms, double(m) * n * 4 / (ms * 1e-3) / 1e9);
  }
  return 0;
}

