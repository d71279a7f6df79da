// Probe of the tcgen05 3xTF32 X-streaming kernels with selector S (Y = X[:, sel]): prints the
// error pattern by output column and by K stage count.  Development aid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1711_02037_b200/csrc \
//        tools/tx_probe.cu paper_1711_02037_b200/csrc/kernels_tc.cu -o tools/tx_probe
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <vector>

#include "kernels.h"
using namespace rnmf_gpu;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

int run(int64_t m, int64_t n, int c, int mode) {
  const int64_t ldx = (n + 31) / 32 * 32;
  std::vector<float> x(size_t(m) * ldx, 0.f), s(size_t(n) * c, 0.f);
  std::mt19937 g(1);
  std::uniform_real_distribution<float> u(0.5f, 1.f);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) x[size_t(i) * ldx + j] = mode == 2 ? float(i / 128) + float(j) / 1024.f + float(i % 128) / 131072.f : u(g);
  // mode 0: S selects column (3 j) % n; mode 1: S = all ones (row sums)
  for (int j = 0; j < c; ++j) {
    if (mode != 1) s[size_t((3 * j) % n) * c + j] = 1.f;
    else for (int64_t kk = 0; kk < n; ++kk) s[size_t(kk) * c + j] = 1.f;
  }
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
  launch_tc_xw(dx, m, n, ldx, dh, dl, c, dy, true, 148, 0);
  CK(cudaDeviceSynchronize());
  std::vector<float> y(size_t(m) * c);
  CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  std::vector<double> colerr(c, 0), rowerr(128, 0), tileerr((m + 127) / 128, 0);
  for (int64_t i = 0; i < m; ++i)
    for (int j = 0; j < c; ++j) {
      double ref = 0;
      if (mode != 1) ref = x[size_t(i) * ldx + (3 * j) % n];
      else for (int64_t kk = 0; kk < n; ++kk) ref += x[size_t(i) * ldx + kk];
      const double e = std::fabs(y[size_t(i) * c + j] - ref) / std::fabs(ref);
      worst = std::max(worst, e);
      colerr[j] = std::max(colerr[j], e);
      rowerr[i % 128] = std::max(rowerr[i % 128], e);
      tileerr[i / 128] = std::max(tileerr[i / 128], e);
    }
  std::printf("m=%lld n=%lld c=%d mode=%d worst rel %.3e\n  cols:", (long long)m, (long long)n, c, mode, worst);
  for (int j = 0; j < c; ++j) std::printf(" %.0e", colerr[j]);
  std::printf("\n  rows%%128 (first 40):");
  for (int r = 0; r < 40; ++r) std::printf(" %.0e", rowerr[r]);
  std::printf("\n  bad tiles:");
  int nb = 0;
  for (size_t t = 0; t < tileerr.size(); ++t)
    if (tileerr[t] > 1e-5 && nb++ < 40) std::printf(" %zu(%.0e)", t, tileerr[t]);
  std::printf(" [%d bad of %zu]\n", nb, tileerr.size());
  // for the first bad tile: which X tile's rows do its outputs match (selector mode)?
  for (size_t t = 0; t < tileerr.size() && mode == 2; ++t) {
    if (tileerr[t] <= 1e-5) continue;
    for (int rr = 0; rr < 128; rr += 37) {
      const int64_t i = int64_t(t) * 128 + rr;
      if (i >= m) break;
      std::printf("  row %lld (tile %lld, r %d): y[j] (tile + col/1024 + r/131072) for j = 0,10,20,..:", (long long)i, (long long)t, rr);
      for (int j = 0; j < c; j += 10) std::printf(" [%d: %.6f]", (3 * j) % (int)n, y[i * c + j]);
      std::printf("\n");
      continue;
      std::printf(" %.6f %.6f %.6f %.6f", x[i * ldx], x[i * ldx + 3], x[i * ldx + 6], x[i * ldx + 9]);
      for (int64_t t2 = 0; t2 < (int64_t)tileerr.size(); ++t2)
        for (int r2 = 0; r2 < 128 && t2 * 128 + r2 < m; ++r2)
          if (std::fabs(x[(t2 * 128 + r2) * ldx] - y[i * c]) < 1e-6 && std::fabs(x[(t2 * 128 + r2) * ldx + 3] - y[i * c + 1]) < 1e-6)
            std::printf("  == x row %lld", (long long)(t2 * 128 + r2));
      std::printf("\n");
    }
    break;
  }
  cudaFree(dx); cudaFree(ds); cudaFree(dh); cudaFree(dl); cudaFree(dy);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 4) return run(atoll(argv[1]), atoll(argv[2]), atoi(argv[3]), atoi(argv[4]));
  run(128, 32, 16, 0);
  run(1024, 512, 60, 1);
  run(4096, 2048, 36, 1);
  return 0;
}
