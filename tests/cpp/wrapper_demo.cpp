// Reference-side use of include/rnmf_gpu.hpp (built and run by tests/test_cpp_wrapper.py):
// rhals_fit on a seeded nonnegative matrix, rqb and rqb_streaming agreement, and the mapping of
// library errors onto the reference exception types.  Prints one line of key=value results.
#include <cmath>
#include <cstdio>
#include <random>

#include "rnmf_gpu.hpp"

using namespace rnmf::gpu;

struct MemSource : ColumnSource {
  const Matrix& a;
  explicit MemSource(const Matrix& x) : a(x) {}
  Index rows() const override { return a.rows(); }
  Index cols() const override { return a.cols(); }
  void read_columns(Index first, Index count, double* dst) const override {
    for (Index i = 0; i < a.rows(); ++i)
      for (Index j = 0; j < count; ++j) dst[i * count + j] = a(i, first + j);
  }
};

int main() {
  const Index m = 400, n = 300, r = 5;
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  Matrix w0(m, r), h0(r, n), x(m, n);
  for (auto& v : w0.a) v = std::fabs(nd(g));
  for (auto& v : h0.a) v = std::fabs(nd(g));
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double s = 0.05 * std::fabs(nd(g));
      for (Index t = 0; t < r; ++t) s += w0(i, t) * h0(t, j);
      x(i, j) = s;
    }
  SolverOptions o;
  o.rank = r;
  o.max_iter = 30;
  o.tol = 1e-300;
  o.oversampling = 5;
  o.seed = 3;
  const FitResult fit = rhals_fit(x, o);
  SketchOptions so;
  so.target_rank = r;
  so.oversampling = 5;
  so.seed = 11;
  so.block_size = 64;
  const SketchResult mem = rqb(x, so);
  const SketchResult st = rqb_streaming(MemSource(x), so);
  double dev = 0.0;  // max |Q B (rqb) - Q B (rqb_streaming)|
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double a = 0.0, b = 0.0;
      for (Index t = 0; t < mem.q.cols(); ++t) a += mem.q(i, t) * mem.b(t, j);
      for (Index t = 0; t < st.q.cols(); ++t) b += st.q(i, t) * st.b(t, j);
      dev = std::fmax(dev, std::fabs(a - b));
    }
  int data_error = 0, param_error = 0;
  Matrix bad = x;
  bad(3, 4) = -1.0;
  try {
    rhals_fit(bad, o);
  } catch (const DataError&) {
    data_error = 1;
  }
  SolverOptions zero = o;
  zero.rank = 0;
  try {
    rhals_fit(x, zero);
  } catch (const ParameterError&) {
    param_error = 1;
  }
  std::printf("records=%zu final_rel_err=%.17g qb_dev=%.3e data_error=%d parameter_error=%d\n", fit.trace.size(),
              fit.trace.back().rel_err, dev, data_error, param_error);
  return 0;
}
