// rnmf_gpu.hpp — header-only C++ face of the B200 path for reference-side callers:
// the reference's types and exceptions, with the work done by the C ABI in rnmf_gpu.h.
//
//   rnmf::gpu::rhals_fit     <- rnmf::rhals_fit     p/include/rnmf/rhals.hpp:40
//   rnmf::gpu::rqb           <- rnmf::rqb           p/include/rnmf/sketch.hpp:64
//   rnmf::gpu::rqb_streaming <- rnmf::rqb_streaming p/include/rnmf/sketch.hpp:71 (any ColumnSource)
//
// Matrix is a minimal row-major double matrix (the reference's Matrix is an Eigen RowMajor
// matrix, p/include/rnmf/types.hpp:17 -- same memory layout, so an Eigen adapter is a copy-free
// Map).  SolverOptions / SketchOptions / TraceRecord / FitResult mirror p/include/rnmf/hals.hpp:15-63
// and sketch.hpp:9-24 field for field; errors are rethrown as the reference exception classes
// (types.hpp:22-39: Shape / Parameter from std::invalid_argument, Data / Io from std::runtime_error).
// Link with -lrnmf_gpu (paper_1711_02037_b200/lib).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnmf_gpu.h"

namespace rnmf {
namespace gpu {

using Index = int64_t;

struct ShapeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ParameterError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {  // CUDA / NCCL failures (no reference counterpart)
  using std::runtime_error::runtime_error;
};

// Row-major dense double matrix.
struct Matrix {
  Index r = 0, c = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(Index rows, Index cols) : r(rows), c(cols), a(size_t(rows) * size_t(cols), 0.0) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
  double& operator()(Index i, Index j) { return a[size_t(i) * size_t(c) + size_t(j)]; }
  double operator()(Index i, Index j) const { return a[size_t(i) * size_t(c) + size_t(j)]; }
};

enum class InitScheme { Random = RNMF_INIT_RANDOM, Svd = RNMF_INIT_SVD };
enum class UpdateOrder { Interleaved = RNMF_ORDER_INTERLEAVED, Grouped = RNMF_ORDER_GROUPED, Shuffled = RNMF_ORDER_SHUFFLED };
enum class StoppingRule { ProjectedGradient = RNMF_STOP_PROJECTED_GRADIENT, Objective = RNMF_STOP_OBJECTIVE };
enum class TestMatrixKind { Uniform = RNMF_TEST_UNIFORM, Gaussian = RNMF_TEST_GAUSSIAN };
enum class MathMode { Exact = RNMF_MATH_EXACT, TF32x3 = RNMF_MATH_TF32X3, TF32 = RNMF_MATH_TF32 };

struct RegConfig {  // p/include/rnmf/hals.hpp:15-20
  double alpha_w = 0.0, alpha_h = 0.0, beta_w = 0.0, beta_h = 0.0;
};

struct SolverOptions {  // p/include/rnmf/hals.hpp:22-38 (+ the GPU-only math mode)
  Index rank = 0;
  Index max_iter = 200;
  double tol = 1e-4;
  InitScheme init = InitScheme::Random;
  UpdateOrder order = UpdateOrder::Grouped;
  StoppingRule stopping = StoppingRule::ProjectedGradient;
  RegConfig reg;
  uint64_t seed = 0;
  bool reseed_dead = false;
  Index trace_full_every = 10;
  Index oversampling = 20;
  Index power_iterations = 2;
  MathMode math_mode = MathMode::Exact;
};

struct SketchOptions {  // p/include/rnmf/sketch.hpp:9-17
  Index target_rank = 0;
  Index oversampling = 20;
  Index power_iterations = 2;
  TestMatrixKind test_matrix = TestMatrixKind::Gaussian;
  Index block_size = 1024;
  uint64_t seed = 0;
};

struct TraceRecord {  // p/include/rnmf/hals.hpp:45-56
  Index iter = 0;
  double elapsed_s = 0.0, objective = 0.0, rel_err = 0.0, pgrad = 0.0, pgrad_full = 0.0,
         objective_compressed = 0.0;
};

struct Factors {
  Matrix w, h;
};

struct FitResult {  // p/include/rnmf/hals.hpp:60-63
  Factors factors;
  std::vector<TraceRecord> trace;
};

struct SketchResult {  // p/include/rnmf/sketch.hpp:19-24
  Matrix q, b;
};

// p/include/rnmf/sketch.hpp:26-33
class ColumnSource {
 public:
  virtual ~ColumnSource() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  // columns [first, first + count) into dst: rows() x count, row-major
  virtual void read_columns(Index first, Index count, double* dst) const = 0;
};

namespace detail {

inline void check(int status, const char* err) {
  switch (status) {
    case RNMF_OK: return;
    case RNMF_SHAPE_ERROR: throw ShapeError(err);
    case RNMF_PARAMETER_ERROR: throw ParameterError(err);
    case RNMF_DATA_ERROR: throw DataError(err);
    case RNMF_IO_ERROR: throw IoError(err);
    default: throw DeviceError(err);
  }
}

// One context per thread and device (contexts own a stream and reusable workspaces).
inline rnmf_gpu_context* context(int device) {
  struct Holder {
    std::vector<rnmf_gpu_context*> ctx;
    ~Holder() {
      for (auto* c : ctx)
        if (c) rnmf_gpu_context_destroy(c);
    }
  };
  static thread_local Holder h;
  if (device < 0) throw ParameterError("rnmf::gpu: negative device index");
  if (h.ctx.size() <= size_t(device)) h.ctx.resize(size_t(device) + 1, nullptr);
  if (!h.ctx[size_t(device)]) {
    char err[1024];
    check(rnmf_gpu_context_create(device, &h.ctx[size_t(device)], err, sizeof err), err);
  }
  return h.ctx[size_t(device)];
}

inline rnmf_solver_options to_c(const SolverOptions& o) {
  rnmf_solver_options c;
  rnmf_default_options(&c);
  c.rank = o.rank;
  c.max_iter = o.max_iter;
  c.tol = o.tol;
  c.init = int32_t(o.init);
  c.order = int32_t(o.order);
  c.stopping = int32_t(o.stopping);
  c.reseed_dead = o.reseed_dead ? 1 : 0;
  c.reg = rnmf_reg_config{o.reg.alpha_w, o.reg.alpha_h, o.reg.beta_w, o.reg.beta_h};
  c.seed = o.seed;
  c.trace_full_every = o.trace_full_every;
  c.oversampling = o.oversampling;
  c.power_iterations = o.power_iterations;
  c.math_mode = int32_t(o.math_mode);
  return c;
}

}  // namespace detail

// rnmf::rhals_fit on GPU `device`: X row-major double on the host.
inline FitResult rhals_fit(const Matrix& x, const SolverOptions& o, int device = 0) {
  rnmf_gpu_context* ctx = detail::context(device);
  const rnmf_solver_options c = detail::to_c(o);
  FitResult r;
  r.factors.w = Matrix(x.rows(), o.rank > 0 ? o.rank : 0);
  r.factors.h = Matrix(o.rank > 0 ? o.rank : 0, x.cols());
  std::vector<rnmf_trace_record> t(size_t(o.max_iter > 0 ? o.max_iter : 0) + 1);
  int64_t len = 0;
  char err[1024];
  detail::check(rnmf_gpu_rhals_fit(ctx, x.data(), RNMF_F64, RNMF_HOST, x.rows(), x.cols(), &c, nullptr, nullptr, nullptr,
                                   r.factors.w.data(), r.factors.h.data(), t.data(), int64_t(t.size()), &len, err,
                                   sizeof err),
                err);
  r.trace.reserve(size_t(len));
  for (int64_t i = 0; i < len; ++i)
    r.trace.push_back(TraceRecord{t[size_t(i)].iter, t[size_t(i)].elapsed_s, t[size_t(i)].objective,
                                  t[size_t(i)].rel_err, t[size_t(i)].pgrad, t[size_t(i)].pgrad_full,
                                  t[size_t(i)].objective_compressed});
  return r;
}

// rnmf::rqb on GPU `device` (fp64, EXACT arithmetic).
inline SketchResult rqb(const Matrix& a, const SketchOptions& o, int device = 0) {
  rnmf_gpu_context* ctx = detail::context(device);
  if (o.block_size < 1) throw ParameterError("sketch: block size must be at least 1");
  char err[1024];
  int64_t l = 0;
  auto call = [&](double* q, double* b) {
    return rnmf_gpu_rqb(ctx, a.data(), RNMF_F64, RNMF_HOST, a.rows(), a.cols(), o.target_rank, o.oversampling,
                        o.power_iterations, int(o.test_matrix), o.seed, nullptr, RNMF_MATH_EXACT, q, b, &l, err,
                        sizeof err);
  };
  detail::check(call(nullptr, nullptr), err);
  SketchResult r{Matrix(a.rows(), l), Matrix(l, a.cols())};
  detail::check(call(r.q.data(), r.b.data()), err);
  return r;
}

// rnmf::rqb_streaming on GPU `device` over any ColumnSource.
inline SketchResult rqb_streaming(const ColumnSource& src, const SketchOptions& o, int device = 0) {
  rnmf_gpu_context* ctx = detail::context(device);
  struct Call {
    const ColumnSource* src;
    std::exception_ptr failure;
  } state{&src, nullptr};
  rnmf_column_reader reader = [](void* user, int64_t first, int64_t count, double* dst) -> int {
    auto* st = static_cast<Call*>(user);
    try {
      st->src->read_columns(first, count, dst);
      return 0;
    } catch (...) {
      st->failure = std::current_exception();
      return 1;
    }
  };
  char err[1024];
  int64_t l = 0;
  auto call = [&](double* q, double* b) {
    return rnmf_gpu_rqb_streaming(ctx, reader, &state, src.rows(), src.cols(), o.target_rank, o.oversampling,
                                  o.power_iterations, int(o.test_matrix), o.block_size, o.seed, nullptr, q, b, &l, err,
                                  sizeof err);
  };
  detail::check(call(nullptr, nullptr), err);
  SketchResult r{Matrix(src.rows(), l), Matrix(l, src.cols())};
  const int st = call(r.q.data(), r.b.data());
  if (st != RNMF_OK && state.failure) std::rethrow_exception(state.failure);
  detail::check(st, err);
  return r;
}

// rqb_streaming over an RNMFMAT1 file (FileColumnSource, p/include/rnmf/data_io.hpp:32-45).
inline SketchResult rqb_streaming_file(const std::string& path, const SketchOptions& o, int device = 0) {
  rnmf_gpu_context* ctx = detail::context(device);
  char err[1024];
  int64_t m = 0, n = 0, l = 0;
  auto call = [&](double* q, double* b) {
    return rnmf_gpu_rqb_streaming_file(ctx, path.c_str(), o.target_rank, o.oversampling, o.power_iterations,
                                       int(o.test_matrix), o.block_size, o.seed, nullptr, q, b, &m, &n, &l, err,
                                       sizeof err);
  };
  detail::check(call(nullptr, nullptr), err);
  SketchResult r{Matrix(m, l), Matrix(l, n)};
  detail::check(call(r.q.data(), r.b.data()), err);
  return r;
}

}  // namespace gpu
}  // namespace rnmf
