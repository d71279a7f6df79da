// rnmf_oracle.cpp — TEST INFRASTRUCTURE ONLY (see rnmf_oracle.h).
//
// fp64 CPU restatement of the reference randomized-HALS path.  Each function cites the
// reference file:line it restates (p/ = /root/reference/proj/).  Written from the reference's
// behaviour, not copied: the reference is Eigen expression code, this is plain loops over
// row-major buffers.  Large loops optionally run on several threads (oracle_set_threads);
// every parallel loop partitions OUTPUT rows, so the result does not depend on the thread
// count.

#include "rnmf_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <thread>

namespace orc {

using Index = int64_t;

// ---------------------------------------------------------------------------------------------
// Exceptions: p/include/rnmf/types.hpp:22-39.
struct ShapeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ParameterError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

static int g_threads = 1;

// Runs f(i0, i1) over a static partition of [0, n) into g_threads contiguous chunks.  Every
// caller partitions OUTPUT rows, so results do not depend on the thread count.
template <typename F>
static void parallel_ranges(Index n, F&& f, Index min_per_thread = 64) {
  const Index T = std::max<Index>(1, std::min<Index>(g_threads, n / std::max<Index>(1, min_per_thread)));
  if (T <= 1) {
    f(Index(0), n);
    return;
  }
  std::vector<std::thread> pool;
  for (Index t = 0; t < T; ++t) pool.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------------------------------------
// Row-major dense matrix (the reference Matrix is RowMajor double, types.hpp:17).
struct Mat {
  Index r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index rows, Index cols, double v = 0.0) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), v) {}
  double& operator()(Index i, Index j) { return a[static_cast<size_t>(i * c + j)]; }
  double operator()(Index i, Index j) const { return a[static_cast<size_t>(i * c + j)]; }
  double* row(Index i) { return a.data() + i * c; }
  const double* row(Index i) const { return a.data() + i * c; }
  Index size() const { return r * c; }
  static Mat from(const double* p, Index rows, Index cols) {
    Mat m(rows, cols);
    if (rows > 0 && cols > 0) std::memcpy(m.a.data(), p, sizeof(double) * static_cast<size_t>(rows * cols));
    return m;
  }
  void to(double* p) const {
    if (size()) std::memcpy(p, a.data(), sizeof(double) * static_cast<size_t>(size()));
  }
};

static std::string shape_string(Index r, Index c) {
  return std::to_string(r) + "x" + std::to_string(c);
}
static std::string shape_string(const Mat& m) { return shape_string(m.r, m.c); }

// C = A * B   (A p x q, B q x s)
static Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw ShapeError("matmul: inner dimensions disagree for " + shape_string(A) +
                                   " * " + shape_string(B));
  Mat C(A.r, B.c);
  const Index p = A.r, q = A.c, s = B.c;
  parallel_ranges(p, [&](Index i0, Index i1) {
    for (Index i = i0; i < i1; ++i) {
      double* ci = C.row(i);
      const double* ai = A.row(i);
      for (Index k = 0; k < q; ++k) {
        const double av = ai[k];
        const double* bk = B.row(k);
        for (Index j = 0; j < s; ++j) ci[j] += av * bk[j];
      }
    }
  });
  return C;
}

// C = A^T * B   (A q x p, B q x s) -> p x s
static Mat matmul_tn(const Mat& A, const Mat& B) {
  if (A.r != B.r) throw ShapeError("matmul: inner dimensions disagree for " +
                                   shape_string(A.c, A.r) + " * " + shape_string(B));
  Mat C(A.c, B.c);
  const Index q = A.r, p = A.c, s = B.c;
  parallel_ranges(p, [&](Index i0, Index i1) {
    for (Index k = 0; k < q; ++k) {
      const double* ak = A.row(k);
      const double* bk = B.row(k);
      for (Index i = i0; i < i1; ++i) {
        const double av = ak[i];
        double* ci = C.row(i);
        for (Index j = 0; j < s; ++j) ci[j] += av * bk[j];
      }
    }
  }, 8);
  return C;
}

// C = A * B^T   (A p x q, B s x q) -> p x s
static Mat matmul_nt(const Mat& A, const Mat& B) {
  if (A.c != B.c) throw ShapeError("matmul: inner dimensions disagree for " + shape_string(A) +
                                   " * " + shape_string(B.c, B.r));
  Mat C(A.r, B.r);
  parallel_ranges(A.r, [&](Index i0, Index i1) {
    for (Index i = i0; i < i1; ++i) {
      const double* ai = A.row(i);
      for (Index j = 0; j < B.r; ++j) {
        const double* bj = B.row(j);
        double s = 0.0;
        for (Index k = 0; k < A.c; ++k) s += ai[k] * bj[k];
        C(i, j) = s;
      }
    }
  });
  return C;
}

static Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (Index i = 0; i < A.r; ++i)
    for (Index j = 0; j < A.c; ++j) T(j, i) = A(i, j);
  return T;
}

static double squared_norm(const Mat& A) {
  double s = 0.0;
  for (double v : A.a) s += v * v;
  return s;
}

// ---------------------------------------------------------------------------------------------
// Rng — restates p/include/rnmf/types.hpp:55-102: mt19937_64 bits, uniform from the top 53
// bits, Box-Muller gaussians with a cached spare, split(tag) = Rng(splitmix64(seed + phi*(tag+1))).
class Rng {
 public:
  explicit Rng(uint64_t seed) : seed_(seed), engine_(seed) {}
  uint64_t seed() const { return seed_; }
  uint64_t next_u64() { return engine_(); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double gaussian() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * kPi * u2;
    spare_ = radius * std::sin(angle);
    has_spare_ = true;
    return radius * std::cos(angle);
  }
  Rng split(uint64_t stream) const {
    return Rng(splitmix64(seed_ + 0x9e3779b97f4a7c15ULL * (stream + 1)));
  }
  static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }

 private:
  static constexpr double kPi = 3.141592653589793238462643383279502884;
  uint64_t seed_;
  std::mt19937_64 engine_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// filled_matrix / uniform_matrix / gaussian_matrix: p/src/core.cpp:20-42 (row-major draw order).
template <typename Draw>
static Mat filled_matrix(Index rows, Index cols, Draw&& draw) {
  if (rows < 1 || cols < 1)
    throw ShapeError("random matrix: dimensions must be positive, got " +
                     shape_string(rows, cols));
  Mat m(rows, cols);
  for (auto& v : m.a) v = draw();
  return m;
}
static Mat uniform_matrix(Index rows, Index cols, Rng& rng) {
  return filled_matrix(rows, cols, [&rng] { return rng.uniform(); });
}
static Mat gaussian_matrix(Index rows, Index cols, Rng& rng) {
  return filled_matrix(rows, cols, [&rng] { return rng.gaussian(); });
}

// economic_qr: p/src/core.cpp:7-16 (Eigen::HouseholderQR, explicit thin Q = householderQ * I).
// Householder vectors follow Eigen's makeHouseholder convention: beta = -sign(c0)*||x||,
// tau = (beta - c0)/beta, essential = x_tail/(c0 - beta); a zero tail gives tau = 0.
struct QrResult {
  Mat q, r;
};
static QrResult economic_qr(const Mat& a) {
  if (a.r < a.c) throw ShapeError("economic_qr: need rows >= cols, got " + shape_string(a));
  const Index m = a.r, l = a.c;
  Mat A = a;
  std::vector<double> tau(static_cast<size_t>(l), 0.0);
  std::vector<double> s(static_cast<size_t>(l));
  for (Index j = 0; j < l; ++j) {
    const double c0 = A(j, j);
    double tail = 0.0;
    for (Index i = j + 1; i < m; ++i) tail += A(i, j) * A(i, j);
    double beta, t;
    if (tail <= std::numeric_limits<double>::min()) {
      t = 0.0;
      beta = c0;
      for (Index i = j + 1; i < m; ++i) A(i, j) = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double inv = 1.0 / (c0 - beta);
      for (Index i = j + 1; i < m; ++i) A(i, j) *= inv;
      t = (beta - c0) / beta;
    }
    tau[static_cast<size_t>(j)] = t;
    A(j, j) = beta;
    if (t != 0.0 && j + 1 < l) {
      // A(j:, j+1:) -= t * v * (v^T A(j:, j+1:)), v = [1; essential]
      for (Index c = j + 1; c < l; ++c) s[static_cast<size_t>(c)] = A(j, c);
      for (Index i = j + 1; i < m; ++i) {
        const double vi = A(i, j);
        const double* ai = A.row(i);
        for (Index c = j + 1; c < l; ++c) s[static_cast<size_t>(c)] += vi * ai[c];
      }
      for (Index c = j + 1; c < l; ++c) {
        s[static_cast<size_t>(c)] *= t;
        A(j, c) -= s[static_cast<size_t>(c)];
      }
      for (Index i = j + 1; i < m; ++i) {
        const double vi = A(i, j);
        double* ai = A.row(i);
        for (Index c = j + 1; c < l; ++c) ai[c] -= s[static_cast<size_t>(c)] * vi;
      }
    }
  }
  QrResult out;
  out.r = Mat(l, l);
  for (Index i = 0; i < l; ++i)
    for (Index j = i; j < l; ++j) out.r(i, j) = A(i, j);
  // Q = H_0 H_1 ... H_{l-1} [I; 0]
  Mat Q(m, l);
  for (Index i = 0; i < l; ++i) Q(i, i) = 1.0;
  for (Index j = l - 1; j >= 0; --j) {
    const double t = tau[static_cast<size_t>(j)];
    if (t == 0.0) continue;
    for (Index c = 0; c < l; ++c) s[static_cast<size_t>(c)] = Q(j, c);
    for (Index i = j + 1; i < m; ++i) {
      const double vi = A(i, j);
      const double* qi = Q.row(i);
      for (Index c = 0; c < l; ++c) s[static_cast<size_t>(c)] += vi * qi[c];
    }
    for (Index c = 0; c < l; ++c) {
      s[static_cast<size_t>(c)] *= t;
      Q(j, c) -= s[static_cast<size_t>(c)];
    }
    for (Index i = j + 1; i < m; ++i) {
      const double vi = A(i, j);
      double* qi = Q.row(i);
      for (Index c = 0; c < l; ++c) qi[c] -= s[static_cast<size_t>(c)] * vi;
    }
  }
  out.q = std::move(Q);
  return out;
}

// synth_lowrank: p/src/data_io.cpp:171-183.
static Mat synth_lowrank(Index rows, Index cols, Index rank, double noise, uint64_t seed) {
  if (rank < 1 || rank > std::min(rows, cols))
    throw ParameterError("synth_lowrank: rank " + std::to_string(rank) + " out of range [1, " +
                         std::to_string(std::min(rows, cols)) + "]");
  if (noise < 0.0) throw ParameterError("synth_lowrank: noise must be nonnegative");
  Rng rng(seed);
  Mat g1 = gaussian_matrix(rows, rank, rng);
  for (auto& v : g1.a) v = std::max(v, 0.0);
  Mat g2 = gaussian_matrix(rank, cols, rng);
  for (auto& v : g2.a) v = std::max(v, 0.0);
  Mat x = matmul(g1, g2);
  if (noise > 0.0) {
    Mat g = gaussian_matrix(rows, cols, rng);
    for (Index i = 0; i < x.size(); ++i) x.a[static_cast<size_t>(i)] += noise * std::max(g.a[static_cast<size_t>(i)], 0.0);
  }
  return x;
}

// ---------------------------------------------------------------------------------------------
// Sketch: p/src/sketch.cpp:30-71.
struct SketchOptions {
  Index target_rank = 0;
  Index oversampling = 20;
  Index power_iterations = 2;
  int test_matrix = RNMF_TEST_GAUSSIAN;
  Index block_size = 1024;
  uint64_t seed = 0;
};

static Index sketch_width(Index rows, Index cols, const SketchOptions& o) {
  const Index bound = std::min(rows, cols);
  if (o.target_rank < 1 || o.target_rank > bound)
    throw ParameterError("sketch: target rank " + std::to_string(o.target_rank) +
                         " out of range [1, " + std::to_string(bound) + "] for a " +
                         shape_string(rows, cols) + " matrix");
  if (o.oversampling < 0 || o.power_iterations < 0)
    throw ParameterError("sketch: oversampling and power iterations must be nonnegative");
  if (o.block_size < 1) throw ParameterError("sketch: block size must be at least 1");
  Index l = o.target_rank + o.oversampling;
  if (l > bound) {
    std::fprintf(stderr, "rnmf: sketch width %lld exceeds min(%lld, %lld); clamping to %lld\n",
                 (long long)l, (long long)rows, (long long)cols, (long long)bound);
    l = bound;
  }
  return l;
}

static bool all_finite(const Mat& a) {
  for (double v : a.a)
    if (!std::isfinite(v)) return false;
  return true;
}

struct SketchResult {
  Mat q, b;
};

// rqb with an optional injected test matrix (omega: n x l) replacing sketch.cpp:57-58.
static SketchResult rqb(const Mat& a, const SketchOptions& o, const double* omega) {
  const Index l = sketch_width(a.r, a.c, o);
  if (!all_finite(a)) throw DataError("rqb: input contains non-finite values");
  Mat om;
  if (omega) {
    om = Mat::from(omega, a.c, l);
  } else {
    Rng rng(o.seed);
    om = o.test_matrix == RNMF_TEST_UNIFORM ? uniform_matrix(a.c, l, rng)
                                            : gaussian_matrix(a.c, l, rng);
  }
  Mat y = matmul(a, om);
  for (Index it = 0; it < o.power_iterations; ++it) {
    const Mat q = economic_qr(y).q;
    const Mat z = economic_qr(matmul_tn(a, q)).q;
    y = matmul(a, z);
  }
  SketchResult out;
  out.q = economic_qr(y).q;
  out.b = matmul_tn(out.q, a);
  return out;
}

// rqb_streaming: p/src/sketch.cpp:73-116 over an in-memory source read in column blocks of bs
// (MatrixColumnSource, p/include/rnmf/sketch.hpp:41-51).  Blocks reduce in ascending order.
static SketchResult rqb_streaming(const Mat& a, const SketchOptions& o, const double* omega) {
  const Index m = a.r, n = a.c;
  const Index l = sketch_width(m, n, o);
  const Index bs = std::min(o.block_size, n);
  Mat om;
  if (omega) {
    om = Mat::from(omega, n, l);
  } else {
    Rng rng(o.seed);
    om = o.test_matrix == RNMF_TEST_UNIFORM ? uniform_matrix(n, l, rng) : gaussian_matrix(n, l, rng);
  }
  auto block = [&](Index c0, Index w) {  // read_columns(c0, w) + the finite check (:86-91)
    Mat b(m, w);
    for (Index i = 0; i < m; ++i)
      for (Index j = 0; j < w; ++j) b(i, j) = a(i, c0 + j);
    if (!all_finite(b))
      throw DataError("rqb_streaming: non-finite values in columns [" + std::to_string(c0) + ", " +
                      std::to_string(c0 + w) + ")");
    return b;
  };
  auto rows_of = [&](const Mat& x, Index r0, Index cnt) {
    Mat s(cnt, x.c);
    for (Index i = 0; i < cnt; ++i)
      for (Index j = 0; j < x.c; ++j) s(i, j) = x(r0 + i, j);
    return s;
  };
  auto add_to = [](Mat& y, const Mat& t) {
    for (size_t e = 0; e < y.a.size(); ++e) y.a[e] += t.a[e];
  };
  Mat y(m, l);
  for (Index c0 = 0; c0 < n; c0 += bs) {
    const Index w = std::min(bs, n - c0);
    add_to(y, matmul(block(c0, w), rows_of(om, c0, w)));  // :95-97
  }
  for (Index it = 0; it < o.power_iterations; ++it) {  // :99-105
    const Mat q = economic_qr(y).q;
    y = Mat(m, l);
    for (Index c0 = 0; c0 < n; c0 += bs) {
      const Index w = std::min(bs, n - c0);
      const Mat b = block(c0, w);
      add_to(y, matmul(b, matmul_tn(b, q)));
    }
  }
  SketchResult out;
  out.q = economic_qr(y).q;  // :108
  out.b = Mat(l, n);
  for (Index c0 = 0; c0 < n; c0 += bs) {  // :109-113
    const Index w = std::min(bs, n - c0);
    const Mat bb = matmul_tn(out.q, block(c0, w));
    for (Index i = 0; i < l; ++i)
      for (Index j = 0; j < w; ++j) out.b(i, c0 + j) = bb(i, j);
  }
  return out;
}

// ---------------------------------------------------------------------------------------------
// Options / helpers: p/include/rnmf/hals.hpp:15-38,101-125 and p/src/hals.cpp:17-124.
static constexpr double kDivisionFloor = 1e-12;  // hals.hpp:67
static constexpr uint64_t kShuffleStream = 1, kReseedStream = 2, kSketchStream = 3;

static void check_nonnegative_finite(const Mat& x) {  // hals.cpp:17-34
  for (Index i = 0; i < x.r; ++i)
    for (Index j = 0; j < x.c; ++j)
      if (!std::isfinite(x(i, j)))
        throw DataError("input contains non-finite entries at (" + std::to_string(i) + "," +
                        std::to_string(j) + ")");
  for (Index i = 0; i < x.r; ++i)
    for (Index j = 0; j < x.c; ++j)
      if (x(i, j) < 0.0)
        throw DataError("input contains negative entries at (" + std::to_string(i) + "," +
                        std::to_string(j) + ")");
}

static void validate_solver_options(const Mat& x, const rnmf_solver_options& o) {  // hals.cpp:36-53
  check_nonnegative_finite(x);
  const Index bound = std::min(x.r, x.c);
  if (o.rank < 1 || o.rank > bound)
    throw ParameterError("rank " + std::to_string(o.rank) + " out of range [1, " +
                         std::to_string(bound) + "] for a " + shape_string(x) + " input");
  if (o.max_iter < 0) throw ParameterError("max_iter must be nonnegative");
  if (!(o.tol > 0.0)) throw ParameterError("tol must be positive");
  if (o.reg.alpha_w < 0.0 || o.reg.alpha_h < 0.0 || o.reg.beta_w < 0.0 || o.reg.beta_h < 0.0)
    throw ParameterError("regularization strengths must be nonnegative");
  if (o.trace_full_every < 1) throw ParameterError("trace_full_every must be at least 1");
  if (o.oversampling < 0 || o.power_iterations < 0)
    throw ParameterError("oversampling and power iterations must be nonnegative");
}

static double projected_sq_norm(const Mat& grad, const Mat& at) {  // hals.cpp:55-65
  double sum = 0.0;
  for (Index i = 0; i < grad.size(); ++i) {
    const double g = grad.a[static_cast<size_t>(i)];
    const double gi = at.a[static_cast<size_t>(i)] > 0.0 ? g : std::min(0.0, g);
    sum += gi * gi;
  }
  return sum;
}

// clamped_col_update: hals.cpp:67-73 (w.col(j) <- [w(:,j) + (t_j - w v_j - a w(:,j) - b)/d]_+)
static void clamped_col_update(Mat& w, Index j, const std::vector<double>& t_j,
                               const std::vector<double>& v_j, double d, double alpha,
                               double beta) {
  const double denom = std::max(d + alpha, kDivisionFloor);
  std::vector<double> num(static_cast<size_t>(w.r));
  for (Index i = 0; i < w.r; ++i) {
    double wv = 0.0;
    for (Index c = 0; c < w.c; ++c) wv += w(i, c) * v_j[static_cast<size_t>(c)];
    num[static_cast<size_t>(i)] = t_j[static_cast<size_t>(i)] - wv - alpha * w(i, j);
    if (beta != 0.0) num[static_cast<size_t>(i)] -= beta;
  }
  for (Index i = 0; i < w.r; ++i) w(i, j) = std::max(w(i, j) + num[static_cast<size_t>(i)] / denom, 0.0);
}

// clamped_row_update: hals.cpp:75-81 (h.row(j) <- [h(j,:) + (r_j^T - s_j^T h - a h(j,:) - b)/d]_+)
static void clamped_row_update(Mat& h, Index j, const double* r_j, Index r_stride,
                               const double* s_j, Index s_stride, double d, double alpha,
                               double beta) {
  const double denom = std::max(d + alpha, kDivisionFloor);
  const Index k = h.r, n = h.c;
  std::vector<double> num(static_cast<size_t>(n));
  for (Index c = 0; c < n; ++c) num[static_cast<size_t>(c)] = r_j[c * r_stride];
  for (Index i = 0; i < k; ++i) {
    const double s = s_j[i * s_stride];
    const double* hi = h.row(i);
    for (Index c = 0; c < n; ++c) num[static_cast<size_t>(c)] -= s * hi[c];
  }
  double* hj = h.row(j);
  for (Index c = 0; c < n; ++c) {
    double v = num[static_cast<size_t>(c)] - alpha * hj[c];
    if (beta != 0.0) v -= beta;
    num[static_cast<size_t>(c)] = v;
  }
  for (Index c = 0; c < n; ++c) hj[c] = std::max(0.0, hj[c] + num[static_cast<size_t>(c)] / denom);
}

static std::vector<Index> sweep_order(Index k, int order, Rng& shuffle_rng) {  // hals.cpp:83-94
  std::vector<Index> idx(static_cast<size_t>(k));
  std::iota(idx.begin(), idx.end(), Index{0});
  if (order == RNMF_ORDER_SHUFFLED) {
    for (Index i = k - 1; i > 0; --i) {
      const Index j = Index(shuffle_rng.next_u64() % uint64_t(i + 1));
      std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(j)]);
    }
  }
  return idx;
}

static void reseed_dead_components(Mat& w, Mat& h, Rng& rng) {  // hals.cpp:96-105
  for (Index j = 0; j < w.c; ++j) {
    double mx = -std::numeric_limits<double>::infinity();
    for (Index i = 0; i < w.r; ++i) mx = std::max(mx, w(i, j));
    if (mx <= 0.0)
      for (Index i = 0; i < w.r; ++i) w(i, j) = rng.uniform() * 1e-4;
    double mh = -std::numeric_limits<double>::infinity();
    for (Index i = 0; i < h.c; ++i) mh = std::max(mh, h(j, i));
    if (mh <= 0.0)
      for (Index i = 0; i < h.c; ++i) h(j, i) = rng.uniform() * 1e-4;
  }
}

struct FactorPair {
  Mat w, h;
};

static double mean(const Mat& x) {
  double s = 0.0;
  for (double v : x.a) s += v;
  return s / double(x.size());
}

// random_init: hals.cpp:118-124, with optional unscaled draws replacing the two uniform_matrix
// calls (W first, then H).
static FactorPair random_init(const Mat& x, Index rank, Rng& rng, const double* w0,
                              const double* h0) {
  const double scale = std::sqrt(mean(x) / double(rank));
  FactorPair f;
  f.w = w0 ? Mat::from(w0, x.r, rank) : uniform_matrix(x.r, rank, rng);
  f.h = h0 ? Mat::from(h0, rank, x.c) : uniform_matrix(rank, x.c, rng);
  for (auto& v : f.w.a) v *= scale;
  for (auto& v : f.h.a) v *= scale;
  return f;
}

// ---- small symmetric eigen / SVD helper for NNDSVD (BDCSVD stand-in, hals.cpp:138) ----------
// Thin SVD of B (l x n, l <= n) by a cyclic one-sided Jacobi on B^T (n x l).  Returns U (l x l),
// singular values (l), V (n x l), sorted descending.  Signs are arbitrary; NNDSVD folds them.
static void jacobi_svd(const Mat& b, Mat& u, std::vector<double>& sv, Mat& v) {
  const Index l = b.r, n = b.c;
  Mat A = transpose(b);  // n x l, columns are rotated until orthogonal
  Mat V(l, l);
  for (Index i = 0; i < l; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (Index p = 0; p < l; ++p)
      for (Index q = p + 1; q < l; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (Index i = 0; i < n; ++i) {
          const double ap = A(i, p), aq = A(i, q);
          alpha += ap * ap;
          beta += aq * aq;
          gamma += ap * aq;
        }
        if (gamma == 0.0) continue;
        const double conv = std::fabs(gamma) / std::sqrt(alpha * beta);
        off = std::max(off, conv);
        if (conv < 1e-15) continue;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (Index i = 0; i < n; ++i) {
          const double ap = A(i, p), aq = A(i, q);
          A(i, p) = c * ap - s * aq;
          A(i, q) = s * ap + c * aq;
        }
        for (Index i = 0; i < l; ++i) {
          const double vp = V(i, p), vq = V(i, q);
          V(i, p) = c * vp - s * vq;
          V(i, q) = s * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> norms(static_cast<size_t>(l));
  for (Index j = 0; j < l; ++j) {
    double s = 0;
    for (Index i = 0; i < n; ++i) s += A(i, j) * A(i, j);
    norms[static_cast<size_t>(j)] = std::sqrt(s);
  }
  std::vector<Index> ord(static_cast<size_t>(l));
  std::iota(ord.begin(), ord.end(), Index{0});
  std::stable_sort(ord.begin(), ord.end(),
                   [&](Index x, Index y) { return norms[static_cast<size_t>(x)] > norms[static_cast<size_t>(y)]; });
  // B = V Sigma U_A^T  ->  left singular vectors of B are columns of V, right are A/sigma.
  u = Mat(l, l);
  v = Mat(n, l);
  sv.assign(static_cast<size_t>(l), 0.0);
  for (Index jj = 0; jj < l; ++jj) {
    const Index j = ord[static_cast<size_t>(jj)];
    sv[static_cast<size_t>(jj)] = norms[static_cast<size_t>(j)];
    for (Index i = 0; i < l; ++i) u(i, jj) = V(i, j);
    const double inv = norms[static_cast<size_t>(j)] > 0 ? 1.0 / norms[static_cast<size_t>(j)] : 0.0;
    for (Index i = 0; i < n; ++i) v(i, jj) = A(i, j) * inv;
  }
}

// nndsvd_init: hals.cpp:129-170.
static FactorPair nndsvd_init(const Mat& x, Index rank, Rng& rng) {
  SketchOptions so;
  so.target_rank = rank;
  so.oversampling = std::min<Index>(20, std::min(x.r, x.c) - rank);
  so.power_iterations = 2;
  so.test_matrix = RNMF_TEST_UNIFORM;
  so.seed = rng.next_u64();
  const SketchResult s = rqb(x, so, nullptr);
  Mat ub, vb;
  std::vector<double> sv;
  jacobi_svd(s.b, ub, sv, vb);
  Mat ubk(ub.r, rank);
  for (Index i = 0; i < ub.r; ++i)
    for (Index j = 0; j < rank; ++j) ubk(i, j) = ub(i, j);
  const Mat u = matmul(s.q, ubk);  // m x rank
  FactorPair f;
  f.w = Mat(x.r, rank);
  f.h = Mat(rank, x.c);
  const double s0 = std::sqrt(sv[0]);
  for (Index i = 0; i < x.r; ++i) f.w(i, 0) = s0 * std::fabs(u(i, 0));
  for (Index c = 0; c < x.c; ++c) f.h(0, c) = s0 * std::fabs(vb(c, 0));
  for (Index j = 1; j < rank; ++j) {
    std::vector<double> up(static_cast<size_t>(x.r)), un(static_cast<size_t>(x.r)), vp(static_cast<size_t>(x.c)), vn(static_cast<size_t>(x.c));
    double nup = 0, nun = 0, nvp = 0, nvn = 0;
    for (Index i = 0; i < x.r; ++i) {
      up[static_cast<size_t>(i)] = std::max(u(i, j), 0.0);
      un[static_cast<size_t>(i)] = std::max(-u(i, j), 0.0);
      nup += up[static_cast<size_t>(i)] * up[static_cast<size_t>(i)];
      nun += un[static_cast<size_t>(i)] * un[static_cast<size_t>(i)];
    }
    for (Index c = 0; c < x.c; ++c) {
      vp[static_cast<size_t>(c)] = std::max(vb(c, j), 0.0);
      vn[static_cast<size_t>(c)] = std::max(-vb(c, j), 0.0);
      nvp += vp[static_cast<size_t>(c)] * vp[static_cast<size_t>(c)];
      nvn += vn[static_cast<size_t>(c)] * vn[static_cast<size_t>(c)];
    }
    nup = std::sqrt(nup), nun = std::sqrt(nun), nvp = std::sqrt(nvp), nvn = std::sqrt(nvn);
    const double mp = nup * nvp, mn = nun * nvn;
    if (std::max(mp, mn) <= 0.0) continue;
    const bool pos = mp >= mn;
    const double mass = std::max(mp, mn);
    const double scale = std::sqrt(sv[static_cast<size_t>(j)] * mass);
    const double un_ = pos ? nup : nun, vn_ = pos ? nvp : nvn;
    for (Index i = 0; i < x.r; ++i) f.w(i, j) = (scale / un_) * (pos ? up[static_cast<size_t>(i)] : un[static_cast<size_t>(i)]);
    for (Index c = 0; c < x.c; ++c) f.h(j, c) = (scale / vn_) * (pos ? vp[static_cast<size_t>(c)] : vn[static_cast<size_t>(c)]);
  }
  const double fill = mean(x) / 100.0;
  for (auto& v : f.w.a)
    if (v <= 0.0) v = fill;
  for (auto& v : f.h.a)
    if (v <= 0.0) v = fill;
  return f;
}

// init_factors: hals.cpp:231-239.
static FactorPair init_factors(const Mat& x, Index rank, int scheme, Rng& rng,
                               const double* w0 = nullptr, const double* h0 = nullptr) {
  check_nonnegative_finite(x);
  const Index bound = std::min(x.r, x.c);
  if (rank < 1 || rank > bound)
    throw ParameterError("init_factors: rank " + std::to_string(rank) + " out of range [1, " +
                         std::to_string(bound) + "]");
  if (scheme == RNMF_INIT_RANDOM) return random_init(x, rank, rng, w0, h0);
  if (w0 || h0) throw ParameterError("init overrides require InitScheme::Random");
  return nndsvd_init(x, rank, rng);
}

static void check_factor_shapes(const Mat& x, const Mat& w, const Mat& h, const char* who) {
  if (w.r != x.r || h.c != x.c || w.c != h.r)
    throw ShapeError(std::string(who) + ": inconsistent shapes X=" + shape_string(x) +
                     ", W=" + shape_string(w) + ", H=" + shape_string(h));
}

// Deterministic HALS (hals.cpp:172-323) — kept in the oracle for the reference's reduction
// tests (identity basis, complete basis, tracking); not on the GPU hot path.
static void hals_w_phase(const Mat& x, Mat& w, const Mat& h, const rnmf_reg_config& reg) {
  const Mat xht = matmul_nt(x, h);  // m x k
  const Mat hht = matmul_nt(h, h);  // k x k
  std::vector<double> tj(static_cast<size_t>(w.r)), vj(static_cast<size_t>(w.c));
  for (Index j = 0; j < w.c; ++j) {
    for (Index i = 0; i < w.r; ++i) tj[static_cast<size_t>(i)] = xht(i, j);
    for (Index i = 0; i < w.c; ++i) vj[static_cast<size_t>(i)] = hht(i, j);
    clamped_col_update(w, j, tj, vj, hht(j, j), reg.alpha_w, reg.beta_w);
  }
}
static void hals_h_phase(const Mat& x, const Mat& w, Mat& h, const rnmf_reg_config& reg,
                         Mat* xtw_out, Mat* wtw_out) {
  Mat xtw = matmul_tn(x, w);  // n x k
  Mat wtw = matmul_tn(w, w);  // k x k
  for (Index j = 0; j < h.r; ++j)
    clamped_row_update(h, j, &xtw(0, j), xtw.c, &wtw(0, j), wtw.c, wtw(j, j), reg.alpha_h,
                       reg.beta_h);
  if (xtw_out) *xtw_out = std::move(xtw);
  if (wtw_out) *wtw_out = std::move(wtw);
}
static void hals_w_component(const Mat& x, Mat& w, const Mat& h, const rnmf_reg_config& reg,
                             Index j) {
  std::vector<double> tj(static_cast<size_t>(x.r), 0.0), vj(static_cast<size_t>(h.r), 0.0);
  for (Index i = 0; i < x.r; ++i) {
    double s = 0;
    for (Index c = 0; c < x.c; ++c) s += x(i, c) * h(j, c);
    tj[static_cast<size_t>(i)] = s;
  }
  for (Index i = 0; i < h.r; ++i) {
    double s = 0;
    for (Index c = 0; c < x.c; ++c) s += h(i, c) * h(j, c);
    vj[static_cast<size_t>(i)] = s;
  }
  clamped_col_update(w, j, tj, vj, vj[static_cast<size_t>(j)], reg.alpha_w, reg.beta_w);
}
static void hals_h_component(const Mat& x, const Mat& w, Mat& h, const rnmf_reg_config& reg,
                             Index j) {
  std::vector<double> rj(static_cast<size_t>(x.c), 0.0), sj(static_cast<size_t>(w.c), 0.0);
  for (Index i = 0; i < x.r; ++i)
    for (Index c = 0; c < x.c; ++c) rj[static_cast<size_t>(c)] += x(i, c) * w(i, j);
  for (Index t = 0; t < w.c; ++t) {
    double s = 0;
    for (Index i = 0; i < w.r; ++i) s += w(i, t) * w(i, j);
    sj[static_cast<size_t>(t)] = s;
  }
  clamped_row_update(h, j, rj.data(), 1, sj.data(), 1, sj[static_cast<size_t>(j)], reg.alpha_h, reg.beta_h);
}

struct SweepScratch {
  Mat xtw, wtw;
  bool valid = false;
};

static SweepScratch run_sweep(const Mat& x, Mat& w, Mat& h, const rnmf_solver_options& o,
                              Rng& shuffle_rng) {
  SweepScratch s;
  if (o.order == RNMF_ORDER_GROUPED) {
    hals_w_phase(x, w, h, o.reg);
    hals_h_phase(x, w, h, o.reg, &s.xtw, &s.wtw);
    s.valid = true;
  } else {
    for (Index j : sweep_order(o.rank, o.order, shuffle_rng)) {
      hals_w_component(x, w, h, o.reg, j);
      hals_h_component(x, w, h, o.reg, j);
    }
  }
  return s;
}

// Full-space residual statistics, streamed over row blocks (no m x n temporary):
// objective = ||X - WH||^2, grad_w = -2 (X - WH) H^T, grad_h = -2 W^T (X - WH).
static void full_space(const Mat& x, const Mat& w, const Mat& h, double* obj, Mat* grad_w,
                       Mat* grad_h) {
  const Index m = x.r, n = x.c, k = w.c;
  const Index RB = 256;
  const Index nblocks = (m + RB - 1) / RB;
  std::vector<double> obj_part(static_cast<size_t>(nblocks), 0.0);
  std::vector<Mat> gh_part(static_cast<size_t>(nblocks));
  if (grad_w) *grad_w = Mat(m, k);
  parallel_ranges(nblocks, [&](Index b0, Index b1) {
  for (Index bidx = b0; bidx < b1; ++bidx) {
    const Index r0 = bidx * RB, r1 = std::min(m, r0 + RB);
    std::vector<double> resid(static_cast<size_t>(n));
    Mat gh(k, n);
    double o = 0.0;
    for (Index i = r0; i < r1; ++i) {
      const double* xi = x.row(i);
      const double* wi = w.row(i);
      for (Index c = 0; c < n; ++c) resid[static_cast<size_t>(c)] = xi[c];
      for (Index t = 0; t < k; ++t) {
        const double wt = wi[t];
        const double* ht = h.row(t);
        for (Index c = 0; c < n; ++c) resid[static_cast<size_t>(c)] -= wt * ht[c];
      }
      for (Index c = 0; c < n; ++c) o += resid[static_cast<size_t>(c)] * resid[static_cast<size_t>(c)];
      if (grad_w) {
        for (Index t = 0; t < k; ++t) {
          const double* ht = h.row(t);
          double s = 0.0;
          for (Index c = 0; c < n; ++c) s += resid[static_cast<size_t>(c)] * ht[c];
          (*grad_w)(i, t) = -2.0 * s;
        }
      }
      if (grad_h) {
        for (Index t = 0; t < k; ++t) {
          const double wt = wi[t];
          double* gt = gh.row(t);
          for (Index c = 0; c < n; ++c) gt[c] += wt * resid[static_cast<size_t>(c)];
        }
      }
    }
    obj_part[static_cast<size_t>(bidx)] = o;
    if (grad_h) gh_part[static_cast<size_t>(bidx)] = std::move(gh);
  }
  }, 1);
  double total = 0.0;
  for (double v : obj_part) total += v;
  *obj = total;
  if (grad_h) {
    *grad_h = Mat(k, n);
    for (Index bidx = 0; bidx < nblocks; ++bidx)
      for (Index i = 0; i < k * n; ++i) grad_h->a[static_cast<size_t>(i)] += gh_part[static_cast<size_t>(bidx)].a[static_cast<size_t>(i)];
    for (auto& v : grad_h->a) v *= -2.0;
  }
}

struct FitResult {
  FactorPair f;
  std::vector<rnmf_trace_record> trace;
};

static FitResult hals_fit(const Mat& x, const rnmf_solver_options& o) {  // hals.cpp:268-323
  validate_solver_options(x, o);
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&t0] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  Rng init_rng(o.seed);
  FactorPair f = init_factors(x, o.rank, o.init, init_rng);
  Rng shuffle_rng = Rng(o.seed).split(kShuffleStream);
  Rng reseed_rng = Rng(o.seed).split(kReseedStream);
  const double x_norm = std::sqrt(squared_norm(x));
  FitResult out;
  auto record = [&](Index iter, const SweepScratch* scratch) {
    rnmf_trace_record r{};
    r.iter = iter;
    Mat gw, gh;
    double obj = 0;
    full_space(x, f.w, f.h, &obj, &gw, &gh);
    r.objective = obj;
    r.rel_err = x_norm > 0.0 ? std::sqrt(obj) / x_norm : 0.0;
    if (scratch && scratch->valid) {  // grad_h = 2 (W^T W H - (X^T W)^T)
      Mat wtwh = matmul(scratch->wtw, f.h);
      for (Index j = 0; j < f.h.r; ++j)
        for (Index c = 0; c < f.h.c; ++c) gh(j, c) = 2.0 * (wtwh(j, c) - scratch->xtw(c, j));
    }
    r.pgrad = projected_sq_norm(gw, f.w) + projected_sq_norm(gh, f.h);
    r.pgrad_full = r.pgrad;
    r.objective_compressed = r.objective;
    r.elapsed_s = elapsed();
    out.trace.push_back(r);
  };
  record(0, nullptr);
  const double pgrad0 = out.trace.front().pgrad;
  const bool stationary = o.stopping == RNMF_STOP_PROJECTED_GRADIENT && !(pgrad0 > 0.0);
  for (Index iter = 1; iter <= o.max_iter && !stationary; ++iter) {
    SweepScratch scratch = run_sweep(x, f.w, f.h, o, shuffle_rng);
    if (o.reseed_dead) {
      reseed_dead_components(f.w, f.h, reseed_rng);
      scratch.valid = false;
    }
    record(iter, &scratch);
    const rnmf_trace_record& last = out.trace.back();
    if (o.stopping == RNMF_STOP_PROJECTED_GRADIENT) {
      if (last.pgrad < o.tol * pgrad0) break;
    } else if (last.objective < o.tol) {
      break;
    }
  }
  out.f = std::move(f);
  return out;
}

// ---------------------------------------------------------------------------------------------
// Randomized HALS: p/src/rhals.cpp.
struct CompressedProblem {  // rhals.hpp:11-17
  Mat q, b, wt, w, h;
};

static void check_problem_shapes(const CompressedProblem& cp, const char* who) {  // rhals.cpp:11-21
  const bool ok = cp.q.r == cp.w.r && cp.q.c == cp.b.r && cp.wt.r == cp.q.c &&
                  cp.wt.c == cp.w.c && cp.h.r == cp.w.c && cp.h.c == cp.b.c;
  if (!ok)
    throw ShapeError(std::string(who) + ": inconsistent compressed problem, Q=" +
                     shape_string(cp.q) + ", B=" + shape_string(cp.b) + ", W~=" +
                     shape_string(cp.wt) + ", W=" + shape_string(cp.w) + ", H=" +
                     shape_string(cp.h));
}

// rhals_w_component: rhals.cpp:23-32.
static void rhals_w_component(CompressedProblem& cp, Index j, const double* t_j, Index t_stride,
                              const double* v_j, Index v_stride, double d,
                              const rnmf_reg_config& reg) {
  const Index l = cp.wt.r, k = cp.wt.c, m = cp.q.r;
  const double denom = std::max(d + reg.alpha_w, kDivisionFloor);
  std::vector<double> step(static_cast<size_t>(l));
  for (Index i = 0; i < l; ++i) {
    double wv = 0.0;
    for (Index c = 0; c < k; ++c) wv += cp.wt(i, c) * v_j[c * v_stride];
    step[static_cast<size_t>(i)] = (t_j[i * t_stride] - wv - reg.alpha_w * cp.wt(i, j)) / denom;
  }
  for (Index i = 0; i < l; ++i) cp.wt(i, j) += step[static_cast<size_t>(i)];
  const double shift = reg.beta_w != 0.0 ? reg.beta_w / denom : 0.0;
  std::vector<double> col(static_cast<size_t>(l));
  for (Index i = 0; i < l; ++i) col[static_cast<size_t>(i)] = cp.wt(i, j);
  for (Index r = 0; r < m; ++r) {
    const double* qr = cp.q.row(r);
    double lifted = 0.0;
    for (Index i = 0; i < l; ++i) lifted += qr[i] * col[static_cast<size_t>(i)];
    if (reg.beta_w != 0.0) lifted -= shift;
    cp.w(r, j) = std::max(lifted, 0.0);
  }
  std::vector<double> acc(static_cast<size_t>(l), 0.0);
  for (Index r = 0; r < m; ++r) {
    const double* qr = cp.q.row(r);
    const double wr = cp.w(r, j);
    for (Index i = 0; i < l; ++i) acc[static_cast<size_t>(i)] += qr[i] * wr;
  }
  for (Index i = 0; i < l; ++i) cp.wt(i, j) = acc[static_cast<size_t>(i)];
}

static double col_sq_norm(const Mat& w, Index j) {
  double s = 0.0;
  for (Index i = 0; i < w.r; ++i) s += w(i, j) * w(i, j);
  return s;
}

// rhals_w_component_fresh / rhals_h_component_fresh: rhals.cpp:34-45.
static void rhals_w_component_fresh(CompressedProblem& cp, const rnmf_reg_config& reg, Index j) {
  const Index l = cp.b.r, n = cp.b.c, k = cp.h.r;
  std::vector<double> t(static_cast<size_t>(l), 0.0), v(static_cast<size_t>(k), 0.0);
  for (Index i = 0; i < l; ++i) {
    double s = 0;
    for (Index c = 0; c < n; ++c) s += cp.b(i, c) * cp.h(j, c);
    t[static_cast<size_t>(i)] = s;
  }
  for (Index i = 0; i < k; ++i) {
    double s = 0;
    for (Index c = 0; c < n; ++c) s += cp.h(i, c) * cp.h(j, c);
    v[static_cast<size_t>(i)] = s;
  }
  rhals_w_component(cp, j, t.data(), 1, v.data(), 1, v[static_cast<size_t>(j)], reg);
}
static void rhals_h_component_fresh(CompressedProblem& cp, const rnmf_reg_config& reg, Index j) {
  const Index l = cp.b.r, n = cp.b.c, k = cp.wt.c;
  std::vector<double> r(static_cast<size_t>(n), 0.0), s(static_cast<size_t>(k), 0.0);
  for (Index i = 0; i < l; ++i)
    for (Index c = 0; c < n; ++c) r[static_cast<size_t>(c)] += cp.b(i, c) * cp.wt(i, j);
  for (Index t = 0; t < k; ++t) {
    double acc = 0;
    for (Index i = 0; i < l; ++i) acc += cp.wt(i, t) * cp.wt(i, j);
    s[static_cast<size_t>(t)] = acc;
  }
  clamped_row_update(cp.h, j, r.data(), 1, s.data(), 1, col_sq_norm(cp.w, j), reg.alpha_h,
                     reg.beta_h);
}

// rhals_h_phase: rhals.cpp:49-58.
static void rhals_h_phase(CompressedProblem& cp, const rnmf_reg_config& reg, Mat* r_out,
                          Mat* st_out) {
  Mat r = matmul_tn(cp.b, cp.wt);    // n x k
  Mat st = matmul_tn(cp.wt, cp.wt);  // k x k
  for (Index j = 0; j < cp.h.r; ++j)
    clamped_row_update(cp.h, j, &r(0, j), r.c, &st(0, j), st.c, col_sq_norm(cp.w, j),
                       reg.alpha_h, reg.beta_h);
  if (r_out) *r_out = std::move(r);
  if (st_out) *st_out = std::move(st);
}

// rhals_update_W: rhals.cpp:107-114.
static void rhals_update_W(CompressedProblem& cp, const rnmf_reg_config& reg) {
  check_problem_shapes(cp, "rhals_update_W");
  const Mat t = matmul_nt(cp.b, cp.h);  // l x k
  const Mat v = matmul_nt(cp.h, cp.h);  // k x k
  for (Index j = 0; j < cp.w.c; ++j)
    rhals_w_component(cp, j, t.row(0) + j, t.c, v.row(0) + j, v.c, v(j, j), reg);
}
static void rhals_update_H(CompressedProblem& cp, const rnmf_reg_config& reg) {
  check_problem_shapes(cp, "rhals_update_H");
  rhals_h_phase(cp, reg, nullptr, nullptr);
}

struct RhalsScratch {
  Mat r, st;
  bool valid = false;
};

static RhalsScratch run_rhals_sweep(CompressedProblem& cp, const rnmf_solver_options& o,
                                    Rng& shuffle_rng) {  // rhals.cpp:66-80
  RhalsScratch s;
  if (o.order == RNMF_ORDER_GROUPED) {
    rhals_update_W(cp, o.reg);
    rhals_h_phase(cp, o.reg, &s.r, &s.st);
    s.valid = true;
  } else {
    for (Index j : sweep_order(o.rank, o.order, shuffle_rng)) {
      rhals_w_component_fresh(cp, o.reg, j);
      rhals_h_component_fresh(cp, o.reg, j);
    }
  }
  return s;
}

// compress: rhals.cpp:84-105 (+ optional Omega / unscaled init overrides).
static CompressedProblem compress(const Mat& x, const rnmf_solver_options& o,
                                  const double* omega, const double* w0, const double* h0) {
  validate_solver_options(x, o);
  SketchOptions so;
  so.target_rank = o.rank;
  so.oversampling = o.oversampling;
  so.power_iterations = o.power_iterations;
  so.test_matrix = RNMF_TEST_UNIFORM;
  so.seed = Rng(o.seed).split(kSketchStream).seed();
  SketchResult s = rqb(x, so, omega);
  Rng init_rng(o.seed);
  FactorPair f = init_factors(x, o.rank, o.init, init_rng, w0, h0);
  CompressedProblem cp;
  cp.q = std::move(s.q);
  cp.b = std::move(s.b);
  cp.w = std::move(f.w);
  cp.h = std::move(f.h);
  cp.wt = matmul_tn(cp.q, cp.w);
  return cp;
}

// The trace loop of rhals_fit: rhals.cpp:128-213.
static FitResult rhals_loop(const Mat& x, CompressedProblem& cp, const rnmf_solver_options& o,
                            std::chrono::steady_clock::time_point t0) {
  auto elapsed = [&t0] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  Rng shuffle_rng = Rng(o.seed).split(kShuffleStream);
  Rng reseed_rng = Rng(o.seed).split(kReseedStream);
  const double x_norm = std::sqrt(squared_norm(x));
  FitResult out;
  double last_objective = 0.0, last_rel_err = 0.0, last_pgrad_full = 0.0;

  auto full_space_metrics = [&] {
    Mat gw, gh;
    double obj = 0;
    full_space(x, cp.w, cp.h, &obj, &gw, &gh);
    last_objective = obj;
    last_rel_err = x_norm > 0.0 ? std::sqrt(obj) / x_norm : 0.0;
    last_pgrad_full = projected_sq_norm(gw, cp.w) + projected_sq_norm(gh, cp.h);
  };
  auto compressed_pgrad = [&](const RhalsScratch* scratch, double& objc) {
    const Index l = cp.b.r, n = cp.b.c, k = cp.h.r;
    Mat residc = cp.b;
    {
      const Mat wth = matmul(cp.wt, cp.h);
      for (Index i = 0; i < l * n; ++i) residc.a[static_cast<size_t>(i)] -= wth.a[static_cast<size_t>(i)];
    }
    objc = squared_norm(residc);
    const Mat rht = matmul_nt(residc, cp.h);  // l x k
    Mat grad_w = matmul(cp.q, rht);           // m x k
    for (auto& v : grad_w.a) v *= -2.0;
    Mat grad_h(k, n);
    if (scratch && scratch->valid) {
      const Mat sh = matmul(scratch->st, cp.h);
      for (Index j = 0; j < k; ++j)
        for (Index c = 0; c < n; ++c) grad_h(j, c) = 2.0 * (sh(j, c) - scratch->r(c, j));
    } else {
      grad_h = matmul_tn(cp.wt, residc);
      for (auto& v : grad_h.a) v *= -2.0;
    }
    return projected_sq_norm(grad_w, cp.w) + projected_sq_norm(grad_h, cp.h);
  };
  auto push_record = [&](Index iter, double objc, double pgradc) {
    rnmf_trace_record r{};
    r.iter = iter;
    r.objective = last_objective;
    r.rel_err = last_rel_err;
    r.pgrad = pgradc;
    r.pgrad_full = last_pgrad_full;
    r.objective_compressed = objc;
    r.elapsed_s = elapsed();
    out.trace.push_back(r);
  };

  full_space_metrics();
  double objc0 = 0.0;
  const double pgrad0 = compressed_pgrad(nullptr, objc0);
  push_record(0, objc0, pgrad0);
  const bool stationary = o.stopping == RNMF_STOP_PROJECTED_GRADIENT && !(pgrad0 > 0.0);
  for (Index iter = 1; iter <= o.max_iter && !stationary; ++iter) {
    RhalsScratch scratch = run_rhals_sweep(cp, o, shuffle_rng);
    if (o.reseed_dead) {
      reseed_dead_components(cp.w, cp.h, reseed_rng);
      cp.wt = matmul_tn(cp.q, cp.w);
      scratch.valid = false;
    }
    double objc = 0.0;
    const double pgradc = compressed_pgrad(&scratch, objc);
    bool full = iter % o.trace_full_every == 0 || iter == o.max_iter ||
                o.stopping == RNMF_STOP_OBJECTIVE;
    if (full) full_space_metrics();
    bool stop = o.stopping == RNMF_STOP_PROJECTED_GRADIENT ? pgradc < o.tol * pgrad0
                                                           : last_objective < o.tol;
    if (stop && !full) {
      full_space_metrics();
      full = true;
    }
    push_record(iter, objc, pgradc);
    if (stop) break;
  }
  out.f.w = std::move(cp.w);
  out.f.h = std::move(cp.h);
  return out;
}

static FitResult rhals_fit(const Mat& x, const rnmf_solver_options& o, const double* omega,
                           const double* w0, const double* h0) {  // rhals.cpp:121-213
  const auto t0 = std::chrono::steady_clock::now();
  CompressedProblem cp = compress(x, o, omega, w0, h0);
  return rhals_loop(x, cp, o, t0);
}

static CompressedProblem make_cp(const rnmf_problem_shape* s, const double* q, const double* b,
                                 const double* wt, const double* w, const double* h) {
  CompressedProblem cp;
  cp.q = Mat::from(q, s->q_rows, s->q_cols);
  cp.b = Mat::from(b, s->b_rows, s->b_cols);
  cp.wt = Mat::from(wt, s->wt_rows, s->wt_cols);
  cp.w = Mat::from(w, s->w_rows, s->w_cols);
  cp.h = Mat::from(h, s->h_rows, s->h_cols);
  return cp;
}

}  // namespace orc

// =============================================================================================
// C ABI
namespace {
void put_err(char* err, size_t cap, const char* msg) {
  if (err && cap) {
    std::strncpy(err, msg, cap - 1);
    err[cap - 1] = '\0';
  }
}
template <typename F>
int guarded(char* err, size_t cap, F&& f) {
  try {
    f();
    put_err(err, cap, "");
    return RNMF_OK;
  } catch (const orc::ShapeError& e) {
    put_err(err, cap, e.what());
    return RNMF_SHAPE_ERROR;
  } catch (const orc::ParameterError& e) {
    put_err(err, cap, e.what());
    return RNMF_PARAMETER_ERROR;
  } catch (const orc::DataError& e) {
    put_err(err, cap, e.what());
    return RNMF_DATA_ERROR;
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return RNMF_CUDA_ERROR;
  }
}
void emit_trace(const orc::FitResult& r, rnmf_trace_record* trace, int64_t cap, int64_t* len) {
  if (int64_t(r.trace.size()) > cap)
    throw orc::ParameterError("trace buffer too small: need " + std::to_string(r.trace.size()) +
                              " records, have " + std::to_string(cap));
  for (size_t i = 0; i < r.trace.size(); ++i) trace[i] = r.trace[i];
  *len = int64_t(r.trace.size());
}
}  // namespace

extern "C" {

void oracle_set_threads(int threads) { orc::g_threads = threads < 1 ? 1 : threads; }

uint64_t oracle_rng_split_seed(uint64_t seed, uint64_t stream) {
  return orc::Rng(seed).split(stream).seed();
}
void oracle_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  orc::Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void oracle_rng_uniform(uint64_t seed, int64_t count, double* out) {
  orc::Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.uniform();
}
void oracle_rng_gaussian(uint64_t seed, int64_t count, double* out) {
  orc::Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.gaussian();
}
int oracle_uniform_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out, char* err,
                          size_t cap) {
  return guarded(err, cap, [&] {
    orc::Rng r(seed);
    orc::uniform_matrix(rows, cols, r).to(out);
  });
}
int oracle_gaussian_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out, char* err,
                           size_t cap) {
  return guarded(err, cap, [&] {
    orc::Rng r(seed);
    orc::gaussian_matrix(rows, cols, r).to(out);
  });
}
int oracle_economic_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r,
                       char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto res = orc::economic_qr(orc::Mat::from(a, rows, cols));
    res.q.to(q);
    res.r.to(r);
  });
}
int oracle_synth_lowrank(int64_t rows, int64_t cols, int64_t rank, double noise, uint64_t seed,
                         double* out, char* err, size_t cap) {
  return guarded(err, cap, [&] { orc::synth_lowrank(rows, cols, rank, noise, seed).to(out); });
}
int oracle_sketch_width(int64_t rows, int64_t cols, int64_t target_rank, int64_t oversampling,
                        int64_t power_iterations, int64_t block_size, int64_t* l_out, char* err,
                        size_t cap) {
  return guarded(err, cap, [&] {
    orc::SketchOptions so;
    so.target_rank = target_rank;
    so.oversampling = oversampling;
    so.power_iterations = power_iterations;
    so.block_size = block_size;
    *l_out = orc::sketch_width(rows, cols, so);
  });
}
int oracle_rqb(const double* a, int64_t m, int64_t n, int64_t target_rank, int64_t oversampling,
               int64_t power_iterations, int test_matrix, uint64_t seed, const double* omega,
               double* q_out, double* b_out, int64_t* l_out, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    orc::SketchOptions so;
    so.target_rank = target_rank;
    so.oversampling = oversampling;
    so.power_iterations = power_iterations;
    so.test_matrix = test_matrix;
    so.seed = seed;
    const orc::Mat x = orc::Mat::from(a, m, n);
    *l_out = orc::sketch_width(m, n, so);
    if (!q_out && !b_out) return;
    auto s = orc::rqb(x, so, omega);
    if (q_out) s.q.to(q_out);
    if (b_out) s.b.to(b_out);
  });
}
int oracle_rqb_streaming(const double* a, int64_t m, int64_t n, int64_t target_rank, int64_t oversampling,
                         int64_t power_iterations, int test_matrix, int64_t block_size, uint64_t seed,
                         const double* omega, double* q_out, double* b_out, int64_t* l_out, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    orc::SketchOptions so;
    so.target_rank = target_rank;
    so.oversampling = oversampling;
    so.power_iterations = power_iterations;
    so.test_matrix = test_matrix;
    so.block_size = block_size;
    so.seed = seed;
    *l_out = orc::sketch_width(m, n, so);
    if (!q_out && !b_out) return;
    auto s = orc::rqb_streaming(orc::Mat::from(a, m, n), so, omega);
    if (q_out) s.q.to(q_out);
    if (b_out) s.b.to(b_out);
  });
}
int oracle_init_factors(const double* x, int64_t m, int64_t n, int64_t rank, int scheme,
                        uint64_t seed, double* w_out, double* h_out, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    orc::Rng rng(seed);
    auto f = orc::init_factors(orc::Mat::from(x, m, n), rank, scheme, rng);
    f.w.to(w_out);
    f.h.to(h_out);
  });
}
int oracle_update_W(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                    const double* h, const rnmf_reg_config* reg, double* w_out, char* err,
                    size_t cap) {
  return guarded(err, cap, [&] {
    const orc::Mat X = orc::Mat::from(x, m, n), H = orc::Mat::from(h, k, n);
    orc::Mat W = orc::Mat::from(w, m, k);
    orc::check_factor_shapes(X, W, H, "update_W");
    orc::hals_w_phase(X, W, H, *reg);
    W.to(w_out);
  });
}
int oracle_update_H(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                    const double* h, const rnmf_reg_config* reg, double* h_out, char* err,
                    size_t cap) {
  return guarded(err, cap, [&] {
    const orc::Mat X = orc::Mat::from(x, m, n), W = orc::Mat::from(w, m, k);
    orc::Mat H = orc::Mat::from(h, k, n);
    orc::check_factor_shapes(X, W, H, "update_H");
    orc::hals_h_phase(X, W, H, *reg, nullptr, nullptr);
    H.to(h_out);
  });
}
int oracle_objective(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                     const double* h, double* out, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    const orc::Mat X = orc::Mat::from(x, m, n), W = orc::Mat::from(w, m, k),
                   H = orc::Mat::from(h, k, n);
    orc::full_space(X, W, H, out, nullptr, nullptr);
  });
}
int oracle_projected_gradient_norm(const double* x, int64_t m, int64_t n, int64_t k,
                                   const double* w, const double* h, double* out, char* err,
                                   size_t cap) {
  return guarded(err, cap, [&] {
    const orc::Mat X = orc::Mat::from(x, m, n), W = orc::Mat::from(w, m, k),
                   H = orc::Mat::from(h, k, n);
    orc::Mat gw, gh;
    double obj;
    orc::full_space(X, W, H, &obj, &gw, &gh);
    *out = orc::projected_sq_norm(gw, W) + orc::projected_sq_norm(gh, H);
  });
}
int oracle_hals_fit(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                    double* w_out, double* h_out, rnmf_trace_record* trace, int64_t trace_cap,
                    int64_t* trace_len, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto r = orc::hals_fit(orc::Mat::from(x, m, n), *opts);
    emit_trace(r, trace, trace_cap, trace_len);
    r.f.w.to(w_out);
    r.f.h.to(h_out);
  });
}
int oracle_compress(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                    const double* omega, const double* w0, const double* h0, double* q_out,
                    double* b_out, double* wt_out, double* w_out, double* h_out, int64_t* l_out,
                    char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto cp = orc::compress(orc::Mat::from(x, m, n), *opts, omega, w0, h0);
    *l_out = cp.q.c;
    if (q_out) cp.q.to(q_out);
    if (b_out) cp.b.to(b_out);
    if (wt_out) cp.wt.to(wt_out);
    if (w_out) cp.w.to(w_out);
    if (h_out) cp.h.to(h_out);
  });
}
int oracle_rhals_update_W(const rnmf_problem_shape* shape, const double* q, const double* b,
                          double* wt, double* w, const double* h, const rnmf_reg_config* reg,
                          char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto cp = orc::make_cp(shape, q, b, wt, w, h);
    orc::rhals_update_W(cp, *reg);
    cp.wt.to(wt);
    cp.w.to(w);
  });
}
int oracle_rhals_update_H(const rnmf_problem_shape* shape, const double* q, const double* b,
                          const double* wt, const double* w, double* h,
                          const rnmf_reg_config* reg, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto cp = orc::make_cp(shape, q, b, wt, w, h);
    orc::rhals_update_H(cp, *reg);
    cp.h.to(h);
  });
}
int oracle_rhals_fit(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                     const double* omega, const double* w0, const double* h0, double* w_out,
                     double* h_out, rnmf_trace_record* trace, int64_t trace_cap,
                     int64_t* trace_len, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    auto r = orc::rhals_fit(orc::Mat::from(x, m, n), *opts, omega, w0, h0);
    emit_trace(r, trace, trace_cap, trace_len);
    r.f.w.to(w_out);
    r.f.h.to(h_out);
  });
}
int oracle_rhals_fit_compressed(const double* x, int64_t m, int64_t n,
                                const rnmf_solver_options* opts, const rnmf_problem_shape* shape,
                                const double* q, const double* b, double* wt, double* w,
                                double* h, rnmf_trace_record* trace, int64_t trace_cap,
                                int64_t* trace_len, char* err, size_t cap) {
  return guarded(err, cap, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    const orc::Mat X = orc::Mat::from(x, m, n);
    orc::validate_solver_options(X, *opts);
    auto cp = orc::make_cp(shape, q, b, wt, w, h);
    orc::check_problem_shapes(cp, "rhals_fit_compressed");
    if (cp.q.r != m || cp.b.c != n || cp.w.c != opts->rank)
      throw orc::ShapeError("rhals_fit_compressed: problem does not match X=" +
                            orc::shape_string(m, n));
    auto r = orc::rhals_loop(X, cp, *opts, t0);
    emit_trace(r, trace, trace_cap, trace_len);
    cp.wt.to(wt);
    r.f.w.to(w);
    r.f.h.to(h);
  });
}

}  // extern "C"
