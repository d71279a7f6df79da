// rnmf_gpu.cu — host orchestration of the B200 randomized-HALS path and its C ABI
// (include/rnmf_gpu.h).  Everything numeric runs in the sm_100a kernels of kernels_*.cu; the host
// validates arguments in the reference's order, draws the reference's random streams, sequences
// the kernels on one CUDA stream and assembles the trace.
#include "../../include/rnmf_gpu.h"
#include "common.cuh"
#include "kernels.h"
#include "tc_metrics.h"

#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is opened at run time (row-sharded contexts)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

namespace rnmf_gpu {

// ---- reference exception classes (p/include/rnmf/types.hpp:22-39) ---------------------------
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

static std::string shape_string(int64_t r, int64_t c) { return std::to_string(r) + "x" + std::to_string(c); }

// ---- the reference random stream (p/include/rnmf/types.hpp:55-102) ---------------------------
// Needed by the product itself: with no overrides, Omega and the initial factors must be the
// reference's own draws.
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
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare_ = radius * std::sin(angle);
    has_spare_ = true;
    return radius * std::cos(angle);
  }
  Rng split(uint64_t stream) const {
    uint64_t x = seed_ + 0x9e3779b97f4a7c15ULL * (stream + 1);
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return Rng(x ^ (x >> 31));
  }

 private:
  uint64_t seed_;
  std::mt19937_64 engine_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

constexpr uint64_t kSketchStream = 3;  // p/include/rnmf/hals.hpp:107
constexpr uint64_t kShuffleStream = 1;
constexpr uint64_t kReseedStream = 2;

// ---- device / pinned buffers owned by a context ----------------------------------------------
struct Buffer {
  void* p = nullptr;
  size_t bytes = 0;
};

// ---- NCCL, opened at run time (only row-sharded contexts need it) --------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // a process that already loaded NCCL (e.g. torch.distributed) shares that copy
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.AllGather || !a.CommDestroy || !a.GetErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.error.empty()) throw CudaError("NCCL: " + api.error);
  return api;
}

#define RNMF_NCCL(call)                                                                             \
  do {                                                                                              \
    const ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) throw CudaError(std::string("NCCL: ") + nccl().GetErrorString(r_) + " at " #call); \
  } while (0)

// Row sharding of one fit over `world` GPUs, one process per GPU (world == 0: not sharded).
struct ShardInfo {
  int rank = 0, world = 0;
  ncclComm_t comm = nullptr;
  unsigned char* peer[kMaxWorld] = {};  // peers' sweep sync blocks mapped by CUDA IPC (own: local)
};

}  // namespace rnmf_gpu

using namespace rnmf_gpu;

struct rnmf_gpu_context {
  ShardInfo shard;
  unsigned char* sync_block = nullptr;  // sweep-kernel sync block (kSweepSyncTotal bytes, own cudaMalloc)
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  int max_smem = 0;
  std::map<std::string, Buffer> dev;
  std::map<std::string, Buffer> pinned;
  std::vector<cudaEvent_t> event_pool;
  size_t event_next = 0;
  rnmf_stage_times last{};

  template <typename V>
  V* d(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(V);
    Buffer& b = dev[name];
    if (b.bytes < bytes) {
      if (b.p) RNMF_CUDA(cudaFree(b.p));
      b.p = nullptr;
      RNMF_CUDA(cudaMalloc(&b.p, bytes));
      b.bytes = bytes;
    }
    return static_cast<V*>(b.p);
  }
  template <typename V>
  V* h(const std::string& name, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(V);
    Buffer& b = pinned[name];
    if (b.bytes < bytes) {
      if (b.p) RNMF_CUDA(cudaFreeHost(b.p));
      b.p = nullptr;
      RNMF_CUDA(cudaMallocHost(&b.p, bytes));
      b.bytes = bytes;
    }
    return static_cast<V*>(b.p);
  }
  cudaEvent_t event() {
    if (event_next == event_pool.size()) {
      cudaEvent_t e;
      RNMF_CUDA(cudaEventCreate(&e));
      event_pool.push_back(e);
    }
    return event_pool[event_next++];
  }
};

namespace rnmf_gpu {

// ---- stage timing -----------------------------------------------------------------------------
enum Stage { kScan, kSketch, kQr, kInit, kSweeps, kMetrics, kXw, kXtw, kH2D, kD2H, kXwK, kXtwK, kNumStages };

struct Timer {
  rnmf_gpu_context* ctx;
  struct Span {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Span> spans;
  cudaEvent_t start{}, stop{};
  int64_t launches = 0;
  explicit Timer(rnmf_gpu_context* c) : ctx(c) {
    ctx->event_next = 0;
    start = ctx->event();
    RNMF_CUDA(cudaEventRecord(start, ctx->stream));
  }
  cudaEvent_t mark() {
    cudaEvent_t e = ctx->event();
    RNMF_CUDA(cudaEventRecord(e, ctx->stream));
    return e;
  }
  template <typename F>
  void span(int stage, F&& f) {
    cudaEvent_t a = mark();
    f();
    cudaEvent_t b = mark();
    spans.push_back({stage, a, b});
  }
  void finish(rnmf_stage_times& out) {
    stop = mark();
    RNMF_CUDA(cudaEventSynchronize(stop));
    double acc[kNumStages] = {};
    int64_t counts[kNumStages] = {};
    for (auto& s : spans) {
      float ms = 0.f;
      RNMF_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
      acc[s.stage] += ms;
      counts[s.stage] += 1;
    }
    float tot = 0.f;
    RNMF_CUDA(cudaEventElapsedTime(&tot, start, stop));
    out.scan_ms = acc[kScan];
    out.sketch_ms = acc[kSketch];
    out.qr_ms = acc[kQr];
    out.init_ms = acc[kInit];
    out.sweeps_ms = acc[kSweeps];
    out.metrics_ms = acc[kMetrics];
    out.h2d_ms = acc[kH2D];
    out.d2h_ms = acc[kD2H];
    out.xw_ms = acc[kXw];
    out.xtw_ms = acc[kXtw];
    out.xw_launches = counts[kXw];
    out.xtw_launches = counts[kXtw];
    out.xw_kernel_ms = acc[kXwK];
    out.xtw_kernel_ms = acc[kXtwK];
    out.total_ms = tot;
    out.kernel_launches = launches;
  }
};

// ---- small host helpers -----------------------------------------------------------------------
static void check_device_ptr(const rnmf_gpu_context* ctx, const void* p, const char* what) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess || attr.type != cudaMemoryTypeDevice ||
      attr.device != ctx->device) {
    cudaGetLastError();
    throw ParameterError(std::string(what) + ": expected device memory of GPU " + std::to_string(ctx->device));
  }
}

static void validate_options_after_data(int64_t m, int64_t n, const rnmf_solver_options& o) {
  // p/src/hals.cpp:36-53 (check_nonnegative_finite already done by the scan)
  const int64_t bound = std::min(m, n);
  if (o.rank < 1 || o.rank > bound)
    throw ParameterError("rank " + std::to_string(o.rank) + " out of range [1, " + std::to_string(bound) +
                         "] for a " + shape_string(m, n) + " input");
  if (o.max_iter < 0) throw ParameterError("max_iter must be nonnegative");
  if (!(o.tol > 0.0)) throw ParameterError("tol must be positive");
  if (o.reg.alpha_w < 0.0 || o.reg.alpha_h < 0.0 || o.reg.beta_w < 0.0 || o.reg.beta_h < 0.0)
    throw ParameterError("regularization strengths must be nonnegative");
  if (o.trace_full_every < 1) throw ParameterError("trace_full_every must be at least 1");
  if (o.oversampling < 0 || o.power_iterations < 0)
    throw ParameterError("oversampling and power iterations must be nonnegative");
}

static void check_supported(const rnmf_solver_options& o) {
  if (o.init != RNMF_INIT_RANDOM && o.init != RNMF_INIT_SVD) throw ParameterError("unknown InitScheme");
  if (o.order != RNMF_ORDER_GROUPED && o.order != RNMF_ORDER_INTERLEAVED && o.order != RNMF_ORDER_SHUFFLED)
    throw ParameterError("unknown UpdateOrder");

  if (o.math_mode != RNMF_MATH_EXACT && o.math_mode != RNMF_MATH_TF32X3 && o.math_mode != RNMF_MATH_TF32)
    throw ParameterError("math_mode must be RNMF_MATH_EXACT, RNMF_MATH_TF32X3 or RNMF_MATH_TF32");
}

// sketch_width, p/src/sketch.cpp:30-50 (block_size is fixed at its default of 1024)
static int64_t sketch_width(int64_t rows, int64_t cols, int64_t target_rank, int64_t oversampling,
                            int64_t power_iterations) {
  const int64_t bound = std::min(rows, cols);
  if (target_rank < 1 || target_rank > bound)
    throw ParameterError("sketch: target rank " + std::to_string(target_rank) + " out of range [1, " +
                         std::to_string(bound) + "] for a " + shape_string(rows, cols) + " matrix");
  if (oversampling < 0 || power_iterations < 0)
    throw ParameterError("sketch: oversampling and power iterations must be nonnegative");
  int64_t l = target_rank + oversampling;
  if (l > bound) {
    std::fprintf(stderr, "rnmf: sketch width %lld exceeds min(%lld, %lld); clamping to %lld\n", (long long)l,
                 (long long)rows, (long long)cols, (long long)bound);
    l = bound;
  }
  return l;
}

static void check_problem_shapes(const rnmf_problem_shape& s, const char* who) {  // p/src/rhals.cpp:11-21
  const bool ok = s.q_rows == s.w_rows && s.q_cols == s.b_rows && s.wt_rows == s.q_cols &&
                  s.wt_cols == s.w_cols && s.h_rows == s.w_cols && s.h_cols == s.b_cols;
  if (!ok)
    throw ShapeError(std::string(who) + ": inconsistent compressed problem, Q=" + shape_string(s.q_rows, s.q_cols) +
                     ", B=" + shape_string(s.b_rows, s.b_cols) + ", W~=" + shape_string(s.wt_rows, s.wt_cols) +
                     ", W=" + shape_string(s.w_rows, s.w_cols) + ", H=" + shape_string(s.h_rows, s.h_cols));
}

// ==============================================================================================
template <typename V>
constexpr ncclDataType_t nccl_type() {
  if constexpr (std::is_same<V, float>::value) return ncclFloat32;
  else if constexpr (std::is_same<V, double>::value) return ncclFloat64;
  else if constexpr (std::is_same<V, unsigned long long>::value) return ncclUint64;
  else return ncclInt64;
}



// dst (rows x ld, pad columns zero) <- src (rows x n, contiguous)
template <typename T>
__global__ void repitch_kernel(const T* __restrict__ src, int64_t rows, int64_t n, T* __restrict__ dst, int64_t ld) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) dst[r * ld + j] = j < n ? src[r * n + j] : T(0);
}
template <typename T>
static int launch_repitch(const T* src, int64_t rows, int64_t n, T* dst, int64_t ld, cudaStream_t st) {
  if (rows <= 0) return 0;
  repitch_kernel<T><<<int(std::min<int64_t>(rows, 148 * 16)), 256, 0, st>>>(src, rows, n, dst, ld);
  RNMF_CUDA_LAUNCH();
  return 1;
}

// ---- streaming sketch helpers (rqb_streaming) -------------------------------------------------
// bad |= 1 when the m x w column block (pitch ld) holds a non-finite value (p/src/sketch.cpp:88-91)
__global__ void block_finite_kernel(const double* __restrict__ blk, int64_t m, int64_t w, int64_t ld, int* bad) {
  int found = 0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m * w; e += int64_t(gridDim.x) * blockDim.x)
    found |= !isfinite(blk[(e / w) * ld + e % w]);
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(bad, 1);
}
// y += t (count doubles)
__global__ void add_inplace_kernel(double* __restrict__ y, const double* __restrict__ t, int64_t count) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
    y[e] += t[e];
}

// Host column reader of the streaming sketch: first, count -> m x count row-major doubles
using ColumnReadFn = std::function<void(int64_t first, int64_t count, double* dst)>;

template <typename T>
class Engine {
 public:
  Engine(rnmf_gpu_context* ctx, Timer& tm) : ctx_(ctx), st_(ctx->stream), tm_(tm) {}
  // arithmetic of the X passes (rnmf_solver_options.math_mode): TF32X3 also moves the full-space
  // metrics onto the tensor cores (metrics_tc)
  void set_math(int math_mode) { math_ = math_mode; }

  // ---- row sharding: this engine holds rows [row_off, row_off + m) of an m_total-row X --------
  bool sharded() const { return ctx_->shard.world > 0; }
  void set_rows(int64_t row_off, int64_t m_total) {
    row_off_ = row_off;
    m_total_ = m_total;
  }
  int64_t m_total() const { return sharded() ? m_total_ : m_; }
  // in-place sum (or min / max) over the GPUs of a device buffer, on the engine's stream
  template <typename V>
  void allreduce(V* buf, size_t count, ncclRedOp_t op = ncclSum) {
    if (!sharded() || count == 0) return;
    RNMF_NCCL(nccl().AllReduce(buf, buf, count, nccl_type<V>(), op, ctx_->shard.comm, st_));
  }

  // X for the X-streaming kernels: rows need a 16-byte aligned pitch (TMA, vector loads).  Device
  // input that already satisfies it is used in place (no copy); otherwise X is copied once into a
  // context buffer whose pad columns are zero (host input: the pitched H2D copy is free).
  const T* import_x(const void* src, int location, int64_t m, int64_t n) {
    constexpr int64_t vn = 16 / sizeof(T);
    m_ = m;
    n_ = n;
    if (location == RNMF_DEVICE) {
      check_device_ptr(ctx_, src, "X");
      if (n % vn == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0) {
        ldx_ = n;
        x_ = static_cast<const T*>(src);
        return x_;
      }
    }
    ldx_ = ceil_div(n, vn) * vn;
    T* dst = ctx_->d<T>("x", size_t(m) * size_t(ldx_));
    const bool padded = ldx_ != n;
    const cudaMemcpyKind kind = location == RNMF_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    auto copy = [&] {
      if (!padded) {
        RNMF_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * size_t(m) * size_t(n), kind, st_));
      } else if (location == RNMF_DEVICE) {
        tm_.launches += launch_repitch<T>(static_cast<const T*>(src), m, n, dst, ldx_, st_);
      } else {
        // host rows of n values into the padded device layout: contiguous 1-D copies of row
        // blocks through a staging buffer (a pitched 2-D copy runs ~10 % below the 1-D PCIe rate),
        // each block re-pitched on the device (pad columns written as zero)
        const int64_t rows_per = std::max<int64_t>(1, (int64_t(64) << 20) / int64_t(sizeof(T) * size_t(n)));
        T* stage = ctx_->d<T>("x.stage", size_t(std::min(rows_per, m)) * size_t(n));
        for (int64_t r0 = 0; r0 < m; r0 += rows_per) {
          const int64_t rc = std::min(rows_per, m - r0);
          RNMF_CUDA(cudaMemcpyAsync(stage, static_cast<const T*>(src) + r0 * n, sizeof(T) * size_t(rc) * size_t(n),
                                    cudaMemcpyHostToDevice, st_));
          tm_.launches += launch_repitch<T>(stage, rc, n, dst + r0 * ldx_, ldx_, st_);
        }
      }
    };
    if (location == RNMF_HOST)
      tm_.span(kH2D, copy);
    else
      copy();
    x_ = dst;
    return x_;
  }
  const T* x() const { return x_; }
  int64_t ldx() const { return ldx_; }

  // Copy a caller matrix (host or device) into a context buffer.
  T* import(const std::string& name, const void* src, int location, size_t count) {
    T* dst = ctx_->d<T>(name, count);
    if (count == 0) return dst;
    if (location == RNMF_DEVICE) {
      check_device_ptr(ctx_, src, name.c_str());
      RNMF_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, st_));
    } else {
      tm_.span(kH2D, [&] { RNMF_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, st_)); });
    }
    return dst;
  }
  void export_(void* dst, int location, const T* src, size_t count) {
    if (count == 0 || dst == nullptr) return;
    if (location == RNMF_DEVICE) {
      check_device_ptr(ctx_, dst, "output");
      RNMF_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, st_));
    } else {
      tm_.span(kD2H, [&] { RNMF_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, st_)); });
    }
  }
  // Upload host doubles converted to T (small matrices: Omega, compressed-problem inputs).
  T* upload_converted(const std::string& name, const double* src, size_t count) {
    T* hst = ctx_->h<T>(name + ".pin", count);
    for (size_t i = 0; i < count; ++i) hst[i] = T(src[i]);
    T* dst = ctx_->d<T>(name, count);
    tm_.span(kH2D, [&] { RNMF_CUDA(cudaMemcpyAsync(dst, hst, count * sizeof(T), cudaMemcpyHostToDevice, st_)); });
    return dst;
  }

  // One pass over X: data checks + sum + sum of squares.  Throws DataError like
  // check_nonnegative_finite (p/src/hals.cpp:17-34), non-finite before negative.
  void scan(bool check_negative, const char* nonfinite_msg) {
    const T* x = x_;
    const int64_t m = m_, n = ldx_;  // pad columns are zero: finite, nonnegative, sum-neutral
    auto* bad = ctx_->d<unsigned long long>("scan.bad", 2);
    auto* part = ctx_->d<double>("scan.part", 2 * scan_grid());
    auto* out = ctx_->d<double>("scan.out", 2);
    tm_.span(kScan, [&] { tm_.launches += launch_scan<T>(x, m * n, bad, part, out, st_); });
    auto* hb = ctx_->h<unsigned long long>("scan.bad.h", 2);
    auto* ho = ctx_->h<double>("scan.out.h", 2);
    RNMF_CUDA(cudaMemcpyAsync(hb, bad, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st_));
    RNMF_CUDA(cudaStreamSynchronize(st_));
    // positions as (row, column) of the whole matrix; sharded: the first offender over all GPUs
    const int64_t nn = n_ > 0 ? n_ : 1;
    for (int e = 0; e < 2; ++e)
      if (hb[e] != ~0ull) hb[e] = (uint64_t(row_off_) + hb[e] / uint64_t(n)) * uint64_t(nn) + hb[e] % uint64_t(n);
    if (sharded()) {
      RNMF_CUDA(cudaMemcpyAsync(bad, hb, 2 * sizeof(unsigned long long), cudaMemcpyHostToDevice, st_));
      allreduce(bad, 2, ncclMin);
      allreduce(out, 2);
      RNMF_CUDA(cudaMemcpyAsync(hb, bad, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st_));
    }
    RNMF_CUDA(cudaMemcpyAsync(ho, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st_));
    RNMF_CUDA(cudaStreamSynchronize(st_));
    if (hb[0] != ~0ull) {
      if (nonfinite_msg) throw DataError(nonfinite_msg);
      const int64_t i = int64_t(hb[0]) / nn, j = int64_t(hb[0]) % nn;
      throw DataError("input contains non-finite entries at (" + std::to_string(i) + "," + std::to_string(j) + ")");
    }
    if (check_negative && hb[1] != ~0ull) {
      const int64_t i = int64_t(hb[1]) / nn, j = int64_t(hb[1]) % nn;
      throw DataError("input contains negative entries at (" + std::to_string(i) + "," + std::to_string(j) + ")");
    }
    sum_ = ho[0];
    sumsq_ = ho[1];
  }

  // Y (m x c) = X S in the engine's math mode (the hals_fit W phase's X H^T, p/src/hals.cpp:173).
  // S is n x c row-major, or (s_rows) given as its c x n transpose -- H itself.
  void gemm_xs(const T* s, int c, bool s_rows, T* out) {
    const T* x = x_;
    const int64_t m = m_, n = n_, ldx = ldx_;
    if constexpr (std::is_same<T, float>::value) {
      if (math_ != RNMF_MATH_EXACT) {
        const bool x3 = math_ == RNMF_MATH_TF32X3;
        const size_t cap = size_t(tc_npad(c)) * size_t(tc_st_pitch(n));
        float* sh = ctx_->d<float>("g.st_hi", cap);
        float* sl = ctx_->d<float>("g.st_lo", cap);
        tm_.launches += s_rows ? launch_tc_prep_rows(s, c, n, sh, sl, st_) : launch_tc_prep_st(s, n, c, sh, sl, st_, x3);
        tm_.launches += launch_tc_xw(x, m, n, ldx, sh, sl, c, out, x3, ctx_->sm_count, st_);
        return;
      }
    }
    const T* sn = s;
    if (s_rows) {
      T* st = ctx_->d<T>("g.s_t", size_t(n) * c);
      tm_.launches += launch_transpose<T>(s, c, n, st, st_);
      sn = st;
    }
    if (sizeof(T) == 4) {
      T* spad = ctx_->d<T>("g.spad", size_t(xw_tma_spad_len(n, c)));
      tm_.launches += launch_xw_tma<T>(x, m, n, ldx, sn, c, out, spad, ctx_->sm_count, st_);
    } else {
      tm_.launches += launch_xw<T>(x, m, n, ldx, sn, c, out, st_);
    }
  }

  // out (n x c) = X^T S, S m x c row-major (the hals_fit H phase's X^T W, p/src/hals.cpp:184).
  void gemm_xts(const T* s, int c, T* out) {
    const T* x = x_;
    const int64_t m = m_, n = n_, ldx = ldx_;
    if constexpr (std::is_same<T, float>::value) {
      if (math_ != RNMF_MATH_EXACT) {
        const bool x3 = math_ == RNMF_MATH_TF32X3;
        const size_t cap = size_t(tc_npad(c)) * size_t(tc_st_pitch(m));
        float* sh = ctx_->d<float>("g.st_hi", cap);
        float* sl = ctx_->d<float>("g.st_lo", cap);
        const int splits = tc_xtw_splits(m, n, ctx_->sm_count);
        float* part = ctx_->d<float>("g.part", size_t(splits) * n * c);
        tm_.launches += launch_tc_prep_st(s, m, c, sh, sl, st_, x3);
        tm_.launches += launch_tc_xtw(x, m, n, ldx, sh, sl, c, part, splits, x3, ctx_->sm_count, st_);
        tm_.launches += launch_splitk_reduce<float>(part, splits, n, c, out, false, st_);
        return;
      }
    }
    if (sizeof(T) == 4) {
      const int sp = xtw_tma_splits(m, n, ctx_->sm_count);
      T* part = ctx_->d<T>("g.part2", size_t(sp) * n * c);
      T* spad = ctx_->d<T>("g.spad2", size_t(xw_tma_spad_len(m, c)));
      tm_.launches += launch_xtw_tma<T>(x, m, n, ldx, s, c, part, sp, out, false, spad, ctx_->sm_count, st_);
    } else {
      const int splits = xtw_default_splits(m, n);
      T* part = ctx_->d<T>("g.part", size_t(splits) * n * c);
      tm_.launches += launch_xtw<T>(x, m, n, ldx, s, c, part, splits, out, false, st_);
    }
  }

  // rqb, p/src/sketch.cpp:52-71 -> Q (m x l), B (l x n) in context buffers.
  // math_mode EXACT: FFMA/DFMA kernels.  TF32 / TF32X3 (fp32 X only): tcgen05 kernels; TF32X3 runs
  // every X pass as 3xTF32 (hi/lo split of both operands, fp32-accurate).
  void rqb(int l, int64_t q_iters, const T* omega_dev, int math_mode, T** q_out, T** b_out) {
    const T* x = x_;
    const int64_t m = m_, n = n_, ldx = ldx_;
    T* y = ctx_->d<T>("rqb.y", size_t(m) * l);
    T* qb = ctx_->d<T>("rqb.q", size_t(m) * l);
    T* p = ctx_->d<T>("rqb.p", size_t(n) * l);
    T* z = ctx_->d<T>("rqb.z", size_t(n) * l);
    T* b = ctx_->d<T>("rqb.b", size_t(l) * n);
    const bool tc = std::is_same<T, float>::value && math_mode != RNMF_MATH_EXACT;
    const bool x3 = math_mode == RNMF_MATH_TF32X3;
    const int splits = tc ? tc_xtw_splits(m, n, ctx_->sm_count) : xtw_default_splits(m, n);
    T* part = ctx_->d<T>("rqb.part", size_t(splits) * n * l);
    const int64_t ws_len = std::max(tsqr_workspace_doubles(m, l, ctx_->max_smem), tsqr_workspace_doubles(n, l, ctx_->max_smem));
    double* ws = ctx_->d<double>("tsqr.ws", size_t(ws_len));
    const double xbytes = double(m) * double(n) * sizeof(T);
    // S^T operands of the tensor-core kernels (hi / lo parts), sized for the larger of m, n
    float* st_hi = nullptr;
    float* st_lo = nullptr;
    if (tc) {
      const size_t cap = size_t(tc_npad(l)) * size_t(tc_st_pitch(std::max(m, n)));
      st_hi = ctx_->d<float>("tc.st_hi", cap);
      st_lo = ctx_->d<float>("tc.st_lo", cap);
    }
    auto xw = [&](const T* s, T* out) {
      tm_.span(kXw, [&] {
        if constexpr (std::is_same<T, float>::value) {
          if (tc) {
            tm_.launches += launch_tc_prep_st(s, n, l, st_hi, st_lo, st_, x3);
            tm_.span(kXwK, [&] { tm_.launches += launch_tc_xw(x, m, n, ldx, st_hi, st_lo, l, out, x3, ctx_->sm_count, st_); });
            return;
          }
        }
        // fp32: TMA-fed tiles; fp64 (BASELINE config 1, rank-deficient: the sketch's trailing
        // columns are rounding noise whose completion the validated register-staged kernels keep)
        // and the RNMF_XW_LEGACY testing knob: the register-staged kernel
        if (sizeof(T) == 4 && !std::getenv("RNMF_XW_LEGACY")) {
          T* spad = ctx_->d<T>("rqb.spad", size_t(xw_tma_spad_len(n, l)));
          tm_.span(kXwK, [&] { tm_.launches += launch_xw_tma<T>(x, m, n, ldx, s, l, out, spad, ctx_->sm_count, st_); });
        } else {
          tm_.span(kXwK, [&] { tm_.launches += launch_xw<T>(x, m, n, ldx, s, l, out, st_); });
        }
      });
      sketch_bytes_ += xbytes;
      ctx_->last.xw_bytes += xbytes;
      sketch_passes_ += 1;
    };
    auto xtw = [&](const T* s, T* out, bool tr) {
      tm_.span(kXtw, [&] {
        if constexpr (std::is_same<T, float>::value) {
          if (tc) {
            tm_.launches += launch_tc_prep_st(s, m, l, st_hi, st_lo, st_, x3);
            tm_.span(kXtwK, [&] {
              tm_.launches += launch_tc_xtw(x, m, n, ldx, st_hi, st_lo, l, part, splits, x3, ctx_->sm_count, st_);
            });
            tm_.launches += launch_splitk_reduce<T>(part, splits, n, l, out, tr, st_);
            return;
          }
        }
        if (sizeof(T) == 4 && !std::getenv("RNMF_XW_LEGACY")) {
          const int sp = xtw_tma_splits(m, n, ctx_->sm_count);
          T* part2 = ctx_->d<T>("rqb.part2", size_t(sp) * n * l);
          T* spad = ctx_->d<T>("rqb.spad2", size_t(xw_tma_spad_len(m, l)));
          // (the FFMA path's span includes its fixed-order split reduction)
          tm_.span(kXtwK, [&] {
            tm_.launches += launch_xtw_tma<T>(x, m, n, ldx, s, l, part2, sp, out, tr, spad, ctx_->sm_count, st_);
          });
        } else {
          tm_.span(kXtwK, [&] { tm_.launches += launch_xtw<T>(x, m, n, ldx, s, l, part, splits, out, tr, st_); });
        }
      });
      sketch_bytes_ += xbytes;
      ctx_->last.xtw_bytes += xbytes;
      sketch_passes_ += 1;
    };
    double* cqws = ctx_->d<double>("cq.ws", size_t(cholqr_workspace_doubles(std::max(m, n), l)));
    int* cqflag = ctx_->d<int>("cq.flag", 1);
    int* hflag = ctx_->h<int>("cq.flag.h", 1);
    // CholeskyQR2 first; Householder TSQR when A is too ill-conditioned (rank-deficient sketches)
    // row-sharded Q (m x l): the Gram of every CholeskyQR pass is summed over the GPUs, and the
    // fallback is shifted CholeskyQR3 (Gram-only, so it shards the same way); the n x l QR of the
    // power iteration is replicated (identical input on every GPU).
    const GramAllreduce gram_ar = [this](double* g, int64_t cnt) { allreduce(g, size_t(cnt)); };
    auto qr = [&](const T* a, int64_t rows, T* out, bool row_sharded) {
      tm_.span(kQr, [&] {
        const GramAllreduce* ar = (row_sharded && sharded()) ? &gram_ar : nullptr;
        tm_.launches += launch_cholqr2<T>(a, rows, l, out, cqws, cqflag, st_, ar);
        RNMF_CUDA(cudaMemcpyAsync(hflag, cqflag, sizeof(int), cudaMemcpyDeviceToHost, st_));
        RNMF_CUDA(cudaStreamSynchronize(st_));
        if (hflag[0] != 0) {
          if (ar) {
            const double shift = 11.0 * (double(m_total()) * l + double(l) * (l + 1)) * 1.1102230246251565e-16;
            tm_.launches += launch_cholqr2<T>(a, rows, l, out, cqws, cqflag, st_, ar, shift);
            // the shifted CholeskyQR3 pivots must hold (all GPUs see the same all-reduced Grams):
            // a Q that is not orthonormal would also void the column reduction's fixed-point bound
            RNMF_CUDA(cudaMemcpyAsync(hflag, cqflag, sizeof(int), cudaMemcpyDeviceToHost, st_));
            RNMF_CUDA(cudaStreamSynchronize(st_));
            if (hflag[0] != 0)
              throw ParameterError("B200 path: the row-sharded sketch of X is numerically rank deficient "
                                   "(shifted CholeskyQR3 failed); run it unsharded (Householder TSQR fallback)");
          } else {
            tm_.launches += launch_tsqr<T>(a, rows, l, out, ws, ctx_->max_smem, st_);
          }
          ++qr_fallbacks_;
        }
        ++qr_calls_;
      });
    };
    xw(omega_dev, y);
    for (int64_t it = 0; it < q_iters; ++it) {
      qr(y, m, qb, true);
      xtw(qb, p, false);
      allreduce(p, size_t(n) * l);  // X^T Q over all rows
      qr(p, n, z, false);
      xw(z, y);
    }
    qr(y, m, qb, true);
    xtw(qb, b, true);
    allreduce(b, size_t(l) * n);  // B = Q^T X over all rows
    *q_out = qb;
    *b_out = b;
  }

  // rqb_streaming (p/src/sketch.cpp:73-116), fp64: X arrives from the host in column blocks of
  // `bs` (ColumnSource::read_columns); 2 + q passes over the source, exactly as the reference:
  //   Y = sum_b X_b Omega_b;  q x { Q = qr(Y); Y = sum_b X_b (X_b^T Q) };  Q = qr(Y);  B_b = Q^T X_b.
  // Each block is copied from a pinned staging buffer (two, alternating: the host reads block
  // b + 1 while the GPU works on block b), checked for non-finite values (DataError naming the
  // block's column range, p/src/sketch.cpp:89-91) and consumed by the FFMA X-streaming kernels.
  void rqb_streaming(const ColumnReadFn& read, int64_t m, int64_t n, int l, int64_t q_iters, int64_t bs,
                     const double* omega_dev, double* q_host, double* b_host) {
    static_assert(std::is_same<T, double>::value, "rqb_streaming is fp64");
    const int64_t ldb = (bs + 1) / 2 * 2;  // 16-byte row pitch
    double* blk = ctx_->d<double>("rs.blk", size_t(m) * size_t(ldb));
    double* stage[2] = {ctx_->h<double>("rs.h0", size_t(m) * size_t(bs)), ctx_->h<double>("rs.h1", size_t(m) * size_t(bs))};
    double* y = ctx_->d<double>("rs.y", size_t(m) * l);
    double* yt = ctx_->d<double>("rs.yt", size_t(m) * l);
    double* q = ctx_->d<double>("rs.q", size_t(m) * l);
    double* z = ctx_->d<double>("rs.z", size_t(bs) * l);
    double* b = ctx_->d<double>("rs.b", size_t(l) * size_t(n));
    double* bt = ctx_->d<double>("rs.bt", size_t(l) * size_t(bs));
    const int splits = xtw_default_splits(m, bs);
    double* part = ctx_->d<double>("rs.part", size_t(splits) * size_t(bs) * l);
    int* bad = ctx_->d<int>("rs.bad", 1);
    int* hbad = ctx_->h<int>("rs.bad.h", 1);
    const int64_t ws_len = tsqr_workspace_doubles(m, l, ctx_->max_smem);
    double* ws = ctx_->d<double>("tsqr.ws", size_t(ws_len));
    double* cqws = ctx_->d<double>("cq.ws", size_t(cholqr_workspace_doubles(m, l)));
    int* cqflag = ctx_->d<int>("cq.flag", 1);
    int* hflag = ctx_->h<int>("cq.flag.h", 1);
    cudaEvent_t copied[2];
    for (auto& e : copied) RNMF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        for (int i = 0; i < 2; ++i) cudaEventDestroy(e[i]);
      }
    } evg{copied};
    auto qr = [&](const double* a, double* out) {
      tm_.span(kQr, [&] {
        tm_.launches += launch_cholqr2<double>(a, m, l, out, cqws, cqflag, st_, nullptr);
        RNMF_CUDA(cudaMemcpyAsync(hflag, cqflag, sizeof(int), cudaMemcpyDeviceToHost, st_));
        RNMF_CUDA(cudaStreamSynchronize(st_));
        if (hflag[0] != 0) tm_.launches += launch_tsqr<double>(a, m, l, out, ws, ctx_->max_smem, st_);
      });
    };
    const int64_t nb = (n + bs - 1) / bs;
    const double xbytes = double(m) * double(n) * sizeof(double);
    // one pass over the source: fn(c0, w) enqueues the block's kernels
    auto each_block = [&](auto&& fn) {
      read(0, std::min(bs, n), stage[0]);
      for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t c0 = ib * bs, w = std::min(bs, n - c0);
        double* hs = stage[ib & 1];
        RNMF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st_));
        RNMF_CUDA(cudaMemcpy2DAsync(blk, size_t(ldb) * sizeof(double), hs, size_t(w) * sizeof(double),
                                    size_t(w) * sizeof(double), size_t(m), cudaMemcpyHostToDevice, st_));
        RNMF_CUDA(cudaEventRecord(copied[ib & 1], st_));
        block_finite_kernel<<<int(std::min<int64_t>(148 * 4, std::max<int64_t>(1, (m * w + 255) / 256))), 256, 0, st_>>>(
            blk, m, w, ldb, bad);
        RNMF_CUDA_LAUNCH();
        RNMF_CUDA(cudaMemcpyAsync(hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st_));
        tm_.launches += 1;
        fn(c0, w);
        if (ib + 1 < nb) {
          // the other staging buffer is free once its previous H2D copy has run
          RNMF_CUDA(cudaEventSynchronize(copied[(ib + 1) & 1]));
          const int64_t c1 = c0 + bs;
          read(c1, std::min(bs, n - c1), stage[(ib + 1) & 1]);
        }
        RNMF_CUDA(cudaStreamSynchronize(st_));
        if (hbad[0] != 0)
          throw DataError("rqb_streaming: non-finite values in columns [" + std::to_string(c0) + ", " +
                          std::to_string(c0 + w) + ")");
      }
      sketch_bytes_ += xbytes;
      sketch_passes_ += 1;
    };
    auto add = [&](double* dst, const double* src, int64_t count) {
      add_inplace_kernel<<<int(std::min<int64_t>(148 * 4, std::max<int64_t>(1, (count + 255) / 256))), 256, 0, st_>>>(
          dst, src, count);
      RNMF_CUDA_LAUNCH();
      tm_.launches += 1;
    };
    tm_.span(kXw, [&] {
      RNMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(m) * l, st_));
      each_block([&](int64_t c0, int64_t w) {
        tm_.launches += launch_xw<double>(blk, m, w, ldb, omega_dev + c0 * l, l, yt, st_);
        add(y, yt, m * l);
      });
    });
    for (int64_t it = 0; it < q_iters; ++it) {
      qr(y, q);
      tm_.span(kXtw, [&] {
        RNMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(m) * l, st_));
        each_block([&](int64_t, int64_t w) {
          tm_.launches += launch_xtw<double>(blk, m, w, ldb, q, l, part, splits, z, false, st_);  // Z = X_b^T Q
          tm_.launches += launch_xw<double>(blk, m, w, ldb, z, l, yt, st_);                     // X_b Z
          add(y, yt, m * l);
        });
      });
    }
    qr(y, q);
    tm_.span(kXtw, [&] {
      each_block([&](int64_t c0, int64_t w) {
        tm_.launches += launch_xtw<double>(blk, m, w, ldb, q, l, part, splits, bt, true, st_);  // Q^T X_b (l x w)
        RNMF_CUDA(cudaMemcpy2DAsync(b + c0, size_t(n) * sizeof(double), bt, size_t(w) * sizeof(double),
                                    size_t(w) * sizeof(double), size_t(l), cudaMemcpyDeviceToDevice, st_));
      });
    });
    RNMF_CUDA(cudaMemcpyAsync(q_host, q, sizeof(double) * size_t(m) * l, cudaMemcpyDeviceToHost, st_));
    RNMF_CUDA(cudaMemcpyAsync(b_host, b, sizeof(double) * size_t(l) * size_t(n), cudaMemcpyDeviceToHost, st_));
    RNMF_CUDA(cudaStreamSynchronize(st_));
  }

  // Full-space metrics (p/src/rhals.cpp:140-148) of the device factors w (m x k), h (k x n):
  // writes [objective, pgrad_full] into res (device).
  // hht_in: H H^T (k x k, fp64) when the caller has it (the sweep kernel's V after every launch)
  void metrics(int k, const T* w, const T* h, double* res, const double* hht_in = nullptr) {
    if constexpr (std::is_same<T, float>::value) {
      if (math_ == RNMF_MATH_TF32X3 && k <= 64 && m_ > 0 && n_ > 0) {
        metrics_tc(k, w, h, res, hht_in);
        return;
      }
    }
    const T* x = x_;
    const int64_t m = m_, n = n_, ldx = ldx_;
    T* ht = ctx_->d<T>("met.ht", size_t(n) * k);
    double* hht = ctx_->d<double>("met.hht", size_t(k) * k);
    double* wtw = ctx_->d<double>("met.wtw", size_t(k) * k);
    double* gpart = ctx_->d<double>("met.gpart", size_t(gram_parts(std::max(m, n))) * k * k);
    double* gpart2 = ctx_->d<double>("met.gpart2", size_t(gram_parts(std::max(m, n))) * k * k);
    const int nb1 = xw_metrics_blocks(m);
    double* pobj = ctx_->d<double>("met.pobj", size_t(nb1));
    double* ppgw = ctx_->d<double>("met.ppgw", size_t(nb1));
    const int splits = xtw_default_splits(m, n);
    T* part = ctx_->d<T>("met.part", size_t(splits) * n * k);
    double* ppgh = ctx_->d<double>("met.ppgh", size_t(grad_h_blocks(n, k)));
    double* tmp = ctx_->d<double>("met.tmp", 4);
    // one fused X pass when the per-tile W^T X partials stay small (<= 1/4 of X), else the fused
    // pass without W^T X plus a split-K X^T W pass
    const bool fused_ok = k <= 64 && (sizeof(T) == 4 || k <= 32);
    const int g1 = metrics_grid(m, k, int(sizeof(T)), ctx_->sm_count);
    const double wtx_bytes = double(g1) * double(n) * k * sizeof(T);
    const bool one_pass = fused_ok && wtx_bytes <= 0.25 * double(m) * double(n) * sizeof(T);
    x_passes_ = 2;
    if (sharded() && !one_pass) throw ParameterError("B200 path: row-sharded metrics need the one-pass kernel (k <= 64)");
    tm_.span(kMetrics, [&] {
      if (hht_in)
        hht = const_cast<double*>(hht_in);
      else
        tm_.launches += launch_gram_cols<T>(h, k, n, gpart, hht, st_);
      tm_.launches += launch_gram_rows<T>(w, m, k, gpart2, wtw, st_);
      allreduce(wtw, size_t(k) * k);  // W^T W over all rows (H H^T is replicated)
      int b1 = 0, b2 = 0;
      if (fused_ok) {
        T* wtx = one_pass ? ctx_->d<T>("met.wtx", size_t(g1) * n * k) : nullptr;
        T* hpad = ctx_->d<T>("met.hpad", size_t(metrics_hpad_len(k, n)));
        double* po = ctx_->d<double>("met.pobj2", size_t(g1));
        double* pw = ctx_->d<double>("met.ppgw2", size_t(g1));
        tm_.launches += launch_metrics_fused<T>(x, m, n, ldx, w, h, k, hht, hpad, wtx, po, pw, ctx_->sm_count, st_);
        b1 = g1;
        pobj = po;
        ppgw = pw;
        if (one_pass) {
          double* pgh = ctx_->d<double>("met.ppgh2", size_t(grad_h_blocks(n, k)));
          if (sharded()) {
            // W^T X: this GPU's CTA partials -> one n x k partial -> summed over the GPUs
            T* wtx1 = ctx_->d<T>("met.wtx1", size_t(n) * k);
            tm_.launches += launch_splitk_reduce<T>(wtx, g1, n, k, wtx1, false, st_);
            allreduce(wtx1, size_t(n) * k);
            tm_.launches += launch_grad_h_reduce<T>(wtx1, 1, n, k, h, wtw, pgh, &b2, st_);
          } else {
            tm_.launches += launch_grad_h_reduce<T>(wtx, g1, n, k, h, wtw, pgh, &b2, st_);
          }
          ppgh = pgh;
          x_passes_ = 1;
        } else {
          double* pgh = ctx_->d<double>("met.ppgh2", size_t(grad_h_blocks(n, k)));
          tm_.launches += launch_xtw_metrics<T>(x, m, n, ldx, w, k, h, wtw, part, splits, pgh, &b2, st_);
          ppgh = pgh;
        }
      } else {
        tm_.launches += launch_transpose<T>(h, k, n, ht, st_);
        tm_.launches += launch_xw_metrics<T>(x, m, n, ldx, ht, w, k, hht, pobj, ppgw, &b1, st_);
        tm_.launches += launch_xtw_metrics<T>(x, m, n, ldx, w, k, h, wtw, part, splits, ppgh, &b2, st_);
      }
      if (!sharded()) {
        tm_.launches += launch_metrics_finalize(pobj, b1, ppgw, b1, ppgh, b2, res, st_);
      } else {
        tm_.launches += launch_sum_parts(pobj, b1, res, st_);
        tm_.launches += launch_sum_parts(ppgw, b1, tmp, st_);
        // objective and the grad_W term are sums over rows: add the GPUs' values (grad_H is replicated)
        allreduce(res, 1);
        allreduce(tmp, 1);
        tm_.launches += launch_sum_parts(ppgh, b2, tmp + 1, st_);
        // res[1] = pgw + pgh, done on device by a 2-element sum
        tm_.launches += launch_sum_parts(tmp, 2, res + 1, st_);
      }
    });
    metrics_bytes_ += double(x_passes_) * double(m) * double(n) * sizeof(T);
    metrics_passes_ += x_passes_;
  }

  // Full-space metrics on the tensor cores (math_mode TF32X3, fp32): tcgen05 3xTF32 kernels with
  // fp32-promoted accumulation (tc_metrics.h):
  //   X H^T -> projected grad_W, X^T W -> projected grad_H, explicit residual -> objective;
  // for k <= 32 the X H^T and residual kernels are one (two X passes per evaluation, else three).
  void metrics_tc(int k, const float* w, const float* h, double* res, const double* hht_in) {
    const float* x = reinterpret_cast<const float*>(x_);
    const int64_t m = m_, n = n_, ldx = ldx_;
    const int sms = ctx_->sm_count;
    double* hht = ctx_->d<double>("met.hht", size_t(k) * k);
    double* wtw = ctx_->d<double>("met.wtw", size_t(k) * k);
    double* gpart = ctx_->d<double>("met.gpart", size_t(gram_parts(std::max(m, n))) * k * k);
    double* gpart2 = ctx_->d<double>("met.gpart2", size_t(gram_parts(std::max(m, n))) * k * k);
    const int npad = tc_npad(k), kw = tc_resid_kw(k);
    float* sth = ctx_->d<float>("tcm.sth", size_t(npad) * size_t(tc_st_pitch(n)));
    float* stl = ctx_->d<float>("tcm.stl", size_t(npad) * size_t(tc_st_pitch(n)));
    float* swh = ctx_->d<float>("tcm.swh", size_t(npad) * size_t(tc_st_pitch(m)));
    float* swl = ctx_->d<float>("tcm.swl", size_t(npad) * size_t(tc_st_pitch(m)));
    float* wh = ctx_->d<float>("tcm.wh", size_t(m) * kw);
    float* wl = ctx_->d<float>("tcm.wl", size_t(m) * kw);
    float* hth = ctx_->d<float>("tcm.hth", size_t(tc_st_pitch(n)) * kw);
    float* htl = ctx_->d<float>("tcm.htl", size_t(tc_st_pitch(n)) * kw);
    float* xht = ctx_->d<float>("tcm.xht", size_t(m) * k);
    const int splits = tc_xtw_splits(m, n, sms);
    float* part = ctx_->d<float>("tcm.part", size_t(splits) * n * k);
    double* pobj = ctx_->d<double>("tcm.pobj", size_t(tc_resid_blocks(m, sms)));
    double* ppgw = ctx_->d<double>("tcm.ppgw", size_t(tc_pgw_blocks(m)));
    double* ppgh = ctx_->d<double>("tcm.ppgh", size_t(grad_h_blocks(n, k)));
    double* tmp = ctx_->d<double>("met.tmp", 4);
    const bool fused = k <= 64 && !std::getenv("RNMF_NO_FUSED_RESID");
    tm_.span(kMetrics, [&] {
      if (hht_in)
        hht = const_cast<double*>(hht_in);
      else
        tm_.launches += launch_gram_cols<float>(h, k, n, gpart, hht, st_);
      tm_.launches += launch_gram_rows<float>(w, m, k, gpart2, wtw, st_);
      allreduce(wtw, size_t(k) * k);  // W^T W over all rows (H H^T is replicated)
      // X H^T (m x k) -> projected grad_W partials
      int b1 = 0, b2 = 0, b0 = 0;
      tm_.launches += launch_tc_metrics_prep(w, m, h, n, k, sth, stl, wh, wl, hth, htl, swh, swl, st_);
      if (fused) {  // X H^T and the residual in one X pass
        tm_.launches += launch_tc_xht_resid(x, m, n, ldx, sth, stl, wh, wl, hth, htl, k, xht, pobj, &b0, sms, st_);
      } else {
        tm_.launches += launch_tc_xw(x, m, n, ldx, sth, stl, k, xht, true, sms, st_);
        tm_.launches += launch_tc_resid(x, m, n, ldx, wh, wl, hth, htl, k, pobj, &b0, sms, st_);
      }
      tm_.launches += launch_tc_pgw(xht, w, m, k, hht, ppgw, &b1, st_);
      // X^T W (n x k split partials) -> projected grad_H partials
      tm_.launches += launch_tc_xtw(x, m, n, ldx, swh, swl, k, part, splits, true, sms, st_);
      if (sharded()) {
        float* wtx1 = ctx_->d<float>("met.wtx1", size_t(n) * k);
        tm_.launches += launch_splitk_reduce<float>(part, splits, n, k, wtx1, false, st_);
        allreduce(wtx1, size_t(n) * k);
        tm_.launches += launch_grad_h_reduce<float>(wtx1, 1, n, k, h, wtw, ppgh, &b2, st_);
      } else {
        tm_.launches += launch_grad_h_reduce<float>(part, splits, n, k, h, wtw, ppgh, &b2, st_);
      }
      if (!sharded()) {
        tm_.launches += launch_metrics_finalize(pobj, b0, ppgw, b1, ppgh, b2, res, st_);
      } else {
        tm_.launches += launch_sum_parts(pobj, b0, res, st_);
        tm_.launches += launch_sum_parts(ppgw, b1, tmp, st_);
        allreduce(res, 1);
        allreduce(tmp, 1);
        tm_.launches += launch_sum_parts(ppgh, b2, tmp + 1, st_);
        tm_.launches += launch_sum_parts(tmp, 2, res + 1, st_);
      }
    });
    x_passes_ = fused ? 2 : 3;
    metrics_bytes_ += double(x_passes_) * double(m) * double(n) * sizeof(float);
    metrics_passes_ += x_passes_;
  }

  double sum() const { return sum_; }
  double sumsq() const { return sumsq_; }
  double sketch_bytes_ = 0, metrics_bytes_ = 0;
  int math_ = RNMF_MATH_EXACT;
  int64_t qr_calls_ = 0, qr_fallbacks_ = 0;
  int64_t sketch_passes_ = 0, metrics_passes_ = 0;

 private:
  rnmf_gpu_context* ctx_;
  cudaStream_t st_;
  Timer& tm_;
  double sum_ = 0.0, sumsq_ = 0.0;
  const T* x_ = nullptr;
  int64_t m_ = 0, n_ = 0, ldx_ = 0;
  int64_t row_off_ = 0, m_total_ = 0;
  int x_passes_ = 2;
};

// ---- the sweep / trace loop shared by rhals_fit and rhals_fit_compressed ---------------------
template <typename T>
struct LoopIO {
  const T* x;
  int64_t m, n;
  int l, k;
  const T* q;
  const T* b;
  T* w;
  T* h;
  double* wt;  // device l x k (in/out)
  bool init_wt;
};

// Sweep-kernel scratch: the fp32 streamed path's float4-column copy of Q (SweepPlan::f32s; once per Q,
// i.e. per fit or stage call) and column-major W, and the wide layout's residc buffer.  Returns the
// kernel launches issued.
template <typename T>
static int attach_sweep_stream(rnmf_gpu_context* ctx, const SweepPlan& plan, SweepArgs<T>& a, cudaStream_t st) {
  if (plan.wide) a.rc = ctx->d<T>("sw.rc", size_t(a.l) * size_t(a.n));
  if constexpr (std::is_same<T, float>::value) {
    if (!plan.f32s) return 0;
    float* q4 = ctx->d<float>("sw.q4", size_t(a.m) * size_t(plan.lreg));
    a.q4 = q4;
    a.wc = ctx->d<float>("sw.wc", size_t(a.m) * size_t(a.k));
    return sweep_relayout_q(a.q, a.m, a.l, plan.lreg, q4, st);
  }
  return 0;
}

// Row-sharded launches: zero this GPU's sync block, then an NCCL all-reduce, so that no GPU's
// kernel can add into a peer's sync block before that peer has zeroed it for this launch.
template <typename T>
static int launch_sweeps_synced(rnmf_gpu_context* ctx, Engine<T>& eng, const SweepArgs<T>& a, const SweepPlan& plan,
                                cudaStream_t st) {
  if (!eng.sharded()) return launch_sweeps<T>(a, plan, st);
  RNMF_CUDA(cudaMemsetAsync(ctx->sync_block, 0, kSweepSyncBytes, st));
  double* tok = ctx->d<double>("sw.launch_token", 1);
  eng.allreduce(tok, 1);
  return launch_sweeps<T>(a, plan, st, false);
}

template <typename T>
static void run_loop(rnmf_gpu_context* ctx, Engine<T>& eng, Timer& tm, const rnmf_solver_options& o, LoopIO<T>& io,
                     std::chrono::steady_clock::time_point t0, double x_norm, rnmf_trace_record* trace,
                     int64_t* trace_len) {
  cudaStream_t st = ctx->stream;
  const int l = io.l, k = io.k;
  const int64_t max_iter = o.max_iter;
  const SweepPlan plan = plan_sweeps<T>(io.m, io.n, l, k, ctx->sm_count, ctx->max_smem);
  if (plan.grid == 0)
    throw ParameterError("B200 path: problem " + shape_string(io.m, io.n) + " with l=" + std::to_string(l) +
                         ", k=" + std::to_string(k) + " does not fit the persistent sweep kernel");
  const int64_t plen = sweep_part_len(l, k);
  SweepArgs<T> a{};
  a.q = io.q;
  a.b = io.b;
  a.w = io.w;
  a.h = io.h;
  a.wt = io.wt;
  a.wn = ctx->d<double>("sw.wn", size_t(k));
  a.tm = ctx->d<double>("sw.tm", size_t(l) * k);
  a.vm = ctx->d<double>("sw.vm", size_t(k) * k);
  a.em = ctx->d<double>("sw.em", size_t(l) * k);
  a.m = io.m;
  a.n = io.n;
  a.l = l;
  a.k = k;
  a.alpha_w = o.reg.alpha_w;
  a.alpha_h = o.reg.alpha_h;
  a.beta_w = o.reg.beta_w;
  a.beta_h = o.reg.beta_h;
  a.stop_rule = o.stopping;
  a.tol = o.tol;
  a.pgrad0 = ctx->d<double>("sw.pgrad0", 1);
  a.trace_objc = ctx->d<double>("sw.tobjc", size_t(max_iter + 1));
  a.trace_pgrad = ctx->d<double>("sw.tpgrad", size_t(max_iter + 1));
  a.trace_time = ctx->d<unsigned long long>("sw.ttime", size_t(max_iter + 1));
  a.status = ctx->d<long long>("sw.status", 3);
  a.barrier = reinterpret_cast<unsigned*>(ctx->sync_block);
  a.part = ctx->d<double>("sw.part", size_t(2 * plen * plan.grid));
  a.fin = ctx->d<double>("sw.fin", size_t(2 * plen));
  tm.launches += attach_sweep_stream<T>(ctx, plan, a, st);
  if (eng.sharded()) {
    // row-sharded: column steps and W-side sums run over every CTA of every GPU
    a.world = ctx->shard.world;
    a.rank = ctx->shard.rank;
    for (int p = 0; p < a.world; ++p) a.peer_sync[p] = ctx->shard.peer[p];
    long long* gs = ctx->d<long long>("sw.gsum", 1);
    long long* hgs = ctx->h<long long>("sw.gsum.h", 1);
    hgs[0] = plan.grid;
    RNMF_CUDA(cudaMemcpyAsync(gs, hgs, sizeof(long long), cudaMemcpyHostToDevice, st));
    eng.allreduce(gs, 1);
    RNMF_CUDA(cudaMemcpyAsync(hgs, gs, sizeof(long long), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaStreamSynchronize(st));
    a.xtotal = hgs[0];
  }
  // RNMF_PROF=1: per-phase cycle counters of CTA 0, printed to stderr (development aid)
  const bool prof = std::getenv("RNMF_PROF") != nullptr && sweep_prof_compiled();
  if (std::getenv("RNMF_PROF") != nullptr && !prof)
    std::fprintf(stderr, "[rnmf prof] library built without RNMF_SWEEP_PROF=1; no cycle profile\n");
  std::vector<long long> prof_sum(kSweepProfSlots, 0);
  long long* hprof = nullptr;
  if (prof) {
    a.prof = ctx->d<long long>("sw.prof", kSweepProfSlots);
    hprof = ctx->h<long long>("sw.prof.h", kSweepProfSlots);
  }

  // Metrics results, one slot per evaluation: [objective, pgrad_full]
  const int64_t max_evals = max_iter / o.trace_full_every + 4 + (o.stopping == RNMF_STOP_OBJECTIVE ? max_iter : 0);
  double* mres = ctx->d<double>("sw.mres", size_t(2 * max_evals));
  std::vector<int64_t> eval_iter;

  // host <-> device clock reference for elapsed_s
  auto* gt_ref = ctx->d<unsigned long long>("sw.gtref", 1);
  RNMF_CUDA(cudaStreamSynchronize(st));
  const double h_ref = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  tm.launches += launch_timestamp(gt_ref, st);

  // record 0: full-space metrics of the initial factors
  eng.metrics(k, io.w, io.h, mres);
  eval_iter.push_back(0);

  auto* hstat = ctx->h<long long>("sw.status.h", 3);
  auto* hmres = ctx->h<double>("sw.mres.h", size_t(2 * max_evals));
  const bool objective_rule = o.stopping == RNMF_STOP_OBJECTIVE;
  const int64_t tfe = o.trace_full_every;
  // Interleaved / Shuffled: the component order of every sweep of a chunk, drawn on the host from
  // the reference shuffle stream (sweep_order, p/src/hals.cpp:83-94: Fisher-Yates with next_u64)
  const bool fresh_order = o.order != RNMF_ORDER_GROUPED;
  Rng shuffle_rng = Rng(o.seed).split(kShuffleStream);
  const int64_t chunk_cap = objective_rule ? 1 : tfe;
  int* hord = fresh_order ? ctx->h<int>("sw.order.h", size_t(chunk_cap * k)) : nullptr;
  int* dord = fresh_order ? ctx->d<int>("sw.order", size_t(chunk_cap * k)) : nullptr;
  int64_t t_begin = 1;
  bool first = true;
  int64_t last = 0;
  // reseed_dead (p/src/rhals.cpp:182-186): liveness stamps per component, the reseed draws from
  // the reference stream on the host when the kernel reports a dead component
  Rng reseed_rng = Rng(o.seed).split(kReseedStream);
  if (o.reseed_dead) {
    a.alive = ctx->d<unsigned>("sw.alive", size_t(2) * k);
    RNMF_CUDA(cudaMemsetAsync(a.alive, 0, sizeof(unsigned) * 2 * k, st));
  }
  while (true) {
    // chunks end at the next full-metrics point (p/src/rhals.cpp:191-193)
    const int64_t t_end = std::min(max_iter, objective_rule ? t_begin : ceil_div(t_begin, tfe) * tfe);
    if (fresh_order) {
      for (int64_t t = t_begin; t <= t_end; ++t) {
        int* idx = hord + (t - t_begin) * k;
        for (int j = 0; j < k; ++j) idx[j] = j;
        if (o.order == RNMF_ORDER_SHUFFLED)
          for (int i = k - 1; i > 0; --i) {
            const int j = int(shuffle_rng.next_u64() % uint64_t(i + 1));
            std::swap(idx[i], idx[j]);
          }
      }
      RNMF_CUDA(cudaMemcpyAsync(dord, hord, sizeof(int) * size_t((t_end - t_begin + 1) * k), cudaMemcpyHostToDevice, st));
    }
    int extra = 0;
    int64_t tb = t_begin;
    bool speculative = false;
    while (true) {
      a.flags = kRecord | kDoW | kDoH | (o.reseed_dead ? kReseed : 0) | extra |
                (first ? (kEval0 | kInitWn | (io.init_wt ? kInitWt : 0)) : 0);
      a.t_begin = tb;
      a.t_end = t_end;
      if (fresh_order) a.order = dord + (tb - t_begin) * k;
      tm.span(kSweeps, [&] { tm.launches += launch_sweeps_synced<T>(ctx, eng, a, plan, st); });
      RNMF_CUDA(cudaMemcpyAsync(hstat, a.status, 3 * sizeof(long long), cudaMemcpyDeviceToHost, st));
      if (prof) RNMF_CUDA(cudaMemcpyAsync(hprof, a.prof, kSweepProfSlots * sizeof(long long), cudaMemcpyDeviceToHost, st));
      // Without reseed_dead the launch never hands control back mid-chunk, so the full-space metrics
      // of the launch's final factors are enqueued before waiting for its status: the GPU goes
      // straight from the sweep kernel into the metrics passes (the record is dropped below if the
      // launch turned out to be a stationary start, last < t_begin).
      speculative = !o.reseed_dead && extra == 0;
      if (speculative) eng.metrics(k, io.w, io.h, mres + 2 * eval_iter.size(), a.vm);
      RNMF_CUDA(cudaStreamSynchronize(st));
      if (prof)
        for (int i = 0; i < kSweepProfSlots; ++i) prof_sum[size_t(i)] += hprof[i];
      first = false;
      if (hstat[2] == 0) break;
      // reseed_dead_components (p/src/hals.cpp:96-105) after sweep t, in the reference's draw order
      const int64_t t = hstat[2];
      std::vector<unsigned> alive(static_cast<size_t>(2 * k));
      RNMF_CUDA(cudaMemcpy(alive.data(), a.alive, sizeof(unsigned) * 2 * k, cudaMemcpyDeviceToHost));
      T* hw = ctx->h<T>("reseed.w", size_t(io.m));
      T* hh = ctx->h<T>("reseed.h", size_t(io.n));
      for (int j = 0; j < k; ++j) {
        if (alive[size_t(j)] != unsigned(t)) {
          for (int64_t i = 0; i < io.m; ++i) hw[i] = T(reseed_rng.uniform() * 1e-4);
          RNMF_CUDA(cudaMemcpy2DAsync(io.w + j, sizeof(T) * k, hw, sizeof(T), sizeof(T), size_t(io.m),
                                      cudaMemcpyHostToDevice, st));
          RNMF_CUDA(cudaStreamSynchronize(st));
        }
        if (alive[size_t(k + j)] != unsigned(t)) {
          for (int64_t c = 0; c < io.n; ++c) hh[c] = T(reseed_rng.uniform() * 1e-4);
          RNMF_CUDA(cudaMemcpyAsync(io.h + int64_t(j) * io.n, hh, sizeof(T) * size_t(io.n), cudaMemcpyHostToDevice, st));
          RNMF_CUDA(cudaStreamSynchronize(st));
        }
      }
      // W~ = Q^T W and the norms from the reseeded W, then the evaluation of sweep t
      extra = kEvalPrev | kInitWt | kInitWn;
      tb = t + 1;
    }
    first = false;
    last = hstat[0];
    const bool stopped = hstat[1] != 0;
    if (last >= t_begin) {
      if (!speculative) eng.metrics(k, io.w, io.h, mres + 2 * eval_iter.size(), a.vm);  // V = H H^T of the final H
      eval_iter.push_back(last);
    }
    bool stop = stopped;
    if (objective_rule && last >= t_begin) {
      RNMF_CUDA(cudaMemcpyAsync(hmres, mres + 2 * (eval_iter.size() - 1), 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      RNMF_CUDA(cudaStreamSynchronize(st));
      stop = hmres[0] < o.tol;  // p/src/rhals.cpp:198-199
    }
    if (stop || last >= max_iter || last < t_end) break;  // last < t_end: stationary start
    t_begin = last + 1;
  }
  // gather the trace
  const int64_t nrec = last + 1;
  auto* hobjc = ctx->h<double>("sw.tobjc.h", size_t(nrec));
  auto* hpg = ctx->h<double>("sw.tpgrad.h", size_t(nrec));
  auto* htime = ctx->h<unsigned long long>("sw.ttime.h", size_t(nrec));
  auto* hgt = ctx->h<unsigned long long>("sw.gtref.h", 1);
  tm.span(kD2H, [&] {
    RNMF_CUDA(cudaMemcpyAsync(hobjc, a.trace_objc, size_t(nrec) * sizeof(double), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaMemcpyAsync(hpg, a.trace_pgrad, size_t(nrec) * sizeof(double), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaMemcpyAsync(htime, a.trace_time, size_t(nrec) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaMemcpyAsync(hgt, gt_ref, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaMemcpyAsync(hmres, mres, 2 * eval_iter.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  });
  RNMF_CUDA(cudaStreamSynchronize(st));
  size_t ev = 0;
  double obj = 0, rel = 0, pgf = 0;
  for (int64_t t = 0; t < nrec; ++t) {
    while (ev < eval_iter.size() && eval_iter[ev] <= t) {
      obj = hmres[2 * ev];
      pgf = hmres[2 * ev + 1];
      rel = x_norm > 0.0 ? std::sqrt(obj) / x_norm : 0.0;
      ++ev;
    }
    rnmf_trace_record& r = trace[t];
    r.iter = t;
    r.objective = obj;
    r.rel_err = rel;
    r.pgrad = hpg[t];
    r.pgrad_full = pgf;
    r.objective_compressed = hobjc[t];
    const double dt = double((long long)(htime[t] - hgt[0])) * 1e-9;
    r.elapsed_s = h_ref + std::max(0.0, dt);
  }
  for (int64_t t = 1; t < nrec; ++t) trace[t].elapsed_s = std::max(trace[t].elapsed_s, trace[t - 1].elapsed_s);
  if (prof) {
    static const char* names[] = {"w_step", "lift", "recompress", "barrier1", "reduce1", "h_cols", "h_products",
                                  "barrier2", "reduce2a", "reduce2b", "pgw", "other", "h_s", "h_init", "h_update",
                                  "kernel_total", "barriers"};
    std::fprintf(stderr, "[rnmf prof] sweeps=%lld grid=%d smem=%zu q_in_smem=%d (cycles of CTA 0 summed over launches)\n",
                 (long long)last, plan.grid, plan.smem, int(plan.q_in_smem));
    for (int i = 0; i < kSweepProfSlots; ++i)
      std::fprintf(stderr, "[rnmf prof] %-12s %14lld  per-sweep %10.1f\n", names[i], prof_sum[size_t(i)],
                   double(prof_sum[size_t(i)]) / double(std::max<int64_t>(last, 1)));
  }
  *trace_len = nrec;
  ctx->last.sweeps = last;
}

// ---- random draws for Omega / init (reference streams unless overridden) ---------------------
static void fill_uniform(Rng& rng, double* out, size_t count) {
  for (size_t i = 0; i < count; ++i) out[i] = rng.uniform();
}
static void fill_gaussian(Rng& rng, double* out, size_t count) {
  for (size_t i = 0; i < count; ++i) out[i] = rng.gaussian();
}

// InitScheme::Svd, nndsvd_init (p/src/hals.cpp:126-170): a second rqb with its own stream
// (seed = the init Rng's first next_u64, uniform test matrix, p = min(20, min(m,n) - k), q = 2), the
// SVD of its B through the Jacobi eigen-decomposition of B B^T, and the NNDSVD split of the leading
// k pairs into w (this GPU's rows) and h; zeros become mean(X)/100.  Runs before the fit's own rqb
// (the two sketches are independent; the rqb buffers are reused).
template <typename T>
static void nndsvd_init_dev(rnmf_gpu_context* ctx, Engine<T>& eng, Timer& tm, const rnmf_solver_options& o, int64_t m,
                            int64_t n, int64_t mt, T* w, T* h) {
  cudaStream_t st = ctx->stream;
  const int k = int(o.rank);
  const int64_t p2 = std::min<int64_t>(20, std::min(mt, n) - k);
  const int l2 = int(sketch_width(mt, n, k, p2, 2));
  if (l2 > 64) throw ParameterError("B200 path: InitScheme::Svd supports a sketch width up to 64");
  Rng init_rng(o.seed);
  Rng orng(init_rng.next_u64());
  std::vector<double> om(size_t(n) * l2);
  fill_uniform(orng, om.data(), om.size());
  T* om_dev = eng.upload_converted("omega.svd", om.data(), om.size());
  T *q2 = nullptr, *b2 = nullptr;
  tm.span(kSketch, [&] { eng.rqb(l2, 2, om_dev, RNMF_MATH_EXACT, &q2, &b2); });
  tm.span(kInit, [&] {
    double* gpart = ctx->d<double>("svd.gpart", size_t(gram_parts(n)) * l2 * l2);
    double* g = ctx->d<double>("svd.g", size_t(l2) * l2);
    double* eval = ctx->d<double>("svd.eval", size_t(l2));
    double* evec = ctx->d<double>("svd.evec", size_t(l2) * l2);
    tm.launches += launch_gram_cols<T>(b2, l2, n, gpart, g, st);
    tm.launches += launch_jacobi_eig(g, l2, eval, evec, st);
    double* heval = ctx->h<double>("svd.eval.h", size_t(l2));
    RNMF_CUDA(cudaMemcpyAsync(heval, eval, sizeof(double) * l2, cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaStreamSynchronize(st));
    std::vector<double> sv(static_cast<size_t>(k));
    for (int j = 0; j < k; ++j) sv[size_t(j)] = std::sqrt(std::max(heval[j], 0.0));
    // u = Q U(:, :k); v = B^T U(:, :k) / s
    double* hcs = ctx->h<double>("svd.cs.h", size_t(2) * k);
    for (int j = 0; j < k; ++j) {
      hcs[j] = 1.0;
      hcs[k + j] = sv[size_t(j)] > 0.0 ? 1.0 / sv[size_t(j)] : 0.0;
    }
    double* cs = ctx->d<double>("svd.cs", size_t(2) * k);
    RNMF_CUDA(cudaMemcpyAsync(cs, hcs, sizeof(double) * 2 * k, cudaMemcpyHostToDevice, st));
    const int bu = nndsvd_norm_blocks(m), bv = nndsvd_norm_blocks(n);
    double* pu = ctx->d<double>("svd.pu", size_t(bu) * 2 * k);
    double* pv = ctx->d<double>("svd.pv", size_t(bv) * 2 * k);
    double* nrm = ctx->d<double>("svd.nrm", size_t(4) * k);
    tm.launches += launch_nndsvd_norms<T>(q2, m, l2, false, evec, k, cs, pu, st);
    tm.launches += launch_nndsvd_norms<T>(b2, n, l2, true, evec, k, cs + k, pv, st);
    tm.launches += launch_reduce_parts(pu, bu, 2 * k, nrm, st);
    tm.launches += launch_reduce_parts(pv, bv, 2 * k, nrm + 2 * k, st);
    eng.allreduce(nrm, size_t(2) * k);  // sharded: u's rows are spread over the GPUs
    double* hn = ctx->h<double>("svd.nrm.h", size_t(4) * k);
    RNMF_CUDA(cudaMemcpyAsync(hn, nrm, sizeof(double) * 4 * k, cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaStreamSynchronize(st));
    // coefficients of the positive / negative parts (p/src/hals.cpp:145-160)
    double* hc = ctx->h<double>("svd.coef.h", size_t(4) * k);
    for (int j = 0; j < k; ++j) {
      double* cu = hc + 2 * j;
      double* cv = hc + 2 * k + 2 * j;
      cu[0] = cu[1] = cv[0] = cv[1] = 0.0;
      if (j == 0) {  // leading pair with the signs folded away: sqrt(s0) |u0|, sqrt(s0) |v0|
        cu[0] = cu[1] = cv[0] = cv[1] = std::sqrt(sv[0]);
        continue;
      }
      const double nup = std::sqrt(hn[2 * j]), nun = std::sqrt(hn[2 * j + 1]);
      const double nvp = std::sqrt(hn[2 * k + 2 * j]), nvn = std::sqrt(hn[2 * k + 2 * j + 1]);
      const double mp = nup * nvp, mn = nun * nvn;
      if (std::max(mp, mn) <= 0.0) continue;  // degenerate pair: left for the fill
      const bool pos = mp >= mn;
      const double scale = std::sqrt(sv[size_t(j)] * std::max(mp, mn));
      if (pos) {
        cu[0] = scale / nup;
        cv[0] = scale / nvp;
      } else {
        cu[1] = scale / nun;
        cv[1] = scale / nvn;
      }
    }
    double* coef = ctx->d<double>("svd.coef", size_t(4) * k);
    RNMF_CUDA(cudaMemcpyAsync(coef, hc, sizeof(double) * 4 * k, cudaMemcpyHostToDevice, st));
    const double fill = eng.sum() / double(mt * n) / 100.0;
    tm.launches += launch_nndsvd_apply<T>(q2, m, l2, false, evec, k, cs, coef, fill, w, false, st);
    tm.launches += launch_nndsvd_apply<T>(b2, n, l2, true, evec, k, cs + k, coef + 2 * k, fill, h, true, st);
    RNMF_CUDA(cudaStreamSynchronize(st));  // host coefficient buffers are reused by later calls
  });
}

// fit_impl: rhals_fit (fit = true) or compress (fit = false).  Row-sharded contexts hold rows
// [row_off, row_off + m) of an m_total-row X (m_total < 0: not sharded, m_total = m).
template <typename T>
static void fit_impl(rnmf_gpu_context* ctx, const void* x_in, int location, int64_t m, int64_t n,
                     const rnmf_solver_options& o, const double* omega, const double* w0, const double* h0,
                     void* w_out, void* h_out, rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len,
                     void* q_out, void* b_out, void* wt_out, int64_t* l_out, bool fit, int64_t row_off = 0,
                     int64_t m_total = -1) {
  const auto t0 = std::chrono::steady_clock::now();
  ctx->last = rnmf_stage_times{};
  Timer tm(ctx);
  Engine<T> eng(ctx, tm);
  eng.set_math(o.math_mode);
  if (m < 0 || n < 0) throw ShapeError("X has negative dimensions " + shape_string(m, n));
  const int64_t mt = m_total < 0 ? m : m_total;
  eng.set_rows(row_off, mt);
  const T* x = nullptr;
  if (mt * n > 0) {
    if (m * n > 0) x = eng.import_x(x_in, location, m, n);
    eng.scan(true, nullptr);
  }
  validate_options_after_data(mt, n, o);
  check_supported(o);
  if (fit && trace_cap < o.max_iter + 1)
    throw ParameterError("trace buffer too small: need " + std::to_string(o.max_iter + 1) + " records, have " +
                         std::to_string(trace_cap));
  const int k = int(o.rank);
  const int64_t l64 = sketch_width(mt, n, o.rank, o.oversampling, o.power_iterations);
  const int l = int(l64);
  if (l > tsqr_max_l(ctx->max_smem) || l > 128)
    throw ParameterError("B200 path: sketch width " + std::to_string(l) + " above the supported maximum " +
                         std::to_string(std::min(128, tsqr_max_l(ctx->max_smem))));
  if (k > 64) throw ParameterError("B200 path: rank above 64 is not supported yet");
  if (l_out) *l_out = l;

  // Omega: p/src/rhals.cpp:87-92 -> uniform from Rng(Rng(seed).split(3).seed())
  std::vector<double> om_host;
  const double* om = omega;
  if (!om) {
    om_host.resize(size_t(n) * l);
    Rng rng(Rng(o.seed).split(kSketchStream).seed());
    fill_uniform(rng, om_host.data(), om_host.size());
    om = om_host.data();
  }
  T* om_dev = eng.upload_converted("omega", om, size_t(n) * l);

  if (eng.sharded() && (o.reseed_dead || o.order != RNMF_ORDER_GROUPED))
    throw ParameterError("B200 path: row-sharded fits support UpdateOrder::Grouped without reseed_dead");
  const bool svd_init = o.init == RNMF_INIT_SVD;
  if (svd_init && (w0 || h0)) throw ParameterError("init overrides require InitScheme::Random");
  if (svd_init && (m * n == 0 || k < 1)) throw ParameterError("InitScheme::Svd needs a non-empty X");
  T* w = ctx->d<T>("w", size_t(m) * k);
  T* h = ctx->d<T>("h", size_t(k) * n);
  if (svd_init) nndsvd_init_dev<T>(ctx, eng, tm, o, m, n, mt, w, h);

  // initial draws on a host thread while the GPU sketches (random_init, p/src/hals.cpp:118-124)
  double* uw = ctx->h<double>("init.uw", size_t(m) * k);
  double* uh = ctx->h<double>("init.uh", size_t(k) * n);
  std::thread drawer([&] {
    if (svd_init) return;
    if (w0 && h0) {
      std::memcpy(uw, w0, sizeof(double) * size_t(m) * k);
      std::memcpy(uh, h0, sizeof(double) * size_t(k) * n);
      return;
    }
    Rng rng(o.seed);
    if (w0) {
      std::memcpy(uw, w0, sizeof(double) * size_t(m) * k);
    } else {
      // the reference draws all m_total x k entries of W, then H: this GPU keeps its rows
      for (int64_t i = 0; i < row_off * k; ++i) rng.uniform();
      fill_uniform(rng, uw, size_t(m) * k);
      for (int64_t i = (row_off + m) * k; i < mt * k; ++i) rng.uniform();
    }
    if (h0)
      std::memcpy(uh, h0, sizeof(double) * size_t(k) * n);
    else
      fill_uniform(rng, uh, size_t(k) * n);
  });
  T *q = nullptr, *b = nullptr;
  try {
    tm.span(kSketch, [&] { eng.rqb(l, o.power_iterations, om_dev, o.math_mode, &q, &b); });
  } catch (...) {
    drawer.join();
    throw;
  }
  drawer.join();

  const double scale = std::sqrt(eng.sum() / double(mt * n) / double(k));
  if (!svd_init) {
    double* uw_d = ctx->d<double>("init.uw.d", size_t(m) * k);
    double* uh_d = ctx->d<double>("init.uh.d", size_t(k) * n);
    tm.span(kH2D, [&] {
      RNMF_CUDA(cudaMemcpyAsync(uw_d, uw, sizeof(double) * size_t(m) * k, cudaMemcpyHostToDevice, ctx->stream));
      RNMF_CUDA(cudaMemcpyAsync(uh_d, uh, sizeof(double) * size_t(k) * n, cudaMemcpyHostToDevice, ctx->stream));
    });
    tm.span(kInit, [&] {
      tm.launches += launch_scale_cast<T>(uw_d, int64_t(m) * k, scale, w, ctx->stream);
      tm.launches += launch_scale_cast<T>(uh_d, int64_t(k) * n, scale, h, ctx->stream);
    });
  }
  double* wt = ctx->d<double>("wt", size_t(l) * k);
  const double x_norm = std::sqrt(eng.sumsq());

  if (fit) {
    LoopIO<T> io{x, m, n, l, k, q, b, w, h, wt, true};
    rnmf_solver_options oo = o;
    run_loop<T>(ctx, eng, tm, oo, io, t0, x_norm, trace, trace_len);
    eng.export_(w_out, location, w, size_t(m) * k);
    eng.export_(h_out, location, h, size_t(k) * n);
  } else {
    // compress: W~ = Q^T W via the sweep kernel's init phase (p/src/rhals.cpp:103)
    const SweepPlan plan = plan_sweeps<T>(m, n, l, k, ctx->sm_count, ctx->max_smem);
    if (plan.grid == 0) throw ParameterError("B200 path: problem does not fit the persistent sweep kernel");
    SweepArgs<T> a{};
    a.q = q;
    a.b = b;
    a.w = w;
    a.h = h;
    a.wt = wt;
    a.wn = ctx->d<double>("sw.wn", size_t(k));
    a.tm = ctx->d<double>("sw.tm", size_t(l) * k);
    a.vm = ctx->d<double>("sw.vm", size_t(k) * k);
    a.em = ctx->d<double>("sw.em", size_t(l) * k);
    a.m = m, a.n = n, a.l = l, a.k = k;
    a.flags = kInitWt | kInitWn;
    a.t_begin = 1, a.t_end = 0;
    a.pgrad0 = ctx->d<double>("sw.pgrad0", 1);
    a.trace_objc = ctx->d<double>("sw.tobjc", 1);
    a.trace_pgrad = ctx->d<double>("sw.tpgrad", 1);
    a.trace_time = ctx->d<unsigned long long>("sw.ttime", 1);
    a.status = ctx->d<long long>("sw.status", 3);
    a.barrier = reinterpret_cast<unsigned*>(ctx->sync_block);
    const int64_t plen = sweep_part_len(l, k);
    a.part = ctx->d<double>("sw.part", size_t(2 * plen * plan.grid));
    a.fin = ctx->d<double>("sw.fin", size_t(2 * plen));
    tm.launches += attach_sweep_stream<T>(ctx, plan, a, ctx->stream);
    tm.span(kInit, [&] { tm.launches += launch_sweeps_synced<T>(ctx, eng, a, plan, ctx->stream); });
    eng.export_(q_out, location, q, size_t(m) * l);
    eng.export_(b_out, location, b, size_t(l) * n);
    if (wt_out) {
      T* wt_t = ctx->d<T>("wt.cast", size_t(l) * k);
      // device-side cast of W~ to the call's dtype
      tm.launches += launch_scale_cast<T>(wt, int64_t(l) * k, 1.0, wt_t, ctx->stream);
      eng.export_(wt_out, location, wt_t, size_t(l) * k);
    }
    eng.export_(w_out, location, w, size_t(m) * k);
    eng.export_(h_out, location, h, size_t(k) * n);
  }
  ctx->last.sketch_bytes = eng.sketch_bytes_;
  ctx->last.metrics_bytes = eng.metrics_bytes_;
  ctx->last.sketch_passes = eng.sketch_passes_;
  ctx->last.metrics_passes = eng.metrics_passes_;
  const double xwb = ctx->last.xw_bytes, xtwb = ctx->last.xtw_bytes;
  const int64_t sweeps = ctx->last.sweeps;
  tm.finish(ctx->last);
  ctx->last.xw_bytes = xwb;
  ctx->last.xtw_bytes = xtwb;
  ctx->last.sweeps = sweeps;
  ctx->last.sketch_bytes = eng.sketch_bytes_;
  ctx->last.metrics_bytes = eng.metrics_bytes_;
  ctx->last.sketch_passes = eng.sketch_passes_;
  ctx->last.metrics_passes = eng.metrics_passes_;
}

// hals_fit, p/src/hals.cpp:268-323: the deterministic full-space HALS solver (the reference CLI's
// `--method hals`, the speed-up baseline of `bench`).  Per sweep (UpdateOrder::Grouped): X H^T
// (X pass) and H H^T, the row-parallel W update (kernels_hals.cu), X^T W (X pass) and W^T W, the
// column-parallel H update; every sweep is recorded with the full-space metrics (objective, rel_err,
// pgrad = pgrad_full, objective_compressed = objective) and tested against the stopping rule.
template <typename T>
static void hals_impl(rnmf_gpu_context* ctx, const void* x_in, int location, int64_t m, int64_t n,
                      const rnmf_solver_options& o, const double* w0, const double* h0, void* w_out, void* h_out,
                      rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len) {
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  ctx->last = rnmf_stage_times{};
  Timer tm(ctx);
  Engine<T> eng(ctx, tm);
  eng.set_math(o.math_mode);
  if (m < 0 || n < 0) throw ShapeError("X has negative dimensions " + shape_string(m, n));
  const T* x = nullptr;
  if (m * n > 0) {
    x = eng.import_x(x_in, location, m, n);
    eng.scan(true, nullptr);
  }
  validate_options_after_data(m, n, o);
  check_supported(o);
  if (o.order != RNMF_ORDER_GROUPED)
    throw ParameterError("B200 path: hals_fit supports UpdateOrder::Grouped");
  if (trace_cap < o.max_iter + 1)
    throw ParameterError("trace buffer too small: need " + std::to_string(o.max_iter + 1) + " records, have " +
                         std::to_string(trace_cap));
  const int k = int(o.rank);
  if (k > 64) throw ParameterError("B200 path: rank above 64 is not supported yet");
  cudaStream_t st = ctx->stream;
  T* w = ctx->d<T>("w", size_t(m) * k);
  T* h = ctx->d<T>("h", size_t(k) * n);
  const bool svd_init = o.init == RNMF_INIT_SVD;
  if (svd_init && (w0 || h0)) throw ParameterError("init overrides require InitScheme::Random");
  if (svd_init) {
    nndsvd_init_dev<T>(ctx, eng, tm, o, m, n, m, w, h);
  } else {
    // random_init (p/src/hals.cpp:118-124) from Rng(seed): W then H, scaled by sqrt(mean(X) / k)
    double* uw = ctx->h<double>("init.uw", size_t(m) * k);
    double* uh = ctx->h<double>("init.uh", size_t(k) * n);
    Rng rng(o.seed);
    if (w0)
      std::memcpy(uw, w0, sizeof(double) * size_t(m) * k);
    else
      fill_uniform(rng, uw, size_t(m) * k);
    if (h0)
      std::memcpy(uh, h0, sizeof(double) * size_t(k) * n);
    else
      fill_uniform(rng, uh, size_t(k) * n);
    const double scale = std::sqrt(eng.sum() / double(m * n) / double(k));
    double* uw_d = ctx->d<double>("init.uw.d", size_t(m) * k);
    double* uh_d = ctx->d<double>("init.uh.d", size_t(k) * n);
    tm.span(kH2D, [&] {
      RNMF_CUDA(cudaMemcpyAsync(uw_d, uw, sizeof(double) * size_t(m) * k, cudaMemcpyHostToDevice, st));
      RNMF_CUDA(cudaMemcpyAsync(uh_d, uh, sizeof(double) * size_t(k) * n, cudaMemcpyHostToDevice, st));
    });
    tm.span(kInit, [&] {
      tm.launches += launch_scale_cast<T>(uw_d, int64_t(m) * k, scale, w, st);
      tm.launches += launch_scale_cast<T>(uh_d, int64_t(k) * n, scale, h, st);
    });
  }
  const double x_norm = std::sqrt(eng.sumsq());
  T* xht = ctx->d<T>("hals.xht", size_t(m) * k);
  T* xtw = ctx->d<T>("hals.xtw", size_t(n) * k);
  double* hht = ctx->d<double>("hals.hht", size_t(k) * k);
  double* wtw = ctx->d<double>("hals.wtw", size_t(k) * k);
  double* gpart = ctx->d<double>("hals.gpart", size_t(gram_parts(std::max(m, n))) * k * k);
  double* mres = ctx->d<double>("hals.mres", 2);
  double* hres = ctx->h<double>("hals.mres.h", 2);
  Rng reseed_rng = Rng(o.seed).split(kReseedStream);

  int64_t len = 0;
  auto record = [&](int64_t iter) {
    eng.metrics(k, w, h, mres);
    RNMF_CUDA(cudaMemcpyAsync(hres, mres, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    RNMF_CUDA(cudaStreamSynchronize(st));
    rnmf_trace_record& r = trace[len++];
    r.iter = iter;
    r.objective = hres[0];
    r.rel_err = x_norm > 0.0 ? std::sqrt(hres[0]) / x_norm : 0.0;
    r.pgrad = hres[1];
    r.pgrad_full = hres[1];
    r.objective_compressed = hres[0];
    r.elapsed_s = elapsed();
  };
  record(0);
  const double pgrad0 = trace[0].pgrad;
  const bool pg_rule = o.stopping == RNMF_STOP_PROJECTED_GRADIENT;
  const bool stationary = pg_rule && !(pgrad0 > 0.0);
  std::vector<T> wh, hh;
  for (int64_t iter = 1; iter <= o.max_iter && !stationary; ++iter) {
    tm.span(kSweeps, [&] {
      // W phase (p/src/hals.cpp:172-178)
      tm.launches += launch_gram_cols<T>(h, k, n, gpart, hht, st);
      tm.span(kXw, [&] { eng.gemm_xs(h, k, true, xht); });
      tm.launches += launch_hals_w_update<T>(w, m, k, xht, hht, o.reg.alpha_w, o.reg.beta_w, st);
      // H phase (p/src/hals.cpp:182-193)
      tm.span(kXtw, [&] { eng.gemm_xts(w, k, xtw); });
      tm.launches += launch_gram_rows<T>(w, m, k, gpart, wtw, st);
      tm.launches += launch_hals_h_update<T>(h, n, k, xtw, wtw, o.reg.alpha_h, o.reg.beta_h, st);
    });
    if (o.reseed_dead) {
      // reseed_dead_components (p/src/hals.cpp:96-105), on the host in the reference's draw order
      wh.resize(size_t(m) * k);
      hh.resize(size_t(k) * n);
      RNMF_CUDA(cudaMemcpyAsync(wh.data(), w, sizeof(T) * wh.size(), cudaMemcpyDeviceToHost, st));
      RNMF_CUDA(cudaMemcpyAsync(hh.data(), h, sizeof(T) * hh.size(), cudaMemcpyDeviceToHost, st));
      RNMF_CUDA(cudaStreamSynchronize(st));
      bool changed = false;
      for (int j = 0; j < k; ++j) {
        bool wlive = false, hlive = false;
        for (int64_t i = 0; i < m && !wlive; ++i) wlive = wh[size_t(i) * k + j] > T(0);
        if (!wlive) {
          for (int64_t i = 0; i < m; ++i) wh[size_t(i) * k + j] = T(reseed_rng.uniform() * 1e-4);
          changed = true;
        }
        for (int64_t c = 0; c < n && !hlive; ++c) hlive = hh[size_t(j) * n + c] > T(0);
        if (!hlive) {
          for (int64_t c = 0; c < n; ++c) hh[size_t(j) * n + c] = T(reseed_rng.uniform() * 1e-4);
          changed = true;
        }
      }
      if (changed) {
        RNMF_CUDA(cudaMemcpyAsync(w, wh.data(), sizeof(T) * wh.size(), cudaMemcpyHostToDevice, st));
        RNMF_CUDA(cudaMemcpyAsync(h, hh.data(), sizeof(T) * hh.size(), cudaMemcpyHostToDevice, st));
      }
    }
    record(iter);
    const rnmf_trace_record& last = trace[len - 1];
    if (pg_rule ? last.pgrad < o.tol * pgrad0 : last.objective < o.tol) break;
  }
  *trace_len = len;
  eng.export_(w_out, location, w, size_t(m) * k);
  eng.export_(h_out, location, h, size_t(k) * n);
  RNMF_CUDA(cudaStreamSynchronize(st));
  tm.finish(ctx->last);
  ctx->last.sweeps = len - 1;
  ctx->last.metrics_bytes = eng.metrics_bytes_;
  ctx->last.metrics_passes = eng.metrics_passes_;
}

template <typename T>
static void rqb_impl(rnmf_gpu_context* ctx, const void* a_in, int location, int64_t m, int64_t n, int64_t rank,
                     int64_t p, int64_t qi, int test_matrix, uint64_t seed, const double* omega, int math_mode, void* q_out,
                     void* b_out, int64_t* l_out) {
  ctx->last = rnmf_stage_times{};
  Timer tm(ctx);
  Engine<T> eng(ctx, tm);
  const int64_t l64 = sketch_width(m, n, rank, p, qi);  // ParameterError before the data check
  if (l_out) *l_out = l64;
  if (!q_out && !b_out) {
    tm.finish(ctx->last);
    return;
  }
  const int l = int(l64);
  if (l > tsqr_max_l(ctx->max_smem) || l > 128)
    throw ParameterError("B200 path: sketch width " + std::to_string(l) + " above the supported maximum");
  eng.import_x(a_in, location, m, n);
  eng.scan(false, "rqb: input contains non-finite values");  // p/src/sketch.cpp:54-56
  std::vector<double> om_host;
  const double* om = omega;
  if (!om) {
    om_host.resize(size_t(n) * l);
    Rng rng(seed);
    if (test_matrix == RNMF_TEST_UNIFORM)
      fill_uniform(rng, om_host.data(), om_host.size());
    else
      fill_gaussian(rng, om_host.data(), om_host.size());
    om = om_host.data();
  }
  T* om_dev = eng.upload_converted("omega", om, size_t(n) * l);
  T *q = nullptr, *b = nullptr;
  tm.span(kSketch, [&] { eng.rqb(l, qi, om_dev, math_mode, &q, &b); });
  eng.export_(q_out, location, q, size_t(m) * l);
  eng.export_(b_out, location, b, size_t(l) * n);
  const double xwb = ctx->last.xw_bytes, xtwb = ctx->last.xtw_bytes;
  tm.finish(ctx->last);
  ctx->last.xw_bytes = xwb;
  ctx->last.xtw_bytes = xtwb;
  ctx->last.sketch_bytes = eng.sketch_bytes_;
  ctx->last.sketch_passes = eng.sketch_passes_;
}

// ---- FileColumnSource (p/src/data_io.cpp:185-223): RNMFMAT1 binary matrix, read by column blocks
// (one strided read per row, as the reference).  Header validated up front with the reference's
// messages.
class FileColumns {
 public:
  explicit FileColumns(const std::string& path) : path_(path) {
    f_ = std::fopen(path.c_str(), "rb");
    if (!f_) throw IoError("cannot open '" + path + "'");
    char magic[8] = {};
    const size_t got = std::fread(magic, 1, 8, f_);
    if (got != 8 || std::memcmp(magic, "RNMFMAT1", 8) != 0)
      throw DataError("'" + path + "': bad magic at byte 0 (expected \"RNMFMAT1\")");
    unsigned char hdr[16];
    if (std::fread(hdr, 1, 16, f_) != 16) throw DataError("'" + path + "': truncated header, file ends before byte 24");
    uint64_t rows = 0, cols = 0;
    for (int i = 7; i >= 0; --i) rows = (rows << 8) | hdr[i];
    for (int i = 7; i >= 0; --i) cols = (cols << 8) | hdr[8 + i];
    std::fseek(f_, 0, SEEK_END);
    const uint64_t size = uint64_t(std::ftell(f_));
    const uint64_t expected = 24 + rows * cols * sizeof(double);
    if (size != expected)
      throw DataError("'" + path + "': file is " + std::to_string(size) + " bytes, expected " + std::to_string(expected) +
                      " for a " + std::to_string(rows) + "x" + std::to_string(cols) + " matrix");
    rows_ = int64_t(rows);
    cols_ = int64_t(cols);
  }
  ~FileColumns() {
    if (f_) std::fclose(f_);
  }
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  void read_columns(int64_t first, int64_t count, double* dst) {
    for (int64_t i = 0; i < rows_; ++i) {
      const uint64_t off = 24 + (uint64_t(i) * uint64_t(cols_) + uint64_t(first)) * sizeof(double);
      if (std::fseek(f_, long(off), SEEK_SET) != 0 ||
          std::fread(dst + i * count, sizeof(double), size_t(count), f_) != size_t(count))
        throw IoError("'" + path_ + "': read failed for columns [" + std::to_string(first) + ", " +
                      std::to_string(first + count) + ") at row " + std::to_string(i));
    }
  }

 private:
  std::string path_;
  std::FILE* f_ = nullptr;
  int64_t rows_ = 0, cols_ = 0;
};

static void rqb_streaming_impl(rnmf_gpu_context* ctx, const ColumnReadFn& read, int64_t m, int64_t n, int64_t rank,
                               int64_t p, int64_t qi, int test_matrix, int64_t block_size, uint64_t seed,
                               const double* omega, double* q_out, double* b_out, int64_t* l_out) {
  ctx->last = rnmf_stage_times{};
  Timer tm(ctx);
  Engine<double> eng(ctx, tm);
  const int64_t l64 = sketch_width(m, n, rank, p, qi);  // p/src/sketch.cpp:30-50 (+ the block size check)
  if (block_size < 1) throw ParameterError("sketch: block size must be at least 1");
  if (l_out) *l_out = l64;
  if (!q_out && !b_out) {
    tm.finish(ctx->last);
    return;
  }
  if (!q_out || !b_out) throw ParameterError("rqb_streaming: q_out and b_out must both be given");
  const int l = int(l64);
  if (l > tsqr_max_l(ctx->max_smem) || l > 128)
    throw ParameterError("B200 path: sketch width " + std::to_string(l) + " above the supported maximum");
  const int64_t bs = std::min(block_size, n);
  // Omega from Rng(seed) directly (p/src/sketch.cpp:79-80), row-major n x l
  std::vector<double> om_host;
  const double* om = omega;
  if (!om) {
    om_host.resize(size_t(n) * l);
    Rng rng(seed);
    if (test_matrix == RNMF_TEST_UNIFORM)
      fill_uniform(rng, om_host.data(), om_host.size());
    else
      fill_gaussian(rng, om_host.data(), om_host.size());
    om = om_host.data();
  }
  const double* om_dev = eng.upload_converted("omega", om, size_t(n) * l);
  tm.span(kSketch, [&] { eng.rqb_streaming(read, m, n, l, qi, bs, om_dev, q_out, b_out); });
  tm.finish(ctx->last);
  ctx->last.sketch_bytes = eng.sketch_bytes_;
  ctx->last.sketch_passes = eng.sketch_passes_;
}


// Stage API: rhals_update_W / rhals_update_H on a caller-supplied compressed problem, and the
// fit loop started from one.
template <typename T>
static void stage_impl(rnmf_gpu_context* ctx, int location, const rnmf_problem_shape& s, const void* q_in,
                       const void* b_in, void* wt_io, void* w_io, void* h_io, const rnmf_reg_config& reg, bool do_w,
                       const char* who) {
  ctx->last = rnmf_stage_times{};
  check_problem_shapes(s, who);
  Timer tm(ctx);
  Engine<T> eng(ctx, tm);
  const int64_t m = s.q_rows, n = s.b_cols;
  const int l = int(s.q_cols), k = int(s.w_cols);
  if (m == 0 || n == 0 || l == 0 || k == 0) {
    tm.finish(ctx->last);
    return;
  }
  if (l > 128 || k > 64) throw ParameterError("B200 path: l <= 128 and k <= 64 supported");
  const T* q = eng.import("st.q", q_in, location, size_t(m) * l);
  const T* b = eng.import("st.b", b_in, location, size_t(l) * n);
  T* wt_t = eng.import("st.wt", wt_io, location, size_t(l) * k);
  T* w = eng.import("st.w", w_io, location, size_t(m) * k);
  T* h = eng.import("st.h", h_io, location, size_t(k) * n);
  double* wt = ctx->d<double>("st.wt.d", size_t(l) * k);
  tm.launches += launch_widen<T>(wt_t, int64_t(l) * k, wt, ctx->stream);
  const SweepPlan plan = plan_sweeps<T>(m, n, l, k, ctx->sm_count, ctx->max_smem);
  if (plan.grid == 0) throw ParameterError("B200 path: problem does not fit the persistent sweep kernel");
  SweepArgs<T> a{};
  a.q = q, a.b = b, a.w = w, a.h = h, a.wt = wt;
  a.wn = ctx->d<double>("sw.wn", size_t(k));
  a.tm = ctx->d<double>("sw.tm", size_t(l) * k);
  a.vm = ctx->d<double>("sw.vm", size_t(k) * k);
  a.em = ctx->d<double>("sw.em", size_t(l) * k);
  a.m = m, a.n = n, a.l = l, a.k = k;
  a.alpha_w = reg.alpha_w, a.alpha_h = reg.alpha_h, a.beta_w = reg.beta_w, a.beta_h = reg.beta_h;
  a.flags = do_w ? (kTvOnly | kDoW) : (kInitWn | kDoH);
  a.t_begin = 1, a.t_end = 1;
  a.pgrad0 = ctx->d<double>("sw.pgrad0", 1);
  a.trace_objc = ctx->d<double>("sw.tobjc", 2);
  a.trace_pgrad = ctx->d<double>("sw.tpgrad", 2);
  a.trace_time = ctx->d<unsigned long long>("sw.ttime", 2);
  a.status = ctx->d<long long>("sw.status", 3);
  a.barrier = reinterpret_cast<unsigned*>(ctx->sync_block);
  const int64_t plen = sweep_part_len(l, k);
  a.part = ctx->d<double>("sw.part", size_t(2 * plen * plan.grid));
  a.fin = ctx->d<double>("sw.fin", size_t(2 * plen));
  tm.launches += attach_sweep_stream<T>(ctx, plan, a, ctx->stream);
  tm.span(kSweeps, [&] { tm.launches += launch_sweeps<T>(a, plan, ctx->stream); });
  if (do_w) {
    T* wt_cast = ctx->d<T>("st.wt.cast", size_t(l) * k);
    tm.launches += launch_scale_cast<T>(wt, int64_t(l) * k, 1.0, wt_cast, ctx->stream);
    eng.export_(wt_io, location, wt_cast, size_t(l) * k);
    eng.export_(w_io, location, w, size_t(m) * k);
  } else {
    eng.export_(h_io, location, h, size_t(k) * n);
  }
  tm.finish(ctx->last);
}

template <typename T>
static void fit_compressed_impl(rnmf_gpu_context* ctx, const void* x_in, int location, int64_t m, int64_t n,
                                const rnmf_solver_options& o, const rnmf_problem_shape& s, const void* q_in,
                                const void* b_in, void* wt_io, void* w_io, void* h_io, rnmf_trace_record* trace,
                                int64_t trace_cap, int64_t* trace_len) {
  const auto t0 = std::chrono::steady_clock::now();
  ctx->last = rnmf_stage_times{};
  Timer tm(ctx);
  Engine<T> eng(ctx, tm);
  eng.set_math(o.math_mode);
  const T* x = nullptr;
  if (m * n > 0) {
    x = eng.import_x(x_in, location, m, n);
    eng.scan(true, nullptr);
  }
  validate_options_after_data(m, n, o);
  check_supported(o);
  check_problem_shapes(s, "rhals_fit_compressed");
  if (s.q_rows != m || s.b_cols != n || s.w_cols != o.rank)
    throw ShapeError("rhals_fit_compressed: problem does not match X=" + shape_string(m, n));
  if (trace_cap < o.max_iter + 1)
    throw ParameterError("trace buffer too small: need " + std::to_string(o.max_iter + 1) + " records, have " +
                         std::to_string(trace_cap));
  const int l = int(s.q_cols), k = int(s.w_cols);
  if (l > 128 || k > 64) throw ParameterError("B200 path: l <= 128 and k <= 64 supported");
  const T* q = eng.import("st.q", q_in, location, size_t(m) * l);
  const T* b = eng.import("st.b", b_in, location, size_t(l) * n);
  T* wt_t = eng.import("st.wt", wt_io, location, size_t(l) * k);
  T* w = eng.import("w", w_io, location, size_t(m) * k);
  T* h = eng.import("h", h_io, location, size_t(k) * n);
  double* wt = ctx->d<double>("wt", size_t(l) * k);
  tm.launches += launch_widen<T>(wt_t, int64_t(l) * k, wt, ctx->stream);
  LoopIO<T> io{x, m, n, l, k, q, b, w, h, wt, false};
  run_loop<T>(ctx, eng, tm, o, io, t0, std::sqrt(eng.sumsq()), trace, trace_len);
  T* wt_cast = ctx->d<T>("st.wt.cast", size_t(l) * k);
  tm.launches += launch_scale_cast<T>(wt, int64_t(l) * k, 1.0, wt_cast, ctx->stream);
  eng.export_(wt_io, location, wt_cast, size_t(l) * k);
  eng.export_(w_io, location, w, size_t(m) * k);
  eng.export_(h_io, location, h, size_t(k) * n);
  const int64_t sweeps = ctx->last.sweeps;
  tm.finish(ctx->last);
  ctx->last.sweeps = sweeps;
  ctx->last.metrics_bytes = eng.metrics_bytes_;
  ctx->last.metrics_passes = eng.metrics_passes_;
}

}  // namespace rnmf_gpu

// =================================================================================================
// C ABI
namespace {

void put_err(char* err, size_t cap, const std::string& msg) {
  if (err && cap) {
    const size_t n = std::min(cap - 1, msg.size());
    std::memcpy(err, msg.data(), n);
    err[n] = '\0';
  }
}

template <typename F>
int guarded(char* err, size_t cap, F&& f) {
  try {
    f();
    put_err(err, cap, "");
    return RNMF_OK;
  } catch (const rnmf_gpu::ShapeError& e) {
    put_err(err, cap, e.what());
    return RNMF_SHAPE_ERROR;
  } catch (const rnmf_gpu::ParameterError& e) {
    put_err(err, cap, e.what());
    return RNMF_PARAMETER_ERROR;
  } catch (const rnmf_gpu::DataError& e) {
    put_err(err, cap, e.what());
    return RNMF_DATA_ERROR;
  } catch (const rnmf_gpu::IoError& e) {
    put_err(err, cap, e.what());
    return RNMF_IO_ERROR;
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return RNMF_CUDA_ERROR;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    RNMF_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void check_ctx(const rnmf_gpu_context* ctx) {
  if (!ctx) throw rnmf_gpu::ParameterError("null rnmf_gpu_context");
}
void check_dtype(int dtype, int location) {
  if (dtype != RNMF_F32 && dtype != RNMF_F64) throw rnmf_gpu::ParameterError("dtype must be RNMF_F32 or RNMF_F64");
  if (location != RNMF_HOST && location != RNMF_DEVICE)
    throw rnmf_gpu::ParameterError("location must be RNMF_HOST or RNMF_DEVICE");
}

}  // namespace

extern "C" {

int rnmf_version(char* buf, size_t cap) {
  put_err(buf, cap, "rnmf-b200 0.1.0 (sm_100a; reference rnmf 0.1.0, p/include/rnmf/version.hpp:7)");
  return RNMF_OK;
}

void rnmf_default_options(rnmf_solver_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->rank = 0;
  o->max_iter = 200;
  o->tol = 1e-4;
  o->init = RNMF_INIT_RANDOM;
  o->order = RNMF_ORDER_GROUPED;
  o->stopping = RNMF_STOP_PROJECTED_GRADIENT;
  o->reseed_dead = 0;
  o->seed = 0;
  o->trace_full_every = 10;
  o->oversampling = 20;
  o->power_iterations = 2;
  o->math_mode = RNMF_MATH_EXACT;
}

int rnmf_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rnmf_gpu_context_create(int device, rnmf_gpu_context** out, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    if (!out) throw rnmf_gpu::ParameterError("null output pointer");
    *out = nullptr;
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw rnmf_gpu::CudaError(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                "); the B200 path has no CPU fallback");
    }
    if (device < 0 || device >= count)
      throw rnmf_gpu::ParameterError("device " + std::to_string(device) + " out of range [0, " +
                                     std::to_string(count) + ")");
    DeviceGuard g(device);
    cudaDeviceProp prop{};
    RNMF_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw rnmf_gpu::CudaError("device " + std::to_string(device) + " (" + prop.name +
                                ") is not a Blackwell sm_100 part; this library is built for sm_100a only");
    auto ctx = std::make_unique<rnmf_gpu_context>();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    ctx->max_smem = int(prop.sharedMemPerBlockOptin);
    RNMF_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    RNMF_CUDA(cudaMalloc(&ctx->sync_block, kSweepSyncTotal));
    *out = ctx.release();
  });
}

int rnmf_gpu_comm_unique_id(unsigned char* id_out, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    if (!id_out) throw rnmf_gpu::ParameterError("null id buffer");
    static_assert(sizeof(ncclUniqueId) == RNMF_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    RNMF_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof id);
  });
}

int rnmf_gpu_context_create_sharded(int device, int rank, int world, const unsigned char* id,
                                    rnmf_gpu_context** out, char* err, size_t err_cap) {
  const int st = rnmf_gpu_context_create(device, out, err, err_cap);
  if (st != RNMF_OK) return st;
  rnmf_gpu_context* ctx = *out;
  const int st2 = guarded(err, err_cap, [&] {
    if (!id) throw rnmf_gpu::ParameterError("null communicator id");
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
      throw rnmf_gpu::ParameterError("sharded context: need 0 <= rank < world <= " + std::to_string(kMaxWorld));
    DeviceGuard g(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    RNMF_NCCL(nccl().CommInitRank(&ctx->shard.comm, world, uid, rank));
    ctx->shard.rank = rank;
    ctx->shard.world = world;
    // map every peer's sweep sync block (CUDA IPC over NVLink); own block stays local
    cudaIpcMemHandle_t mine;
    RNMF_CUDA(cudaIpcGetMemHandle(&mine, ctx->sync_block));
    unsigned char* dh = nullptr;
    RNMF_CUDA(cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * (world + 1)));
    RNMF_CUDA(cudaMemcpyAsync(dh + sizeof(cudaIpcMemHandle_t) * world, &mine, sizeof mine, cudaMemcpyHostToDevice,
                              ctx->stream));
    RNMF_NCCL(nccl().AllGather(dh + sizeof(cudaIpcMemHandle_t) * world, dh, sizeof(cudaIpcMemHandle_t), ncclUint8,
                               ctx->shard.comm, ctx->stream));
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(world));
    RNMF_CUDA(cudaMemcpyAsync(all.data(), dh, sizeof(cudaIpcMemHandle_t) * world, cudaMemcpyDeviceToHost, ctx->stream));
    RNMF_CUDA(cudaStreamSynchronize(ctx->stream));
    RNMF_CUDA(cudaFree(dh));
    for (int p = 0; p < world; ++p) {
      if (p == rank) {
        ctx->shard.peer[p] = ctx->sync_block;
      } else {
        void* ptr = nullptr;
        RNMF_CUDA(cudaIpcOpenMemHandle(&ptr, all[size_t(p)], cudaIpcMemLazyEnablePeerAccess));
        ctx->shard.peer[p] = static_cast<unsigned char*>(ptr);
      }
    }
  });
  if (st2 != RNMF_OK) {
    rnmf_gpu_context_destroy(ctx);
    *out = nullptr;
  }
  return st2;
}

void rnmf_gpu_context_destroy(rnmf_gpu_context* ctx) {
  if (!ctx) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->dev)
    if (kv.second.p) cudaFree(kv.second.p);
  for (auto& kv : ctx->pinned)
    if (kv.second.p) cudaFreeHost(kv.second.p);
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  for (int p = 0; p < ctx->shard.world; ++p)
    if (p != ctx->shard.rank && ctx->shard.peer[p]) cudaIpcCloseMemHandle(ctx->shard.peer[p]);
  if (ctx->shard.comm) nccl().CommDestroy(ctx->shard.comm);
  if (ctx->sync_block) cudaFree(ctx->sync_block);
  cudaStreamDestroy(ctx->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete ctx;
}

int rnmf_gpu_last_stage_times(const rnmf_gpu_context* ctx, rnmf_stage_times* out) {
  if (!ctx || !out) return RNMF_PARAMETER_ERROR;
  *out = ctx->last;
  return RNMF_OK;
}

int rnmf_gpu_rhals_fit(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m, int64_t n,
                       const rnmf_solver_options* opts, const double* omega, const double* w0, const double* h0,
                       void* w_out, void* h_out, rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len,
                       char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!opts || !trace || !trace_len) throw rnmf_gpu::ParameterError("null options / trace pointer");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      fit_impl<float>(ctx, x, location, m, n, *opts, omega, w0, h0, w_out, h_out, trace, trace_cap, trace_len,
                      nullptr, nullptr, nullptr, nullptr, true);
    else
      fit_impl<double>(ctx, x, location, m, n, *opts, omega, w0, h0, w_out, h_out, trace, trace_cap, trace_len,
                       nullptr, nullptr, nullptr, nullptr, true);
  });
}

int rnmf_gpu_hals_fit(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m, int64_t n,
                      const rnmf_solver_options* opts, const double* w0, const double* h0, void* w_out, void* h_out,
                      rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!opts || !trace || !trace_len) throw rnmf_gpu::ParameterError("null options / trace pointer");
    if (ctx->shard.world > 0) throw rnmf_gpu::ParameterError("hals_fit runs on a single-GPU context");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      hals_impl<float>(ctx, x, location, m, n, *opts, w0, h0, w_out, h_out, trace, trace_cap, trace_len);
    else
      hals_impl<double>(ctx, x, location, m, n, *opts, w0, h0, w_out, h_out, trace, trace_cap, trace_len);
  });
}

int rnmf_gpu_rhals_fit_sharded(rnmf_gpu_context* ctx, const void* x_local, int dtype, int location,
                               int64_t m_local, int64_t row_offset, int64_t m_total, int64_t n,
                               const rnmf_solver_options* opts, const double* omega, const double* w0_local,
                               const double* h0, void* w_out, void* h_out, rnmf_trace_record* trace,
                               int64_t trace_cap, int64_t* trace_len, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!opts || !trace || !trace_len) throw rnmf_gpu::ParameterError("null options / trace pointer");
    if (ctx->shard.world < 1) throw rnmf_gpu::ParameterError("context is not sharded (rnmf_gpu_context_create_sharded)");
    if (m_local < 1 || row_offset < 0 || m_total < row_offset + m_local || n < 0)
      throw rnmf_gpu::ShapeError("sharded X: rows [" + std::to_string(row_offset) + ", " +
                                 std::to_string(row_offset + m_local) + ") of " + std::to_string(m_total));
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      fit_impl<float>(ctx, x_local, location, m_local, n, *opts, omega, w0_local, h0, w_out, h_out, trace, trace_cap,
                      trace_len, nullptr, nullptr, nullptr, nullptr, true, row_offset, m_total);
    else
      fit_impl<double>(ctx, x_local, location, m_local, n, *opts, omega, w0_local, h0, w_out, h_out, trace,
                       trace_cap, trace_len, nullptr, nullptr, nullptr, nullptr, true, row_offset, m_total);
  });
}

int rnmf_gpu_rhals_fit_compressed(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m,
                                  int64_t n, const rnmf_solver_options* opts, const rnmf_problem_shape* shape,
                                  const void* q, const void* b, void* wt, void* w, void* h, rnmf_trace_record* trace,
                                  int64_t trace_cap, int64_t* trace_len, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!opts || !shape || !trace || !trace_len) throw rnmf_gpu::ParameterError("null argument");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      fit_compressed_impl<float>(ctx, x, location, m, n, *opts, *shape, q, b, wt, w, h, trace, trace_cap, trace_len);
    else
      fit_compressed_impl<double>(ctx, x, location, m, n, *opts, *shape, q, b, wt, w, h, trace, trace_cap, trace_len);
  });
}

int rnmf_gpu_compress(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m, int64_t n,
                      const rnmf_solver_options* opts, const double* omega, const double* w0, const double* h0,
                      void* q_out, void* b_out, void* wt_out, void* w_out, void* h_out, int64_t* l_out, char* err,
                      size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!opts) throw rnmf_gpu::ParameterError("null options");
    DeviceGuard g(ctx->device);
    int64_t dummy_len = 0;
    if (dtype == RNMF_F32)
      fit_impl<float>(ctx, x, location, m, n, *opts, omega, w0, h0, w_out, h_out, nullptr, 0, &dummy_len, q_out,
                      b_out, wt_out, l_out, false);
    else
      fit_impl<double>(ctx, x, location, m, n, *opts, omega, w0, h0, w_out, h_out, nullptr, 0, &dummy_len, q_out,
                       b_out, wt_out, l_out, false);
  });
}

int rnmf_gpu_rqb(rnmf_gpu_context* ctx, const void* a, int dtype, int location, int64_t m, int64_t n,
                 int64_t target_rank, int64_t oversampling, int64_t power_iterations, int test_matrix, uint64_t seed,
                 const double* omega, int math_mode, void* q_out, void* b_out, int64_t* l_out, char* err,
                 size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (math_mode < RNMF_MATH_EXACT || math_mode > RNMF_MATH_TF32) throw rnmf_gpu::ParameterError("invalid math_mode");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      rqb_impl<float>(ctx, a, location, m, n, target_rank, oversampling, power_iterations, test_matrix, seed, omega,
                      math_mode, q_out, b_out, l_out);
    else
      rqb_impl<double>(ctx, a, location, m, n, target_rank, oversampling, power_iterations, test_matrix, seed, omega,
                       math_mode, q_out, b_out, l_out);
  });
}

int rnmf_gpu_rqb_streaming(rnmf_gpu_context* ctx, rnmf_column_reader reader, void* user, int64_t m, int64_t n,
                           int64_t target_rank, int64_t oversampling, int64_t power_iterations, int test_matrix,
                           int64_t block_size, uint64_t seed, const double* omega, double* q_out, double* b_out,
                           int64_t* l_out, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    if (!reader) throw rnmf_gpu::ParameterError("rqb_streaming: reader is NULL");
    if (m < 0 || n < 0) throw rnmf_gpu::ShapeError("rqb_streaming: negative dimensions " + rnmf_gpu::shape_string(m, n));
    DeviceGuard g(ctx->device);
    const rnmf_gpu::ColumnReadFn read = [&](int64_t first, int64_t count, double* dst) {
      if (reader(user, first, count, dst) != 0)
        throw rnmf_gpu::IoError("read_columns: the column source failed for columns [" + std::to_string(first) + ", " +
                                std::to_string(first + count) + ")");
    };
    rnmf_gpu::rqb_streaming_impl(ctx, read, m, n, target_rank, oversampling, power_iterations, test_matrix, block_size,
                                 seed, omega, q_out, b_out, l_out);
  });
}

int rnmf_gpu_rqb_streaming_file(rnmf_gpu_context* ctx, const char* path, int64_t target_rank, int64_t oversampling,
                                int64_t power_iterations, int test_matrix, int64_t block_size, uint64_t seed,
                                const double* omega, double* q_out, double* b_out, int64_t* m_out, int64_t* n_out,
                                int64_t* l_out, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    if (!path) throw rnmf_gpu::ParameterError("rqb_streaming: path is NULL");
    rnmf_gpu::FileColumns src(path);
    if (m_out) *m_out = src.rows();
    if (n_out) *n_out = src.cols();
    DeviceGuard g(ctx->device);
    const rnmf_gpu::ColumnReadFn read = [&](int64_t first, int64_t count, double* dst) {
      src.read_columns(first, count, dst);
    };
    rnmf_gpu::rqb_streaming_impl(ctx, read, src.rows(), src.cols(), target_rank, oversampling, power_iterations,
                                 test_matrix, block_size, seed, omega, q_out, b_out, l_out);
  });
}

int rnmf_gpu_rhals_update_W(rnmf_gpu_context* ctx, int dtype, int location, const rnmf_problem_shape* shape,
                            const void* q, const void* b, void* wt, void* w, const void* h, const rnmf_reg_config* reg,
                            char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!shape || !reg) throw rnmf_gpu::ParameterError("null argument");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      stage_impl<float>(ctx, location, *shape, q, b, wt, w, const_cast<void*>(h), *reg, true, "rhals_update_W");
    else
      stage_impl<double>(ctx, location, *shape, q, b, wt, w, const_cast<void*>(h), *reg, true, "rhals_update_W");
  });
}

int rnmf_gpu_rhals_update_H(rnmf_gpu_context* ctx, int dtype, int location, const rnmf_problem_shape* shape,
                            const void* q, const void* b, const void* wt, const void* w, void* h,
                            const rnmf_reg_config* reg, char* err, size_t err_cap) {
  return guarded(err, err_cap, [&] {
    check_ctx(ctx);
    check_dtype(dtype, location);
    if (!shape || !reg) throw rnmf_gpu::ParameterError("null argument");
    DeviceGuard g(ctx->device);
    if (dtype == RNMF_F32)
      stage_impl<float>(ctx, location, *shape, q, b, const_cast<void*>(wt), const_cast<void*>(w), h, *reg, false,
                        "rhals_update_H");
    else
      stage_impl<double>(ctx, location, *shape, q, b, const_cast<void*>(wt), const_cast<void*>(w), h, *reg, false,
                         "rhals_update_H");
  });
}

}  // extern "C"
