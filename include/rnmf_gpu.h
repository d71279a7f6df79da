/*
 * rnmf_gpu.h — C-ABI drop-in boundary for the randomized HALS NMF hot path on B200 (sm_100a).
 *
 * Every entry point below replaces one entry of the reference C++ library `rnmf`
 * (citations are path:line into the reference, `p/` = proj/):
 *
 *   rnmf_gpu_rhals_fit            <- rnmf::rhals_fit            p/include/rnmf/rhals.hpp:40, p/src/rhals.cpp:121-213
 *   rnmf_gpu_rhals_fit_compressed <- the sweep/trace loop of rhals_fit started from a given
 *                                    CompressedProblem           p/src/rhals.cpp:128-213
 *   rnmf_gpu_compress             <- rnmf::compress             p/include/rnmf/rhals.hpp:22, p/src/rhals.cpp:84-105
 *   rnmf_gpu_rhals_update_W       <- rnmf::rhals_update_W       p/include/rnmf/rhals.hpp:33, p/src/rhals.cpp:107-114
 *   rnmf_gpu_rhals_update_H       <- rnmf::rhals_update_H       p/include/rnmf/rhals.hpp:27, p/src/rhals.cpp:116-119
 *   rnmf_gpu_rqb                  <- rnmf::rqb                  p/include/rnmf/sketch.hpp:64, p/src/sketch.cpp:52-71
 *   rnmf_gpu_rqb_streaming        <- rnmf::rqb_streaming        p/include/rnmf/sketch.hpp:71, p/src/sketch.cpp:73-116
 *   rnmf_gpu_rqb_streaming_file   <- rqb_streaming(FileColumnSource) p/include/rnmf/data_io.hpp:32-45
 *
 * Types mirror the reference field for field:
 *   rnmf_reg_config      <- RegConfig      p/include/rnmf/hals.hpp:15-20
 *   rnmf_solver_options  <- SolverOptions  p/include/rnmf/hals.hpp:22-38 (+ GPU-only math_mode)
 *   rnmf_trace_record    <- TraceRecord    p/include/rnmf/hals.hpp:45-56
 *
 * Errors: the reference throws ShapeError / ParameterError (std::invalid_argument) and
 * DataError / IoError (std::runtime_error), p/include/rnmf/types.hpp:22-39.  Here every
 * function returns an int status (RNMF_OK or one of the error codes) and writes the same
 * message text the reference would put in e.what() into the caller's `err` buffer.
 *
 * Matrices are dense row-major (the reference Matrix is RowMajor, types.hpp:17).  `dtype`
 * selects the element type of every matrix argument of a call (RNMF_F32 or RNMF_F64);
 * `location` says whether those matrix pointers are host memory or device memory of the
 * context's GPU.  Overrides (omega, w0, h0) are always host double.
 *
 * Calls are synchronous and single-threaded per context (the reference is synchronous and
 * re-entrant on distinct inputs); distinct contexts are independent.
 */
#ifndef RNMF_GPU_H
#define RNMF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------- */
#define RNMF_OK 0
#define RNMF_SHAPE_ERROR 1     /* rnmf::ShapeError      types.hpp:22 */
#define RNMF_PARAMETER_ERROR 2 /* rnmf::ParameterError  types.hpp:27 */
#define RNMF_DATA_ERROR 3      /* rnmf::DataError       types.hpp:32 */
#define RNMF_IO_ERROR 4        /* rnmf::IoError         types.hpp:37 */
#define RNMF_CUDA_ERROR 5      /* CUDA / NCCL runtime failure (no reference equivalent) */

/* ---- enums (values are the C ABI, names follow the reference) -------------------------- */
#define RNMF_INIT_RANDOM 0 /* InitScheme::Random  hals.hpp:9 */
#define RNMF_INIT_SVD 1    /* InitScheme::Svd */

#define RNMF_ORDER_INTERLEAVED 0 /* UpdateOrder  hals.hpp:10 */
#define RNMF_ORDER_GROUPED 1
#define RNMF_ORDER_SHUFFLED 2

#define RNMF_STOP_PROJECTED_GRADIENT 0 /* StoppingRule  hals.hpp:11 */
#define RNMF_STOP_OBJECTIVE 1

#define RNMF_TEST_UNIFORM 0 /* TestMatrixKind  sketch.hpp:7 */
#define RNMF_TEST_GAUSSIAN 1

#define RNMF_F32 0
#define RNMF_F64 1

#define RNMF_HOST 0
#define RNMF_DEVICE 1

/* GPU-only: arithmetic used by the X-streaming GEMMs (the sketch and full-space metrics).
 * EXACT  = plain FMA in the working precision (the verification mode; TF32 disallowed).
 * TF32X3 = tcgen05 kind::tf32 with a 3-term hi/lo split (fp32-equivalent accuracy).
 * TF32   = single-pass tcgen05 kind::tf32. */
#define RNMF_MATH_EXACT 0
#define RNMF_MATH_TF32X3 1
#define RNMF_MATH_TF32 2

/* ---- POD types ------------------------------------------------------------------------- */
typedef struct rnmf_reg_config {
  double alpha_w;
  double alpha_h;
  double beta_w;
  double beta_h;
} rnmf_reg_config;

typedef struct rnmf_solver_options {
  int64_t rank;             /* default 0 (must be set) */
  int64_t max_iter;         /* default 200 */
  double tol;               /* default 1e-4 */
  int32_t init;             /* RNMF_INIT_*, default Random */
  int32_t order;            /* RNMF_ORDER_*, default Grouped */
  int32_t stopping;         /* RNMF_STOP_*, default ProjectedGradient */
  int32_t reseed_dead;      /* bool, default 0 */
  rnmf_reg_config reg;      /* default all zero */
  uint64_t seed;            /* default 0 */
  int64_t trace_full_every; /* default 10 */
  int64_t oversampling;     /* default 20 */
  int64_t power_iterations; /* default 2 */
  int32_t math_mode;        /* GPU-only, RNMF_MATH_*, default EXACT */
  int32_t reserved0;
} rnmf_solver_options;

typedef struct rnmf_trace_record {
  int64_t iter;
  double elapsed_s;
  double objective;            /* ||X - W H||_F^2 */
  double rel_err;              /* ||X - W H||_F / ||X||_F */
  double pgrad;                /* compressed projected-gradient norm^2 */
  double pgrad_full;           /* full-space projected-gradient norm^2 */
  double objective_compressed; /* ||B - W~ H||_F^2 */
} rnmf_trace_record;

/* Shapes of a CompressedProblem (p/include/rnmf/rhals.hpp:11-17) as the caller holds them:
 * Q m x l, B l x n, W~ l x k, W m x k, H k x n.  Checked like check_problem_shapes,
 * p/src/rhals.cpp:11-21. */
typedef struct rnmf_problem_shape {
  int64_t q_rows, q_cols;
  int64_t b_rows, b_cols;
  int64_t wt_rows, wt_cols;
  int64_t w_rows, w_cols;
  int64_t h_rows, h_cols;
} rnmf_problem_shape;

/* Per-stage device timings of the last call on a context (CUDA events, milliseconds).
 * Bytes are algorithmic bytes of X streamed by the X-passes of that call. */
typedef struct rnmf_stage_times {
  double scan_ms;      /* validation / mean / norm pass over X */
  double sketch_ms;    /* all X-streaming GEMMs of rqb */
  double qr_ms;        /* tall-skinny QRs */
  double init_ms;      /* init + W~ = Q^T W */
  double sweeps_ms;    /* persistent HALS sweep kernel(s) */
  double metrics_ms;   /* full-space metrics passes */
  double total_ms;     /* whole call on the device */
  double h2d_ms;       /* host->device copies inside the call */
  double d2h_ms;       /* device->host copies inside the call */
  double sketch_bytes; /* X bytes streamed by sketch GEMMs */
  double metrics_bytes;
  int64_t sketch_passes;
  int64_t metrics_passes;
  int64_t sweeps;
  int64_t kernel_launches; /* kernels of this library launched by the call */
  double xw_ms;            /* time in the X*S kernel (Y = X Omega, Y = X Z) */
  double xtw_ms;           /* time in the X^T*S kernel (X^T Q, Q^T X) */
  int64_t xw_launches;
  int64_t xtw_launches;
  double xw_bytes;
  double xtw_bytes;
  double xw_kernel_ms;     /* the X*S GEMM kernels alone (xw_ms minus operand prep) */
  double xtw_kernel_ms;    /* the X^T*S GEMM kernels alone (xtw_ms minus operand prep and split reduction) */
} rnmf_stage_times;

typedef struct rnmf_gpu_context rnmf_gpu_context;

/* ---- library ----------------------------------------------------------------------------- */
/* Version string, e.g. "rnmf-b200 0.1.0 (reference rnmf 0.1.0, p/include/rnmf/version.hpp:7)". */
int rnmf_version(char* buf, size_t cap);

/* Reference defaults, p/include/rnmf/hals.hpp:22-38. */
void rnmf_default_options(rnmf_solver_options* opts);

/* Number of CUDA devices visible (0 when no driver / no GPU). */
int rnmf_gpu_device_count(void);

/* ---- context ------------------------------------------------------------------------------ */
int rnmf_gpu_context_create(int device, rnmf_gpu_context** out, char* err, size_t err_cap);
void rnmf_gpu_context_destroy(rnmf_gpu_context* ctx);
/* Timings of the most recent call on this context. */
int rnmf_gpu_last_stage_times(const rnmf_gpu_context* ctx, rnmf_stage_times* out);

/* ---- hot path ----------------------------------------------------------------------------- */
/* rhals_fit(X, opts) -> {W, H, trace}.
 * x: m x n (dtype, location).  w_out: m x k, h_out: k x n (same dtype and location as x).
 * omega: optional host double n x l test matrix replacing the draw at p/src/sketch.cpp:57-58
 *        (l = sketch width after clamping).  NULL -> the reference stream: uniform [0,1) from
 *        Rng(Rng(seed).split(3).seed()), p/src/rhals.cpp:89-92.
 * w0, h0: optional host double m x k / k x n unscaled initial draws replacing the two
 *        uniform_matrix calls of random_init, p/src/hals.cpp:118-124 (they are multiplied by
 *        sqrt(mean(X)/k) exactly as there).  NULL -> uniform from Rng(seed), W then H.
 * trace: caller buffer of trace_cap records; *trace_len receives the number written
 *        (<= max_iter + 1).  Fails with RNMF_PARAMETER_ERROR if trace_cap is too small. */
int rnmf_gpu_rhals_fit(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m,
                       int64_t n, const rnmf_solver_options* opts, const double* omega,
                       const double* w0, const double* h0, void* w_out, void* h_out,
                       rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len,
                       char* err, size_t err_cap);

/* rnmf::hals_fit (p/include/rnmf/hals.hpp:92, p/src/hals.cpp:268-323): the deterministic
 * full-space HALS solver, the baseline the reference CLI's `bench` times rHALS against.  Same
 * arguments and trace semantics as rnmf_gpu_rhals_fit without Omega (every record carries the
 * full-space metrics; pgrad = pgrad_full, objective_compressed = objective).  UpdateOrder::Grouped
 * only (ParameterError otherwise); single-GPU contexts. */
int rnmf_gpu_hals_fit(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m,
                      int64_t n, const rnmf_solver_options* opts, const double* w0, const double* h0,
                      void* w_out, void* h_out, rnmf_trace_record* trace, int64_t trace_cap,
                      int64_t* trace_len, char* err, size_t err_cap);

/* The sweep / trace loop of rhals_fit (p/src/rhals.cpp:128-213) started from a caller-supplied
 * compressed problem (Q, B, W~, W, H) instead of compress(X).  W~, W, H are in/out.
 * Used for the two-stage parity of rank-deficient inputs. */
int rnmf_gpu_rhals_fit_compressed(rnmf_gpu_context* ctx, const void* x, int dtype, int location,
                                  int64_t m, int64_t n, const rnmf_solver_options* opts,
                                  const rnmf_problem_shape* shape, const void* q, const void* b,
                                  void* wt, void* w, void* h, rnmf_trace_record* trace,
                                  int64_t trace_cap, int64_t* trace_len, char* err,
                                  size_t err_cap);

/* compress(X, opts) -> {Q m x l, B l x n, W~ l x k, W m x k, H k x n}; *l_out = l.
 * Output buffers must hold m*min(k+p, min(m,n)) etc.  Overrides as in rnmf_gpu_rhals_fit. */
int rnmf_gpu_compress(rnmf_gpu_context* ctx, const void* x, int dtype, int location, int64_t m,
                      int64_t n, const rnmf_solver_options* opts, const double* omega,
                      const double* w0, const double* h0, void* q_out, void* b_out,
                      void* wt_out, void* w_out, void* h_out, int64_t* l_out, char* err,
                      size_t err_cap);

/* rqb(A, SketchOptions{target_rank, oversampling, power_iterations, test_matrix, seed})
 * -> {Q m x l, B l x n}.  omega: optional host double n x l override of the test matrix.
 * When q_out/b_out are NULL only *l_out is computed (sketch_width, p/src/sketch.cpp:30-50). */
int rnmf_gpu_rqb(rnmf_gpu_context* ctx, const void* a, int dtype, int location, int64_t m,
                 int64_t n, int64_t target_rank, int64_t oversampling, int64_t power_iterations,
                 int test_matrix, uint64_t seed, const double* omega, int math_mode,
                 void* q_out, void* b_out, int64_t* l_out, char* err, size_t err_cap);

/* ColumnSource::read_columns (p/include/rnmf/sketch.hpp:26-33): write columns [first, first +
 * count) of the m x n source into dst as an m x count row-major double block; return 0 on
 * success, nonzero on failure (reported as RNMF_IO_ERROR). */
typedef int (*rnmf_column_reader)(void* user, int64_t first, int64_t count, double* dst);

/* rqb_streaming(src, SketchOptions{..., block_size, ...}) -> {Q m x l, B l x n}, fp64
 * (p/include/rnmf/sketch.hpp:71, p/src/sketch.cpp:73-116).  The source is read in column blocks
 * of block_size, 2 + power_iterations passes; Omega from Rng(seed) (or the n x l `omega`
 * override).  q_out (m x l) / b_out (l x n) are host row-major doubles; both NULL: only *l_out. */
int rnmf_gpu_rqb_streaming(rnmf_gpu_context* ctx, rnmf_column_reader reader, void* user, int64_t m,
                           int64_t n, int64_t target_rank, int64_t oversampling,
                           int64_t power_iterations, int test_matrix, int64_t block_size,
                           uint64_t seed, const double* omega, double* q_out, double* b_out,
                           int64_t* l_out, char* err, size_t err_cap);

/* rqb_streaming over FileColumnSource(path) (p/include/rnmf/data_io.hpp:32-45,
 * p/src/data_io.cpp:185-223): the RNMFMAT1 binary format (8-byte magic, rows and cols as
 * little-endian u64, row-major float64 payload).  *m_out / *n_out receive the file's shape; call
 * with q_out = b_out = NULL first to size the outputs. */
int rnmf_gpu_rqb_streaming_file(rnmf_gpu_context* ctx, const char* path, int64_t target_rank,
                                int64_t oversampling, int64_t power_iterations, int test_matrix,
                                int64_t block_size, uint64_t seed, const double* omega,
                                double* q_out, double* b_out, int64_t* m_out, int64_t* n_out,
                                int64_t* l_out, char* err, size_t err_cap);

/* rhals_update_W(cp, reg): in place on wt and w (p/src/rhals.cpp:107-114). */
int rnmf_gpu_rhals_update_W(rnmf_gpu_context* ctx, int dtype, int location,
                            const rnmf_problem_shape* shape, const void* q, const void* b,
                            void* wt, void* w, const void* h, const rnmf_reg_config* reg,
                            char* err, size_t err_cap);

/* rhals_update_H(cp, reg): in place on h (p/src/rhals.cpp:116-119 -> :49-58). */
int rnmf_gpu_rhals_update_H(rnmf_gpu_context* ctx, int dtype, int location,
                            const rnmf_problem_shape* shape, const void* q, const void* b,
                            const void* wt, const void* w, void* h, const rnmf_reg_config* reg,
                            char* err, size_t err_cap);

/* ---- multi-GPU: X sharded by rows, one process per GPU ------------------------ *
 * The reference is single-process/single-node; these entries extend rhals_fit to X row-sharded
 * over `world` GPUs of one node.  Rank 0 calls rnmf_gpu_comm_unique_id and the host program
 * hands the 128 bytes to every rank (e.g. torch.distributed.broadcast_object_list); each rank
 * then creates its context (collective: NCCL communicator + CUDA IPC mapping of the peers' sweep
 * sync blocks) and calls rnmf_gpu_rhals_fit_sharded with the same options (collective).
 * Exchanges: Gram all-reduces inside CholeskyQR (shifted CholeskyQR3 replaces the TSQR fallback),
 * NCCL all-reduces of X^T Q, Q^T X, W^T W, W^T X and the metrics scalars; inside the persistent
 * sweep kernel every column step adds its fixed-point partials into every GPU's accumulators with
 * integer atomics over NVLink (order-free: all GPUs hold bitwise-identical W~), and the
 * W~-init / grad_W sums go through a rank-ordered exchange buffer.  H, B, T, V, E are replicated. */
#define RNMF_COMM_ID_BYTES 128
int rnmf_gpu_comm_unique_id(unsigned char* id_out, char* err, size_t err_cap);
int rnmf_gpu_context_create_sharded(int device, int rank, int world, const unsigned char* id,
                                    rnmf_gpu_context** out, char* err, size_t err_cap);
/* Rows [row_offset, row_offset + m_local) of an m_total x n matrix on this rank.  w0_local: this
 * rank's rows of the unscaled W draw (NULL: the reference stream, of which this rank keeps its
 * rows); omega, h0 as in rnmf_gpu_rhals_fit (identical on every rank).  w_out: m_local x k rows,
 * h_out: k x n (replicated), trace identical on every rank. */
int rnmf_gpu_rhals_fit_sharded(rnmf_gpu_context* ctx, const void* x_local, int dtype, int location,
                               int64_t m_local, int64_t row_offset, int64_t m_total, int64_t n,
                               const rnmf_solver_options* opts, const double* omega,
                               const double* w0_local, const double* h0, void* w_out, void* h_out,
                               rnmf_trace_record* trace, int64_t trace_cap, int64_t* trace_len,
                               char* err, size_t err_cap);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* RNMF_GPU_H */
