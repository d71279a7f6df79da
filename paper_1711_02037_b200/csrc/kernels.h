// kernels.h — host-side launch wrappers of the rnmf-b200 sm_100a kernels.
// Every wrapper enqueues on `stream` and returns the number of kernels it launched.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

namespace rnmf_gpu {

// ---- validation / mean / norm pass over X (kernels_scan.cu) ---------------------------------
// out[0] = sum(X), out[1] = sum(X^2) (fp64, fixed-order reduction).  bad[0] = linear index of
// the first non-finite entry, bad[1] = of the first negative entry (UINT64_MAX if none).
// `part` must hold 2 * scan_grid() doubles.
int scan_grid();
template <typename T>
int launch_scan(const T* x, int64_t count, unsigned long long* bad, double* part, double* out,
                cudaStream_t stream);

// ---- X-streaming GEMMs (kernels_xgemm.cu) ----------------------------------------------------
// Y (m x c) = X (m x n) * S (n x c).  All row-major, leading dims = column counts.
template <typename T>
int launch_xw(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, cudaStream_t stream);
// The same through TMA-fed, register-blocked FMA tiles (kernels_xw.cu); X rows 16-byte aligned.
// spad: scratch of xw_tma_spad_len(n, c) elements (S zero-padded to the kernel's column count).
int64_t xw_tma_spad_len(int64_t n, int c);
// P = X^T S through TMA-fed FMA panels (kernels_xw.cu): part holds splits * n * c, then the fixed
// order split reduction into out (n x c, or c x n with transpose_out); spad: xw_tma_spad_len(m, c)
int xtw_tma_splits(int64_t m, int64_t n, int sm_count);
template <typename T>
int launch_xtw_tma(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits, T* out,
                   bool transpose_out, T* spad, int sm_count, cudaStream_t stream);
template <typename T>
int launch_xw_tma(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* y, T* spad, int sm_count,
                  cudaStream_t stream);

// Fused full-space metrics pass 1 over X: with S = H^T (n x k) and W (m x k):
//   part_obj[b]  = partial sum of (X - W H)^2 over CTA b's rows
//   part_pgw[b]  = partial sum of projected (grad_W)^2, grad_W = -2 (X H^T - W (H H^T))
// hht: k x k fp64.  Returns launches; *nblocks receives the number of partials written.
template <typename T>
int launch_xw_metrics(const T* x, int64_t m, int64_t n, int64_t ldx, const T* ht, const T* w, int k,
                      const double* hht, double* part_obj, double* part_pgw, int* nblocks,
                      cudaStream_t stream);
int xw_metrics_blocks(int64_t m);

// P (n x c) = X^T (n x m) * S (m x c), split over m into `splits` partial sums (part holds
// splits * n * c values of T), then reduced in fixed order into `out` (n x c, or c x n when
// transpose_out).  splits = 0 picks a default.
template <typename T>
int launch_xtw(const T* x, int64_t m, int64_t n, int64_t ldx, const T* s, int c, T* part, int splits, T* out,
               bool transpose_out, cudaStream_t stream);
// fixed-order reduction of split partials part[s][n][c] -> out (n x c, or c x n)
template <typename T>
int launch_splitk_reduce(const T* part, int splits, int64_t n, int c, T* out, bool transpose_out, cudaStream_t stream);
int xtw_default_splits(int64_t m, int64_t n);

// Metrics pass 2: with S = W (m x k): part_pgh[b] = partial sums of projected (grad_H)^2,
// grad_H = -2 (W^T X - (W^T W) H), wtw: k x k fp64.  part holds splits*n*k values of T.
template <typename T>
int launch_xtw_metrics(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, int k, const T* h,
                       const double* wtw, T* part, int splits, double* part_pgh, int* nblocks,
                       cudaStream_t stream);

// grad_H projected norm from W^T X split partials part[s][n][k] (fixed-order sum over s);
// writes grad_h_blocks(n, k) partial sums to part_pgh
int64_t grad_h_blocks(int64_t n, int k);
template <typename T>
int launch_grad_h_reduce(const T* part, int splits, int64_t n, int k, const T* h, const double* wtw, double* part_pgh,
                         int* nblocks, cudaStream_t stream);

// ---- fused one-pass metrics (kernels_metrics.cu): objective from the explicit residual, projected
// grad_W, and (when wtx_part != nullptr) per-CTA partials of W^T X (metrics_grid(m) x n x k).
// X (pitch ldx, 16-byte aligned rows) and a zero-padded copy of H (metrics_hpad_len(k, n) elements of
// scratch `hpad`) are streamed by TMA.
int metrics_grid(int64_t m, int k, int elem_bytes, int sm_count);
int64_t metrics_hpad_len(int k, int64_t n);
template <typename T>
int launch_metrics_fused(const T* x, int64_t m, int64_t n, int64_t ldx, const T* w, const T* h, int k,
                         const double* hht, T* hpad, T* wtx_part, double* part_obj, double* part_pgw, int sm_count,
                         cudaStream_t stream);
// 2-D row-major tensor map (rows x cols, pitch in elements), box = box_rows x box_cols, zero fill
// out of bounds; swizzle128: SWIZZLE_128B (box rows of 128 bytes, 16-byte chunk index XOR row % 8)
CUtensorMap make_tma_2d(const void* base, int elem_bytes, int64_t rows, int64_t cols, int64_t pitch, int box_cols,
                        int box_rows, bool swizzle128 = false);

// ---- small dense helpers (kernels_xgemm.cu) ---------------------------------------------------
// G (c x c, fp64) = A^T A for A (rows x c) row-major.  part: gram_parts(rows)*c*c doubles.
template <typename T>
int launch_gram_rows(const T* a, int64_t rows, int c, double* part, double* g, cudaStream_t stream);
// G (c x c, fp64) = A A^T for A (c x cols) row-major.
template <typename T>
int launch_gram_cols(const T* a, int c, int64_t cols, double* part, double* g, cudaStream_t stream);
int gram_parts(int64_t len);
// out (cols x rows) = in (rows x cols)^T
template <typename T>
int launch_transpose(const T* in, int64_t rows, int64_t cols, T* out, cudaStream_t stream);
// out[i] = (T)(in[i] * scale)
template <typename T>
int launch_scale_cast(const double* in, int64_t count, double scale, T* out, cudaStream_t stream);
// out[i] = (double)in[i]
template <typename T>
int launch_widen(const T* in, int64_t count, double* out, cudaStream_t stream);
// sum of `count` doubles in fixed order -> out[0]
int launch_sum_parts(const double* part, int count, double* out, cudaStream_t stream);
// res[0] = sum of pobj, res[1] = sum of ppgw + sum of ppgh (one launch)
int launch_metrics_finalize(const double* pobj, int nobj, const double* ppgw, int npgw, const double* ppgh, int npgh,
                            double* res, cudaStream_t stream);
// out[e] = sum_p part[p * len + e], fixed order
int launch_reduce_parts(const double* part, int nparts, int len, double* out, cudaStream_t stream);
// writes %globaltimer to *out
int launch_timestamp(unsigned long long* out, cudaStream_t stream);

// ---- tcgen05 tensor-core X-streaming GEMMs (kernels_tc.cu, fp32 X only) ------------------------
int tc_npad(int c);               // UMMA N for c output columns (multiple of 16)
void tc_set_chunk(int stages);    // K stages per TMEM accumulation chunk (tests / probes)
int64_t tc_st_pitch(int64_t n);   // pitch of the S^T operand
// S (n x c) -> S^T split into tf32 hi and fp32 lo parts (tc_npad(c) x tc_st_pitch(n) each)
int launch_tc_prep_st(const float* s, int64_t n, int c, float* st_hi, float* st_lo, cudaStream_t stream,
                      bool raw);
// Y (m x c) = X (m x n, pitch ldx) * S; x3 = 3xTF32 (fp32-accurate), else 1xTF32
int launch_tc_xw(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo, int c,
                 float* y, bool x3, int sm_count, cudaStream_t stream);

// part[split] (n x c) = X[rows of split]^T S[rows of split]; S^T given as st (tc_npad(c) x
// tc_st_pitch(m), K-major).  The caller reduces the splits.
int tc_xtw_splits(int64_t m, int64_t n, int sm_count);
int launch_tc_xtw(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st, const float* st_lo, int c,
                  float* part, int splits, bool x3, int sm_count, cudaStream_t stream);

// ---- tall-skinny QR (kernels_tsqr.cu) ---------------------------------------------------------
// Householder TSQR of A (rows x l, row-major) -> explicit thin Q (rows x l, written to q_out in
// T).  Workspace sized by tsqr_workspace_doubles.  Requires rows >= l.
int64_t tsqr_workspace_doubles(int64_t rows, int l, int max_smem);
template <typename T>
int launch_tsqr(const T* a, int64_t rows, int l, T* q_out, double* ws, int max_smem,
                cudaStream_t stream);
int tsqr_max_l(int max_smem);

// ---- CholeskyQR2 fast path (kernels_cholqr.cu) -------------------------------------------------
// Q (rows x l) of A via two fp64-Gram CholeskyQR passes; *flag (device) is set non-zero when A is
// too ill-conditioned for CholeskyQR2 (the caller then runs TSQR).  l <= 128.
int64_t cholqr_workspace_doubles(int64_t rows, int l);
// Row-sharded QR: `allreduce` sums the l x l fp64 Gram (device) over the GPUs holding the other
// rows before every Cholesky.  shift_rel > 0: shifted CholeskyQR3 (G + shift_rel * trace(G) * I in
// the first pass, then two plain passes) -- the sharded replacement of the TSQR fallback.
using GramAllreduce = std::function<void(double* gram, int64_t count)>;
template <typename T>
int launch_cholqr2(const T* a, int64_t rows, int l, T* q_out, double* ws, int* flag, cudaStream_t stream,
                   const GramAllreduce* allreduce = nullptr, double shift_rel = 0.0);

// ---- NNDSVD init (kernels_nndsvd.cu) ------------------------------------------------------------
// eigen-decomposition of a symmetric l x l fp64 matrix (l <= 64): eval descending, evec columns
int launch_jacobi_eig(const double* g, int l, double* eval, double* evec, cudaStream_t stream);
int nndsvd_norm_blocks(int64_t rows);
// part[b][j][2] = block partial sums of squares of the positive / negative parts of column j of
// u = S U(:, :k) diag(colscale) (S rows x l, or l x rows when `transpose`); U is l x l.
template <typename T>
int launch_nndsvd_norms(const T* s, int64_t rows, int l, bool transpose, const double* u, int k,
                        const double* colscale, double* part, cudaStream_t stream);
// out = coef-weighted positive / negative part of u, zeros -> fill (rows x k, or k x rows)
template <typename T>
int launch_nndsvd_apply(const T* s, int64_t rows, int l, bool transpose, const double* u, int k,
                        const double* colscale, const double* coef, double fill, T* out, bool out_transposed,
                        cudaStream_t stream);

// ---- deterministic full-space HALS factor updates (kernels_hals.cu) -----------------------------
// W (m x k) <- clamped_col_update over j with P = X H^T (m x k), G = H H^T (k x k, fp64)
template <typename T>
int launch_hals_w_update(T* w, int64_t m, int k, const T* xht, const double* hht, double alpha, double beta,
                         cudaStream_t st);
// H (k x n) <- clamped_row_update over j with P = X^T W (n x k), G = W^T W
template <typename T>
int launch_hals_h_update(T* h, int64_t n, int k, const T* xtw, const double* wtw, double alpha, double beta,
                         cudaStream_t st);

// ---- persistent compressed-HALS sweep kernel (kernels_sweeps.cuh) ----------------------------
enum SweepFlags : int {
  kInitWt = 1,    // W~ <- Q^T W
  kInitWn = 2,    // wn <- diag(W^T W)
  kEval0 = 4,     // record 0: objc0, pgrad0 (grad_h = -2 W~^T residc), T, V, E
  kTvOnly = 8,    // T, V from the current H (no record)
  kDoW = 16,      // W phase in each sweep
  kDoH = 32,      // H phase (+ evaluation) in each sweep
  kRecord = 64,   // write trace entries / stop checks
  kColOrdered = 128,  // column-step reduction through ordered fp64 partials (else fixed-point atomics)
  kReseed = 256,      // reseed_dead: liveness stamps per sweep, stop at a dead component (host reseeds)
  kEvalPrev = 512,    // evaluate + record sweep t_begin - 1 first (after a host-side reseed)
  kXFlat = 1024,      // row-sharded column step: every CTA exchanges with every GPU (testing knob)
  kHWarpCols = 2048,  // H phase on the warp-per-column path even where lane-per-column fits (testing knob)
};
// Sync block of the sweep kernel (zeroed before every launch): the legacy grid-barrier counter at
// byte 0 (cross-GPU counter at byte 64), a 3-slot ring of 64-bit fixed-point accumulators for the
// column step, then the replicated grid-barrier counters.  Both the accumulators and the barrier
// counter are replicated on separate 128-byte L2 lines (CTA g uses replica g % reps; readers sum
// the replicas -- integer sums, so the result is exact and order-free): the 148 same-address
// atomics of one column step become 148 / reps per line.
constexpr int kColAccMax = 136;      // entries per slot, >= l + 1
constexpr int kColAccSpacing = 16;   // words between entries: one 128-byte L2 line per entry (the
                                     // atomics of different entries do not serialise on a line)
constexpr int kColAccReps = 4;       // accumulator replicas per entry
constexpr int kColAccStride = kColAccReps * kColAccMax * kColAccSpacing;  // words per slot
constexpr int kBarReps = 8;          // grid-barrier counter replicas (one 128-byte line each)
constexpr size_t kSweepBarOffset = 128 + 3 * size_t(kColAccStride) * sizeof(unsigned long long);
// Row-sharded column step (hierarchical): every GPU's CTA 0 adds its GPU's column sums into every
// GPU's global accumulators (3-slot ring, one line per entry), arrives on every GPU's CTA-0
// counter, and releases its own GPU's CTAs through the flag.
constexpr size_t kSweepGaccOffset = kSweepBarOffset + size_t(kBarReps) * 128;
constexpr size_t kSweepXcolOffset = kSweepGaccOffset + 3 * size_t(kColAccMax) * kColAccSpacing * sizeof(unsigned long long);
constexpr size_t kSweepFlagOffset = kSweepXcolOffset + 128;
// zeroed part: counters (bytes 0 / 64), accumulators, replicated barrier counters, the sharded
// column-step accumulators / counter / flag
constexpr size_t kSweepSyncBytes = kSweepFlagOffset + 128;
// Row-sharded runs (one process per GPU): after the zeroed part, a 2-slot exchange buffer of
// kMaxWorld x kXMax doubles per slot that peers write into (never needs clearing).
constexpr int kMaxWorld = 8;
constexpr int kXMax = 128 * 64 + 64;  // >= l * k + k
constexpr size_t kSweepXbufOffset = kSweepSyncBytes;
constexpr size_t kSweepSyncTotal = kSweepSyncBytes + 2 * size_t(kMaxWorld) * kXMax * sizeof(double);

template <typename T>
struct SweepArgs {
  const T* q;  // m x l
  const T* b;  // l x n
  T* w;        // m x k (in/out)
  T* h;        // k x n (in/out)
  double* wt;  // l x k (in/out state)
  double* wn;  // k
  double* tm;  // l x k  (T = B H^T)
  double* vm;  // k x k  (V = H H^T)
  double* em;  // l x k  (E = residc H^T)
  int64_t m, n;
  int l, k;
  double alpha_w, alpha_h, beta_w, beta_h;
  int flags;
  int64_t t_begin, t_end;  // sweeps t_begin..t_end (inclusive)
  int stop_rule;           // RNMF_STOP_*
  double tol;
  double* pgrad0;          // device scalar (written by kEval0)
  double* trace_objc;      // [max_iter + 1]
  double* trace_pgrad;     // [max_iter + 1]
  unsigned long long* trace_time;  // [max_iter + 1]
  long long* status;       // [0] = last recorded sweep, [1] = stopped flag, [2] = sweep to reseed (0: none)
  unsigned* alive;         // reseed_dead: [2k] last sweep in which W(:,j) / H(j,:) had a positive entry
  unsigned* barrier;       // sync block (kSweepSyncTotal; the first kSweepSyncBytes zeroed before launch)
  // row sharding: this process is `rank` of `world` GPUs; peer_sync[p] = GPU p's sync block mapped
  // into this process (peer_sync[rank] = barrier); xtotal = sum of the grids of all ranks.
  // world == 0: single-GPU kernel (no cross-GPU steps).
  int world, rank;
  long long xtotal;
  unsigned char* peer_sync[kMaxWorld];
  double* part;            // [2 * sweep_part_len(l,k) * grid]  (two alternating slots)
  double* fin;             // [2 * sweep_part_len(l,k)]
  long long* prof;         // optional: per-phase cycle counters of CTA 0 (kSweepProfSlots)
  const int* order;        // Interleaved / Shuffled: component order, k per sweep of t_begin..t_end
                           // (nullptr: Grouped)
  // fp32 streamed-Q path (SweepPlan::f32s): Q re-laid out as float4 columns, q4[i4 * m + r] =
  // Q(r, 4 i4 .. 4 i4 + 3) (zero past l; sweep_relayout_q), and a k x m column-major W scratch the
  // launch works in (W is transposed in at the start of the launch and back at the end)
  const float* q4;
  float* wc;
  // SweepPlan::wide: residc (l x n) in global memory
  T* rc;
};
// q4 (ceil(l_pad / 4) float4 columns of m rows) from row-major Q (m x l); l_pad = SweepPlan::lreg
int sweep_relayout_q(const float* q, int64_t m, int l, int l_pad, float* q4, cudaStream_t stream);
bool sweep_prof_compiled();  // built with RNMF_SWEEP_PROF=1
constexpr int kSweepProfSlots = 17;  // 16 buckets + barrier count

__host__ __device__ inline int64_t sweep_part_len(int l, int k) {
  const int64_t a = 2 * int64_t(l) * k + int64_t(k) * k + 2;
  const int64_t b = int64_t(l) * k + k;
  const int64_t c = a > b ? a : b;
  return c > l + 1 ? c : int64_t(l) + 1;
}
// Returns the cooperative grid size that will be used (0 if the problem does not fit).
struct SweepPlan {
  int grid = 0;
  bool q_in_smem = false;
  size_t smem = 0;
  int64_t rows_per_cta = 0;
  int64_t cols_per_cta = 0;
  int lreg = 0;  // > 0: Q rows register-resident (rows_per_cta <= 256, l + 1 <= lreg <= 64)
  int qring = 0;  // > 0: streamed slabs through a shared-memory bulk-copy ring of that many stages
  bool f32s = false;  // fp32 X, Q slab not resident: coalesced float4-column Q (SweepArgs::q4), fp32
                      // FMA lift / recompress, column-major W scratch (SweepArgs::wc); lreg = padded l
  bool wide = false;  // B / H / residc column slabs in global memory (SweepArgs::rc), no P = W~ V in
                      // shared memory: for n or l x k too large for the shared-memory slabs (C5)
};
template <typename T>
SweepPlan plan_sweeps(int64_t m, int64_t n, int l, int k, int sm_count, int max_smem);
template <typename T>
// zero_sync = false: the caller has zeroed the sync block (row-sharded runs zero it, then pass an
// NCCL all-reduce so no GPU's kernel can touch a peer's block before the peer zeroed it)
int launch_sweeps(const SweepArgs<T>& args, const SweepPlan& plan, cudaStream_t stream, bool zero_sync = true);

}  // namespace rnmf_gpu
