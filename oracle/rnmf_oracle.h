/*
 * rnmf_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of the CPU oracle: an fp64 C++ restatement of the reference rnmf hot path
 * (p/src/rhals.cpp, p/src/sketch.cpp, p/src/hals.cpp, p/src/core.cpp, p/include/rnmf/types.hpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it; the product (paper_1711_02037_b200/, librnmf_gpu.so) never does.
 *
 * Parity status: the reference itself cannot be compiled in this container (Eigen3, CLI11 and
 * doctest are absent), so there are no reference-produced output vectors.  The
 * oracle is pinned against (1) the C++ standard's mt19937_64 known answer and the SURVEY's Rng
 * known answers, (2) every known-answer test of the reference suites on this path (hand
 * examples, QR 3-4-5, objective 14, pgrad 16), and (3) the reference's property tests
 * (p/tests/test_rhals.cpp, test_sketch.cpp, test_hals.cpp, acceptance.cpp), re-run against
 * this oracle in tests/test_oracle_*.py.  Bitwise Eigen parity is not claimed.
 *
 * Matrices are row-major double.  Status codes and structs are those of include/rnmf_gpu.h.
 */
#ifndef RNMF_ORACLE_H
#define RNMF_ORACLE_H

#include "../include/rnmf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* threads used by the large GEMM-like loops (1 = the reference's single-threaded Eigen). */
void oracle_set_threads(int threads);

/* ---- Rng (p/include/rnmf/types.hpp:55-102) ---- */
uint64_t oracle_rng_split_seed(uint64_t seed, uint64_t stream);
void oracle_rng_u64(uint64_t seed, int64_t count, uint64_t* out);
void oracle_rng_uniform(uint64_t seed, int64_t count, double* out);
void oracle_rng_gaussian(uint64_t seed, int64_t count, double* out);
/* uniform_matrix / gaussian_matrix (p/src/core.cpp:20-42), row-major draw order. */
int oracle_uniform_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out, char* err,
                          size_t cap);
int oracle_gaussian_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out, char* err,
                           size_t cap);

/* ---- core ---- */
/* economic_qr (p/src/core.cpp:7-16): Householder thin QR, explicit Q (rows x cols), R. */
int oracle_economic_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r,
                       char* err, size_t cap);
/* synth_lowrank (p/src/data_io.cpp:171-183). */
int oracle_synth_lowrank(int64_t rows, int64_t cols, int64_t rank, double noise, uint64_t seed,
                         double* out, char* err, size_t cap);

/* ---- sketch ---- */
int oracle_sketch_width(int64_t rows, int64_t cols, int64_t target_rank, int64_t oversampling,
                        int64_t power_iterations, int64_t block_size, int64_t* l_out, char* err,
                        size_t cap);
int oracle_rqb(const double* a, int64_t m, int64_t n, int64_t target_rank, int64_t oversampling,
               int64_t power_iterations, int test_matrix, uint64_t seed, const double* omega,
               double* q_out, double* b_out, int64_t* l_out, char* err, size_t cap);

/* rqb_streaming over an in-memory column source (p/src/sketch.cpp:73-116) */
int oracle_rqb_streaming(const double* a, int64_t m, int64_t n, int64_t target_rank, int64_t oversampling,
                         int64_t power_iterations, int test_matrix, int64_t block_size, uint64_t seed,
                         const double* omega, double* q_out, double* b_out, int64_t* l_out, char* err,
                         size_t cap);

/* ---- deterministic HALS helpers (p/src/hals.cpp) ---- */
int oracle_init_factors(const double* x, int64_t m, int64_t n, int64_t rank, int scheme,
                        uint64_t seed, double* w_out, double* h_out, char* err, size_t cap);
int oracle_update_W(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                    const double* h, const rnmf_reg_config* reg, double* w_out, char* err,
                    size_t cap);
int oracle_update_H(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                    const double* h, const rnmf_reg_config* reg, double* h_out, char* err,
                    size_t cap);
int oracle_objective(const double* x, int64_t m, int64_t n, int64_t k, const double* w,
                     const double* h, double* out, char* err, size_t cap);
int oracle_projected_gradient_norm(const double* x, int64_t m, int64_t n, int64_t k,
                                   const double* w, const double* h, double* out, char* err,
                                   size_t cap);
int oracle_hals_fit(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                    double* w_out, double* h_out, rnmf_trace_record* trace, int64_t trace_cap,
                    int64_t* trace_len, char* err, size_t cap);

/* ---- randomized HALS (p/src/rhals.cpp) ---- */
int oracle_compress(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                    const double* omega, const double* w0, const double* h0, double* q_out,
                    double* b_out, double* wt_out, double* w_out, double* h_out, int64_t* l_out,
                    char* err, size_t cap);
int oracle_rhals_update_W(const rnmf_problem_shape* shape, const double* q, const double* b,
                          double* wt, double* w, const double* h, const rnmf_reg_config* reg,
                          char* err, size_t cap);
int oracle_rhals_update_H(const rnmf_problem_shape* shape, const double* q, const double* b,
                          const double* wt, const double* w, double* h,
                          const rnmf_reg_config* reg, char* err, size_t cap);
int oracle_rhals_fit(const double* x, int64_t m, int64_t n, const rnmf_solver_options* opts,
                     const double* omega, const double* w0, const double* h0, double* w_out,
                     double* h_out, rnmf_trace_record* trace, int64_t trace_cap,
                     int64_t* trace_len, char* err, size_t cap);
int oracle_rhals_fit_compressed(const double* x, int64_t m, int64_t n,
                                const rnmf_solver_options* opts, const rnmf_problem_shape* shape,
                                const double* q, const double* b, double* wt, double* w,
                                double* h, rnmf_trace_record* trace, int64_t trace_cap,
                                int64_t* trace_len, char* err, size_t cap);

#ifdef __cplusplus
}
#endif

#endif
