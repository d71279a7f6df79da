// tc_metrics.h — full-space metrics on the tcgen05 tensor cores (math_mode TF32X3, fp32 X),
// kernels_tc.cu.  Three X passes instead of the FFMA kernel's one, each at tensor-core rates:
//   X H^T (m x k)   launch_tc_xw with S^T = H            -> projected grad_W (launch_tc_pgw)
//   X^T W (n x k)   launch_tc_xtw with S = W             -> projected grad_H (launch_grad_h_reduce)
//   ||X - W H||^2   launch_tc_resid (explicit residual, as p/src/rhals.cpp:141 computes it)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rnmf_gpu {

// S^T operand of launch_tc_xw from rows that are already transposed: src (c x n, pitch n) ->
// st_hi / st_lo (tc_npad(c) x tc_st_pitch(n)), hi = rna_tf32, lo = rna_tf32(v - hi)
int launch_tc_prep_rows(const float* src, int c, int64_t n, float* st_hi, float* st_lo, cudaStream_t stream);

// Residual pass.  K extent of the W tile (32 or 64; k <= 64)
int tc_resid_kw(int k);
// hi / lo split operands: W (m x k) -> w_hi / w_lo (m x kw), H (k x n) -> H^T hi / lo
// (tc_st_pitch(n) x kw), zero padded
int launch_tc_resid_prep(const float* w, int64_t m, const float* h, int64_t n, int k, float* w_hi, float* w_lo,
                         float* ht_hi, float* ht_lo, cudaStream_t stream);
// part_obj[b] (fp64) = sum over CTA b's 128-row tiles of (X - W H)^2, W H by 3xTF32 UMMAs;
// returns the number of partials via *nblocks
int launch_tc_resid(const float* x, int64_t m, int64_t n, int64_t ldx, const float* w_hi, const float* w_lo,
                    const float* ht_hi, const float* ht_lo, int k, double* part_obj, int* nblocks, int sm_count,
                    cudaStream_t stream);
int tc_resid_blocks(int64_t m, int sm_count);

// part_pgw[b] = partial sums of the projected grad_W^2, grad_W = -2 (XH^T - W (H H^T)) (fp64 math
// on the fp32 X H^T, W and the fp64 H H^T); returns the number of partials via *nblocks
// k <= 32: X H^T and the residual partials in ONE X pass (operands as for launch_tc_xw with
// S^T = H via launch_tc_prep_rows, and launch_tc_resid_prep); part_obj holds tc_resid_blocks(m)
int launch_tc_xht_resid(const float* x, int64_t m, int64_t n, int64_t ldx, const float* st_hi, const float* st_lo,
                        const float* w_hi, const float* w_lo, const float* ht_hi, const float* ht_lo, int k, float* xht,
                        double* part_obj, int* nblocks, int sm_count, cudaStream_t stream);

// every operand split of one evaluation in one launch: launch_tc_prep_rows(H) + launch_tc_resid_prep
// + launch_tc_prep_st(W) (sw_hi / sw_lo: tc_npad(k) x tc_st_pitch(m))
int launch_tc_metrics_prep(const float* w, int64_t m, const float* h, int64_t n, int k, float* st_hi, float* st_lo,
                           float* w_hi, float* w_lo, float* ht_hi, float* ht_lo, float* sw_hi, float* sw_lo,
                           cudaStream_t stream);

int launch_tc_pgw(const float* xht, const float* w, int64_t m, int k, const double* hht, double* part_pgw,
                  int* nblocks, cudaStream_t stream);
int tc_pgw_blocks(int64_t m);

}  // namespace rnmf_gpu
