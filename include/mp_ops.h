/*
 * mp_ops.h -- kernel-level entry points of the PTD-P hot path (arXiv 2104.04473).
 *
 * These are the individual steps that mp_layer_fwd / mp_layer_bwd compose
 * (SURVEY.md Sec. 8(a) rows a3-a18), exported so that each kernel can be
 * parity-tested against the fp64 oracle on the same inputs.  All pointers
 * are DEVICE pointers owned by the caller; all calls are asynchronous on
 * `stream` (cudaStream_t as void*).  `dtype` selects the storage precision
 * of activations and weights (MP_BF16: bf16 storage, fp32 math; MP_FP32:
 * fp32 everywhere).  Matrices are row-major.  Errors: MP_EINVAL for bad
 * shapes / alignment, MP_ECUDA for launch failures.
 */
#ifndef MP_OPS_H_
#define MP_OPS_H_

#include "mp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Batched GEMM  C_z[m, n] (+)= alpha * sum_k A_z(m, k) B_z(k, n) + bias[n]
 * (Appendix: every linear layer and both attention products are
 * such a GEMM; the attention ones are strided-batched over the b*a/t heads
 * without transposes).
 *   A K-major  (a_major = 0): A_z(m, k) = A[z*strideA + m*lda + k]
 *   A MN-major (a_major = 1): A_z(m, k) = A[z*strideA + k*lda + m]
 *   B K-major  (b_major = 0): B_z(k, n) = B[z*strideB + n*ldb + k]
 *   B MN-major (b_major = 1): B_z(k, n) = B[z*strideB + k*ldb + n]
 *   C_z[m, n] = C[z*strideC + m*ldc + n]
 * A, B, bias are in `dtype`; C is fp32 if c_fp32 else `dtype`.
 * accumulate = 1 adds into the existing C (fp32 C only).
 * causal (square attention GEMMs, blocks of 128 rows):
 *   0 full;
 *   1 output tiles entirely above the diagonal are skipped (not written):
 *     scores S = Q K^T and dP = dO V^T, "implicit causal masking";
 *   2 reduction limited to k < min(K, 128*(floor(m/128)+1)): P V and dS K,
 *     whose A operand is zero above the diagonal;
 *   3 reduction limited to k >= 128*floor(m/128): P^T dO and dS^T Q.
 * bf16 runs on the tcgen05 tensor cores (TMA-fed, TMEM accumulators);
 * fp32 runs a SIMT FFMA kernel (tcgen05 has no fp32 kind). */
typedef struct {
  int M, N, K, batch;
  int a_major, b_major;
  const void* A; long long lda, strideA;
  const void* B; long long ldb, strideB;
  void* C; long long ldc, strideC;
  const void* bias;
  int c_fp32;
  int accumulate;
  int causal;
  float alpha;
} mp_gemm_desc;

mp_status mp_op_gemm(mp_dtype dtype, const mp_gemm_desc* g, void* stream);

/* Number of SMs used for persistent grids and the GEMM tile config chosen
 * for a shape (for tests and the bench's roofline bookkeeping):
 * out[0] = BN, out[1] = stages, out[2] = grid size. */
mp_status mp_op_gemm_config(const mp_gemm_desc* g, int* out3);

#ifdef __cplusplus
}
#endif
#endif /* MP_OPS_H_ */
