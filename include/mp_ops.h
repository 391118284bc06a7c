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
 * act = 1 (bf16 only; the fused bias-GeLU of a15): C = x, C2 = gelu(x)
 *   with x = alpha A B + bias in fp32, both bf16 [M, N] with ldc / strideC
 *   (tanh form of GeLU, as in the oracle); act = 0: C2 unused.
 * act = 2 (bf16 only; the GeLU backward of a17 fused into the FC2 dgrad GEMM):
 *   C = bf16(x * gelu'(C2)) with x = alpha A B in fp32 and C2 the stored bf16
 *   pre-activation U [M, N] (same ldc / strideC); if colsum != NULL, also
 *   colsum[n] += sum_m C[m, n] (of the stored bf16 values: the FC1 bias
 *   gradient), fp32 atomics.  No bias, no accumulate.
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
  int act;
  void* C2;
  float* colsum;
} mp_gemm_desc;

mp_status mp_op_gemm(mp_dtype dtype, const mp_gemm_desc* g, void* stream);

/* Number of SMs used for persistent grids and the GEMM tile config chosen
 * for a shape (for tests and the bench's roofline bookkeeping):
 * out[0] = BN, out[1] = stages, out[2] = grid size. */
mp_status mp_op_gemm_config(const mp_gemm_desc* g, int* out3);

/* Algorithmic FLOPs of a GEMM call: 2 M N K batch, or for the causal modes
 * only the defined lower-triangular part (Appendix P:574 counts 2Bs^2h per
 * attention product; the causal kernels never execute the upper half). */
double mp_gemm_flops(const mp_gemm_desc* g);

/* Live GEMM profile: while enabled, every bf16 GEMM launch is bracketed by
 * CUDA events on its own stream.  mp_profile_gemm(1) enables and resets,
 * (0) disables; mp_profile_gemm_read synchronises the device and returns the
 * summed algorithmic FLOPs, summed kernel seconds and the launch count. */
mp_status mp_profile_gemm(int enable);
mp_status mp_profile_gemm_read(double* flops, double* seconds, long long* launches);

/* Number of kernels launched by this library since it was loaded. */
long long mp_launch_count(void);

/* LayerNorm over rows of x [R, h] (implied by Eq. (1)'s 13h term, P:344;
 * pre-LN GPT layer, reading #1; biased variance, eps): y = g * xhat + b;
 * per-row fp32 mean / rstd saved for the backward.  h <= 16384 (bf16), 8192 (fp32);
 * the backward takes h <= 8192 (bf16), 4096 (fp32). */
mp_status mp_op_layernorm_fwd(mp_dtype dt, const void* x, const void* g, const void* b, void* y, float* mean,
                              float* rstd, int R, int h, float eps, void* stream);

/* Fused bias-dropout-add + LayerNorm (P:312 fusion; dropout p = 0 here):
 * x1 = r + (y + bias) (stored), out = LN(x1; g, b). */
mp_status mp_op_bda_layernorm_fwd(mp_dtype dt, const void* y, const void* bias, const void* r, void* x1,
                                  const void* g, const void* b, void* out, float* mean, float* rstd, int R, int h,
                                  float eps, void* stream);

/* LayerNorm backward (a17; P:574 counts it with the layer): dx = LN'(dy)
 * (+ dres if non-NULL); dgamma, dbeta (fp32 [h]) are ACCUMULATED (+=).
 * A row kernel (dx) and a column-tile kernel (the column sums). */
mp_status mp_op_layernorm_bwd(mp_dtype dt, const void* dy, const void* x, const void* g, const float* mean,
                              const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta, int R, int h,
                              void* stream);
/* Same, also accumulating the column sums of dres (dres_sum) and of the
 * stored dx (dx_sum), either may be NULL, both need dres: in the layer
 * backward around LN2 these are the bias gradients of FC2 (b2: column sum of
 * the layer's output gradient, P:146 bias added after g) and of the
 * projection (bo: column sum of dX1), taken in the column kernel's pass, so
 * no separate column-sum launches run. */
mp_status mp_op_layernorm_bwd_sums(mp_dtype dt, const void* dy, const void* x, const void* g, const float* mean,
                                   const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta,
                                   float* dres_sum, float* dx_sum, int R, int h, void* stream);

/* Fused bias + tanh-GeLU (reading #3): out = gelu(y + b), y [R, N]. */
mp_status mp_op_bias_gelu_fwd(mp_dtype dt, const void* y, const void* b, void* out, long long R, int N,
                              void* stream);
/* Its backward: du = dh * gelu'(y + b); db (fp32 [N]) += column sums of du. */
mp_status mp_op_bias_gelu_bwd(mp_dtype dt, const void* dh, const void* y, const void* b, void* du, float* db, int R,
                              int N, void* stream);

/* Implicit-causal scale-mask-softmax in place over z matrices
 * [s, s]: P[i, j] = exp(scale S[i,j]) / sum_{k<=i} exp(scale S[i,k]) for
 * j <= i; reads only j <= i; writes j < kend(i) = min(s, 128 (floor(i/128)+1)),
 * zeros for j > i.  s <= 4096 (bf16). */
mp_status mp_op_softmax_causal_fwd(mp_dtype dt, void* S, long long z, int s, float scale, void* stream);
/* Backward in place on dP: dS = P (dP - rowsum(dP P)) scale, same masking. */
mp_status mp_op_softmax_causal_bwd(mp_dtype dt, void* dP, const void* P, long long z, int s, float scale,
                                   void* stream);

/* Fused causal attention core (same result as the
 * scores GEMM + scale-mask-softmax + P.V GEMM of P:312 without materialising
 * the s x s scores): qkv bf16 [s, b, heads, 3, hd] (head-major [q|k|v]),
 * ctx bf16 [s, b, heads, hd] = softmax_causal(Q K^T / sqrt(hd)) V, and lse2
 * fp32 [b*heads, s] = log2 sum_j exp2(log2(e) S[i,j] / sqrt(hd)) (base-2
 * log-sum-exp of each row, kept for the backward).  hd in {32, 64, 96, 128};
 * MP_EUNSUPPORTED otherwise.  bf16 only. */
mp_status mp_op_flash_attn_fwd(const void* qkv, void* ctx, float* lse2, int s, int b, int heads, int hd,
                               void* stream);

/* Backward of mp_op_flash_attn_fwd: writes dQ, dK, dV into the q/k/v slots of
 * dqkv (bf16, same layout as qkv) from qkv, ctx, dctx and lse2; ws is an fp32
 * workspace of mp_op_flash_attn_bwd_ws_floats(s, b, heads, hd) floats (dQ
 * accumulator, D = rowsum(dO o O), and the dK / dV accumulators used when the
 * kernel splits each key tile's query range over several CTAs to fill the SMs
 * at small b * heads).  dK / dV accumulation order then varies run to run. */
long long mp_op_flash_attn_bwd_ws_floats(int s, int b, int heads, int hd);
mp_status mp_op_flash_attn_bwd(const void* qkv, const void* ctx, const void* dctx, const float* lse2, void* dqkv,
                               float* ws, int s, int b, int heads, int hd, void* stream);

/* out[n] += sum_r X[r, n] (bias gradients, fp32 out). */
mp_status mp_op_colsum_accum(mp_dtype dt, const void* X, float* out, int R, int N, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MP_OPS_H_ */
