// Memory-bound kernels of the hot path (SURVEY 8(a) rows a3, a4, a8, a12,
// a13, a15, a17, a18, a20): LayerNorm, fused bias-dropout-add(+LayerNorm),
// fused bias-GeLU, implicit-causal scale-mask-softmax, vocab-parallel
// embedding and cross-entropy, column reductions for bias gradients, Adam.
// All are coalesced, 16-byte vectorised, fp32 math with warp-shuffle
// reductions; templated on the storage type T (float or __nv_bfloat16).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/mp.h"
#include "dropout.cuh"

namespace mp {

// Rows of the causal softmax output that later GEMMs may read: P[i, j] is
// written for j < kend(i) = min(s, 128 (floor(i/128) + 1)), zero for j > i.
__host__ __device__ inline int causal_kend(int i, int s) { return min(s, ((i >> 7) + 1) << 7); }

template <class T>
mp_status layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int R, int h,
                        float eps, cudaStream_t st);
// X1 = r + y + bias (written to x1), then A = LN(X1; g, b) (written to y).
// red: yv is the multicast address of a TP-symmetric buffer and y is the NVLS
// reduce-load of the t partial products (the g all-reduce fused into the load).
template <class T>
mp_status bda_layernorm_fwd(const T* yv, const T* bias, const T* r, T* x1, const T* g, const T* b, T* out,
                            float* mean, float* rstd, int R, int h, float eps, cudaStream_t st, Dropout dp = Dropout{},
                            bool red = false);
// out = r + dropout(y + bias)   (red: as above)
template <class T>
mp_status bias_add_residual(const T* yv, const T* bias, const T* r, T* out, long long R, int h, cudaStream_t st,
                            Dropout dp = Dropout{}, bool red = false);
// dZ = dropout mask * dY, db += colsum(dZ)   (hidden dropout backward)
template <class T>
mp_status dropout_colsum(const T* dY, T* dZ, float* db, int R, int N, Dropout dp, cudaStream_t st);
// Pd = dropout(P) over the causal written region (unfused attention dropout)
template <class T>
mp_status attn_dropout(const T* P, T* Pd, long long z, int s, Dropout dp, cudaStream_t st);
// dx = LN backward of dy (+ dres if non-null); dgamma/dbeta accumulated (fp32, +=).
// dy_copy non-null: dy is a multicast address, dy = NVLS reduce-load of the t
// partials (the f all-reduce fused into the load), stored to dy_copy [R, h].
// dres_sum / dx_sum (optional, need dres): += column sums of dres and of the
// stored dx (the bias gradients of the row-parallel outputs around LN2, a17).
template <class T>
mp_status layernorm_bwd(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* dres,
                        T* dx, float* dgamma, float* dbeta, int R, int h, cudaStream_t st,
                        T* dy_copy = nullptr, float* dres_sum = nullptr, float* dx_sum = nullptr);
// H = gelu(Y + b)
template <class T>
mp_status bias_gelu_fwd(const T* yv, const T* b, T* out, long long R, int N, cudaStream_t st);
// dU = dH * gelu'(Y + b) (written to du), db += colsum(dU); b may be null (Y already biased)
template <class T>
mp_status bias_gelu_bwd(const T* dh, const T* yv, const T* b, T* du, float* db, int R, int N, cudaStream_t st);
// out[n] += sum_r X[r, n]
template <class T>
mp_status colsum_accum(const T* X, float* out, int R, int N, cudaStream_t st);
// In-place causal scale-mask-softmax over z*s rows of length s.
template <class T>
mp_status softmax_causal_fwd(T* S, long long z, int s, float scale, cudaStream_t st);
// In-place dS = P * (dP - rowsum(dP * P)) * scale on dP.
template <class T>
mp_status softmax_causal_bwd(T* dP, const T* P, long long z, int s, float scale, cudaStream_t st,
                             Dropout dp = Dropout{});
// X[i*b + beta] = (tok in [v0, v0+Vr) ? E[tok - v0] : 0) + (pos ? pos[i] : 0)
template <class T>
mp_status embed_fwd(const int* tok, int tok_ld, const T* E, int v0, int Vr, const T* pos, T* X, int s, int b, int h,
                    cudaStream_t st);
// dE[tok - v0] += dX[row] (owned rows), dpos[i] += sum_beta dX[i*b + beta] (if dpos)
template <class T>
mp_status embed_bwd(const int* tok, int tok_ld, const T* dX, int v0, int Vr, float* dE, float* dpos, int s, int b,
                    int h, cudaStream_t st);
// Cross-entropy over vocab-parallel fp32 logits [R, Vr].
mp_status ce_rowmax(const float* logits, float* rowmax, int R, int Vr, cudaStream_t st);
mp_status ce_sumexp_target(const float* logits, const float* rowmax, const int* lab, int lab_ld, int s, int b,
                           int v0, float* sum_tgt, int R, int Vr, cudaStream_t st);
template <class T>
mp_status ce_loss_grad(const float* logits, const float* rowmax, const float* sum_tgt, const int* lab, int lab_ld,
                       int s, int b, int v0, float scale, T* dlogits, float* loss_acc, int R, int Vr,
                       cudaStream_t st);
// bf16 path: the logit GEMM's statistics epilogue feeds these (a18).
mp_status ce_stats(const float2* part, int np, const float* tgt, const int* lab, int lab_ld, int b, int v0, int Vr,
                   float* mx, float* mx_local, float* stt, int R, cudaStream_t st);
mp_status ce_rescale(const float* mx, const float* mx_local, float* stt, int R, cudaStream_t st);
mp_status ce_grad_inplace(__nv_bfloat16* logits, const float* rowmax, const float* sum_tgt, const int* lab,
                          int lab_ld, int b, int v0, float scale, float* loss_acc, int R, int Vr, cudaStream_t st);
// Adam over flat fp32 arrays; writes the storage copy w_store.
template <class T>
mp_status adam_step(float* w, const float* g, float* m1, float* m2, T* w_store, long long n, float lr, float b1,
                    float b2, float eps, float bc1, float bc2, cudaStream_t st);
template <class T>
mp_status cast_from_f32(const float* src, T* dst, long long n, cudaStream_t st);

}  // namespace mp
