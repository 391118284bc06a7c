// C-ABI wrappers of the memory-bound kernels (include/mp_ops.h): dtype
// dispatch and argument checks only.
#include "kernels.cuh"
#include "common.h"
#include "../../include/mp_ops.h"

using namespace mp;
using bf16 = __nv_bfloat16;

#define DISPATCH(dt, FN, ...)                                                          \
  do {                                                                                 \
    MP_REQUIRE_DEVICE();                                                               \
    cudaStream_t _st = reinterpret_cast<cudaStream_t>(stream);                         \
    if ((dt) == MP_BF16) return FN<bf16> __VA_ARGS__;                                  \
    if ((dt) == MP_FP32) return FN<float> __VA_ARGS__;                                 \
    return set_err(MP_EINVAL, "bad dtype");                                            \
  } while (0)

template <class T> static const T* C(const void* p) { return reinterpret_cast<const T*>(p); }
template <class T> static T* M(void* p) { return reinterpret_cast<T*>(p); }

template <class T>
static mp_status ln_fwd_(const void* x, const void* g, const void* b, void* y, float* mu, float* rs, int R, int h,
                         float eps, cudaStream_t st) {
  return layernorm_fwd<T>(C<T>(x), C<T>(g), C<T>(b), M<T>(y), mu, rs, R, h, eps, st);
}
template <class T>
static mp_status bda_ln_(const void* y, const void* bias, const void* r, void* x1, const void* g, const void* b,
                         void* out, float* mu, float* rs, int R, int h, float eps, cudaStream_t st) {
  return bda_layernorm_fwd<T>(C<T>(y), C<T>(bias), C<T>(r), M<T>(x1), C<T>(g), C<T>(b), M<T>(out), mu, rs, R, h, eps,
                              st);
}
template <class T>
static mp_status ln_bwd_(const void* dy, const void* x, const void* g, const float* mu, const float* rs,
                         const void* dres, void* dx, float* dg, float* db, float* dres_sum, float* dx_sum, int R,
                         int h, cudaStream_t st) {
  return layernorm_bwd<T>(C<T>(dy), C<T>(x), C<T>(g), mu, rs, C<T>(dres), M<T>(dx), dg, db, R, h, st, nullptr,
                          dres_sum, dx_sum);
}
template <class T>
static mp_status gelu_fwd_(const void* y, const void* b, void* out, long long R, int N, cudaStream_t st) {
  return bias_gelu_fwd<T>(C<T>(y), C<T>(b), M<T>(out), R, N, st);
}
template <class T>
static mp_status gelu_bwd_(const void* dh, const void* y, const void* b, void* du, float* db, int R, int N,
                           cudaStream_t st) {
  return bias_gelu_bwd<T>(C<T>(dh), C<T>(y), C<T>(b), M<T>(du), db, R, N, st);
}
template <class T>
static mp_status sm_fwd_(void* S, long long z, int s, float scale, cudaStream_t st) {
  return softmax_causal_fwd<T>(M<T>(S), z, s, scale, st);
}
template <class T>
static mp_status sm_bwd_(void* dP, const void* P, long long z, int s, float scale, cudaStream_t st) {
  return softmax_causal_bwd<T>(M<T>(dP), C<T>(P), z, s, scale, st);
}
template <class T>
static mp_status colsum_(const void* X, float* out, int R, int N, cudaStream_t st) {
  return colsum_accum<T>(C<T>(X), out, R, N, st);
}

extern "C" {

mp_status mp_op_layernorm_fwd(mp_dtype dt, const void* x, const void* g, const void* b, void* y, float* mean,
                              float* rstd, int R, int h, float eps, void* stream) {
  DISPATCH(dt, ln_fwd_, (x, g, b, y, mean, rstd, R, h, eps, _st));
}

mp_status mp_op_bda_layernorm_fwd(mp_dtype dt, const void* y, const void* bias, const void* r, void* x1,
                                  const void* g, const void* b, void* out, float* mean, float* rstd, int R, int h,
                                  float eps, void* stream) {
  DISPATCH(dt, bda_ln_, (y, bias, r, x1, g, b, out, mean, rstd, R, h, eps, _st));
}

mp_status mp_op_layernorm_bwd(mp_dtype dt, const void* dy, const void* x, const void* g, const float* mean,
                              const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta, int R, int h,
                              void* stream) {
  DISPATCH(dt, ln_bwd_, (dy, x, g, mean, rstd, dres, dx, dgamma, dbeta, nullptr, nullptr, R, h, _st));
}

mp_status mp_op_layernorm_bwd_sums(mp_dtype dt, const void* dy, const void* x, const void* g, const float* mean,
                                   const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta,
                                   float* dres_sum, float* dx_sum, int R, int h, void* stream) {
  DISPATCH(dt, ln_bwd_, (dy, x, g, mean, rstd, dres, dx, dgamma, dbeta, dres_sum, dx_sum, R, h, _st));
}

mp_status mp_op_bias_gelu_fwd(mp_dtype dt, const void* y, const void* b, void* out, long long R, int N,
                              void* stream) {
  DISPATCH(dt, gelu_fwd_, (y, b, out, R, N, _st));
}

mp_status mp_op_bias_gelu_bwd(mp_dtype dt, const void* dh, const void* y, const void* b, void* du, float* db, int R,
                              int N, void* stream) {
  DISPATCH(dt, gelu_bwd_, (dh, y, b, du, db, R, N, _st));
}

mp_status mp_op_softmax_causal_fwd(mp_dtype dt, void* S, long long z, int s, float scale, void* stream) {
  DISPATCH(dt, sm_fwd_, (S, z, s, scale, _st));
}

mp_status mp_op_softmax_causal_bwd(mp_dtype dt, void* dP, const void* P, long long z, int s, float scale,
                                   void* stream) {
  DISPATCH(dt, sm_bwd_, (dP, P, z, s, scale, _st));
}

mp_status mp_op_colsum_accum(mp_dtype dt, const void* X, float* out, int R, int N, void* stream) {
  DISPATCH(dt, colsum_, (X, out, R, N, _st));
}

}  // extern "C"
