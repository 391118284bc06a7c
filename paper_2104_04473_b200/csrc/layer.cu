// Tensor-parallel GPT transformer layer (Megatron partitioning),
// model ends (vocab-parallel embedding, final LayerNorm + tied logit layer +
// cross-entropy), forward and backward, on one rank of a TP group.
//
// Forward (per rank, T = s*b rows, [s, b, h] layout):
//   A   = LN1(X)                               replicated          (a4)
//   QKV = A Wqkv_r^T + bqkv_r                  column-parallel     (a6)
//   S   = Q K^T per head (causal tile skip)    strided batched     (a7)
//   P   = softmax(S / sqrt(hd)), in place      fused kernel        (a8)
//   ctx = P V                                  strided batched     (a9)
//   Z   = ctx Wo_r^T                           row-parallel        (a10)
//   g: all-reduce(Z)                           NCCL, TP comm       (a11)
//   X1 = X + Z + bo; A2 = LN2(X1)              fused kernel        (a12, a13)
//   Y1 = A2 W1_r^T; H = gelu(Y1 + b1)          column-parallel + fused (a14, a15)
//   Z   = H W2_r^T; g: all-reduce; Y = X1 + Z + b2                  (a16)
// Backward mirrors it (a17); the two f all-reduces of the LayerNorm-input
// gradients run on a side stream concurrently with the matching dW GEMM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.h"
#include "kernels.cuh"
#include "layer.h"
#include "gemm.h"
#include "../../include/mp_ops.h"

namespace mp {

mp_status flash_attn_fwd(const void* QKV, void* O, float* L2, int s, int b, int heads, int hd, cudaStream_t st,
                         Dropout dp);
long long flash_bwd_ws_floats(int s, int b, int heads, int hd);
mp_status flash_attn_bwd(const void* QKV, const void* O, const void* dO, const float* L2, void* dQKV, float* ws,
                         int s, int b, int heads, int hd, cudaStream_t st, Dropout dp);

// Dropout streams of layer `layer` (reading #6): tensor 0 attention
// probabilities, 1 hidden after the projection, 2 hidden after FC2.
static Dropout make_dropout(const mp_ctx* c, int layer, int tensor, int seq0, int b) {
  Dropout d;
  const float p = tensor == 0 ? c->cfg.p_drop_attn : c->cfg.p_drop_hidden;
  if (p <= 0.f) return d;
  d.seed = c->cfg.seed;
  d.stream = (uint32_t)(layer * 8 + tensor);
  d.thresh = (uint32_t)std::floor((1.0 - (double)p) * 16777216.0);
  d.scale = 1.f / (1.f - p);
  d.seq0 = seq0;
  d.b = b;
  d.heads = c->cfg.a / c->t;
  d.head0 = c->tp * d.heads;
  return d;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

mp_status nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) return set_err(MP_ENCCL, "%s: %s", what, ncclGetErrorString(r));
  return MP_OK;
}

// Y[T, N] = X[T, K] W[N, K]^T (+ bias)
static mp_status lin_fwd(mp_ctx* c, const void* X, const void* W, const void* bias, void* Y, int T, int N, int K) {
  mp_gemm_desc g{};
  g.M = T; g.N = N; g.K = K; g.batch = 1;
  g.A = X; g.lda = K; g.B = W; g.ldb = K; g.C = Y; g.ldc = N;
  g.bias = bias; g.alpha = 1.f;
  g.c_fp32 = c->cfg.dtype == MP_FP32;
  return gemm(c->cfg.dtype, g, c->cs);
}
// bf16: U = X W^T + bias and H = gelu(U) from one GEMM epilogue (a14 + a15 fused)
static mp_status lin_fwd_gelu(mp_ctx* c, const void* X, const void* W, const void* bias, void* U, void* H, int T,
                              int N, int K) {
  mp_gemm_desc g{};
  g.M = T; g.N = N; g.K = K; g.batch = 1;
  g.A = X; g.lda = K; g.B = W; g.ldb = K; g.C = U; g.ldc = N;
  g.bias = bias; g.alpha = 1.f;
  g.act = 1; g.C2 = H;
  return gemm(c->cfg.dtype, g, c->cs);
}
// dX[T, K] = dY[T, N] W[N, K]
static mp_status lin_dgrad(mp_ctx* c, const void* dY, const void* W, void* dX, int T, int N, int K) {
  mp_gemm_desc g{};
  g.M = T; g.N = K; g.K = N; g.batch = 1;
  g.A = dY; g.lda = N; g.a_major = 0;
  g.B = W; g.ldb = K; g.b_major = 1;
  g.C = dX; g.ldc = K; g.alpha = 1.f;
  g.c_fp32 = c->cfg.dtype == MP_FP32;
  return gemm(c->cfg.dtype, g, c->cs);
}
// dU[T, K] = (dY[T, N] W[N, K]) * gelu'(U) and db[K] += colsum(dU): the FC2 dgrad GEMM with the
// GeLU backward and the FC1 bias gradient in its epilogue (bf16)
static mp_status lin_dgrad_dgelu(mp_ctx* c, const void* dY, const void* W, const void* U, void* dU, float* db, int T,
                                 int N, int K) {
  mp_gemm_desc g{};
  g.M = T; g.N = K; g.K = N; g.batch = 1;
  g.A = dY; g.lda = N; g.a_major = 0;
  g.B = W; g.ldb = K; g.b_major = 1;
  g.C = dU; g.ldc = K; g.alpha = 1.f;
  g.act = 2; g.C2 = const_cast<void*>(U); g.colsum = db;
  return gemm(c->cfg.dtype, g, c->cs);
}
// dW[N, K] += dY[T, N]^T X[T, K]  (fp32 accumulators)
static mp_status lin_wgrad(mp_ctx* c, const void* dY, const void* X, float* dW, int T, int N, int K,
                           cudaStream_t st = nullptr) {
  mp_gemm_desc g{};
  g.M = N; g.N = K; g.K = T; g.batch = 1;
  g.A = dY; g.lda = N; g.a_major = 1;
  g.B = X; g.ldb = K; g.b_major = 1;
  g.C = dW; g.ldc = K; g.c_fp32 = 1; g.accumulate = 1; g.alpha = 1.f;
  return gemm(c->cfg.dtype, g, st ? st : c->cs);
}

template <class T> static T* ptr(mp_ctx* c, int pidx) {
  return reinterpret_cast<T*>(c->wstore) + c->params[pidx].off;
}
static float* gptr(mp_ctx* c, int pidx) { return c->grads + c->params[pidx].off; }

enum { P_LN1G, P_LN1B, P_WQKV, P_BQKV, P_WO, P_BO, P_LN2G, P_LN2B, P_W1, P_B1, P_W2, P_B2 };

struct Dims {
  int T, h, ht, h3t, h4t, heads, hd, s, b;
  long long z, sq;
};
static Dims dims(mp_ctx* c, int b) {
  Dims d;
  d.s = c->cfg.s; d.b = b; d.T = c->cfg.s * b; d.h = c->cfg.h;
  d.ht = d.h / c->t; d.h3t = 3 * d.ht; d.h4t = 4 * d.ht;
  d.heads = c->cfg.a / c->t; d.hd = d.h / c->cfg.a;
  d.z = (long long)b * d.heads; d.sq = (long long)d.s * d.s;
  return d;
}

// FC1 bias + GeLU in the GEMM epilogue (bf16 path)?
static bool fuse_gelu(const mp_ctx* c) {
  static const bool off = getenv("MP_NO_GELU_EPILOGUE") != nullptr;   // ablation
  return c->cfg.dtype == MP_BF16 && !off;
}

// fused tcgen05 attention core usable for this configuration?
static bool use_fused(const mp_ctx* c) {
  const int hd = c->cfg.h / c->cfg.a;
  return c->cfg.attn_impl == 1 && c->cfg.dtype == MP_BF16 && hd % 32 == 0 && hd >= 32 && hd <= 128;
}

mp_status alloc_async(mp_ctx* c, void** p, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMallocFromPoolAsync(p, bytes ? bytes : 256, c->pool, st);
  if (e != cudaSuccess) return set_err(MP_ENOMEM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  return MP_OK;
}

mp_status ensure_workspace(mp_ctx* c, int b) {
  if (c->t > 1) MP_TRY(tp_sym_ensure(c, (size_t)c->cfg.s * b * c->cfg.h * c->esz));
  if (c->ws_b >= b) return MP_OK;
  MP_CUDA(cudaStreamSynchronize(c->cs));
  void** bufs[] = {&c->ws_z, &c->ws_dsq, &c->ws_d4h, &c->ws_dh1, &c->ws_dh2, &c->ws_dqkv, &c->ws_dctx};
  for (void** q : bufs)
    if (*q) { cudaFree(*q); *q = nullptr; }
  if (c->ws_fa) { cudaFree(c->ws_fa); c->ws_fa = nullptr; }
  Dims d = dims(c, b);
  const bool fused = use_fused(c);
  const size_t es = c->esz;
  size_t sizes[] = {(size_t)d.T * d.h * es, fused ? 256 : (size_t)(d.z * d.sq) * es, (size_t)d.T * d.h4t * es,
                    (size_t)d.T * d.h * es, (size_t)d.T * d.h * es, (size_t)d.T * d.h3t * es,
                    (size_t)d.T * d.ht * es};
  for (int i = 0; i < 7; ++i) MP_CUDA(cudaMalloc(bufs[i], al256(sizes[i])));
  if (fused) MP_CUDA(cudaMalloc(&c->ws_fa, al256(sizeof(float) * (size_t)flash_bwd_ws_floats(d.s, d.b, d.heads, d.hd))));
  c->ws_b = b;
  return MP_OK;
}

static mp_status allreduce(mp_ctx* c, void* buf, size_t n, cudaStream_t st) {
  if (c->t == 1) return MP_OK;
  // timing experiments only (results are wrong): MP_DEBUG_SKIP_TP_AR=1 drops the layer all-reduces
  static const bool skip = getenv("MP_DEBUG_SKIP_TP_AR") && atoi(getenv("MP_DEBUG_SKIP_TP_AR"));
  if (skip) return MP_OK;
  return nccl_check(ncclAllReduce(buf, buf, n, c->nccl_dt, ncclSum, c->tp_comm, st), "tp all-reduce");
}

// ------------------------------------------------------------ attention
template <class T>
static mp_status attention_fwd(mp_ctx* c, const Dims& d, const void* QKV, void* P, void* ctx, const Dropout& dp) {
  const mp_dtype dt = c->cfg.dtype;
  const long long ldq = (long long)d.b * d.h3t;
  mp_gemm_desc g{};
  // S = Q K^T  [z, s, s] (tiles above the diagonal skipped)
  g.M = d.s; g.N = d.s; g.K = d.hd; g.batch = (int)d.z;
  g.A = QKV; g.lda = ldq; g.strideA = 3LL * d.hd;
  g.B = reinterpret_cast<const T*>(QKV) + d.hd; g.ldb = ldq; g.strideB = 3LL * d.hd;
  g.C = P; g.ldc = d.s; g.strideC = d.sq; g.alpha = 1.f; g.causal = 1;
  g.c_fp32 = dt == MP_FP32;
  MP_TRY(gemm(dt, g, c->cs));
  MP_TRY(softmax_causal_fwd<T>(reinterpret_cast<T*>(P), d.z, d.s, 1.f / std::sqrt((float)d.hd), c->cs));
  // attention-probability dropout: the P.V product reads dropout(P); P itself is stashed
  const void* Pv = P;
  if (dp.on()) {
    MP_TRY(attn_dropout<T>(reinterpret_cast<const T*>(P), reinterpret_cast<T*>(c->ws_dsq), d.z, d.s, dp, c->cs));
    Pv = c->ws_dsq;
  }
  // ctx = P V  [s, b, heads, hd]
  g = mp_gemm_desc{};
  g.M = d.s; g.N = d.hd; g.K = d.s; g.batch = (int)d.z;
  g.A = Pv; g.lda = d.s; g.strideA = d.sq;
  g.B = reinterpret_cast<const T*>(QKV) + 2 * d.hd; g.ldb = ldq; g.strideB = 3LL * d.hd; g.b_major = 1;
  g.C = ctx; g.ldc = (long long)d.b * d.ht; g.strideC = d.hd; g.alpha = 1.f; g.causal = 2;
  g.c_fp32 = dt == MP_FP32;
  return gemm(dt, g, c->cs);
}

template <class T>
static mp_status attention_bwd(mp_ctx* c, const Dims& d, const void* QKV, const void* P, const void* dctx,
                               void* dP, void* dQKV, const Dropout& dp) {
  const mp_dtype dt = c->cfg.dtype;
  const bool f32 = dt == MP_FP32;
  const long long ldq = (long long)d.b * d.h3t, ldc = (long long)d.b * d.ht;
  const T* Q = reinterpret_cast<const T*>(QKV);
  T* dQ = reinterpret_cast<T*>(dQKV);
  mp_gemm_desc g{};
  // dV = dropout(P)^T dO  (dropout(P) regenerated into the dP workspace first)
  const void* Pv = P;
  if (dp.on()) {
    MP_TRY(attn_dropout<T>(reinterpret_cast<const T*>(P), reinterpret_cast<T*>(dP), d.z, d.s, dp, c->cs));
    Pv = dP;
  }
  g.M = d.s; g.N = d.hd; g.K = d.s; g.batch = (int)d.z;
  g.A = Pv; g.lda = d.s; g.strideA = d.sq; g.a_major = 1;
  g.B = dctx; g.ldb = ldc; g.strideB = d.hd; g.b_major = 1;
  g.C = dQ + 2 * d.hd; g.ldc = ldq; g.strideC = 3LL * d.hd; g.alpha = 1.f; g.causal = 3; g.c_fp32 = f32;
  MP_TRY(gemm(dt, g, c->cs));
  // dP = dO V^T (causal tiles)
  g = mp_gemm_desc{};
  g.M = d.s; g.N = d.s; g.K = d.hd; g.batch = (int)d.z;
  g.A = dctx; g.lda = ldc; g.strideA = d.hd;
  g.B = Q + 2 * d.hd; g.ldb = ldq; g.strideB = 3LL * d.hd;
  g.C = dP; g.ldc = d.s; g.strideC = d.sq; g.alpha = 1.f; g.causal = 1; g.c_fp32 = f32;
  MP_TRY(gemm(dt, g, c->cs));
  // dS = P (dP - rowsum(dP P)) / sqrt(hd), in place (dP masked by the dropout first)
  MP_TRY(softmax_causal_bwd<T>(reinterpret_cast<T*>(dP), reinterpret_cast<const T*>(P), d.z, d.s,
                               1.f / std::sqrt((float)d.hd), c->cs, dp));
  // dQ = dS K
  g = mp_gemm_desc{};
  g.M = d.s; g.N = d.hd; g.K = d.s; g.batch = (int)d.z;
  g.A = dP; g.lda = d.s; g.strideA = d.sq;
  g.B = Q + d.hd; g.ldb = ldq; g.strideB = 3LL * d.hd; g.b_major = 1;
  g.C = dQ; g.ldc = ldq; g.strideC = 3LL * d.hd; g.alpha = 1.f; g.causal = 2; g.c_fp32 = f32;
  MP_TRY(gemm(dt, g, c->cs));
  // dK = dS^T Q
  g = mp_gemm_desc{};
  g.M = d.s; g.N = d.hd; g.K = d.s; g.batch = (int)d.z;
  g.A = dP; g.lda = d.s; g.strideA = d.sq; g.a_major = 1;
  g.B = Q; g.ldb = ldq; g.strideB = 3LL * d.hd; g.b_major = 1;
  g.C = dQ + d.hd; g.ldc = ldq; g.strideC = 3LL * d.hd; g.alpha = 1.f; g.causal = 3; g.c_fp32 = f32;
  return gemm(dt, g, c->cs);
}

// ------------------------------------------------------------- layer
template <class T>
static mp_status layer_fwd_t(mp_ctx* c, int layer, int b, const void* x, void* y, LayerStash& st) {
  const Dims d = dims(c, b);
  const auto& lp = c->layer_params.at(layer).idx;
  MP_TRY(ensure_workspace(c, b));
  const size_t es = c->esz;
  // one block for every stashed activation of this layer
  size_t off[13], tot = 0;
  size_t sz[13] = {4ull * d.T, 4ull * d.T, 4ull * d.T, 4ull * d.T, es * d.T * d.h, es * d.T * d.h3t,
                   use_fused(c) ? 4ull * d.z * d.s : es * (size_t)(d.z * d.sq), es * d.T * d.ht, es * d.T * d.h, es * d.T * d.h, es * d.T * d.h4t,
                   es * d.T * d.h4t, 0};
  for (int i = 0; i < 12; ++i) { off[i] = tot; tot += al256(sz[i]); }
  MP_TRY(alloc_async(c, &st.block, tot, c->cs));
  char* base = reinterpret_cast<char*>(st.block);
  st.mu1 = (float*)(base + off[0]); st.rs1 = (float*)(base + off[1]);
  st.mu2 = (float*)(base + off[2]); st.rs2 = (float*)(base + off[3]);
  st.A = base + off[4]; st.QKV = base + off[5]; st.P = base + off[6]; st.ctx = base + off[7];
  st.X1 = base + off[8]; st.A2 = base + off[9]; st.Y1 = base + off[10]; st.H = base + off[11];
  st.b = b;
  st.seq0 = c->cur_seq0;
  const Dropout dpa = make_dropout(c, layer, 0, st.seq0, b), dp1 = make_dropout(c, layer, 1, st.seq0, b),
                dp2 = make_dropout(c, layer, 2, st.seq0, b);
  const float eps = c->cfg.ln_eps;
  const T* X = reinterpret_cast<const T*>(x);
  MP_TRY(layernorm_fwd<T>(X, ptr<T>(c, lp[P_LN1G]), ptr<T>(c, lp[P_LN1B]), (T*)st.A, st.mu1, st.rs1, d.T, d.h, eps,
                          c->cs));
  MP_TRY(lin_fwd(c, st.A, ptr<T>(c, lp[P_WQKV]), ptr<T>(c, lp[P_BQKV]), st.QKV, d.T, d.h3t, d.h));
  if (use_fused(c))      // P holds the per-row base-2 log-sum-exp [z, s] instead of the scores
    MP_TRY(flash_attn_fwd(st.QKV, st.ctx, (float*)st.P, d.s, d.b, d.heads, d.hd, c->cs, dpa));
  else
    MP_TRY(attention_fwd<T>(c, d, st.QKV, st.P, st.ctx, dpa));
  const bool nv = c->tps.on, two = nv && tp_sym_two_shot(c), nvr = nv && !two && !tp_sym_debug_local();
  void* zw; const void* zr;   // partial-product buffer: GEMM writes zw, the consumer reads zr
  // g (a11): NCCL all-reduce in place; NVLS one-shot: barrier + reduce-load inside the consumer;
  // NVLS two-shot: slab reduce-load + multicast store, the consumer reads the local sum
  auto g_op = [&]() -> mp_status {
    if (!nv) return allreduce(c, zw, (size_t)d.T * d.h, c->cs);
    if (two) return tp_sym_reduce_two_shot(c, (size_t)d.T * d.h, c->cs, &zr);
    return tp_sym_barrier(c, c->cs);
  };
  auto z_next = [&]() {
    if (nv) tp_sym_next(c, &zw, &zr); else { zw = c->ws_z; zr = c->ws_z; }
    if (nv && !nvr) zr = zw;
  };
  z_next();
  MP_TRY(lin_fwd(c, st.ctx, ptr<T>(c, lp[P_WO]), nullptr, zw, d.T, d.h, d.ht));
  MP_TRY(g_op());
  MP_TRY(bda_layernorm_fwd<T>((const T*)zr, ptr<T>(c, lp[P_BO]), X, (T*)st.X1, ptr<T>(c, lp[P_LN2G]),
                              ptr<T>(c, lp[P_LN2B]), (T*)st.A2, st.mu2, st.rs2, d.T, d.h, eps, c->cs, dp1, nvr));
  if (fuse_gelu(c)) {      // Y1 holds the biased pre-activation
    MP_TRY(lin_fwd_gelu(c, st.A2, ptr<T>(c, lp[P_W1]), ptr<T>(c, lp[P_B1]), st.Y1, st.H, d.T, d.h4t, d.h));
  } else {
    MP_TRY(lin_fwd(c, st.A2, ptr<T>(c, lp[P_W1]), nullptr, st.Y1, d.T, d.h4t, d.h));
    MP_TRY(bias_gelu_fwd<T>((const T*)st.Y1, ptr<T>(c, lp[P_B1]), (T*)st.H, d.T, d.h4t, c->cs));
  }
  z_next();
  MP_TRY(lin_fwd(c, st.H, ptr<T>(c, lp[P_W2]), nullptr, zw, d.T, d.h, d.h4t));
  MP_TRY(g_op());
  MP_TRY(bias_add_residual<T>((const T*)zr, ptr<T>(c, lp[P_B2]), (const T*)st.X1, (T*)y, d.T, d.h, c->cs, dp2, nvr));
  return MP_OK;
}

// SMs the side-stream dW GEMM may use while the NVLS LayerNorm backward runs
// (MP_WGRAD_SM_RESERVE SMs are left to it; default 0 = share every SM).
static int wgrad_ctas() {
  static const int reserve = getenv("MP_WGRAD_SM_RESERVE") ? atoi(getenv("MP_WGRAD_SM_RESERVE")) : 0;
  return reserve > 0 ? std::max(1, num_sms() - reserve) : 0;
}

template <class T>
static mp_status layer_bwd_t(mp_ctx* c, int layer, const LayerStash& st, const void* dy, void* dx) {
  const Dims d = dims(c, st.b);
  const auto& lp = c->layer_params.at(layer).idx;
  MP_TRY(ensure_workspace(c, st.b));
  const T* dY = reinterpret_cast<const T*>(dy);
  T* dU = (T*)c->ws_d4h;
  T* dA2 = (T*)c->ws_dh1;
  T* dX1 = (T*)c->ws_dh2;
  cudaEvent_t ev_a = c->events.at(0), ev_b = c->events.at(1);
  const Dropout dpa = make_dropout(c, layer, 0, st.seq0, st.b), dp1 = make_dropout(c, layer, 1, st.seq0, st.b),
                dp2 = make_dropout(c, layer, 2, st.seq0, st.b);
  // MLP: dZ2 = dropout mask * dY; db2; dH = dZ2 W2; dW2 += H^T dZ2
  // without dropout db2 = colsum(dY) is taken by the LN2 backward, which reads dY as its residual input
  const T* dZ2 = dY;
  if (dp2.on()) {
    MP_TRY(dropout_colsum<T>(dY, (T*)c->ws_z, gptr(c, lp[P_B2]), d.T, d.h, dp2, c->cs));
    dZ2 = (const T*)c->ws_z;
  }
  if (fuse_gelu(c)) {      // Y1 holds the biased pre-activation; GeLU backward + db1 in the dgrad epilogue
    MP_TRY(lin_dgrad_dgelu(c, dZ2, ptr<T>(c, lp[P_W2]), st.Y1, dU, gptr(c, lp[P_B1]), d.T, d.h, d.h4t));
    MP_TRY(lin_wgrad(c, dZ2, st.H, gptr(c, lp[P_W2]), d.T, d.h, d.h4t));
  } else {
    MP_TRY(lin_dgrad(c, dZ2, ptr<T>(c, lp[P_W2]), dU, d.T, d.h, d.h4t));
    MP_TRY(lin_wgrad(c, dZ2, st.H, gptr(c, lp[P_W2]), d.T, d.h, d.h4t));
    MP_TRY(bias_gelu_bwd<T>(dU, (const T*)st.Y1, ptr<T>(c, lp[P_B1]), dU, gptr(c, lp[P_B1]), d.T, d.h4t, c->cs));
  }
  // f (a17): NVLS -- dgrad writes its partial into the symmetric buffer, dW1 accumulates, one barrier,
  // and the LayerNorm backward reduce-loads the sum; NCCL -- all-reduce dA2 on the side stream during dW1
  const bool nv = c->tps.on, two = nv && tp_sym_two_shot(c), nvr = nv && !two && !tp_sym_debug_local();
  void* fw = dA2; const void* fr = dA2;
  if (nv) tp_sym_next(c, &fw, &fr);
  if (nv && !nvr) fr = fw;
  MP_TRY(lin_dgrad(c, dU, ptr<T>(c, lp[P_W1]), fw, d.T, d.h4t, d.h));
  if (c->t > 1) {
    // the f all-reduce (NCCL) or the barrier + reduce-loading LayerNorm backward (NVLS) overlaps dW1
    MP_CUDA(cudaEventRecord(ev_a, c->cs));
    MP_CUDA(cudaStreamWaitEvent(c->side, ev_a, 0));
  }
  if (c->t > 1 && !nv) {
    MP_TRY(allreduce(c, dA2, (size_t)d.T * d.h, c->side));
    MP_CUDA(cudaEventRecord(ev_b, c->side));
    MP_TRY(lin_wgrad(c, dU, st.A2, gptr(c, lp[P_W1]), d.T, d.h4t, d.h));
    MP_CUDA(cudaStreamWaitEvent(c->cs, ev_b, 0));
  } else if (nv) {
    gemm_set_max_ctas(wgrad_ctas());
    MP_TRY(lin_wgrad(c, dU, st.A2, gptr(c, lp[P_W1]), d.T, d.h4t, d.h, c->side));
    gemm_set_max_ctas(0);
    MP_CUDA(cudaEventRecord(ev_b, c->side));
    if (two) MP_TRY(tp_sym_reduce_two_shot(c, (size_t)d.T * d.h, c->cs, &fr));
    else MP_TRY(tp_sym_barrier(c, c->cs));
  } else {
    MP_TRY(lin_wgrad(c, dU, st.A2, gptr(c, lp[P_W1]), d.T, d.h4t, d.h));
  }
  // dX1 = LN2'(dA2) + dY, with db2 = colsum(dY) and dbo = colsum(dX1) (no dropout) in the same pass
  MP_TRY(layernorm_bwd<T>((const T*)fr, (const T*)st.X1, ptr<T>(c, lp[P_LN2G]), st.mu2, st.rs2, dY, dX1,
                          gptr(c, lp[P_LN2G]), gptr(c, lp[P_LN2B]), d.T, d.h, c->cs,
                          nvr ? dA2 : nullptr, dp2.on() ? nullptr : gptr(c, lp[P_B2]),
                          dp1.on() ? nullptr : gptr(c, lp[P_BO])));
  // attention block: dZ1 = dropout mask * dX1; dbo; dctx = dZ1 Wo; dWo += ctx^T dZ1
  const T* dZ1 = dX1;
  if (dp1.on()) {
    MP_TRY(dropout_colsum<T>(dX1, (T*)c->ws_z, gptr(c, lp[P_BO]), d.T, d.h, dp1, c->cs));
    dZ1 = (const T*)c->ws_z;
  }
  if (nv) MP_CUDA(cudaStreamWaitEvent(c->cs, ev_b, 0));   // dW1 done before dU / A2 are reused
  MP_TRY(lin_dgrad(c, dZ1, ptr<T>(c, lp[P_WO]), c->ws_dctx, d.T, d.h, d.ht));
  MP_TRY(lin_wgrad(c, dZ1, st.ctx, gptr(c, lp[P_WO]), d.T, d.h, d.ht));
  if (use_fused(c))
    MP_TRY(flash_attn_bwd(st.QKV, st.ctx, c->ws_dctx, (const float*)st.P, c->ws_dqkv, c->ws_fa, d.s, d.b, d.heads,
                          d.hd, c->cs, dpa));
  else
    MP_TRY(attention_bwd<T>(c, d, st.QKV, st.P, c->ws_dctx, c->ws_dsq, c->ws_dqkv, dpa));
  MP_TRY(colsum_accum<T>((const T*)c->ws_dqkv, gptr(c, lp[P_BQKV]), d.T, d.h3t, c->cs));
  T* dA = (T*)c->ws_dh1;
  fw = dA; fr = dA;
  if (nv) tp_sym_next(c, &fw, &fr);
  if (nv && !nvr) fr = fw;
  MP_TRY(lin_dgrad(c, c->ws_dqkv, ptr<T>(c, lp[P_WQKV]), fw, d.T, d.h3t, d.h));
  if (c->t > 1) {
    MP_CUDA(cudaEventRecord(ev_a, c->cs));
    MP_CUDA(cudaStreamWaitEvent(c->side, ev_a, 0));
  }
  if (c->t > 1 && !nv) {
    MP_TRY(allreduce(c, dA, (size_t)d.T * d.h, c->side));
    MP_CUDA(cudaEventRecord(ev_b, c->side));
    MP_TRY(lin_wgrad(c, c->ws_dqkv, st.A, gptr(c, lp[P_WQKV]), d.T, d.h3t, d.h));
    MP_CUDA(cudaStreamWaitEvent(c->cs, ev_b, 0));
  } else if (nv) {
    gemm_set_max_ctas(wgrad_ctas());
    MP_TRY(lin_wgrad(c, c->ws_dqkv, st.A, gptr(c, lp[P_WQKV]), d.T, d.h3t, d.h, c->side));
    gemm_set_max_ctas(0);
    MP_CUDA(cudaEventRecord(ev_b, c->side));
    if (two) MP_TRY(tp_sym_reduce_two_shot(c, (size_t)d.T * d.h, c->cs, &fr));
    else MP_TRY(tp_sym_barrier(c, c->cs));
  } else {
    MP_TRY(lin_wgrad(c, c->ws_dqkv, st.A, gptr(c, lp[P_WQKV]), d.T, d.h3t, d.h));
  }
  MP_TRY(layernorm_bwd<T>((const T*)fr, (const T*)st.x, ptr<T>(c, lp[P_LN1G]), st.mu1, st.rs1, dX1, (T*)dx,
                          gptr(c, lp[P_LN1G]), gptr(c, lp[P_LN1B]), d.T, d.h, c->cs,
                          nvr ? dA : nullptr));
  if (nv) MP_CUDA(cudaStreamWaitEvent(c->cs, ev_b, 0));   // dWqkv done before the stash is released
  return MP_OK;
}

// Calibration of the fused g / f reduction as the layer runs it (NVLS path): per repetition
// next buffer -> barrier (one-shot) or slab reduce-load + multicast store + barrier
// (two-shot) -> the consuming bias-residual kernel reading the sum.  Collective over the
// TP group.  Returns seconds per reduction (CUDA events on the compute stream).
template <class T>
static mp_status tp_probe_t(mp_ctx* c, int b, int iters, double* seconds) {
  const Dims d = dims(c, b);
  MP_TRY(ensure_workspace(c, b));
  if (!c->tps.on) return set_err(MP_EUNSUPPORTED, "tp probe: the NVLS path is not active on this context");
  const size_t n = (size_t)d.T * d.h;
  void* blk = nullptr;
  MP_TRY(alloc_async(c, &blk, al256(n * c->esz) + al256(d.h * c->esz) + al256(n * c->esz), c->cs));
  char* base = (char*)blk;
  T* out = (T*)base;
  T* zb = (T*)(base + al256(n * c->esz));
  T* zr = (T*)(base + al256(n * c->esz) + al256(d.h * c->esz));
  MP_CUDA(cudaMemsetAsync(zb, 0, d.h * c->esz, c->cs));
  MP_CUDA(cudaMemsetAsync(zr, 0, n * c->esz, c->cs));
  const bool two = tp_sym_two_shot(c);
  auto one = [&]() -> mp_status {
    void* w; const void* r;
    tp_sym_next(c, &w, &r);
    if (two) MP_TRY(tp_sym_reduce_two_shot(c, n, c->cs, &r));
    else MP_TRY(tp_sym_barrier(c, c->cs));
    return bias_add_residual<T>((const T*)r, zb, zr, out, d.T, d.h, c->cs, Dropout{}, !two);
  };
  for (int i = 0; i < 3; ++i) MP_TRY(one());
  cudaEvent_t e0 = nullptr, e1 = nullptr;   // timing events (the context's own are sync-only)
  MP_CUDA(cudaEventCreate(&e0));
  MP_CUDA(cudaEventCreate(&e1));
  mp_status s = MP_OK;
  if (cudaEventRecord(e0, c->cs) != cudaSuccess) s = set_err(MP_ECUDA, "tp probe: event record");
  for (int i = 0; i < iters && s == MP_OK; ++i) s = one();
  float ms = 0.f;
  if (s == MP_OK && (cudaEventRecord(e1, c->cs) != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess ||
                     cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess))
    s = set_err(MP_ECUDA, "tp probe: event timing");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  MP_TRY(s);
  *seconds = ms * 1e-3 / iters;
  MP_CUDA(cudaFreeAsync(blk, c->cs));
  return MP_OK;
}
mp_status tp_reduce_probe(mp_ctx* c, int b, int iters, double* seconds) {
  return c->cfg.dtype == MP_BF16 ? tp_probe_t<__nv_bfloat16>(c, b, iters, seconds)
                                 : tp_probe_t<float>(c, b, iters, seconds);
}

mp_status layer_fwd(mp_ctx* c, int layer, int b, const void* x, void* y, LayerStash& st) {
  return c->cfg.dtype == MP_BF16 ? layer_fwd_t<__nv_bfloat16>(c, layer, b, x, y, st)
                                 : layer_fwd_t<float>(c, layer, b, x, y, st);
}
mp_status layer_bwd(mp_ctx* c, int layer, const LayerStash& st, const void* dy, void* dx) {
  return c->cfg.dtype == MP_BF16 ? layer_bwd_t<__nv_bfloat16>(c, layer, st, dy, dx)
                                 : layer_bwd_t<float>(c, layer, st, dy, dx);
}
mp_status stash_release(mp_ctx* c, LayerStash& st, cudaStream_t s) {
  if (st.block) MP_CUDA(cudaFreeAsync(st.block, s));
  if (st.own_x && st.x) MP_CUDA(cudaFreeAsync(st.x, s));
  st = LayerStash{};
  return MP_OK;
}

// ------------------------------------------------------------ model ends
// Embedding (stage 0): X0 = E_r[tok] (vocab-parallel, rows [tp V/t, (tp+1) V/t))
// + pos (added by tp rank 0), then all-reduce over the TP group.
template <class T>
static mp_status embed_fwd_t(mp_ctx* c, const int* dtok, int tok_ld, int b, void* X) {
  const int Vr = c->cfg.V / c->t;
  const int ie = c->param_index.at("emb#-1"), ip = c->param_index.at("pos#-1");
  MP_TRY(embed_fwd<T>(dtok, tok_ld, ptr<T>(c, ie), c->tp * Vr, Vr, c->tp == 0 ? ptr<T>(c, ip) : nullptr, (T*)X,
                      c->cfg.s, b, c->cfg.h, c->cs));
  return allreduce(c, X, (size_t)c->cfg.s * b * c->cfg.h, c->cs);
}
template <class T>
static mp_status embed_bwd_t(mp_ctx* c, const int* dtok, int tok_ld, int b, const void* dX) {
  const int Vr = c->cfg.V / c->t;
  const int ie = c->param_index.at("emb#-1"), ip = c->param_index.at("pos#-1");
  return embed_bwd<T>(dtok, tok_ld, (const T*)dX, c->tp * Vr, Vr, gptr(c, ie), gptr(c, ip), c->cfg.s, b, c->cfg.h,
                      c->cs);
}
mp_status embed_forward(mp_ctx* c, const int* dtok, int tok_ld, int b, void* X) {
  return c->cfg.dtype == MP_BF16 ? embed_fwd_t<__nv_bfloat16>(c, dtok, tok_ld, b, X)
                                 : embed_fwd_t<float>(c, dtok, tok_ld, b, X);
}
mp_status embed_backward(mp_ctx* c, const int* dtok, int tok_ld, int b, const void* dX) {
  return c->cfg.dtype == MP_BF16 ? embed_bwd_t<__nv_bfloat16>(c, dtok, tok_ld, b, dX)
                                 : embed_bwd_t<float>(c, dtok, tok_ld, b, dX);
}

// Head (last stage): Z = LN_f(X); logits = Z E_r^T (fp32, [T, V/t]);
// vocab-parallel cross-entropy (TP all-reduces of row max, sum-exp and
// target logit); dlogits = (softmax - onehot) * scale; dZ = dlogits E_r
// (f: all-reduce); dE_r += dlogits^T Z; dX = LN_f'(dZ).  loss += scale * sum.
// bf16 head: the logit GEMM writes bf16 logits and, in its epilogue, the
// cross-entropy row statistics of the fp32 accumulators (max and sum-exp
// partials per column block, target logit); one combine kernel and one
// in-place gradient pass follow (HBM: logits written once, read once, dlogits
// written once -- instead of fp32 logits read by three passes).
static mp_status head_bf16(mp_ctx* c, const void* X, const int* dlab, int lab_ld, int b, float scale, void* dX,
                           int defer_slot) {
  using T = __nv_bfloat16;
  const int s = c->cfg.s, h = c->cfg.h, Tn = s * b, Vr = c->cfg.V / c->t;
  const bool defer = defer_slot >= 0;
  const int ie = c->param_index.at("emb#-1"), ig = c->param_index.at("lnf_g#-1"), ib = c->param_index.at("lnf_b#-1");
  mp_gemm_desc lg{};
  lg.M = Tn; lg.N = Vr; lg.K = h; lg.batch = 1;
  lg.B = ptr<T>(c, ie); lg.lda = h; lg.ldb = h; lg.ldc = Vr; lg.alpha = 1.f;
  const int np = 2 * gemm_ce_nblocks(lg);
  size_t o_Z = 0, o_mu = o_Z + al256(defer ? 0 : 2ull * Tn * h), o_rs = o_mu + al256(4ull * Tn),
         o_L = o_rs + al256(4ull * Tn), o_P = o_L + al256(defer ? 0 : 2ull * Tn * Vr), o_tg = o_P + al256(8ull * Tn * np), o_mx = o_tg + al256(4ull * Tn),
         o_ml = o_mx + al256(4ull * Tn), o_st = o_ml + al256(4ull * Tn), o_dZ = o_st + al256(8ull * Tn),
         tot = o_dZ + al256(2ull * Tn * h);
  void* blk = nullptr;
  MP_TRY(alloc_async(c, &blk, tot, c->cs));
  char* base = (char*)blk;
  T* Z = defer ? (T*)c->head_z + (size_t)defer_slot * Tn * h : (T*)(base + o_Z);
  float *mu = (float*)(base + o_mu), *rs = (float*)(base + o_rs);
  T* L = defer ? (T*)c->head_dl + (size_t)defer_slot * Tn * Vr : (T*)(base + o_L);
  float2* part = (float2*)(base + o_P);
  float *tgt = (float*)(base + o_tg), *mx = (float*)(base + o_mx), *mxl = (float*)(base + o_ml),
        *stt = (float*)(base + o_st);
  T* dZ = (T*)(base + o_dZ);
  MP_TRY(layernorm_fwd<T>((const T*)X, ptr<T>(c, ig), ptr<T>(c, ib), Z, mu, rs, Tn, h, c->cfg.ln_eps, c->cs));
  lg.A = Z; lg.C = L;
  const GemmCe ce{part, tgt, dlab, lab_ld, b, c->tp * Vr};
  MP_TRY(gemm(c->cfg.dtype, lg, c->cs, &ce));   // logits = Z E_r^T (+ CE statistics)
  MP_TRY(ce_stats(part, np, tgt, dlab, lab_ld, b, c->tp * Vr, Vr, mx, c->t > 1 ? mxl : nullptr, stt, Tn, c->cs));
  if (c->t > 1) {
    MP_TRY(nccl_check(ncclAllReduce(mx, mx, Tn, ncclFloat32, ncclMax, c->tp_comm, c->cs), "ce max"));
    MP_TRY(ce_rescale(mx, mxl, stt, Tn, c->cs));
    MP_TRY(nccl_check(ncclAllReduce(stt, stt, 2 * Tn, ncclFloat32, ncclSum, c->tp_comm, c->cs), "ce sum"));
  }
  MP_TRY(ce_grad_inplace(L, mx, stt, dlab, lab_ld, b, c->tp * Vr, scale, c->d_loss, Tn, Vr, c->cs));
  T* dL = L;
  {  // dZ = dlogits E_r
    mp_gemm_desc g{};
    g.M = Tn; g.N = h; g.K = Vr; g.batch = 1;
    g.A = dL; g.lda = Vr; g.B = ptr<T>(c, ie); g.ldb = h; g.b_major = 1; g.C = dZ; g.ldc = h; g.alpha = 1.f;
    MP_TRY(gemm(c->cfg.dtype, g, c->cs));
  }
  MP_TRY(allreduce(c, dZ, (size_t)Tn * h, c->cs));                              // f
  if (!defer) {  // dE_r += dlogits^T Z
    mp_gemm_desc g{};
    g.M = Vr; g.N = h; g.K = Tn; g.batch = 1;
    g.A = dL; g.lda = Vr; g.a_major = 1; g.B = Z; g.ldb = h; g.b_major = 1;
    g.C = gptr(c, ie); g.ldc = h; g.c_fp32 = 1; g.accumulate = 1; g.alpha = 1.f;
    MP_TRY(gemm(c->cfg.dtype, g, c->cs));
  }
  MP_TRY(layernorm_bwd<T>(dZ, (const T*)X, ptr<T>(c, ig), mu, rs, nullptr, (T*)dX,
                          gptr(c, ig), gptr(c, ib), Tn, h, c->cs));
  MP_CUDA(cudaFreeAsync(blk, c->cs));
  return MP_OK;
}

// The logit layer's weight gradient of a whole batch as one GEMM at the flush: the
// microbatches' dlogits / Z row blocks are contiguous, so sum_mb dL_mb^T Z_mb =
// [dL_1; ..; dL_m]^T [Z_1; ..; Z_m] (K = m b s): the fp32 dE_r accumulator is read and
// written once per batch instead of once per microbatch, and the GEMM leaves the
// last stage's forward tasks (it fills that device's cool-down idle instead).
mp_status head_dE_deferred(mp_ctx* c, int b, int n_slots) {
  const int h = c->cfg.h, Vr = c->cfg.V / c->t;
  const long long K = (long long)n_slots * c->cfg.s * b;
  if (K > 0x7fffffffLL) return set_err(MP_EINVAL, "deferred dE: K too large");
  mp_gemm_desc g{};
  g.M = Vr; g.N = h; g.K = (int)K; g.batch = 1;
  g.A = c->head_dl; g.lda = Vr; g.a_major = 1; g.B = c->head_z; g.ldb = h; g.b_major = 1;
  g.C = gptr(c, c->param_index.at("emb#-1")); g.ldc = h; g.c_fp32 = 1; g.accumulate = 1; g.alpha = 1.f;
  return gemm(c->cfg.dtype, g, c->cs);
}

template <class T>
static mp_status head_t(mp_ctx* c, const void* X, const int* dlab, int lab_ld, int b, float scale, void* dX) {
  const int s = c->cfg.s, h = c->cfg.h, Tn = s * b, Vr = c->cfg.V / c->t;
  const int ie = c->param_index.at("emb#-1"), ig = c->param_index.at("lnf_g#-1"), ib = c->param_index.at("lnf_b#-1");
  const size_t es = c->esz;
  size_t o_Z = 0, o_mu = o_Z + al256(es * Tn * h), o_rs = o_mu + al256(4ull * Tn), o_L = o_rs + al256(4ull * Tn),
         o_dL = o_L + al256(4ull * Tn * Vr), o_mx = o_dL + al256(es * Tn * Vr), o_st = o_mx + al256(4ull * Tn),
         o_dZ = o_st + al256(8ull * Tn), tot = o_dZ + al256(es * Tn * h);
  void* blk = nullptr;
  MP_TRY(alloc_async(c, &blk, tot, c->cs));
  char* base = (char*)blk;
  T* Z = (T*)(base + o_Z);
  float *mu = (float*)(base + o_mu), *rs = (float*)(base + o_rs), *L = (float*)(base + o_L);
  T* dL = (T*)(base + o_dL);
  float *mx = (float*)(base + o_mx), *stt = (float*)(base + o_st);
  T* dZ = (T*)(base + o_dZ);
  MP_TRY(layernorm_fwd<T>((const T*)X, ptr<T>(c, ig), ptr<T>(c, ib), Z, mu, rs, Tn, h, c->cfg.ln_eps, c->cs));
  {  // logits = Z E_r^T  (fp32 out)
    mp_gemm_desc g{};
    g.M = Tn; g.N = Vr; g.K = h; g.batch = 1;
    g.A = Z; g.lda = h; g.B = ptr<T>(c, ie); g.ldb = h; g.C = L; g.ldc = Vr; g.c_fp32 = 1; g.alpha = 1.f;
    MP_TRY(gemm(c->cfg.dtype, g, c->cs));
  }
  MP_TRY(ce_rowmax(L, mx, Tn, Vr, c->cs));
  if (c->t > 1) MP_TRY(nccl_check(ncclAllReduce(mx, mx, Tn, ncclFloat32, ncclMax, c->tp_comm, c->cs), "ce max"));
  MP_TRY(ce_sumexp_target(L, mx, dlab, lab_ld, s, b, c->tp * Vr, stt, Tn, Vr, c->cs));
  if (c->t > 1) MP_TRY(nccl_check(ncclAllReduce(stt, stt, 2 * Tn, ncclFloat32, ncclSum, c->tp_comm, c->cs), "ce sum"));
  MP_TRY(ce_loss_grad<T>(L, mx, stt, dlab, lab_ld, s, b, c->tp * Vr, scale, dL, c->d_loss, Tn, Vr, c->cs));
  {  // dZ = dlogits E_r
    mp_gemm_desc g{};
    g.M = Tn; g.N = h; g.K = Vr; g.batch = 1;
    g.A = dL; g.lda = Vr; g.B = ptr<T>(c, ie); g.ldb = h; g.b_major = 1; g.C = dZ; g.ldc = h; g.alpha = 1.f;
    g.c_fp32 = c->cfg.dtype == MP_FP32;
    MP_TRY(gemm(c->cfg.dtype, g, c->cs));
  }
  MP_TRY(allreduce(c, dZ, (size_t)Tn * h, c->cs));                              // f
  {  // dE_r += dlogits^T Z
    mp_gemm_desc g{};
    g.M = Vr; g.N = h; g.K = Tn; g.batch = 1;
    g.A = dL; g.lda = Vr; g.a_major = 1; g.B = Z; g.ldb = h; g.b_major = 1;
    g.C = gptr(c, ie); g.ldc = h; g.c_fp32 = 1; g.accumulate = 1; g.alpha = 1.f;
    MP_TRY(gemm(c->cfg.dtype, g, c->cs));
  }
  MP_TRY(layernorm_bwd<T>(dZ, (const T*)X, ptr<T>(c, ig), mu, rs, nullptr, (T*)dX,
                          gptr(c, ig), gptr(c, ib), Tn, h, c->cs));
  MP_CUDA(cudaFreeAsync(blk, c->cs));
  return MP_OK;
}

mp_status head_fwd_bwd(mp_ctx* c, const void* X, const int* dlab, int lab_ld, int b, float scale, void* dX,
                       int defer_slot) {
  MP_TRY(ensure_workspace(c, b));
  static const bool legacy = getenv("MP_HEAD_FP32_LOGITS") != nullptr;   // A/B: round-1 three-pass head
  if (c->cfg.dtype == MP_BF16 && !legacy) return head_bf16(c, X, dlab, lab_ld, b, scale, dX, defer_slot);
  if (defer_slot >= 0) return set_err(MP_EINVAL, "deferred dE needs the bf16 head");
  return c->cfg.dtype == MP_BF16 ? head_t<__nv_bfloat16>(c, X, dlab, lab_ld, b, scale, dX)
                                 : head_t<float>(c, X, dlab, lab_ld, b, scale, dX);
}

}  // namespace mp
