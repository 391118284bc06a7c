// Memory-bound kernels of the hot path; see kernels.cuh for the contracts.
// Design: every kernel streams 16-byte vectors (8 bf16 or 4 fp32) with the
// thread index on the contiguous dimension, keeps one row in registers where
// the op is a row reduction (LayerNorm forward: a group of threads per row,
// several groups per persistent CTA; LayerNorm backward dx: one CTA per row;
// causal softmax: one CTA per row), reduces with warp shuffles, and computes
// in fp32.  Every kernel is launched with programmatic dependent launch
// (launch.cuh) and starts with pdl_entry().
#include "kernels.cuh"
#include "common.h"
#include "launch.cuh"
#include "dropout.cuh"

#include <algorithm>
#include <cfloat>

namespace mp {

// ------------------------------------------------------------ vector I/O
template <class T> struct VW;
template <> struct VW<float> { static constexpr int N = 4; };
template <> struct VW<__nv_bfloat16> { static constexpr int N = 8; };

__device__ __forceinline__ void ld_vec(const float* p, float* o) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void st_vec(float* p, const float* o) {
  *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
}
__device__ __forceinline__ void ld_vec(const __nv_bfloat16* p, float* o) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void st_vec(__nv_bfloat16* p, const float* o) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}

// NVLS reduce-loads: `p` is a multicast address of a
// TP-symmetric buffer; the NVSwitch returns the sum over the TP group's copies
// (fp32 accumulation, one rounding to the storage type for bf16).
__device__ __forceinline__ void ld_vec_red(const float* p, float* o) {
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_vec_red(const __nv_bfloat16* p, float* o) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
}
template <bool RED, class T>
__device__ __forceinline__ void ld_in(const T* p, float* o) {
  if constexpr (RED) ld_vec_red(p, o); else ld_vec(p, o);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Sum of two values over the block (<= 32 warps); result broadcast to all threads.
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, nw = (blockDim.x + 31) / 32;
  __syncthreads();
  if (l == 0) red[w] = make_float2(a, b);
  __syncthreads();
  float2 r = make_float2(0.f, 0.f);
  for (int i = 0; i < nw; ++i) { r.x += red[i].x; r.y += red[i].y; }
  return r;
}
__device__ __forceinline__ float block_max(float a, float* red) {
  a = warp_max(a);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, nw = (blockDim.x + 31) / 32;
  __syncthreads();
  if (l == 0) red[w] = a;
  __syncthreads();
  float r = -FLT_MAX;
  for (int i = 0; i < nw; ++i) r = fmaxf(r, red[i]);
  return r;
}

// keep bits of the V consecutive elements e0 .. e0+V-1 (e0 a multiple of V)
template <int V>
__device__ __forceinline__ uint32_t keep_bits(const Dropout& d, unsigned long long e0, uint32_t lane_hi, uint32_t n) {
  uint32_t m = keep4(d, e0 / 4, lane_hi, n);
  if (V == 8) m |= keep4(d, e0 / 4 + 1, lane_hi, n) << 4;
  return m;
}

#define LAUNCH_CHECK()                                                                         \
  do {                                                                                         \
    count_launch();                                                                            \
    cudaError_t _e = cudaGetLastError();                                                       \
    if (_e != cudaSuccess) return set_err(MP_ECUDA, "%s: %s", __func__, cudaGetErrorString(_e)); \
    return MP_OK;                                                                              \
  } while (0)

// ------------------------------------------------------------ LayerNorm
// Row-group layout shared by the LayerNorm kernels (coalesced,
// warp-shuffle rows).  A row of h elements (nvec 16-byte vectors) belongs to a
// group of RG threads (a multiple of 32); thread lt of the group holds vectors
// lt + k RG (k < NV) in registers.  A CTA runs NG groups on different rows and
// is persistent (grid = resident CTAs, rows visited in a grid-stride loop), so
// a thread owns the same columns for every row it visits -- the backward keeps
// its dgamma / dbeta / bias-gradient column partials in registers across rows.
// Per-row sums: warp shuffles, then one shared-memory exchange under the
// group's named barrier (double-buffered, so one barrier per reduction).
struct RowCfg { int nvec, NV, RG, NG; };
constexpr int ROW_THREADS = 256;                   // CTA size bound (<= 255 registers per thread)
constexpr int ROW_MAX_NG = 8, ROW_MAX_WARPS = 8;   // named barriers 1..8; RG <= 256

// NV in {1, 2, 3, 4, 8} with RG = roundup32(ceil(nvec / NV)) <= 256 and the fewest idle
// lanes (h = 2304 bf16: NV = 3, RG = 96; h = 4096: 2 x 256; h = 8192: 4 x 256).
template <class T>
static RowCfg row_cfg(int h) {
  constexpr int V = VW<T>::N;
  RowCfg r;
  r.nvec = h / V;
  r.NV = 8;
  r.RG = ROW_THREADS;
  long long best = -1;
  for (int nv : {1, 2, 3, 4, 8}) {
    const int rg = ((r.nvec + nv - 1) / nv + 31) / 32 * 32;
    if (rg > ROW_THREADS) continue;
    const long long waste = (long long)rg * nv - r.nvec;
    if (best < 0 || waste < best) { best = waste; r.NV = nv; r.RG = rg; }
  }
  r.NG = std::max(1, std::min(ROW_MAX_NG, ROW_THREADS / r.RG));
  return r;
}

template <class T>
static mp_status check_row_dims(int R, int h) {
  constexpr int V = VW<T>::N;
  if (R <= 0 || h <= 0 || h % V) return set_err(MP_EINVAL, "row kernel: h=%d must be a multiple of %d", h, V);
  if (h / V > 8 * ROW_THREADS) return set_err(MP_EINVAL, "row kernel: h=%d too large", h);
  return MP_OK;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// (a, b) summed over the RG threads of the caller's row group; red holds
// RG / 32 float2 of this group and is not reused before the group's next
// barrier (callers alternate two buffers).
__device__ __forceinline__ float2 group_sum2(float a, float b, float2* red, int lt, int RG, int bar) {
  a = warp_sum(a);
  b = warp_sum(b);
  if (RG == 32) return make_float2(a, b);
  if ((lt & 31) == 0) red[lt >> 5] = make_float2(a, b);
  named_bar(bar, RG);
  float2 r = make_float2(0.f, 0.f);
  for (int i = 0; i < RG / 32; ++i) { r.x += red[i].x; r.y += red[i].y; }
  return r;
}
// values as stored in T (bf16 rounding of an fp32 result, identity for fp32)
template <class T, int V>
__device__ __forceinline__ void round_as(float (&o)[V]) {
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int e = 0; e < V; ++e) o[e] = __bfloat162float(__float2bfloat16_rn(o[e]));
  }
}

template <class K>
static int resident_ctas(K kernel, int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  return std::max(1, n);
}

// mode 0: x = in; mode 1: x1 = r + dropout(in + bias) is stored and x = x1 as stored.
template <class T, int NV, int MODE, bool RED>
__global__ void __launch_bounds__(ROW_THREADS) ln_fwd_kernel(const T* __restrict__ in, const T* __restrict__ bias,
                                                      const T* __restrict__ res, T* __restrict__ x1,
                                                      const T* __restrict__ g, const T* __restrict__ b,
                                                      T* __restrict__ out, float* __restrict__ mean,
                                                      float* __restrict__ rstd, int h, float eps, Dropout dp, int R,
                                                      int RG, int NG) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float2 red[2][ROW_MAX_NG][ROW_MAX_WARPS];
  const int grp = threadIdx.x / RG, lt = threadIdx.x - grp * RG;
  const int nvec = h / V;
  for (long long row = (long long)blockIdx.x * NG + grp; row < R; row += (long long)gridDim.x * NG) {
    float v[NV][V];
    float s1 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int vi = lt + k * RG;
      if (vi < nvec) {
        ld_in<RED>(in + row * h + vi * V, v[k]);
        if constexpr (MODE == 1) {
          float bb[V], rr[V];
          ld_vec(bias + vi * V, bb);
          ld_vec(res + row * h + vi * V, rr);
          if (dp.on()) {   // x1 = r + dropout(y + bias), mask keyed by (sequence, position, feature)
            const int pos = (int)(row / dp.b), seq = dp.seq0 + (int)(row % dp.b);
            const uint32_t km = keep_bits<V>(dp, (unsigned long long)pos * h + vi * V, 0, seq);
#pragma unroll
            for (int e = 0; e < V; ++e) v[k][e] = rr[e] + ((km >> e) & 1 ? (v[k][e] + bb[e]) * dp.scale : 0.f);
          } else {
#pragma unroll
            for (int e = 0; e < V; ++e) v[k][e] = rr[e] + (v[k][e] + bb[e]);
          }
          st_vec(x1 + row * h + vi * V, v[k]);
          round_as<T>(v[k]);   // LayerNorm consumes the stored residual-stream value
        }
#pragma unroll
        for (int e = 0; e < V; ++e) s1 += v[k][e];
      }
    }
    const float mu = group_sum2(s1, 0.f, red[0][grp], lt, RG, 1 + grp).x / h;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int vi = lt + k * RG;
      if (vi < nvec)
#pragma unroll
        for (int e = 0; e < V; ++e) { const float d = v[k][e] - mu; s2 += d * d; }
    }
    const float var = group_sum2(s2, 0.f, red[1][grp], lt, RG, 1 + grp).x / h;
    const float rs = rsqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int vi = lt + k * RG;
      if (vi < nvec) {
        float gg[V], bb[V], o[V];
        ld_vec(g + vi * V, gg);
        ld_vec(b + vi * V, bb);
#pragma unroll
        for (int e = 0; e < V; ++e) o[e] = (v[k][e] - mu) * rs * gg[e] + bb[e];
        st_vec(out + row * h + vi * V, o);
      }
    }
    if (lt == 0) { mean[row] = mu; rstd[row] = rs; }
  }
}

template <class T, int MODE, bool RED>
static mp_status launch_ln_fwd(const T* in, const T* bias, const T* res, T* x1, const T* g, const T* b, T* out,
                               float* mean, float* rstd, int R, int h, float eps, Dropout dp, cudaStream_t st) {
  MP_TRY(check_row_dims<T>(R, h));
  const RowCfg rc = row_cfg<T>(h);
  auto go = [&](auto kern) {
    const int threads = rc.RG * rc.NG;
    const long long need = (R + rc.NG - 1) / rc.NG;
    const int grid = (int)std::min<long long>(need, (long long)num_sms() * resident_ctas(kern, threads, 0));
    pdl_launch(kern, grid, threads, 0, st, in, bias, res, x1, g, b, out, mean, rstd, h, eps, dp, R, rc.RG, rc.NG);
  };
  switch (rc.NV) {
    case 1: go(ln_fwd_kernel<T, 1, MODE, RED>); break;
    case 2: go(ln_fwd_kernel<T, 2, MODE, RED>); break;
    case 3: go(ln_fwd_kernel<T, 3, MODE, RED>); break;
    case 4: go(ln_fwd_kernel<T, 4, MODE, RED>); break;
    default: go(ln_fwd_kernel<T, 8, MODE, RED>); break;
  }
  LAUNCH_CHECK();
}

template <class T>
mp_status layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int R, int h, float eps,
                        cudaStream_t st) {
  return launch_ln_fwd<T, 0, false>(x, nullptr, nullptr, nullptr, g, b, y, mean, rstd, R, h, eps, Dropout{}, st);
}

template <class T>
mp_status bda_layernorm_fwd(const T* yv, const T* bias, const T* r, T* x1, const T* g, const T* b, T* out,
                            float* mean, float* rstd, int R, int h, float eps, cudaStream_t st, Dropout dp,
                            bool red) {
  if (red) return launch_ln_fwd<T, 1, true>(yv, bias, r, x1, g, b, out, mean, rstd, R, h, eps, dp, st);
  return launch_ln_fwd<T, 1, false>(yv, bias, r, x1, g, b, out, mean, rstd, R, h, eps, dp, st);
}

// ------------------------------------------------------ bias + residual add
template <class T, bool RED = false>
__global__ void bias_add_residual_kernel(const T* __restrict__ yv, const T* __restrict__ bias,
                                         const T* __restrict__ r, T* __restrict__ out, long long nvec, int hv,
                                         Dropout dp) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    float a[V], bb[V], rr[V];
    ld_in<RED>(yv + i * V, a);
    ld_vec(bias + (i % hv) * V, bb);
    ld_vec(r + i * V, rr);
    if (dp.on()) {
      const long long row = i / hv;
      const int pos = (int)(row / dp.b), seq = dp.seq0 + (int)(row % dp.b);
      const uint32_t km = keep_bits<V>(dp, (unsigned long long)pos * hv * V + (i % hv) * V, 0, seq);
#pragma unroll
      for (int e = 0; e < V; ++e) a[e] = rr[e] + ((km >> e) & 1 ? (a[e] + bb[e]) * dp.scale : 0.f);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) a[e] = rr[e] + (a[e] + bb[e]);
    }
    st_vec(out + i * V, a);
  }
}

static int ew_grid(long long nvec) {
  long long g = (nvec + 255) / 256;
  return (int)std::max(1LL, std::min<long long>(g, (long long)num_sms() * 8));
}

template <class T>
mp_status bias_add_residual(const T* yv, const T* bias, const T* r, T* out, long long R, int h, cudaStream_t st,
                            Dropout dp, bool red) {
  constexpr int V = VW<T>::N;
  if (h % V) return set_err(MP_EINVAL, "bias_add_residual: h %% %d", V);
  long long nvec = R * h / V;
  if (red)
    pdl_launch(bias_add_residual_kernel<T, true>, ew_grid(nvec), 256, 0, st, yv, bias, r, out, nvec, h / V, dp);
  else
    pdl_launch(bias_add_residual_kernel<T>, ew_grid(nvec), 256, 0, st, yv, bias, r, out, nvec, h / V, dp);
  LAUNCH_CHECK();
}

// ------------------------------------------------------------ LayerNorm bwd
// Two kernels: the row kernel (dx; one CTA per row, ~20 resident CTAs per SM so
// many rows' loads are in flight) and the column-tile kernel below (dgamma,
// dbeta and, around LN2, the two bias gradients b2 = colsum(dres) and bo =
// colsum(dx) in the same pass over the rows).
static int row_threads(int nvec) {
  int t = ((nvec + 3) / 4 + 31) / 32 * 32;   // <= 4 vectors per thread
  return std::max(32, std::min(256, t));
}
constexpr int LNB_MAXV = 4;
// Grid of a row kernel: every row handled by one CTA in a grid-stride loop, the grid
// sized to the CTAs that are resident at once (<= 64 warps / 32 CTAs per SM), so there
// is no partial last wave (T = 4096 rows of 96 threads would be 1.3 waves).
static int row_grid(long long R, int nvec) {
  const int warps = row_threads(nvec) / 32;
  const int per_sm = std::max(1, std::min(32, 64 / warps));
  return (int)std::max(1LL, std::min<long long>(R, (long long)num_sms() * per_sm));
}

// dx: one CTA per row (fp32 block sums of dxhat and dxhat*xhat).
// RED: dy is a multicast address (NVLS reduce-load of the TP partial sums); the
// reduced rows are also stored to dy_copy for the gamma/beta kernel.
template <class T, bool RED = false>
__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                        const T* __restrict__ g, const float* __restrict__ mean,
                                                        const float* __restrict__ rstd, const T* __restrict__ dres,
                                                        T* __restrict__ dx, int h, T* __restrict__ dy_copy, int R) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float2 red[32];
  const int nvec = h / V;
  for (long long row = blockIdx.x; row < R; row += gridDim.x) {
  const float mu = mean[row], rs = rstd[row];
  float xh[LNB_MAXV][V], dxh[LNB_MAXV][V];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < LNB_MAXV; ++k) {
    const int vi = threadIdx.x + k * blockDim.x;
    if (vi < nvec) {
      float d[V], xv[V], gg[V];
      ld_in<RED>(dy + row * h + vi * V, d);
      if constexpr (RED) st_vec(dy_copy + row * h + vi * V, d);
      ld_vec(x + row * h + vi * V, xv);
      ld_vec(g + vi * V, gg);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        xh[k][e] = (xv[e] - mu) * rs;
        dxh[k][e] = d[e] * gg[e];
        s1 += dxh[k][e];
        s2 += dxh[k][e] * xh[k][e];
      }
    }
  }
  const float2 sm = block_sum2(s1, s2, red);
  const float m1 = sm.x / h, m2 = sm.y / h;
#pragma unroll
  for (int k = 0; k < LNB_MAXV; ++k) {
    const int vi = threadIdx.x + k * blockDim.x;
    if (vi < nvec) {
      float o[V];
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] = rs * (dxh[k][e] - m1 - xh[k][e] * m2);
      if (dres) {
        float q[V];
        ld_vec(dres + row * h + vi * V, q);
#pragma unroll
        for (int e = 0; e < V; ++e) o[e] += q[e];
      }
      st_vec(dx + row * h + vi * V, o);
    }
  }
  }
}

// Column-reduction tiling shared by the bias / gamma / beta gradient kernels:
// a CTA is CT_X column vectors x CT_Y row groups and covers CT_ROWS rows; a
// thread accumulates its column vector over rows r0 + ty + CT_Y j, the CT_Y
// partials are summed through shared memory and one fp32 atomic per column
// per CTA adds the result into the gradient accumulator.
constexpr int CT_X = 32, CT_Y = 8, CT_ROWS = 64;

template <int V>
__device__ __forceinline__ void ct_reduce_add(float (&acc)[V], float* red /* [CT_Y][CT_X][V] */, float* out,
                                              int vi, int nv) {
  const int tx = threadIdx.x % CT_X, ty = threadIdx.x / CT_X;
#pragma unroll
  for (int e = 0; e < V; ++e) red[(ty * CT_X + tx) * V + e] = acc[e];
  __syncthreads();
  if (ty == 0 && vi < nv) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      float sum = 0.f;
#pragma unroll
      for (int y = 0; y < CT_Y; ++y) sum += red[(y * CT_X + tx) * V + e];
      atomicAdd(out + vi * V + e, sum);
    }
  }
}

static inline dim3 ct_grid(int nv, int R) { return dim3((nv + CT_X - 1) / CT_X, (R + CT_ROWS - 1) / CT_ROWS); }

// out[n] += sum_r X[r, n]
template <class T>
__global__ void __launch_bounds__(CT_X * CT_Y) colsum_kernel(const T* __restrict__ X, float* __restrict__ out, int R,
                                                            int N) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float red[CT_Y * CT_X * V];
  const int tx = threadIdx.x % CT_X, ty = threadIdx.x / CT_X;
  const int nv = N / V, vi = blockIdx.x * CT_X + tx;
  const int r0 = blockIdx.y * CT_ROWS, r1 = min(R, r0 + CT_ROWS);
  float acc[V] = {};
  if (vi < nv) {
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += CT_Y) {
      float v[V];
      ld_vec(X + (long long)r * N + vi * V, v);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] += v[e];
    }
  }
  ct_reduce_add<V>(acc, red, out, vi, nv);
}

template <class T>
mp_status colsum_accum(const T* X, float* out, int R, int N, cudaStream_t st) {
  constexpr int V = VW<T>::N;
  if (N % V) return set_err(MP_EINVAL, "colsum: N %% %d", V);
  pdl_launch(colsum_kernel<T>, ct_grid(N / V, R), CT_X * CT_Y, 0, st, X, out, R, N);
  LAUNCH_CHECK();
}

// dZ = dropout mask * dY (written) and db[n] += sum_r dZ[r, n]   (hidden dropout backward)
template <class T>
__global__ void __launch_bounds__(CT_X * CT_Y) dropout_colsum_kernel(const T* __restrict__ dY, T* __restrict__ dZ,
                                                                    float* __restrict__ out, int R, int N, Dropout dp) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float red[CT_Y * CT_X * V];
  const int tx = threadIdx.x % CT_X, ty = threadIdx.x / CT_X;
  const int nv = N / V, vi = blockIdx.x * CT_X + tx;
  const int r0 = blockIdx.y * CT_ROWS, r1 = min(R, r0 + CT_ROWS);
  float acc[V] = {};
  if (vi < nv) {
    for (int r = r0 + ty; r < r1; r += CT_Y) {
      float v[V];
      ld_vec(dY + (long long)r * N + vi * V, v);
      const int pos = r / dp.b, seq = dp.seq0 + r % dp.b;
      const uint32_t km = keep_bits<V>(dp, (unsigned long long)pos * N + vi * V, 0, seq);
#pragma unroll
      for (int e = 0; e < V; ++e) v[e] = (km >> e) & 1 ? v[e] * dp.scale : 0.f;
      st_vec(dZ + (long long)r * N + vi * V, v);
      ld_vec(dZ + (long long)r * N + vi * V, v);   // the bias gradient sums the stored values
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] += v[e];
    }
  }
  ct_reduce_add<V>(acc, red, out, vi, nv);
}

template <class T>
mp_status dropout_colsum(const T* dY, T* dZ, float* out, int R, int N, Dropout dp, cudaStream_t st) {
  constexpr int V = VW<T>::N;
  if (N % V) return set_err(MP_EINVAL, "dropout_colsum: N %% %d", V);
  pdl_launch(dropout_colsum_kernel<T>, ct_grid(N / V, R), CT_X * CT_Y, 0, st, dY, dZ, out, R, N, dp);
  LAUNCH_CHECK();
}

// dgamma[n] += sum_r dy[r,n] (x[r,n] - mean[r]) rstd[r];  dbeta[n] += sum_r dy[r,n];
// SUMS: also dres_sum[n] += sum_r dres[r,n], dx_sum[n] += sum_r dx[r,n] (stored values)
template <class T, bool SUMS>
__global__ void __launch_bounds__(CT_X * CT_Y) ln_bwd_gb_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                               const float* __restrict__ mean,
                                                               const float* __restrict__ rstd,
                                                               const T* __restrict__ dres, const T* __restrict__ dx,
                                                               float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                               float* __restrict__ dres_sum, float* __restrict__ dx_sum,
                                                               int R, int h) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float red[CT_Y * CT_X * V];
  const int tx = threadIdx.x % CT_X, ty = threadIdx.x / CT_X;
  const int nv = h / V, vi = blockIdx.x * CT_X + tx;
  const int r0 = blockIdx.y * CT_ROWS, r1 = min(R, r0 + CT_ROWS);
  float ag[V] = {}, ab[V] = {}, ar[V] = {}, ax[V] = {};
  if (vi < nv) {
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += CT_Y) {
      float d[V], xv[V];
      ld_vec(dy + (long long)r * h + vi * V, d);
      ld_vec(x + (long long)r * h + vi * V, xv);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        ag[e] += d[e] * (xv[e] - mu) * rs;
        ab[e] += d[e];
      }
      if constexpr (SUMS) {
        float q[V], o[V];
        ld_vec(dres + (long long)r * h + vi * V, q);
        ld_vec(dx + (long long)r * h + vi * V, o);
#pragma unroll
        for (int e = 0; e < V; ++e) { ar[e] += q[e]; ax[e] += o[e]; }
      }
    }
  }
  ct_reduce_add<V>(ag, red, dgamma, vi, nv);
  __syncthreads();
  ct_reduce_add<V>(ab, red, dbeta, vi, nv);
  if constexpr (SUMS) {
    __syncthreads();
    if (dres_sum) ct_reduce_add<V>(ar, red, dres_sum, vi, nv);
    __syncthreads();
    if (dx_sum) ct_reduce_add<V>(ax, red, dx_sum, vi, nv);
  }
}

template <class T>
mp_status layernorm_bwd(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* dres,
                        T* dx, float* dgamma, float* dbeta, int R, int h, cudaStream_t st, T* dy_copy,
                        float* dres_sum, float* dx_sum) {
  MP_TRY(check_row_dims<T>(R, h));
  if ((dres_sum || dx_sum) && !dres) return set_err(MP_EINVAL, "layernorm_bwd: column sums need dres");
  const int nv = h / VW<T>::N;
  if (nv > LNB_MAXV * 256) return set_err(MP_EINVAL, "layernorm_bwd: h=%d too large", h);
  if (dy_copy) {
    pdl_launch(ln_bwd_dx_kernel<T, true>, row_grid(R, nv), row_threads(nv), 0, st, dy, x, g, mean, rstd, dres, dx, h,
                                                                            dy_copy, R);
    dy = dy_copy;
  } else {
    pdl_launch(ln_bwd_dx_kernel<T>, row_grid(R, nv), row_threads(nv), 0, st, dy, x, g, mean, rstd, dres, dx, h, nullptr, R);
  }
  count_launch();
  if (dres_sum || dx_sum)
    pdl_launch(ln_bwd_gb_kernel<T, true>, ct_grid(nv, R), CT_X * CT_Y, 0, st, dy, x, mean, rstd, dres, dx, dgamma, dbeta,
                                                                      dres_sum, dx_sum, R, h);
  else
    pdl_launch(ln_bwd_gb_kernel<T, false>, ct_grid(nv, R), CT_X * CT_Y, 0, st, dy, x, mean, rstd, nullptr, nullptr, dgamma,
                                                                       dbeta, nullptr, nullptr, R, h);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------- GeLU
__device__ __forceinline__ float gelu_f(float u, float* dgelu) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float th = tanhf(c * (u + a * u * u * u));
  if (dgelu) *dgelu = 0.5f * (1.f + th) + 0.5f * u * (1.f - th * th) * c * (1.f + 3.f * a * u * u);
  return 0.5f * u * (1.f + th);
}

template <class T>
__global__ void bias_gelu_fwd_kernel(const T* __restrict__ yv, const T* __restrict__ b, T* __restrict__ out,
                                     long long nvec, int nv_row) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    float a[V], bb[V];
    ld_vec(yv + i * V, a);
    ld_vec(b + (i % nv_row) * V, bb);
#pragma unroll
    for (int e = 0; e < V; ++e) a[e] = gelu_f(a[e] + bb[e], nullptr);
    st_vec(out + i * V, a);
  }
}

template <class T>
mp_status bias_gelu_fwd(const T* yv, const T* b, T* out, long long R, int N, cudaStream_t st) {
  constexpr int V = VW<T>::N;
  if (N % V) return set_err(MP_EINVAL, "bias_gelu: N %% %d", V);
  long long nvec = R * N / V;
  pdl_launch(bias_gelu_fwd_kernel<T>, ew_grid(nvec), 256, 0, st, yv, b, out, nvec, N / V);
  LAUNCH_CHECK();
}

template <class T>
__global__ void __launch_bounds__(CT_X * CT_Y) bias_gelu_bwd_kernel(const T* dh, const T* __restrict__ yv,
                                                                   const T* __restrict__ b, T* du,
                                                                   float* __restrict__ db, int R, int N) {
  pdl_entry();
  // du may alias dh (each element is read, then written, by the same thread)
  constexpr int V = VW<T>::N;
  __shared__ float red[CT_Y * CT_X * V];
  const int tx = threadIdx.x % CT_X, ty = threadIdx.x / CT_X;
  const int nv = N / V, vi = blockIdx.x * CT_X + tx;
  const int r0 = blockIdx.y * CT_ROWS, r1 = min(R, r0 + CT_ROWS);
  float acc[V] = {};
  if (vi < nv) {
    float bb[V] = {};
    if (b) ld_vec(b + vi * V, bb);     // null: yv already holds the biased pre-activation
#pragma unroll 2
    for (int r = r0 + ty; r < r1; r += CT_Y) {
      float d[V], y[V];
      const long long off = (long long)r * N + vi * V;
      ld_vec(dh + off, d);
      ld_vec(yv + off, y);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        float gd;
        gelu_f(y[e] + bb[e], &gd);
        d[e] *= gd;
      }
      st_vec(du + off, d);
      // the bias gradient is the column sum of the stored (rounded) dU
      ld_vec(du + off, d);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] += d[e];
    }
  }
  ct_reduce_add<V>(acc, red, db, vi, nv);
}

template <class T>
mp_status bias_gelu_bwd(const T* dh, const T* yv, const T* b, T* du, float* db, int R, int N, cudaStream_t st) {
  constexpr int V = VW<T>::N;
  if (N % V) return set_err(MP_EINVAL, "bias_gelu_bwd: N %% %d", V);
  pdl_launch(bias_gelu_bwd_kernel<T>, ct_grid(N / V, R), CT_X * CT_Y, 0, st, dh, yv, b, du, db, R, N);
  LAUNCH_CHECK();
}

// ----------------------------------------------------- causal softmax
// One 128-thread CTA per row i of a [z, s, s] score tensor; each thread holds
// VPT 16-byte vectors of the row in registers (high occupancy, all loads of
// the row in flight at once).  Reads columns j <= i only, writes columns
// j < kend(i) (zeros for i < j < kend).  exp2 with the scale folded into log2e.
constexpr int SM_THREADS = 128;

__device__ __forceinline__ float block_max128(float a, float* red) {
  a = warp_max(a);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = a;
  __syncthreads();
  const float r = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  return r;
}
__device__ __forceinline__ float block_sum128(float a, float* red) {
  a = warp_sum(a);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = a;
  __syncthreads();
  const float r = (red[0] + red[1]) + (red[2] + red[3]);
  __syncthreads();
  return r;
}

template <class T, int VPT>
__global__ void __launch_bounds__(SM_THREADS) softmax_fwd_kernel(T* __restrict__ S, int s, float scale_log2) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float red[4];
  const long long rg = blockIdx.x;
  const int i = (int)(rg % s);
  T* p = S + rg * s;
  const int nv_read = i / V + 1;
  const int nv_write = causal_kend(i, s) / V;
  float v[VPT][V];
  float mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + SM_THREADS * k;
    if (vi < nv_read) {
      ld_vec(p + vi * V, v[k]);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[k][e] = vi * V + e <= i ? v[k][e] * scale_log2 : -FLT_MAX;
        mx = fmaxf(mx, v[k][e]);
      }
    }
  }
  mx = block_max128(mx, red);
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + SM_THREADS * k;
    if (vi < nv_read)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[k][e] = vi * V + e <= i ? exp2f(v[k][e] - mx) : 0.f;
        sum += v[k][e];
      }
  }
  const float inv = 1.f / block_sum128(sum, red);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + SM_THREADS * k;
    if (vi < nv_write) {
      float o[V];
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] = vi < nv_read ? v[k][e] * inv : 0.f;
      st_vec(p + vi * V, o);
    }
  }
}

template <class T, int VPT>
__global__ void __launch_bounds__(SM_THREADS) softmax_bwd_kernel(T* __restrict__ dP, const T* __restrict__ P, int s,
                                                                 float scale, Dropout dp) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  __shared__ float red[4];
  const long long rg = blockIdx.x;
  const int i = (int)(rg % s);
  T* dpr = dP + rg * s;
  const T* pp = P + rg * s;
  const int nv_read = i / V + 1;
  const int nv_write = causal_kend(i, s) / V;
  float d[VPT][V], pv[VPT][V];
  float dot = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + SM_THREADS * k;
    if (vi < nv_read) {
      ld_vec(dpr + vi * V, d[k]);
      ld_vec(pp + vi * V, pv[k]);
      if (dp.on()) {   // dP = dropout mask * d(P_dropped)
        const int zz = (int)(rg / s), bb = zz / dp.heads, jj = zz % dp.heads;
        const uint32_t km = keep_bits<V>(dp, (unsigned long long)i * s + vi * V, dp.head0 + jj, dp.seq0 + bb);
#pragma unroll
        for (int e = 0; e < V; ++e) d[k][e] = (km >> e) & 1 ? d[k][e] * dp.scale : 0.f;
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        if (vi * V + e > i) { d[k][e] = 0.f; pv[k][e] = 0.f; }
        dot += d[k][e] * pv[k][e];
      }
    }
  }
  dot = block_sum128(dot, red);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + SM_THREADS * k;
    if (vi < nv_write) {
      float o[V];
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] = vi < nv_read ? pv[k][e] * (d[k][e] - dot) * scale : 0.f;
      st_vec(dpr + vi * V, o);
    }
  }
}

template <class T>
static int softmax_vpt(int s) {
  constexpr int V = VW<T>::N;
  const int need = (s / V + SM_THREADS - 1) / SM_THREADS;
  for (int k : {1, 2, 4})
    if (k >= need) return k;
  return -1;
}

template <class T>
mp_status softmax_causal_fwd(T* S, long long z, int s, float scale, cudaStream_t st) {
  constexpr int V = VW<T>::N;
  if (s % V) return set_err(MP_EINVAL, "softmax: s %% %d", V);
  const int vpt = softmax_vpt<T>(s);
  if (vpt < 0) return set_err(MP_EINVAL, "softmax: s=%d too long", s);
  const long long rows = z * s;
  if (rows > 0x7fffffffLL) return set_err(MP_EINVAL, "softmax: too many rows");
  const float sl2 = scale * 1.4426950408889634f;
  if (vpt == 1) pdl_launch(softmax_fwd_kernel<T, 1>, (unsigned)rows, SM_THREADS, 0, st, S, s, sl2);
  else if (vpt == 2) pdl_launch(softmax_fwd_kernel<T, 2>, (unsigned)rows, SM_THREADS, 0, st, S, s, sl2);
  else pdl_launch(softmax_fwd_kernel<T, 4>, (unsigned)rows, SM_THREADS, 0, st, S, s, sl2);
  LAUNCH_CHECK();
}

template <class T>
mp_status softmax_causal_bwd(T* dP, const T* P, long long z, int s, float scale, cudaStream_t st, Dropout dp) {
  constexpr int V = VW<T>::N;
  if (s % V) return set_err(MP_EINVAL, "softmax: s %% %d", V);
  const int vpt = softmax_vpt<T>(s);
  if (vpt < 0) return set_err(MP_EINVAL, "softmax: s=%d too long", s);
  const long long rows = z * s;
  if (rows > 0x7fffffffLL) return set_err(MP_EINVAL, "softmax: too many rows");
  if (vpt == 1) pdl_launch(softmax_bwd_kernel<T, 1>, (unsigned)rows, SM_THREADS, 0, st, dP, P, s, scale, dp);
  else if (vpt == 2) pdl_launch(softmax_bwd_kernel<T, 2>, (unsigned)rows, SM_THREADS, 0, st, dP, P, s, scale, dp);
  else pdl_launch(softmax_bwd_kernel<T, 4>, (unsigned)rows, SM_THREADS, 0, st, dP, P, s, scale, dp);
  LAUNCH_CHECK();
}

// Pd = dropout(P) over the written region j < kend(i) of a causal [z, s, s]
// probability tensor (attention-probability dropout, unfused path).
template <class T>
__global__ void __launch_bounds__(SM_THREADS) attn_dropout_kernel(const T* __restrict__ P, T* __restrict__ Pd, int s,
                                                                  Dropout dp) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  const long long rg = blockIdx.x;
  const int i = (int)(rg % s);
  const int zz = (int)(rg / s), bb = zz / dp.heads, jj = zz % dp.heads;
  const int nv_write = causal_kend(i, s) / V;
  for (int vi = threadIdx.x; vi < nv_write; vi += SM_THREADS) {
    float v[V];
    ld_vec(P + rg * s + vi * V, v);
    const uint32_t km = keep_bits<V>(dp, (unsigned long long)i * s + vi * V, dp.head0 + jj, dp.seq0 + bb);
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = (km >> e) & 1 ? v[e] * dp.scale : 0.f;
    st_vec(Pd + rg * s + vi * V, v);
  }
}

template <class T>
mp_status attn_dropout(const T* P, T* Pd, long long z, int s, Dropout dp, cudaStream_t st) {
  const long long rows = z * s;
  if (rows > 0x7fffffffLL) return set_err(MP_EINVAL, "attn_dropout: too many rows");
  pdl_launch(attn_dropout_kernel<T>, (unsigned)rows, SM_THREADS, 0, st, P, Pd, s, dp);
  LAUNCH_CHECK();
}

// ------------------------------------------------------------- embedding
template <class T>
__global__ void embed_fwd_kernel(const int* __restrict__ tok, int tok_ld, const T* __restrict__ E, int v0, int Vr,
                                 const T* __restrict__ pos, T* __restrict__ X, int b, int h) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  const int row = blockIdx.x;           // row = i*b + beta
  const int i = row / b, beta = row % b;
  const int id = tok[(long long)beta * tok_ld + i] - v0;
  const bool own = id >= 0 && id < Vr;
  for (int vi = threadIdx.x; vi < h / V; vi += blockDim.x) {
    float o[V] = {};
    if (own) ld_vec(E + (long long)id * h + vi * V, o);
    if (pos) {
      float q[V];
      ld_vec(pos + (long long)i * h + vi * V, q);
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] += q[e];
    }
    st_vec(X + (long long)row * h + vi * V, o);
  }
}

template <class T>
mp_status embed_fwd(const int* tok, int tok_ld, const T* E, int v0, int Vr, const T* pos, T* X, int s, int b, int h,
                    cudaStream_t st) {
  if (h % VW<T>::N) return set_err(MP_EINVAL, "embed: h");
  pdl_launch(embed_fwd_kernel<T>, s * b, std::min(256, std::max(32, h / VW<T>::N)), 0, st, tok, tok_ld, E, v0, Vr, pos, X, b,
                                                                                    h);
  LAUNCH_CHECK();
}

__device__ __forceinline__ void red_v4(float* p, const float* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
               : "memory");
}

template <class T>
__global__ void embed_bwd_kernel(const int* __restrict__ tok, int tok_ld, const T* __restrict__ dX, int v0, int Vr,
                                 float* __restrict__ dE, float* __restrict__ dpos, int b, int h) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  const int row = blockIdx.x;
  const int i = row / b, beta = row % b;
  const int id = tok[(long long)beta * tok_ld + i] - v0;
  const bool own = id >= 0 && id < Vr;
  for (int vi = threadIdx.x; vi < h / V; vi += blockDim.x) {
    float d[V];
    ld_vec(dX + (long long)row * h + vi * V, d);
    // vector reductions (red.global.add.v4.f32): a quarter of the atomic operations
#pragma unroll
    for (int e = 0; e < V; e += 4) {
      if (own) red_v4(dE + (long long)id * h + vi * V + e, d + e);
      if (dpos) red_v4(dpos + (long long)i * h + vi * V + e, d + e);
    }
  }
}

template <class T>
mp_status embed_bwd(const int* tok, int tok_ld, const T* dX, int v0, int Vr, float* dE, float* dpos, int s, int b,
                    int h, cudaStream_t st) {
  if (h % VW<T>::N) return set_err(MP_EINVAL, "embed: h");
  pdl_launch(embed_bwd_kernel<T>, s * b, std::min(256, std::max(32, h / VW<T>::N)), 0, st, tok, tok_ld, dX, v0, Vr, dE, dpos,
                                                                                    b, h);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------- cross-entropy
__global__ void ce_rowmax_kernel(const float* __restrict__ L, float* __restrict__ rowmax, int Vr) {
  pdl_entry();
  __shared__ float red[32];
  const float* p = L + (long long)blockIdx.x * Vr;
  float m = -FLT_MAX;
  for (int j = threadIdx.x * 4; j < Vr; j += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(p + j);
    m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
  }
  m = block_max(m, red);
  if (threadIdx.x == 0) rowmax[blockIdx.x] = m;
}

mp_status ce_rowmax(const float* logits, float* rowmax, int R, int Vr, cudaStream_t st) {
  if (Vr % 4) return set_err(MP_EINVAL, "ce: Vr %% 4");
  pdl_launch(ce_rowmax_kernel, R, 256, 0, st, logits, rowmax, Vr);
  LAUNCH_CHECK();
}

__device__ __forceinline__ int ce_label(const int* lab, int lab_ld, int row, int b) {
  return lab[(long long)(row % b) * lab_ld + row / b];
}

__global__ void ce_sum_kernel(const float* __restrict__ L, const float* __restrict__ rowmax,
                              const int* __restrict__ lab, int lab_ld, int b, int v0, float* __restrict__ out, int R,
                              int Vr) {
  pdl_entry();
  __shared__ float2 red[32];
  const int row = blockIdx.x;
  const float* p = L + (long long)row * Vr;
  const float mx = rowmax[row];
  float s = 0.f;
  for (int j = threadIdx.x * 4; j < Vr; j += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(p + j);
    s += __expf(v.x - mx) + __expf(v.y - mx) + __expf(v.z - mx) + __expf(v.w - mx);
  }
  s = block_sum2(s, 0.f, red).x;
  if (threadIdx.x == 0) {
    const int id = ce_label(lab, lab_ld, row, b) - v0;
    out[row] = s;
    out[R + row] = (id >= 0 && id < Vr) ? p[id] : 0.f;
  }
}

mp_status ce_sumexp_target(const float* logits, const float* rowmax, const int* lab, int lab_ld, int s, int b, int v0,
                           float* sum_tgt, int R, int Vr, cudaStream_t st) {
  pdl_launch(ce_sum_kernel, R, 256, 0, st, logits, rowmax, lab, lab_ld, b, v0, sum_tgt, R, Vr);
  LAUNCH_CHECK();
}

template <class T>
__global__ void ce_grad_kernel(const float* __restrict__ L, const float* __restrict__ rowmax,
                               const float* __restrict__ st, const int* __restrict__ lab, int lab_ld, int b, int v0,
                               float scale, T* __restrict__ dL, float* __restrict__ loss_acc, int R, int Vr) {
  pdl_entry();
  constexpr int V = VW<T>::N;
  const int row = blockIdx.x;
  const float* p = L + (long long)row * Vr;
  const float mx = rowmax[row], sum = st[row];
  const float inv = 1.f / sum;
  const int id = ce_label(lab, lab_ld, row, b) - v0;
  if (threadIdx.x == 0) atomicAdd(loss_acc, scale * (logf(sum) + mx - st[R + row]));
  for (int j = threadIdx.x * V; j < Vr; j += blockDim.x * V) {
    float o[V];
#pragma unroll
    for (int e = 0; e < V; ++e) o[e] = (__expf(p[j + e] - mx) * inv - (j + e == id ? 1.f : 0.f)) * scale;
    st_vec(dL + (long long)row * Vr + j, o);
  }
}

template <class T>
mp_status ce_loss_grad(const float* logits, const float* rowmax, const float* sum_tgt, const int* lab, int lab_ld,
                       int s, int b, int v0, float scale, T* dlogits, float* loss_acc, int R, int Vr, cudaStream_t st) {
  if (Vr % VW<T>::N) return set_err(MP_EINVAL, "ce: Vr");
  pdl_launch(ce_grad_kernel<T>, R, 256, 0, st, logits, rowmax, sum_tgt, lab, lab_ld, b, v0, scale, dlogits, loss_acc, R, Vr);
  LAUNCH_CHECK();
}

// Cross-entropy on the bf16 path (a18): the logit GEMM's epilogue has
// written bf16 logits, per-(row, column block) partials (max, sum exp(x - max))
// of the unrounded fp32 logits and the fp32 target logit of owned labels.
// ce_stats: one warp per row combines the np partials into this shard's row
// max (mx, and mx_local when a TP max-reduction follows) and sum-exp relative
// to it (stt[r]); stt[R + r] = the target logit if the label is in the shard.
__global__ void ce_stats_kernel(const float2* __restrict__ part, int np, const float* __restrict__ tgt,
                                const int* __restrict__ lab, int lab_ld, int b, int v0, int Vr,
                                float* __restrict__ mx, float* __restrict__ mx_local, float* __restrict__ stt,
                                int R) {
  pdl_entry();
  const int lane = threadIdx.x % 32;
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= R) return;
  const float2* p = part + (long long)row * np;
  float m = -FLT_MAX;
  for (int j = lane; j < np; j += 32) m = fmaxf(m, p[j].x);
  m = warp_max(m);
  float s = 0.f;
  for (int j = lane; j < np; j += 32) {
    const float2 q = p[j];
    if (q.y > 0.f) s += q.y * exp2f((q.x - m) * 1.4426950408889634f);
  }
  s = warp_sum(s);
  if (lane == 0) {
    mx[row] = m;
    if (mx_local) mx_local[row] = m;
    stt[row] = s;
    const int id = ce_label(lab, lab_ld, row, b) - v0;
    stt[R + row] = (id >= 0 && id < Vr) ? tgt[row] : 0.f;
  }
}

// after the TP max-reduction of mx: sum-exp relative to the global row max
__global__ void ce_rescale_kernel(const float* __restrict__ mx, const float* __restrict__ mx_local,
                                  float* __restrict__ stt, int R) {
  pdl_entry();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) stt[r] *= exp2f((mx_local[r] - mx[r]) * 1.4426950408889634f);
}

mp_status ce_stats(const float2* part, int np, const float* tgt, const int* lab, int lab_ld, int b, int v0, int Vr,
                   float* mx, float* mx_local, float* stt, int R, cudaStream_t st) {
  pdl_launch(ce_stats_kernel, (R + 7) / 8, 256, 0, st, part, np, tgt, lab, lab_ld, b, v0, Vr, mx, mx_local, stt, R);
  LAUNCH_CHECK();
}
mp_status ce_rescale(const float* mx, const float* mx_local, float* stt, int R, cudaStream_t st) {
  pdl_launch(ce_rescale_kernel, (R + 255) / 256, 256, 0, st, mx, mx_local, stt, R);
  LAUNCH_CHECK();
}

// dlogits = (softmax - onehot) * scale, in place over the bf16 logits (one read
// and one write of the shard, 16-byte vectors); loss += scale (log S + max - target).
__global__ void __launch_bounds__(256) ce_grad_inplace_kernel(__nv_bfloat16* __restrict__ L,
                                                              const float* __restrict__ rowmax,
                                                              const float* __restrict__ st, const int* __restrict__ lab,
                                                              int lab_ld, int b, int v0, float scale,
                                                              float* __restrict__ loss_acc, int R, int Vr) {
  pdl_entry();
  const int row = blockIdx.x;
  __nv_bfloat16* p = L + (long long)row * Vr;
  const float mxl2 = rowmax[row] * 1.4426950408889634f, sum = st[row];
  const float inv = scale / sum;
  const int id = ce_label(lab, lab_ld, row, b) - v0;
  if (threadIdx.x == 0) atomicAdd(loss_acc, scale * (logf(sum) + rowmax[row] - st[R + row]));
  for (int j = threadIdx.x * 8; j < Vr; j += blockDim.x * 8) {
    float v[8];
    ld_vec(p + j, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = exp2f(fmaf(v[e], 1.4426950408889634f, -mxl2)) * inv - (j + e == id ? scale : 0.f);
    st_vec(p + j, v);
  }
}

mp_status ce_grad_inplace(__nv_bfloat16* logits, const float* rowmax, const float* sum_tgt, const int* lab, int lab_ld,
                          int b, int v0, float scale, float* loss_acc, int R, int Vr, cudaStream_t st) {
  if (Vr % 8) return set_err(MP_EINVAL, "ce: Vr %% 8");
  pdl_launch(ce_grad_inplace_kernel, R, 256, 0, st, logits, rowmax, sum_tgt, lab, lab_ld, b, v0, scale, loss_acc, R, Vr);
  LAUNCH_CHECK();
}

// ------------------------------------------------------------------ Adam
template <class T>
__device__ __forceinline__ void adam_elem(float& w, float g, float& m1, float& m2, T& ws, float lr, float b1, float b2,
                                          float eps, float bc1, float bc2) {
  m1 = b1 * m1 + (1.f - b1) * g;
  m2 = b2 * m2 + (1.f - b2) * g * g;
  w = w - lr * (m1 / bc1) / (sqrtf(m2 / bc2) + eps);
  if constexpr (sizeof(T) == 2) ws = __float2bfloat16_rn(w); else ws = w;
}

// 4 parameters per thread per step through 16-byte loads / stores (30 B of
// traffic per bf16-stored parameter); the n % 4 tail is done scalar.
template <class T>
__global__ void adam_kernel(float* w, const float* __restrict__ g, float* __restrict__ m1,
                            float* __restrict__ m2, T* ws /* may alias w (fp32) */, long long n, float lr, float b1, float b2,
                            float eps, float bc1, float bc2) {
  pdl_entry();
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 a = reinterpret_cast<float4*>(m1)[i], c = reinterpret_cast<float4*>(m2)[i];
    T o[4];
    adam_elem(wv.x, gv.x, a.x, c.x, o[0], lr, b1, b2, eps, bc1, bc2);
    adam_elem(wv.y, gv.y, a.y, c.y, o[1], lr, b1, b2, eps, bc1, bc2);
    adam_elem(wv.z, gv.z, a.z, c.z, o[2], lr, b1, b2, eps, bc1, bc2);
    adam_elem(wv.w, gv.w, a.w, c.w, o[3], lr, b1, b2, eps, bc1, bc2);
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(m1)[i] = a;
    reinterpret_cast<float4*>(m2)[i] = c;
    if constexpr (sizeof(T) == 2) {
      uint2 u;
      __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&u);
      h[0] = o[0]; h[1] = o[1]; h[2] = o[2]; h[3] = o[3];
      reinterpret_cast<uint2*>(ws)[i] = u;
    } else {
      reinterpret_cast<float4*>(ws)[i] = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - 4 * n4) {
    const long long i = 4 * n4 + threadIdx.x;
    adam_elem(w[i], g[i], m1[i], m2[i], ws[i], lr, b1, b2, eps, bc1, bc2);
  }
}

template <class T>
mp_status adam_step(float* w, const float* g, float* m1, float* m2, T* w_store, long long n, float lr, float b1,
                    float b2, float eps, float bc1, float bc2, cudaStream_t st) {
  auto al = [](const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
  if (!al(w, 16) || !al(g, 16) || !al(m1, 16) || !al(m2, 16) || !al(w_store, sizeof(T) * 4))
    return set_err(MP_EINVAL, "adam_step: arrays must be 16-byte aligned");
  pdl_launch(adam_kernel<T>, ew_grid(n / 4 + 1), 256, 0, st, w, g, m1, m2, w_store, n, lr, b1, b2, eps, bc1, bc2);
  LAUNCH_CHECK();
}

template <class T>
__global__ void cast_kernel(const float* __restrict__ s, T* __restrict__ d, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 2) d[i] = __float2bfloat16_rn(s[i]); else d[i] = s[i];
  }
}

template <class T>
mp_status cast_from_f32(const float* src, T* dst, long long n, cudaStream_t st) {
  pdl_launch(cast_kernel<T>, ew_grid(n), 256, 0, st, src, dst, n);
  LAUNCH_CHECK();
}

// ------------------------------------------------------ instantiations
#define INST(T)                                                                                                     \
  template mp_status layernorm_fwd<T>(const T*, const T*, const T*, T*, float*, float*, int, int, float,             \
                                      cudaStream_t);                                                                \
  template mp_status bda_layernorm_fwd<T>(const T*, const T*, const T*, T*, const T*, const T*, T*, float*, float*,  \
                                          int, int, float, cudaStream_t, Dropout, bool);                            \
  template mp_status bias_add_residual<T>(const T*, const T*, const T*, T*, long long, int, cudaStream_t, Dropout,   \
                                          bool);                                                                    \
  template mp_status dropout_colsum<T>(const T*, T*, float*, int, int, Dropout, cudaStream_t);                      \
  template mp_status attn_dropout<T>(const T*, T*, long long, int, Dropout, cudaStream_t);                          \
  template mp_status layernorm_bwd<T>(const T*, const T*, const T*, const float*, const float*, const T*, T*,        \
                                      float*, float*, int, int, cudaStream_t, T*, float*, float*);                  \
  template mp_status bias_gelu_fwd<T>(const T*, const T*, T*, long long, int, cudaStream_t);                         \
  template mp_status bias_gelu_bwd<T>(const T*, const T*, const T*, T*, float*, int, int, cudaStream_t);             \
  template mp_status colsum_accum<T>(const T*, float*, int, int, cudaStream_t);                                     \
  template mp_status softmax_causal_fwd<T>(T*, long long, int, float, cudaStream_t);                                \
  template mp_status softmax_causal_bwd<T>(T*, const T*, long long, int, float, cudaStream_t, Dropout);             \
  template mp_status embed_fwd<T>(const int*, int, const T*, int, int, const T*, T*, int, int, int, cudaStream_t);  \
  template mp_status embed_bwd<T>(const int*, int, const T*, int, int, float*, float*, int, int, int, cudaStream_t); \
  template mp_status ce_loss_grad<T>(const float*, const float*, const float*, const int*, int, int, int, int,      \
                                     float, T*, float*, int, int, cudaStream_t);                                    \
  template mp_status adam_step<T>(float*, const float*, float*, float*, T*, long long, float, float, float, float,  \
                                  float, float, cudaStream_t);                                                      \
  template mp_status cast_from_f32<T>(const float*, T*, long long, cudaStream_t);

INST(float)
INST(__nv_bfloat16)

}  // namespace mp
