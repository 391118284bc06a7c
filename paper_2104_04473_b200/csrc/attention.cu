// Fused causal attention core on tcgen05 (replaces the
// a7 scores GEMM + a8 scale-mask-softmax + a9 P.V GEMM when enabled).
//
// Computes, per (batch*head z, query tile of 128 rows), the same result as
// the unfused path ("implicit causal masking", scale 1/sqrt(hd)):
//   O = softmax_causal(Q K^T / sqrt(hd)) V,   L2 = log2-sum-exp of each row
// without ever writing the s x s scores to HBM (online softmax over 128-wide
// key/value tiles).  Reads Q, K, V straight from the [s, b, a/t, 3, hd] QKV
// layout through 3-D TMA maps; writes O into the [s, b, a/t, hd] context
// layout and L2 (fp32 [z, s]) for the backward.
//
// CTA = 6 warps: warp 0 TMA producer (Q once, K/V tiles through a 2-stage
// ring), warp 1 MMA issuer (S = Q K^T into a double-buffered TMEM tile,
// O += P V into a TMEM accumulator), warps 2-5 softmax: each thread owns one
// query row, reads its S row from TMEM, keeps the running max / sum, rescales
// its O row in TMEM when the max grows, and writes P (bf16) into a 128-byte
// swizzled shared-memory tile that is the A operand of the P V product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <queue>
#include <tuple>
#include <vector>

#include "common.h"
#include "launch.cuh"
#include "ptx.cuh"
#include "tma_host.h"
#include "dropout.cuh"
#include "../../include/mp_ops.h"

namespace mp {
extern long long* g_fa_trace;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

namespace fa {
constexpr int BQ = 128, BKV = 128;
constexpr int THREADS = 192;
// shared memory carve-up (bytes)
constexpr int Q_BYTES = 2 * BQ * 128;        // 2 hd-blocks of 64 (hd <= 128)
constexpr int K_BYTES = 2 * BKV * 128;
constexpr int V_BYTES = 2 * 2 * 64 * 128;    // [hd block][kv block] boxes of 64 x 64
constexpr int P_BYTES = 2 * BQ * 128;        // 2 kv-blocks of 64
constexpr int SMEM = Q_BYTES + 2 * (K_BYTES + V_BYTES) + 2 * P_BYTES + 1024 + 512;   // P double buffered
// Lazy rescaling: P is computed against a running reference max that is only
// raised (and O, l rescaled) when the true row max exceeds it by more than
// 2^8, so P <= 256 and most tiles never touch O (bf16 P / fp32 O have the range).
constexpr float RESCALE_LOG2 = 8.f;
constexpr int TMEM_COLS = 512;               // S[2] at 0 / 128, O at 256
}  // namespace fa

struct FaArgs {
  int s, heads, hd, nq, nhb;   // nhb = hd blocks of 64
  __nv_bfloat16* O;
  long long ldo;               // row stride of O (b * heads * hd)
  float* L2;                   // [z, s]
  float scale_log2;
  Dropout dp;                  // attention-probability dropout (off when dp.thresh == 0)
  long long* trace;            // debug: per-tile event timestamps of CTA 0 (null = off)
  const int4* work;            // split-KV mode: per CTA ((z << 16) | q tile, first kv tile, end kv tile, slot)
  float* Opart;                // split-KV: unnormalised fp32 O [slot][128][hd]
  float2* ml;                  // split-KV: (reference max m, sum l) [slot][128]
};

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FA_TRACE(ev, j)                                                         \
  do {                                                                          \
    if (g.trace && blockIdx.x == 0 && (j) < 64) g.trace[(ev) * 64 + (j)] = gtime(); \
  } while (0)

template <bool DROP>
__global__ void __launch_bounds__(fa::THREADS, 1)
flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, FaArgs g) {
  using namespace fa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;                  // [2 stages]
  uint8_t* sV = sK + 2 * K_BYTES;              // [2 stages]
  uint8_t* sP = sV + 2 * V_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * P_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* v_full = bar + 3;    // [2]
  uint64_t* kv_empty = bar + 5;  // [2] K tile free (after its S product) -- V uses v_empty
  uint64_t* v_empty = bar + 14;  // [2] V tile free (after its P.V product)
  uint64_t* s_full = bar + 7;    // [2]
  uint64_t* s_empty = bar + 9;   // [2]
  uint64_t* p_full = bar + 11;
  uint64_t* pv_done = bar + 12;  // [2]: PV of P buffer b complete (buffer reusable, O updated)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // heaviest (longest causal range) query tiles first across the whole grid
  // (longest-processing-time-first list scheduling of the CTAs onto the SMs);
  // split-KV mode: the CTA covers kv tiles j0 .. j0+nkv-1 of its query tile
  int qt, z, j0 = 0, nkv, slot = -1;
  if (g.work) {
    const int4 w = g.work[blockIdx.x];
    z = w.x >> 16; qt = w.x & 0xffff; j0 = w.y; nkv = w.z - w.y; slot = w.w;
  } else {
    const int zn = (int)(gridDim.x / g.nq);
    qt = g.nq - 1 - (int)(blockIdx.x / zn);
    z = (int)(blockIdx.x % zn);
    nkv = qt + 1;
  }

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&v_full[i], 1); mbar_init(&kv_empty[i], 1); mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(&pv_done[0], 1);
    mbar_init(&pv_done[1], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();   // prologue above overlaps the previous kernel's tail

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------- producer
      mbar_arrive_expect_tx(q_full, g.nhb * BQ * 128);
      for (int hb = 0; hb < g.nhb; ++hb) tma_load_3d(sQ + hb * BQ * 128, &tmQ, q_full, 64 * hb, qt * BQ, z);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], g.nhb * BKV * 128);
        for (int hb = 0; hb < g.nhb; ++hb)
          tma_load_3d(sK + st * K_BYTES + hb * BKV * 128, &tmK, &k_full[st], 64 * hb, (j0 + j) * BKV, z);
        FA_TRACE(0, j);
        if (j >= 2) mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        FA_TRACE(1, j);
        mbar_arrive_expect_tx(&v_full[st], g.nhb * 2 * 64 * 128);
        for (int hb = 0; hb < g.nhb; ++hb)
          for (int kb = 0; kb < 2; ++kb)
            tma_load_3d(sV + st * V_BYTES + hb * 2 * 8192 + kb * 8192, &tmV, &v_full[st], 64 * hb,
                        (j0 + j) * BKV + 64 * kb, z);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------ MMA issuer
      const uint32_t idesc_s = idesc_bf16(BQ, BKV, 0, 0);
      const uint32_t idesc_o = idesc_bf16(BQ, g.hd, 0, 1);
      const int ksteps_s = g.hd / 16;
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        const int st = jj & 1;
        mbar_wait(p_full, jj & 1);
        mbar_wait(&v_full[st], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(sP + (jj & 1) * P_BYTES), vb = smem_u32(sV + st * V_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          // P: K-major, 64-wide kv blocks 16 KB apart; V: MN-major, hd blocks 16 KB apart (LBO)
          const uint64_t ad = smem_desc_sw128(pa + (k / 4) * (BQ * 128) + (k % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(vb + (k / 4) * 8192 + (k % 4) * 2048, 16384, 1024);
          umma_f16(tmem + 256, ad, bd, idesc_o, (jj > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[jj & 1]);
        umma_commit(&v_empty[st]);
        FA_TRACE(3, jj);
      };
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1, sb = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ), kb = smem_u32(sK + st * K_BYTES);
        for (int k = 0; k < ksteps_s; ++k) {
          const uint64_t ad = smem_desc_sw128(qa + (k / 4) * (BQ * 128) + (k % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(kb + (k / 4) * (BKV * 128) + (k % 4) * 32, 16, 1024);
          umma_f16(tmem + sb * 128, ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        umma_commit(&kv_empty[st]);       // K(j) consumed: the producer may refill this stage's K
        FA_TRACE(2, j);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nkv - 1);
    }
  } else {
    // ---------------------------------------------------------- softmax
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;                 // row within the tile
    const int qrow = qt * BQ + r;                      // query index
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float m = -FLT_MAX, l = 0.f;      // m: reference max (log2 units) P is computed against
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      const bool diag = j0 + j == qt;
      const uint32_t sa = tmem + lane_off + sb * 128;
      // the whole S row (128 fp32) into registers with one wait; the TMEM tile is then free
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(sa + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&s_empty[sb]);
      if (threadIdx.x == 64) FA_TRACE(4, j);
      // row max over 8 independent chains (a single 128-long fmax chain is latency-bound:
      // ncu r02 "stalled_wait" dominated the softmax warps)
      float mxa[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mxa[k] = -FLT_MAX;
      if (diag) {
#pragma unroll
        for (int e = 0; e < 128; ++e)
          if (e <= r) mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(sv[e]));
      } else {
#pragma unroll
        for (int e = 0; e < 128; ++e) mxa[e & 7] = fmaxf(mxa[e & 7], __uint_as_float(sv[e]));
      }
      const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                             fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
      const float mt = mx * g.scale_log2;
      // raise the reference max only when this tile exceeds it by more than 2^RESCALE_LOG2
      const bool need = __any_sync(0xffffffffu, mt > m + RESCALE_LOG2);
      float alpha = 1.f;
      if (need) {
        const float m_new = fmaxf(m, mt);
        alpha = ex2f(m - m_new);
        m = m_new;
        if (j > 0) {          // O holds P(0..j-1) V: wait for PV(j-1), then rescale it
          mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
          for (int c = 0; c < g.hd; c += 32) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tmem + lane_off + 256 + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_off + 256 + c, o);
          }
          tmem_st_wait();
        }
      }
      if (threadIdx.x == 64) FA_TRACE(5, j);
      // the P buffer of tile j was last read by PV(j-2)
      if (j >= 2) mbar_wait(&pv_done[sb], ((j - 2) >> 1) & 1);
      const uint32_t prow = smem_u32(sP + sb * P_BYTES) + r * 128;
      // P = exp2(s * scale_log2 - m) -> bf16 into the swizzled P tile (dropped
      // entries zeroed and kept ones scaled; the row sum uses the undropped values)
      float rsa[4] = {0.f, 0.f, 0.f, 0.f};   // row sum over 4 independent chains
      constexpr bool drop = DROP;
      const int zb = z / g.dp.heads, zj = z % g.dp.heads;
      const int cut = diag ? r : 127;          // columns > cut are masked (causal diagonal tile)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t km = 0xffffffffu;
        if (drop) {
          km = 0;
          const unsigned long long e0 = (unsigned long long)qrow * g.s + (j0 + j) * BKV + 32 * c;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            km |= keep4(g.dp, e0 / 4 + q4, g.dp.head0 + zj, g.dp.seq0 + zb) << (4 * q4);
        }
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int col = 32 * c + e;
          float p0 = ex2f(fmaf(__uint_as_float(sv[col]), g.scale_log2, -m));
          float p1 = ex2f(fmaf(__uint_as_float(sv[col + 1]), g.scale_log2, -m));
          if (col > cut) p0 = 0.f;
          if (col + 1 > cut) p1 = 0.f;
          rsa[(e >> 1) & 3] += p0 + p1;
          if (drop) {
            p0 = (km >> e) & 1 ? p0 * g.dp.scale : 0.f;
            p1 = (km >> (e + 1)) & 1 ? p1 * g.dp.scale : 0.f;
          }
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          w[e / 2] = *reinterpret_cast<uint32_t*>(&pr);
        }
        // columns 32c..32c+31 = kv block (c/2), 16-byte chunks 4(c%2)..4(c%2)+3
        const uint32_t blk = prow + (c / 2) * (BQ * 128);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = 4 * (c % 2) + q;
          st_shared_v4(blk + ((chunk ^ (r & 7)) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      }
      tc_fence_before();
      l = l * alpha + ((rsa[0] + rsa[1]) + (rsa[2] + rsa[3]));
      fence_proxy_async_smem();        // P written by the generic proxy, read by tcgen05.mma
      mbar_arrive(p_full);
      if (threadIdx.x == 64) FA_TRACE(6, j);
    }
    // epilogue: O / l -> bf16 context row, L2 = m + log2(l)
    mbar_wait(&pv_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
    tc_fence_after();
    if (g.work) {
      // partial result of kv tiles j0 .. j0+nkv-1: unnormalised O, reference max, sum
      // layout [slot][hd / 4][128 rows] of float4: a warp's stores are contiguous
      float4* op = reinterpret_cast<float4*>(g.Opart) + (long long)slot * (g.hd / 4) * BQ + r;
      for (int c = 0; c < g.hd; c += 32) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + lane_off + 256 + c, o);
        tmem_ld_wait();
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          op[(c / 4 + q4) * BQ] = make_float4(__uint_as_float(o[4 * q4]), __uint_as_float(o[4 * q4 + 1]),
                                              __uint_as_float(o[4 * q4 + 2]), __uint_as_float(o[4 * q4 + 3]));
      }
      g.ml[(long long)slot * BQ + r] = make_float2(m, l);
    } else {
    const float inv = 1.f / l;
    const bool ok = qrow < g.s;
    __nv_bfloat16* orow = g.O + (long long)qrow * g.ldo + (long long)z * g.hd;
    for (int c = 0; c < g.hd; c += 32) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tmem + lane_off + 256 + c, o);
      tmem_ld_wait();
      if (ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 pr = __floats2bfloat162_rn(__uint_as_float(o[8 * q + 2 * e]) * inv,
                                                      __uint_as_float(o[8 * q + 2 * e + 1]) * inv);
            w[e] = *reinterpret_cast<uint32_t*>(&pr);
          }
          *reinterpret_cast<uint4*>(orow + c + 8 * q) = u;
        }
      }
    }
    if (ok) g.L2[(long long)z * g.s + qrow] = m + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<fa::TMEM_COLS>(tmem);
}

// ------------------------------------------------- forward, query-tile pairs
// Two consecutive 128-row query tiles A = 2w, B = 2w + 1 of one head per CTA
// (the K / V tiles are loaded once for both), with one softmax warpgroup per
// tile so the tensor core and the two softmax groups ping-pong: while group A
// turns S_A(j) into P_A(j), the MMA warp runs P_B(j-1) V and S_B(j), and the
// other way round.  P is written back into TMEM over S (packed bf16) and read
// from there as the A operand of O += P V, so no shared-memory P tiles exist.
// Warps: 0 TMA, 1 MMA, 2-5 softmax A, 6-9 softmax B.
// TMEM: S_A [0,128), S_B [128,256), O_A [256, 256+hd), O_B [384, 384+hd).
// Same arithmetic as flash_fwd_kernel (lazy 2^8 rescaling, exp2, fp32 O).
namespace fa2 {
constexpr int THREADS = 320;
constexpr int Q_BYTES = 2 * fa::BQ * 128;              // one Q tile (2 hd blocks of 64)
constexpr int K_BYTES = 2 * fa::BKV * 128;
constexpr int V_BYTES = 2 * 2 * 64 * 128;
constexpr int SMEM = 2 * Q_BYTES + 2 * (K_BYTES + V_BYTES) + 1024 + 512;
}  // namespace fa2

template <bool DROP>
__global__ void __launch_bounds__(fa2::THREADS, 1)
flash_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, FaArgs g) {
  using namespace fa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // [2 tiles]
  uint8_t* sK = sQ + 2 * fa2::Q_BYTES;                  // [2 stages]
  uint8_t* sV = sK + 2 * fa2::K_BYTES;                  // [2 stages]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 2 * fa2::V_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* v_full = bar + 3;    // [2]
  uint64_t* k_empty = bar + 5;   // [2] both S products of K(j) done
  uint64_t* v_empty = bar + 7;   // [2] both P.V products of V(j) done
  uint64_t* s_full = bar + 9;    // [2 tiles]
  uint64_t* p_ready = bar + 11;  // [2 tiles] P written into TMEM (S read out)
  uint64_t* pv_done = bar + 13;  // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int npair = (g.nq + 1) / 2;
  const int zn = (int)(gridDim.x / npair);
  const int w = npair - 1 - (int)(blockIdx.x / zn);     // heaviest pairs first
  const int z = (int)(blockIdx.x % zn);
  const int qa = 2 * w, qb = 2 * w + 1;
  const int nA = qa + 1, nB = qb < g.nq ? qb + 1 : 0;   // kv tiles per query tile (causal)
  const int nkv = nB > 0 ? nB : nA;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&v_full[i], 1); mbar_init(&k_empty[i], 1); mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&p_ready[i], 128); mbar_init(&pv_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();   // the prologue above overlaps the previous kernel's tail

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------- producer
      const int ntile = nB > 0 ? 2 : 1;
      mbar_arrive_expect_tx(q_full, ntile * g.nhb * BQ * 128);
      for (int t = 0; t < ntile; ++t)
        for (int hb = 0; hb < g.nhb; ++hb)
          tma_load_3d(sQ + t * fa2::Q_BYTES + hb * BQ * 128, &tmQ, q_full, 64 * hb, (qa + t) * BQ, z);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], g.nhb * BKV * 128);
        for (int hb = 0; hb < g.nhb; ++hb)
          tma_load_3d(sK + st * fa2::K_BYTES + hb * BKV * 128, &tmK, &k_full[st], 64 * hb, j * BKV, z);
        if (j >= 2) mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[st], g.nhb * 2 * 64 * 128);
        for (int hb = 0; hb < g.nhb; ++hb)
          for (int kb = 0; kb < 2; ++kb)
            tma_load_3d(sV + st * fa2::V_BYTES + hb * 2 * 8192 + kb * 8192, &tmV, &v_full[st], 64 * hb,
                        j * BKV + 64 * kb, z);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------ MMA issuer
      // order: S_A(0) S_B(0) | PV_A(0) S_A(1) | PV_B(0) S_B(1) | PV_A(1) S_A(2) | ...
      const uint32_t idesc_s = idesc_bf16(BQ, BKV, 0, 0);
      const uint32_t idesc_o = idesc_bf16(BQ, g.hd, 0, 1);
      const int ksteps_s = g.hd / 16;
      mbar_wait(q_full, 0);
      const uint32_t qbase = smem_u32(sQ);
      auto issue_s = [&](int t, int j) {        // S_t = Q_t K_j^T into TMEM [128 t, +128)
        const int st = j & 1;
        const uint32_t qa_ = qbase + t * fa2::Q_BYTES, kb = smem_u32(sK + st * fa2::K_BYTES);
        for (int k = 0; k < ksteps_s; ++k) {
          const uint64_t ad = smem_desc_sw128(qa_ + (k / 4) * (BQ * 128) + (k % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(kb + (k / 4) * (BKV * 128) + (k % 4) * 32, 16, 1024);
          umma_f16(tmem + 128 * t, ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {       // O_t += P_t V_j, P_t packed bf16 in TMEM [128 t, +64)
        const int st = j & 1;
        mbar_wait(&p_ready[t], j & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(sV + st * fa2::V_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint64_t bd = smem_desc_sw128(vb + (k / 4) * 8192 + (k % 4) * 2048, 16384, 1024);
          umma_f16_ts(tmem + 256 + 128 * t, tmem + 128 * t + 8 * k, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[t]);
      };
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const bool a_on = j < nA, b_on = j < nB;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        tc_fence_after();
        if (j == 0) {
          if (a_on) issue_s(0, 0);
          if (b_on) issue_s(1, 0);
        }
        umma_commit(&k_empty[st]);   // (j > 0: S(j) of both tiles was issued in iteration j - 1)
        mbar_wait(&v_full[st], (j >> 1) & 1);
        tc_fence_after();
        const bool next = j + 1 < nkv;
        if (next) {                  // K(j+1) for the S products issued behind this tile's P.V
          mbar_wait(&k_full[st ^ 1], ((j + 1) >> 1) & 1);
          tc_fence_after();
        }
        if (a_on) {
          issue_pv(0, j);
          if (next && j + 1 < nA) issue_s(0, j + 1);
        }
        if (b_on) {
          issue_pv(1, j);
          if (next && j + 1 < nB) issue_s(1, j + 1);
        }
        umma_commit(&v_empty[st]);
      }
    }
  } else {
    // ---------------------------------------------------------- softmax
    const int t = (warp - 2) / 4;                      // query tile of this warpgroup
    const int nt = t == 0 ? nA : nB;
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const int qt = qa + t;
    const int qrow = qt * BQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t scol = 128 * t, ocol = 256 + 128 * t;
    float m = -FLT_MAX, l = 0.f;
    const int zb = z / g.dp.heads, zj = z % g.dp.heads;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const bool diag = j == qt;
      const int cut = diag ? r : 127;            // columns > cut are masked (causal diagonal tile)
      // two passes over the S row in TMEM (32-column chunks, two loads in flight): the
      // softmax state stays ~100 registers per thread, so both warpgroups fit the register
      // file and alternate on the schedulers
      float mxa[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
      for (int c2 = 0; c2 < 4; c2 += 2) {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(tmem + lane_off + scol + 32 * c2, va);
        tmem_ld_32x32b_x32(tmem + lane_off + scol + 32 * (c2 + 1), vb);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          if (32 * c2 + e <= cut) mxa[e & 3] = fmaxf(mxa[e & 3], __uint_as_float(va[e]));
          if (32 * (c2 + 1) + e <= cut) mxa[e & 3] = fmaxf(mxa[e & 3], __uint_as_float(vb[e]));
        }
      }
      const float mx = fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3]));
      const float mt = mx * g.scale_log2;
      const bool need = __any_sync(0xffffffffu, mt > m + RESCALE_LOG2);
      float alpha = 1.f;
      if (need) {
        const float m_new = fmaxf(m, mt);
        alpha = ex2f(m - m_new);
        m = m_new;
        if (j > 0) {          // O holds P(0..j-1) V: wait for PV(j-1), then rescale it
          mbar_wait(&pv_done[t], (j - 1) & 1);
          tc_fence_after();
          for (int c = 0; c < g.hd; c += 32) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tmem + lane_off + ocol + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_off + ocol + c, o);
          }
        }
      }
      // P = exp2(s scale_log2 - m) -> packed bf16 pairs over S (chunks c2, c2+1 land in the
      // columns of S chunk c2/2, already read); dropped entries zeroed, kept ones scaled, the
      // row sum uses the undropped values
      float rsa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c2 = 0; c2 < 4; c2 += 2) {
        uint32_t vv[2][32];
        tmem_ld_32x32b_x32(tmem + lane_off + scol + 32 * c2, vv[0]);
        tmem_ld_32x32b_x32(tmem + lane_off + scol + 32 * (c2 + 1), vv[1]);
        tmem_ld_wait();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = c2 + h2;
          uint32_t km = 0xffffffffu;
          if (DROP) {
            km = 0;
            const unsigned long long e0 = (unsigned long long)qrow * g.s + j * BKV + 32 * c;
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4)
              km |= keep4(g.dp, e0 / 4 + q4, g.dp.head0 + zj, g.dp.seq0 + zb) << (4 * q4);
          }
          uint32_t wv[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int col = 32 * c + e;
            float p0 = ex2f(fmaf(__uint_as_float(vv[h2][e]), g.scale_log2, -m));
            float p1 = ex2f(fmaf(__uint_as_float(vv[h2][e + 1]), g.scale_log2, -m));
            if (col > cut) p0 = 0.f;
            if (col + 1 > cut) p1 = 0.f;
            rsa[(e >> 1) & 3] += p0 + p1;
            if (DROP) {
              p0 = (km >> e) & 1 ? p0 * g.dp.scale : 0.f;
              p1 = (km >> (e + 1)) & 1 ? p1 * g.dp.scale : 0.f;
            }
            __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
            wv[e / 2] = *reinterpret_cast<uint32_t*>(&pr);
          }
          tmem_st_32x32b_x16(tmem + lane_off + scol + 16 * c, wv);
        }
      }
      const float rs = (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
      l = l * alpha + rs;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_ready[t]);
    }
    // epilogue: O / l -> bf16 context row, L2 = m + log2(l)
    if (nt > 0) {
      mbar_wait(&pv_done[t], (nt - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      const bool ok = qrow < g.s;
      __nv_bfloat16* orow = g.O + (long long)qrow * g.ldo + (long long)z * g.hd;
      for (int c = 0; c < g.hd; c += 32) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + lane_off + ocol + c, o);
        tmem_ld_wait();
        if (ok) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            uint32_t* wq = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 pr = __floats2bfloat162_rn(__uint_as_float(o[8 * q + 2 * e]) * inv,
                                                        __uint_as_float(o[8 * q + 2 * e + 1]) * inv);
              wq[e] = *reinterpret_cast<uint32_t*>(&pr);
            }
            *reinterpret_cast<uint4*>(orow + c + 8 * q) = u;
          }
        }
      }
      if (ok) g.L2[(long long)z * g.s + qrow] = m + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<fa::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------- backward
// Per (head z, key/value tile j) CTA, looping over the query tiles i >= j:
//   S = Q_i K_j^T, dP = dO_i V_j^T                       (TMEM [0,128), [128,256))
//   P = exp2(S log2e/sqrt(hd) - L2_i), dS = P (dP - D_i) / sqrt(hd)   (compute warps)
//   dV_j += P^T dO_i, dK_j += dS^T Q_i                   (TMEM accumulators)
//   dQ_i  = dS K_j -> fp32 vector reductions into a dQ accumulator
// D_i = rowsum(dO_i * O_i) is precomputed.  Q_i / dO_i / K_j tiles serve both
// as K-major and (via the MN-major descriptor view) MN-major operands, and P
// / dS as K-major (dQ) and MN-major (dV, dK) operands: no transposes.
namespace fab {
// warp 0 TMA, warp 1 MMA, warps 2-9 compute: two warps per TMEM lane quarter,
// each taking half of the 128 key columns (P / dS) and of the dQ chunks
constexpr int THREADS = 320;
constexpr int CW = 256;                      // compute threads
constexpr int T_BYTES = 2 * 128 * 128;       // one [128 rows x hd<=128] bf16 tile (2 hd blocks)
constexpr int SMEM = 6 * T_BYTES + 1024 + 512;
}  // namespace fab

struct FabArgs {
  int s, heads, hd, nq, nhb;
  const float* L2;     // [z, s]
  const float* D;      // [z, s]
  float* dQacc;        // [z, s, hd] fp32 (zeroed)
  __nv_bfloat16* dQKV; // [s, b, heads, 3, hd]
  long long ldq;       // b * heads * 3 * hd
  float scale_log2, scale;
  Dropout dp;
  long long* trace;
  const int4* work;    // split mode: per CTA (z, kv tile, first, end query-tile offset); null = whole ranges
  float* dKacc;        // split mode: fp32 [z, s, hd] accumulators of dK / dV (zeroed)
  float* dVacc;
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <bool DROP>
__global__ void __maxnreg__(168)
flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                 const __grid_constant__ CUtensorMap tmdQ, FabArgs g) {
  using namespace fab;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + T_BYTES;
  uint8_t* sQ = sV + T_BYTES;
  uint8_t* sdO = sQ + T_BYTES;
  uint8_t* sP = sdO + T_BYTES;
  uint8_t* sdS = sP + T_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sdS + T_BYTES);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;     // Q_i landed
  uint64_t* q_empty = bar + 2;    // Q_i's last products (dK += dS^T Q_i) complete
  uint64_t* do_full = bar + 7;    // dO_i landed
  uint64_t* do_empty = bar + 9;   // dO_i's last products (dV += P^T dO_i) complete
  uint64_t* sdp_full = bar + 3;
  uint64_t* ds_ready = bar + 4;
  uint64_t* dq_full = bar + 5;
  uint64_t* tmem_free = bar + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // key/value tile, heaviest (most query tiles) first across the whole grid;
  // split mode: a CTA takes query tiles kt+it0 .. kt+it1-1 of its kv tile
  int kt, z, it0 = 0, niter;
  if (g.work) {
    const int4 w = g.work[blockIdx.x];
    z = w.x; kt = w.y; it0 = w.z; niter = w.w - w.z;
  } else {
    const int zn = (int)(gridDim.x / g.nq);
    kt = (int)(blockIdx.x / zn);
    z = (int)(blockIdx.x % zn);
    niter = g.nq - kt;                              // query tiles kt .. nq-1
  }
  const int tile_bytes = g.nhb * 128 * 128;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1); mbar_init(q_full, 1); mbar_init(q_empty, 1); mbar_init(sdp_full, 1);
    mbar_init(do_full, 1); mbar_init(do_empty, 1);
    mbar_init(ds_ready, CW); mbar_init(dq_full, 1); mbar_init(tmem_free, CW);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmdO); tma_prefetch(&tmdQ);
  }
  if (warp == 1) tmem_alloc<fa::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();   // prologue above overlaps the previous kernel's tail

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * tile_bytes);
      for (int hb = 0; hb < g.nhb; ++hb) {
        tma_load_3d(sK + hb * 16384, &tmK, kv_full, 64 * hb, kt * 128, z);
        tma_load_3d(sV + hb * 16384, &tmV, kv_full, 64 * hb, kt * 128, z);
      }
      for (int it = 0; it < niter; ++it) {
        const int qi = kt + it0 + it;
        // dO_i as soon as the dV products of i-1 are done, Q_i after its dK products
        // (the MMA issuer runs the dV products first): the loads overlap the tail of i-1
        if (it > 0) mbar_wait(do_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(do_full, tile_bytes);
        for (int hb = 0; hb < g.nhb; ++hb) tma_load_3d(sdO + hb * 16384, &tmdO, do_full, 64 * hb, qi * 128, z);
        if (it > 0) mbar_wait(q_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(q_full, tile_bytes);
        for (int hb = 0; hb < g.nhb; ++hb) tma_load_3d(sQ + hb * 16384, &tmQ, q_full, 64 * hb, qi * 128, z);
        FA_TRACE(0, it);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_sdp = idesc_bf16(128, 128, 0, 0);
      const uint32_t id_dkv = idesc_bf16(128, g.hd, 1, 1);
      const uint32_t id_dq = idesc_bf16(128, g.hd, 0, 1);
      const int kh = g.hd / 16;
      mbar_wait(kv_full, 0);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), adO = smem_u32(sdO);
      const uint32_t aP = smem_u32(sP), adS = smem_u32(sdS);
      for (int it = 0; it < niter; ++it) {
        if (it > 0) mbar_wait(tmem_free, (it - 1) & 1);
        mbar_wait(do_full, it & 1);
        tc_fence_after();
        for (int k = 0; k < kh; ++k) {       // dP = dO V^T (K-major operands over hd)
          const uint32_t off = (k / 4) * 16384 + (k % 4) * 32;
          umma_f16(tmem + 128, smem_desc_sw128(adO + off, 16, 1024), smem_desc_sw128(aV + off, 16, 1024), id_sdp,
                   k > 0 ? 1u : 0u);
        }
        mbar_wait(q_full, it & 1);
        tc_fence_after();
        for (int k = 0; k < kh; ++k) {       // S = Q K^T
          const uint32_t off = (k / 4) * 16384 + (k % 4) * 32;
          umma_f16(tmem + 0, smem_desc_sw128(aQ + off, 16, 1024), smem_desc_sw128(aK + off, 16, 1024), id_sdp,
                   k > 0 ? 1u : 0u);
        }
        umma_commit(sdp_full);
        FA_TRACE(1, it);
        mbar_wait(ds_ready, it & 1);
        tc_fence_after();
        // reductions over the 128 query rows / 128 keys; MN-major views step K rows by 2 KB,
        // K-major views step 16 columns.  dV first (frees dO_i), then dK (frees Q_i), then dQ.
        for (int k = 0; k < 8; ++k)          // dV += P^T dO
          umma_f16(tmem + 256, smem_desc_sw128(aP + k * 2048, 16384, 1024), smem_desc_sw128(adO + k * 2048, 16384, 1024),
                   id_dkv, (it > 0 || k > 0) ? 1u : 0u);
        umma_commit(do_empty);
        for (int k = 0; k < 8; ++k)          // dK += dS^T Q
          umma_f16(tmem + 384, smem_desc_sw128(adS + k * 2048, 16384, 1024), smem_desc_sw128(aQ + k * 2048, 16384, 1024),
                   id_dkv, (it > 0 || k > 0) ? 1u : 0u);
        umma_commit(q_empty);
        for (int k = 0; k < 8; ++k) {        // dQ_i = dS K  (into the dP columns, already consumed)
          const uint32_t km = (k / 4) * 16384 + (k % 4) * 32;
          umma_f16(tmem + 128, smem_desc_sw128(adS + km, 16, 1024), smem_desc_sw128(aK + k * 2048, 16384, 1024), id_dq,
                   k > 0 ? 1u : 0u);
        }
        umma_commit(dq_full);
        FA_TRACE(2, it);
      }
    }
  } else {
    const int quarter = warp % 4;
    const int half = (warp - 2) / 4;               // key columns 64 half .. +63, dQ chunks c0 + half
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float l2n = 0.f, ddn = 0.f;
    {
      const int q0 = (kt + it0) * 128 + r;
      if (q0 < g.s) { l2n = g.L2[(long long)z * g.s + q0]; ddn = g.D[(long long)z * g.s + q0]; }
    }
    for (int it = 0; it < niter; ++it) {
      const int qi = kt + it0 + it;
      const int q = qi * 128 + r;
      const bool qok = q < g.s;
      const float l2 = l2n, dd = ddn;
      if (it + 1 < niter && q + 128 < g.s) {        // prefetch the next tile's row statistics
        l2n = g.L2[(long long)z * g.s + q + 128];
        ddn = g.D[(long long)z * g.s + q + 128];
      }
      const bool diag = qi == kt;
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      if (threadIdx.x == 64) FA_TRACE(3, it);
      const uint32_t prow = smem_u32(sP) + r * 128, dsrow = smem_u32(sdS) + r * 128;
      constexpr bool drop = DROP;
      const int zb = z / g.dp.heads, zj = z % g.dp.heads;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * half + cc;
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tmem + lane_off + 32 * c, sv);
        tmem_ld_32x32b_x32(tmem + lane_off + 128 + 32 * c, dv);
        tmem_ld_wait();
        uint32_t km = 0xffffffffu;
        if (drop) {
          km = 0;
          const unsigned long long e0 = (unsigned long long)q * g.s + kt * 128 + 32 * c;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            km |= keep4(g.dp, e0 / 4 + q4, g.dp.head0 + zj, g.dp.seq0 + zb) << (4 * q4);
        }
        uint32_t wp[16], wd[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int col = 32 * c + e + u;
            const bool vis = qok && (!diag || col <= r);
            const float pr = vis ? ex2f(fmaf(__uint_as_float(sv[e + u]), g.scale_log2, -l2)) : 0.f;
            const bool keep = (km >> (e + u)) & 1;
            // dV uses the dropped probabilities; dP = mask * d(P_dropped)
            const float dpv = drop ? (keep ? __uint_as_float(dv[e + u]) * g.dp.scale : 0.f) : __uint_as_float(dv[e + u]);
            ds[u] = pr * (dpv - dd) * g.scale;
            p[u] = drop ? (keep ? pr * g.dp.scale : 0.f) : pr;
          }
          __nv_bfloat162 pp = __floats2bfloat162_rn(p[0], p[1]);
          __nv_bfloat162 pd = __floats2bfloat162_rn(ds[0], ds[1]);
          wp[e / 2] = *reinterpret_cast<uint32_t*>(&pp);
          wd[e / 2] = *reinterpret_cast<uint32_t*>(&pd);
        }
        const uint32_t boff = (c / 2) * 16384;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = 4 * (c % 2) + u;
          const uint32_t sw = (uint32_t)((chunk ^ (r & 7)) << 4);
          st_shared_v4(prow + boff + sw, wp[4 * u], wp[4 * u + 1], wp[4 * u + 2], wp[4 * u + 3]);
          st_shared_v4(dsrow + boff + sw, wd[4 * u], wd[4 * u + 1], wd[4 * u + 2], wd[4 * u + 3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_ready);
      if (threadIdx.x == 64) FA_TRACE(4, it);
      // dQ_i tile -> fp32 TMA reduce-add into the dQ accumulator, staged through
      // the P tile (free: the dV product that read it has completed)
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      if (threadIdx.x == 64) FA_TRACE(5, it);
      const int nchunk = g.hd / 32;
      const uint32_t stg = smem_u32(sP) + half * 16384;
      for (int c0 = 0; c0 < nchunk; c0 += 2) {
        const int c = c0 + half;
        const bool has = c < nchunk;                 // warp-uniform
        uint32_t dqv[32];
        if (has) {
          tmem_ld_32x32b_x32(tmem + lane_off + 128 + 32 * c, dqv);
          tmem_ld_wait();
        }
        if (c0 + 2 >= nchunk) {
          tc_fence_before();
          mbar_arrive(tmem_free);      // the next S / dP products may now overwrite TMEM
        }
        if (c0 >= 2) {                 // the previous boxes (same staging halves) must have been read
          if (threadIdx.x == 64) bulk_wait_read<0>();
          named_bar_sync(1, CW);
        }
        if (has) {
          const uint32_t rowa = stg + r * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(rowa + ((j ^ (r & 7)) << 4), dqv[4 * j], dqv[4 * j + 1], dqv[4 * j + 2], dqv[4 * j + 3]);
        }
        fence_proxy_async_smem();
        named_bar_sync(1, CW);
        if (threadIdx.x == 64) {
          for (int u = 0; u < 2 && c0 + u < nchunk; ++u)
            tma_reduce_add_3d(&tmdQ, sP + u * 16384, 32 * (c0 + u), qi * 128, z);
          bulk_commit();
        }
      }
      // the P tile is rewritten by the next iteration: wait until the TMA has read it
      if (threadIdx.x == 64) bulk_wait_read<0>();
      named_bar_sync(1, CW);
      if (threadIdx.x == 64) FA_TRACE(6, it);
    }
    if (threadIdx.x == 64) bulk_wait_all();
    // dK_j, dV_j rows (TMEM lane = key row) -> bf16 into the K / V slots of dQKV
    const int kvrow = kt * 128 + r;
    if (niter > 0) {
      // the last dq_full also covers the final dV / dK products
      const bool ok = kvrow < g.s;
      const int zb = z / g.heads, zh = z % g.heads;
      (void)zb; (void)zh;
      __nv_bfloat16* base = g.dQKV + (long long)kvrow * g.ldq + (long long)z * 3 * g.hd;
      const int part = half;                            // 0: dK (cols 384), 1: dV (cols 256)
      const uint32_t col0 = part == 0 ? 384 : 256;
      if (g.work) {
        // partial sums over this CTA's query tiles: fp32 reductions into the accumulators
        float* acc = (part == 0 ? g.dKacc : g.dVacc) + ((long long)z * g.s + kvrow) * g.hd;
        for (int c = 0; c < g.hd; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem + lane_off + col0 + c, v);
          tmem_ld_wait();
          if (ok) {
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4)
              red_add_v4(acc + c + 4 * q4, __uint_as_float(v[4 * q4]), __uint_as_float(v[4 * q4 + 1]),
                         __uint_as_float(v[4 * q4 + 2]), __uint_as_float(v[4 * q4 + 3]));
          }
        }
      } else {
        __nv_bfloat16* dst = base + (part == 0 ? g.hd : 2 * g.hd);
        for (int c = 0; c < g.hd; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem + lane_off + col0 + c, v);
          tmem_ld_wait();
          if (ok) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint4 u;
              uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 pr = __floats2bfloat162_rn(__uint_as_float(v[8 * q4 + 2 * e]),
                                                          __uint_as_float(v[8 * q4 + 2 * e + 1]));
                w[e] = *reinterpret_cast<uint32_t*>(&pr);
              }
              *reinterpret_cast<uint4*>(dst + c + 8 * q4) = u;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<fa::TMEM_COLS>(tmem);
}

// D[z, q] = sum_d dO[q, z, d] O[q, z, d]   (one warp per row)
__global__ void flash_bwd_dot_kernel(const __nv_bfloat16* __restrict__ dO, const __nv_bfloat16* __restrict__ O,
                                     float* __restrict__ D, int s, int zn, int hd, long long ldo) {
  pdl_entry();
  // 16 lanes per row, one 16-byte vector (8 elements) per lane (hd <= 128); rows taken in
  // memory order (q major, z minor), so a warp streams contiguous [q, z, hd] data
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 16;   // = q * zn + z
  const int j = threadIdx.x % 16;
  const bool ok = row < (long long)zn * s;
  float acc = 0.f;
  if (ok && 8 * j < hd) {
    const long long off = (row / zn) * ldo + (row % zn) * hd + 8 * j;
    const uint4 a = *reinterpret_cast<const uint4*>(dO + off), b = *reinterpret_cast<const uint4*>(O + off);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = __bfloat1622float2(pa[k]), y = __bfloat1622float2(pb[k]);
      acc += x.x * y.x + x.y * y.y;
    }
  }
#pragma unroll
  for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (ok && j == 0) D[(row % zn) * s + row / zn] = acc;
}

// dQacc fp32 [z, s, hd] -> bf16 Q slot of dQKV [s, b, heads, 3, hd]
// (dQ: slot 0; split mode also dK: slot 1, dV: slot 2); 8 elements per thread
__global__ void flash_bwd_dq_kernel(const float* __restrict__ acc0, __nv_bfloat16* __restrict__ dQKV, int s, int zn,
                                    int hd, long long ldq, int slot0, long long slot_stride) {
  pdl_entry();
  const int slot = slot0 + (int)blockIdx.y;        // destination slot; accumulators slot_stride floats apart
  const float* acc = acc0 + blockIdx.y * slot_stride;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;   // one group of 8 elements
  const long long n = (long long)zn * s * hd / 8;
  if (i >= n) return;
  const long long e = 8 * i;
  const int d = (int)(e % hd);
  const long long zq = e / hd;
  const int q = (int)(zq % s), z = (int)(zq / s);
  const float4 v0 = *reinterpret_cast<const float4*>(acc + e), v1 = *reinterpret_cast<const float4*>(acc + e + 4);
  uint4 u;
  __nv_bfloat162* w = reinterpret_cast<__nv_bfloat162*>(&u);
  w[0] = __floats2bfloat162_rn(v0.x, v0.y); w[1] = __floats2bfloat162_rn(v0.z, v0.w);
  w[2] = __floats2bfloat162_rn(v1.x, v1.y); w[3] = __floats2bfloat162_rn(v1.z, v1.w);
  *reinterpret_cast<uint4*>(dQKV + (long long)q * ldq + (long long)z * 3 * hd + slot * hd + d) = u;
}

// Split-Q work decomposition of the backward (few heads per rank, e.g. t >= 2):
// a kv tile's query range [kt, nq) is cut into chunks of L tiles so that the
// grid fills the SMs; L is chosen by list-scheduling the CTAs (heaviest
// first) onto the SMs under a cost model of one unit per query tile plus
// per-CTA overheads, against the unsplit decomposition.  Cached per shape.
struct BwdWork { int4* dev = nullptr; int n = 0; };
static double makespan(std::vector<double> jobs, int M) {
  std::sort(jobs.begin(), jobs.end(), std::greater<double>());
  std::priority_queue<double, std::vector<double>, std::greater<double>> h;
  for (int i = 0; i < M; ++i) h.push(0.0);
  double mx = 0;
  for (double j : jobs) { double t = h.top(); h.pop(); t += j; mx = std::max(mx, t); h.push(t); }
  return mx;
}
static const BwdWork* bwd_work(int zn, int nq, cudaStream_t st) {
  static std::map<std::pair<int, int>, BwdWork> cache;
  auto key = std::make_pair(zn, nq);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second.dev ? &it->second : nullptr;
  const int M = num_sms();
  auto jobs_for = [&](int L) {
    std::vector<double> j;
    for (int z = 0; z < zn; ++z)
      for (int kt = 0; kt < nq; ++kt)
        for (int c = 0; c < nq - kt; c += L) j.push_back(std::min(L, nq - kt - c) + 0.5 + (L < nq ? 0.3 : 0.0));
    return j;
  };
  int bestL = nq;
  double best = makespan(jobs_for(nq), M);
  for (int L : {8, 6, 5, 4, 3, 2}) {
    if (L >= nq) continue;
    const double m = makespan(jobs_for(L), M) + 1.5;   // + zeroing / converting the dK, dV accumulators
    if (m < 0.85 * best) { best = m; bestL = L; }
  }
  if (const char* e = getenv("MP_FA_BWD_SPLIT_L")) bestL = std::max(1, std::min(nq, atoi(e)));   // tuning sweeps
  BwdWork w;
  if (bestL < nq) {
    std::vector<int4> items;
    for (int z = 0; z < zn; ++z)
      for (int kt = 0; kt < nq; ++kt)
        for (int c = 0; c < nq - kt; c += bestL) items.push_back(make_int4(z, kt, c, std::min(nq - kt, c + bestL)));
    std::stable_sort(items.begin(), items.end(), [](const int4& a, const int4& b) { return a.w - a.z > b.w - b.z; });
    if (cudaMalloc(&w.dev, items.size() * sizeof(int4)) == cudaSuccess &&
        cudaMemcpy(w.dev, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice) == cudaSuccess)
      w.n = (int)items.size();
    else
      w.dev = nullptr;
  }
  (void)st;
  auto& ref = cache[key] = w;
  return ref.dev ? &ref : nullptr;
}

// D region padded to 32 floats so the dK / dV accumulators after it stay 128-byte aligned
// (their float4 reduce-adds and loads need 16-byte alignment for any zn * s)
static inline long long d_pad(long long n) { return (n + 31) & ~31LL; }

long long flash_bwd_ws_floats(int s, int b, int heads, int hd) {
  // dQ accumulator, D, and (split mode) dK / dV accumulators
  const long long zs = (long long)b * heads * s;
  return 3LL * zs * hd + d_pad(zs);
}

// dQKV = d/dQKV of the fused attention, given O (= ctx), dO (= dctx), L2 from the forward.
// workspace: fp32 [b*heads*s*hd + b*heads*s] (dQ accumulator, D).
mp_status flash_attn_bwd(const void* QKV, const void* O, const void* dO, const float* L2, void* dQKV, float* ws,
                         int s, int b, int heads, int hd, cudaStream_t st, Dropout dp) {
  if (dp.on() && s % 4) return set_err(MP_EUNSUPPORTED, "fused attention dropout needs s %% 4 == 0");
  if (hd % 32 || hd > 128 || hd < 32) return set_err(MP_EUNSUPPORTED, "flash attention needs hd in {32,64,96,128}");
  const long long ldq = (long long)b * heads * 3 * hd, ldo = (long long)b * heads * hd;
  const long long zn = (long long)b * heads;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(QKV);
  CUtensorMap tq, tk, tv, tdo, tdq;
  bool ok = make_map(&tq, q, hd, s, zn, ldq, 3LL * hd, 128) && make_map(&tk, q + hd, hd, s, zn, ldq, 3LL * hd, 128) &&
            make_map(&tv, q + 2 * hd, hd, s, zn, ldq, 3LL * hd, 128) &&
            make_map(&tdo, dO, hd, s, zn, ldo, (long long)hd, 128) &&
            make_map(&tdq, ws, hd, s, zn, hd, (long long)s * hd, 128, 4);
  if (!ok) return set_err(MP_ECUDA, "flash attention bwd: tensor map encode failed");
  float* dqacc = ws;
  float* D = ws + zn * s * hd;
  float* dkacc = D + d_pad(zn * s);
  float* dvacc = dkacc + zn * s * hd;
  const int nq = (s + 127) / 128;
  const BwdWork* work = bwd_work((int)zn, nq, st);
  MP_CUDA(cudaMemsetAsync(dqacc, 0, sizeof(float) * zn * s * hd, st));
  if (work) MP_CUDA(cudaMemsetAsync(dkacc, 0, sizeof(float) * 2 * zn * s * hd, st));
  {
    const long long rows = zn * s;
    pdl_launch(flash_bwd_dot_kernel, (unsigned)((rows + 15) / 16), 256, 0, st, reinterpret_cast<const __nv_bfloat16*>(dO),
                                                                   reinterpret_cast<const __nv_bfloat16*>(O), D, s,
                                                                   (int)zn, hd, ldo);
    count_launch();
  }
  FabArgs a;
  a.s = s; a.heads = heads; a.hd = hd; a.nq = (s + 127) / 128; a.nhb = (hd + 63) / 64;
  a.L2 = L2; a.D = D; a.dQacc = dqacc; a.dQKV = reinterpret_cast<__nv_bfloat16*>(dQKV); a.ldq = ldq;
  a.scale = 1.f / std::sqrt((float)hd);
  a.scale_log2 = 1.4426950408889634f * a.scale;
  a.dp = dp;
  a.trace = nullptr;
  a.work = work ? work->dev : nullptr;
  a.dKacc = dkacc;
  a.dVacc = dvacc;
  {
    static long long* dtrace = nullptr;
    if (getenv("MP_FA_TRACE")) {
      if (!dtrace) cudaMalloc(&dtrace, 8 * 64 * sizeof(long long));
      cudaMemsetAsync(dtrace, 0, 8 * 64 * sizeof(long long), st);
      a.trace = dtrace;
      g_fa_trace = dtrace;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(flash_bwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fab::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(flash_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fab::SMEM);
    if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention bwd smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  const unsigned grid = work ? (unsigned)work->n : (unsigned)(zn * a.nq);
  if (dp.on()) pdl_launch(flash_bwd_kernel<true>, grid, fab::THREADS, fab::SMEM, st, tq, tk, tv, tdo, tdq, a);
  else pdl_launch(flash_bwd_kernel<false>, grid, fab::THREADS, fab::SMEM, st, tq, tk, tv, tdo, tdq, a);
  count_launch();
  {
    const long long n = zn * s * hd / 8;
    if (work) {   // dQ, dK, dV (dK / dV accumulators are contiguous after D)
      pdl_launch(flash_bwd_dq_kernel, dim3((unsigned)((n + 255) / 256), 1), 256, 0, st, 
          dqacc, reinterpret_cast<__nv_bfloat16*>(dQKV), s, (int)zn, hd, ldq, 0, 0);
      pdl_launch(flash_bwd_dq_kernel, dim3((unsigned)((n + 255) / 256), 2), 256, 0, st, 
          dkacc, reinterpret_cast<__nv_bfloat16*>(dQKV), s, (int)zn, hd, ldq, 1, zn * s * hd);
      count_launch(2);
    } else {
      pdl_launch(flash_bwd_dq_kernel, dim3((unsigned)((n + 255) / 256), 1), 256, 0, st, 
          dqacc, reinterpret_cast<__nv_bfloat16*>(dQKV), s, (int)zn, hd, ldq, 0, 0);
      count_launch();
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa_attr{};
    cudaFuncGetAttributes(&fa_attr, flash_bwd_kernel<false>);
    return set_err(MP_ECUDA, "flash attention bwd launch: %s (kernel: %d regs, max %d threads, %zu local B)",
                   cudaGetErrorString(e), fa_attr.numRegs, fa_attr.maxThreadsPerBlock, fa_attr.localSizeBytes);
  }
  return MP_OK;
}

// Split-KV combine: per (z, query tile) and row, merge the partial results
// (O_p, m_p, l_p) of its nsplit CTAs: M = max m_p, l = sum l_p 2^(m_p - M),
// O = sum O_p 2^(m_p - M) / l, L2 = M + log2 l.  first[zq] = first slot, the
// slots of one tile are consecutive.
__global__ void flash_fwd_combine_kernel(const float* __restrict__ Opart, const float2* __restrict__ ml,
                                         const int2* __restrict__ tiles, __nv_bfloat16* __restrict__ O, float* L2,
                                         int s, int nq, int hd, long long ldo) {
  pdl_entry();
  // block (tile zq, 4-column chunk c4), thread = row: all loads independent across threads
  const int zq = blockIdx.x, c4 = blockIdx.y, r = threadIdx.x;
  const int z = zq / nq, qt = zq % nq;
  const int q = qt * 128 + r;
  if (q >= s) return;
  const int2 t = tiles[zq];               // (first slot, count <= 16)
  float2 v[16];
  float M = -FLT_MAX;
#pragma unroll
  for (int p = 0; p < 16; ++p)
    if (p < t.y) { v[p] = ml[(long long)(t.x + p) * 128 + r]; M = fmaxf(M, v[p].x); }
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 16; ++p)
    if (p < t.y) {
      const float w = ex2f(v[p].x - M);
      l += v[p].y * w;
      const float4 o = reinterpret_cast<const float4*>(Opart)[((long long)(t.x + p) * (hd / 4) + c4) * 128 + r];
      acc.x += o.x * w; acc.y += o.y * w; acc.z += o.z * w; acc.w += o.w * w;
    }
  const float inv = 1.f / l;
  __nv_bfloat16* orow = O + (long long)q * ldo + (long long)z * hd + 4 * c4;
  *reinterpret_cast<__nv_bfloat162*>(orow) = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
  *reinterpret_cast<__nv_bfloat162*>(orow + 2) = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  if (c4 == 0) L2[(long long)z * s + q] = M + log2f(l);
}

// Split-KV decomposition of the forward for small b * heads (cf. bwd_work):
// a query tile's causal kv range [0, qt] is cut into <= 16 chunks of L tiles.
struct FwdWork { int4* dev = nullptr; int2* tiles = nullptr; int n = 0; float* Opart = nullptr; float2* ml = nullptr; };
static const FwdWork* fwd_work(int zn, int nq, int hd) {
  static std::map<std::tuple<int, int, int>, FwdWork> cache;
  auto key = std::make_tuple(zn, nq, hd);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second.dev ? &it->second : nullptr;
  const int M = num_sms();
  auto jobs_for = [&](int L) {
    std::vector<double> j;
    for (int z = 0; z < zn; ++z)
      for (int qt = 0; qt < nq; ++qt)
        for (int c = 0; c <= qt; c += L) j.push_back(std::min(L, qt + 1 - c) + 1.0 + (L < nq ? 0.5 : 0.0));
    return j;
  };
  int bestL = nq;
  double best = makespan(jobs_for(nq), M);
  for (int L : {8, 6, 5, 4, 3, 2}) {
    if (L >= nq || (nq + L - 1) / L > 16) continue;
    const double m = makespan(jobs_for(L), M) + 3.0;   // + the combine pass
    if (m < 0.85 * best) { best = m; bestL = L; }
  }
  if (const char* e = getenv("MP_FA_FWD_SPLIT_L")) bestL = std::max(1, std::min(nq, atoi(e)));   // tuning sweeps
  FwdWork w;
  if (bestL < nq) {
    std::vector<int4> items;
    std::vector<int2> tiles;
    for (int z = 0; z < zn; ++z)
      for (int qt = 0; qt < nq; ++qt) {
        tiles.push_back(make_int2((int)items.size(), (qt + bestL) / bestL));
        for (int c = 0; c <= qt; c += bestL)
          items.push_back(make_int4((z << 16) | qt, c, std::min(qt + 1, c + bestL), (int)items.size()));
      }
    std::stable_sort(items.begin(), items.end(), [](const int4& a, const int4& b) { return a.z - a.y > b.z - b.y; });
    bool ok = cudaMalloc(&w.dev, items.size() * sizeof(int4)) == cudaSuccess &&
              cudaMalloc(&w.tiles, tiles.size() * sizeof(int2)) == cudaSuccess &&
              cudaMalloc(&w.Opart, items.size() * 128 * (size_t)hd * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&w.ml, items.size() * 128 * sizeof(float2)) == cudaSuccess &&
              cudaMemcpy(w.dev, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(w.tiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) w.n = (int)items.size(); else w.dev = nullptr;
  }
  auto& ref = cache[key] = w;
  return ref.dev ? &ref : nullptr;
}

// QKV: [s, b, heads, 3, hd] bf16; O: [s, b, heads, hd] bf16; L2: [b*heads, s] fp32.
mp_status flash_attn_fwd(const void* QKV, void* O, float* L2, int s, int b, int heads, int hd, cudaStream_t st,
                         Dropout dp) {
  if (dp.on() && s % 4) return set_err(MP_EUNSUPPORTED, "fused attention dropout needs s %% 4 == 0");
  if (hd % 32 || hd > 128 || hd < 32) return set_err(MP_EUNSUPPORTED, "flash attention needs hd in {32,64,96,128}");
  if (s < 1 || b < 1 || heads < 1) return set_err(MP_EINVAL, "flash attention: bad shape");
  const long long ldq = (long long)b * heads * 3 * hd;
  const long long z = (long long)b * heads;
  const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(QKV);
  CUtensorMap tq, tk, tv;
  bool ok = make_map(&tq, q, hd, s, z, ldq, 3LL * hd, fa::BQ) && make_map(&tk, q + hd, hd, s, z, ldq, 3LL * hd, fa::BKV) &&
            make_map(&tv, q + 2 * hd, hd, s, z, ldq, 3LL * hd, 64);
  if (!ok) return set_err(MP_ECUDA, "flash attention: tensor map encode failed");
  FaArgs a;
  a.s = s; a.heads = heads; a.hd = hd;
  a.nq = (s + fa::BQ - 1) / fa::BQ;
  a.nhb = (hd + 63) / 64;
  a.O = reinterpret_cast<__nv_bfloat16*>(O);
  a.ldo = (long long)b * heads * hd;
  a.L2 = L2;
  a.scale_log2 = 1.4426950408889634f / std::sqrt((float)hd);
  a.dp = dp;
  if (!dp.on()) a.dp.heads = 1;
  a.trace = nullptr;
  {
    static long long* dtrace = nullptr;
    if (getenv("MP_FA_TRACE")) {
      if (!dtrace) cudaMalloc(&dtrace, 8 * 64 * sizeof(long long));
      cudaMemsetAsync(dtrace, 0, 8 * 64 * sizeof(long long), st);
      a.trace = dtrace;
      extern long long* g_fa_trace;
      g_fa_trace = dtrace;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(flash_fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(flash_fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
    if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  const FwdWork* work = (z < 65536 && a.nq < 65536) ? fwd_work((int)z, a.nq, hd) : nullptr;
  // whole causal ranges: query-tile pairs (one K / V stream, two ping-ponging softmax groups)
  // unless that leaves fewer than two CTAs per SM; MP_FA_FWD_PAIR=0 forces the single-tile kernel
  const char* pe = getenv("MP_FA_FWD_PAIR");   // read per call (tests force both kernels)
  const int pair_env = pe ? atoi(pe) : -1;
  const long long pair_grid = z * ((a.nq + 1) / 2);
  const bool pair = !work && pair_env != 0 && (pair_env == 1 || pair_grid >= 2LL * num_sms());
  if (pair) {
    static bool attr2 = false;
    if (!attr2) {
      cudaError_t e = cudaFuncSetAttribute(flash_fwd_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           fa2::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(flash_fwd_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa2::SMEM);
      if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention smem attr: %s", cudaGetErrorString(e));
      attr2 = true;
    }
    a.work = nullptr;
    if (dp.on()) pdl_launch(flash_fwd_pair_kernel<true>, (unsigned)pair_grid, fa2::THREADS, fa2::SMEM, st, tq, tk, tv, a);
    else pdl_launch(flash_fwd_pair_kernel<false>, (unsigned)pair_grid, fa2::THREADS, fa2::SMEM, st, tq, tk, tv, a);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention launch: %s", cudaGetErrorString(e));
    return MP_OK;
  }
  a.work = work ? work->dev : nullptr;
  a.Opart = work ? work->Opart : nullptr;
  a.ml = work ? work->ml : nullptr;
  const long long grid = work ? work->n : z * a.nq;
  if (grid > 0x7fffffffLL) return set_err(MP_EINVAL, "flash attention: grid too large");
  if (dp.on()) pdl_launch(flash_fwd_kernel<true>, (unsigned)grid, fa::THREADS, fa::SMEM, st, tq, tk, tv, a);
  else pdl_launch(flash_fwd_kernel<false>, (unsigned)grid, fa::THREADS, fa::SMEM, st, tq, tk, tv, a);
  count_launch();
  if (work) {
    pdl_launch(flash_fwd_combine_kernel, dim3((unsigned)(z * a.nq), (unsigned)(hd / 4)), 128, 0, st, 
        work->Opart, work->ml, work->tiles, a.O, L2, s, a.nq, hd, a.ldo);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention launch: %s", cudaGetErrorString(e));
  return MP_OK;
}

long long* g_fa_trace = nullptr;

}  // namespace mp

extern "C" long long mp_op_flash_attn_bwd_ws_floats(int s, int b, int heads, int hd) {
  return mp::flash_bwd_ws_floats(s, b, heads, hd);
}

extern "C" mp_status mp_op_flash_attn_bwd(const void* qkv, const void* ctx, const void* dctx, const float* lse2,
                                          void* dqkv, float* ws, int s, int b, int heads, int hd, void* stream) {
  MP_REQUIRE_DEVICE();
  return mp::flash_attn_bwd(qkv, ctx, dctx, lse2, dqkv, ws, s, b, heads, hd, reinterpret_cast<cudaStream_t>(stream),
                            mp::Dropout{});
}

extern "C" void mp_debug_fa_trace(long long* host512) {
  if (mp::g_fa_trace) cudaMemcpy(host512, mp::g_fa_trace, 8 * 64 * sizeof(long long), cudaMemcpyDeviceToHost);
}

extern "C" mp_status mp_op_flash_attn_fwd(const void* qkv, void* ctx, float* lse2, int s, int b, int heads, int hd,
                                          void* stream) {
  MP_REQUIRE_DEVICE();
  return mp::flash_attn_fwd(qkv, ctx, lse2, s, b, heads, hd, reinterpret_cast<cudaStream_t>(stream), mp::Dropout{});
}
