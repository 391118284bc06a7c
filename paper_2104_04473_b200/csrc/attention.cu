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

#include "common.h"
#include "ptx.cuh"
#include "tma_host.h"
#include "../../include/mp_ops.h"

namespace mp {

namespace fa {
constexpr int BQ = 128, BKV = 128;
constexpr int THREADS = 192;
// shared memory carve-up (bytes)
constexpr int Q_BYTES = 2 * BQ * 128;        // 2 hd-blocks of 64 (hd <= 128)
constexpr int K_BYTES = 2 * BKV * 128;
constexpr int V_BYTES = 2 * 2 * 64 * 128;    // [hd block][kv block] boxes of 64 x 64
constexpr int P_BYTES = 2 * BQ * 128;        // 2 kv-blocks of 64
constexpr int SMEM = Q_BYTES + 2 * (K_BYTES + V_BYTES) + P_BYTES + 1024 + 512;
constexpr int TMEM_COLS = 512;               // S[2] at 0 / 128, O at 256
}  // namespace fa

struct FaArgs {
  int s, heads, hd, nq, nhb;   // nhb = hd blocks of 64
  __nv_bfloat16* O;
  long long ldo;               // row stride of O (b * heads * hd)
  float* L2;                   // [z, s]
  float scale_log2;
};

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
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + P_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* v_full = bar + 3;    // [2]
  uint64_t* kv_empty = bar + 5;  // [2]
  uint64_t* s_full = bar + 7;    // [2]
  uint64_t* s_empty = bar + 9;   // [2]
  uint64_t* p_full = bar + 11;
  uint64_t* o_ready = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // heaviest (longest causal range) query tiles first
  const int qt = g.nq - 1 - (int)(blockIdx.x % g.nq);
  const int z = (int)(blockIdx.x / g.nq);
  const int nkv = qt + 1;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&v_full[i], 1); mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_ready, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

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
          tma_load_3d(sK + st * K_BYTES + hb * BKV * 128, &tmK, &k_full[st], 64 * hb, j * BKV, z);
        mbar_arrive_expect_tx(&v_full[st], g.nhb * 2 * 64 * 128);
        for (int hb = 0; hb < g.nhb; ++hb)
          for (int kb = 0; kb < 2; ++kb)
            tma_load_3d(sV + st * V_BYTES + hb * 2 * 8192 + kb * 8192, &tmV, &v_full[st], 64 * hb, j * BKV + 64 * kb, z);
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
        const uint32_t pa = smem_u32(sP), vb = smem_u32(sV + st * V_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          // P: K-major, 64-wide kv blocks 16 KB apart; V: MN-major, hd blocks 16 KB apart (LBO)
          const uint64_t ad = smem_desc_sw128(pa + (k / 4) * (BQ * 128) + (k % 4) * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(vb + (k / 4) * 8192 + (k % 4) * 2048, 16384, 1024);
          umma_f16(tmem + 256, ad, bd, idesc_o, (jj > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(o_ready);
        umma_commit(&kv_empty[st]);
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
    float m = -FLT_MAX, l = 0.f;
    const uint32_t prow = smem_u32(sP) + r * 128;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      const bool diag = j == qt;
      const uint32_t sa = tmem + lane_off + sb * 128;
      // pass 1: row max of the scaled, masked scores
      float mx = -FLT_MAX;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(sa + 32 * c, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int col = 32 * c + e;
          if (!diag || col <= r) mx = fmaxf(mx, __uint_as_float(v[e]));
        }
      }
      const float m_new = fmaxf(m, mx * g.scale_log2);
      const float alpha = exp2f(m - m_new);
      // P(j-1) has been consumed and O(j-1) is complete: rescale O and reuse the P tile
      if (j > 0) {
        mbar_wait(o_ready, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha < 1.f)) {
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
      // pass 2: P = exp2(s * scale_log2 - m_new) -> bf16 into the swizzled P tile
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(sa + 32 * c, v);
        tmem_ld_wait();
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int col = 32 * c + e;
          float p0 = (!diag || col <= r) ? exp2f(__uint_as_float(v[e]) * g.scale_log2 - m_new) : 0.f;
          float p1 = (!diag || col + 1 <= r) ? exp2f(__uint_as_float(v[e + 1]) * g.scale_log2 - m_new) : 0.f;
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          // the row sum uses the rounded values the P.V product consumes
          const float2 f = __bfloat1622float2(pr);
          rs += f.x + f.y;
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
      mbar_arrive(&s_empty[sb]);
      l = l * alpha + rs;
      m = m_new;
      fence_proxy_async_smem();        // P written by the generic proxy, read by tcgen05.mma
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 context row, L2 = m + log2(l)
    mbar_wait(o_ready, (nkv - 1) & 1);
    tc_fence_after();
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<fa::TMEM_COLS>(tmem);
}

// QKV: [s, b, heads, 3, hd] bf16; O: [s, b, heads, hd] bf16; L2: [b*heads, s] fp32.
mp_status flash_attn_fwd(const void* QKV, void* O, float* L2, int s, int b, int heads, int hd, cudaStream_t st) {
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
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(flash_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
    if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  const long long grid = z * a.nq;
  if (grid > 0x7fffffffLL) return set_err(MP_EINVAL, "flash attention: grid too large");
  flash_fwd_kernel<<<(unsigned)grid, fa::THREADS, fa::SMEM, st>>>(tq, tk, tv, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MP_ECUDA, "flash attention launch: %s", cudaGetErrorString(e));
  return MP_OK;
}

}  // namespace mp

extern "C" mp_status mp_op_flash_attn_fwd(const void* qkv, void* ctx, float* lse2, int s, int b, int heads, int hd,
                                          void* stream) {
  MP_REQUIRE_DEVICE();
  return mp::flash_attn_fwd(qkv, ctx, lse2, s, b, heads, hd, reinterpret_cast<cudaStream_t>(stream));
}
