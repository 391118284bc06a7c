// Batched GEMM engine of the hot path (SURVEY 8(a) rows a6, a7, a9, a10,
// a14, a16, a17, a18): C_z (+)= alpha * A_z B_z + bias.
//
// bf16: persistent, warp-specialised tcgen05 kernel for sm_100a.
//   warp 0  : TMA producer (one elected lane), 128B-swizzled tiles into a
//             STAGES-deep shared-memory ring guarded by full/empty mbarriers;
//   warp 1  : TMEM allocator + MMA issuer (one lane issues tcgen05.mma
//             128 x BN x 16, fp32 accumulators in TMEM, double buffered so
//             the epilogue of tile i overlaps the main loop of tile i+1);
//   warps 2-9: epilogue (two warps per TMEM lane quarter, alternate 128-byte
//             column boxes), tcgen05.ld 32 columns per thread (one TMEM lane =
//             one output row), + bias / GeLU / GeLU' / cross-entropy row
//             statistics, convert, 128B-swizzled staging box -> TMA store, or
//             TMA reduce-add into fp32 accumulators (weight gradients).
// CTA pairs (cta_group::2) for large GEMMs; whole-tile waves + a stream-K tail
// for accumulate GEMMs; raster by estimated DRAM traffic; launched with PDL.
// Operands may be K-major or MN-major (the dX and dW GEMMs of the backward
// and the P V / P^T dO attention products read MN-major tiles directly, so
// no transpose is ever materialised -- the point of the paper's [s,b,a,h]
// layout).
// fp32: a plain SIMT FFMA tiled kernel with the same semantics (parity mode).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <algorithm>

#include "ptx.cuh"
#include "common.h"
#include "tma_host.h"
#include "gemm.h"
#include "launch.cuh"
#include "../../include/mp_ops.h"

namespace mp {

constexpr int BM = 128;
constexpr int BK = 64;              // 64 bf16 = 128 B = one swizzle row
constexpr int EPI_WARPS = 8;               // two warps per TMEM lane quarter
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

// PAIR: CTA pair (cta_group::2) tile of 256 x BN; each CTA holds 128 rows of A
// and BN/2 rows of B per stage and accumulates its 128 x BN half in its TMEM.
template <int BN, bool PAIR = false>
struct TcCfg {
  static constexpr int STAGES = PAIR ? (BN == 256 ? 6 : 8) : (BN == 256 ? 4 : (BN == 128 ? 6 : 8));
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  // epilogue staging: per epilogue warp one 32-row x 128-byte box (TMA store)
  static constexpr int STAGE_OUT_BYTES = EPI_WARPS * 4096;
  static constexpr int SMEM = STAGES * STAGE_BYTES + STAGE_OUT_BYTES + 1024 + 256;
};

struct TcArgs {
  int M, N, K, batch;
  int m_blocks, n_blocks, num_tiles;
  void* C;
  long long ldc, strideC;
  const __nv_bfloat16* bias;
  int c_fp32, accumulate, causal, vec_ok;
  int tma_out;          // epilogue through shared memory + TMA store / reduce-add (tmC valid)
  int stream_k;         // accumulate mode: CTAs split the (tile, k-block) iterations evenly
  int n_fast;           // tile order n-block fastest (consecutive tiles share the A panel)
  int act;              // 1: bf16 C = x and C2 = gelu(x) (tmC2 valid); 2: C = x * gelu'(U), U = aux
  const __nv_bfloat16* aux;   // act 2: pre-activation U, same layout as C
  float* colsum;        // act 2: colsum[n] += sum_m C[m, n] (optional)
  int pair;             // CTA-pair kernel: m_blocks count 256-row pair tiles
  int kb_per_tile;      // k-blocks per tile (stream_k)
  int sk_first;         // stream_k: tiles [0, sk_first) run whole (full waves), the rest is split
  float alpha;
  // act 3 (logit layer + cross-entropy statistics, a18 / P:577): besides the bf16
  // logits, per (row, n-block, epilogue half) the fp32 max and sum of exp(x - max)
  // of the unrounded logits -> ce_part[row][2 n_blocks] (float2), and the fp32
  // target logit of rows whose label falls in this shard -> ce_tgt[row]
  float2* ce_part;
  float* ce_tgt;
  const int* ce_lab;    // labels, row r = i*b + beta -> ce_lab[beta * ce_lab_ld + i] - ce_v0
  int ce_lab_ld, ce_b, ce_v0;
};

__device__ __forceinline__ bool tile_skipped(const TcArgs& g, int m_blk, int n_blk, int BN) {
  return g.causal == 1 && n_blk * BN > m_blk * BM + BM - 1;
}
__device__ __forceinline__ void k_range(const TcArgs& g, int m_blk, int& kb0, int& kb1) {
  int kend = g.K;
  kb0 = 0;
  if (g.causal == 2) kend = min(g.K, (m_blk + 1) * BM);
  if (g.causal == 3) kb0 = (m_blk * BM) / BK;
  kb1 = (kend + BK - 1) / BK;
}

// GeLU, tanh form (P:146 / oracle.layer.gelu), tanh on the SFU (tanh.approx:
// |rel err| ~ 2^-11, below the bf16 rounding of the stored result)
__device__ __forceinline__ float gelu_fast(float u) {
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(0.7978845608028654f * (u + 0.044715f * u * u * u)));
  return 0.5f * u * (1.f + th);
}
// d gelu / du, tanh form (oracle.layer.gelu_grad)
__device__ __forceinline__ float dgelu_fast(float u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(c * (u + a * u * u * u)));
  return 0.5f * (1.f + th) + 0.5f * u * (1.f - th * th) * c * (1.f + 3.f * a * u * u);
}

// Work sequence of one CTA, identical for the producer, MMA and epilogue roles.
// Tile mode: tiles blockIdx.x, +gridDim.x, ... with their (causal) k-block ranges.
// Stream-K mode (accumulate GEMMs, whose epilogue is a TMA reduce-add into the
// fp32 accumulator): the tiles of the full waves [0, sk_first) run whole in tile
// order (concurrent CTAs work on neighbouring tiles, so operand panels are
// shared in L2 at the same k position), then the remaining tiles' (tile,
// k-block) iterations are cut into gridDim.x equal contiguous ranges, so every
// SM gets the same number of k-blocks (no partial last wave); a tile split
// between CTAs is simply reduce-added twice.
struct WorkIter {
  long long i, i1;
  int t, nb;
  __device__ __forceinline__ explicit WorkIter(const TcArgs& g) {
    // CTA pairs walk the tiles together: logical block = cluster index
    const int b = g.pair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    nb = g.pair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    if (g.stream_k) {
      const long long I = (long long)(g.num_tiles - g.sk_first) * g.kb_per_tile;
      const long long i0 = (long long)g.sk_first * g.kb_per_tile;
      i = i0 + I * b / nb;
      i1 = i0 + I * (b + 1) / nb;
    }
    t = b;
  }
  template <int BN>
  __device__ __forceinline__ bool next(const TcArgs& g, int& tile, int& kb0, int& kb1) {
    if (g.stream_k) {
      if (t < g.sk_first) {   // full waves: whole tiles
        tile = t;
        t += nb;
        kb0 = 0;
        kb1 = g.kb_per_tile;
        return true;
      }
      if (i >= i1) return false;
      tile = (int)(i / g.kb_per_tile);
      kb0 = (int)(i % g.kb_per_tile);
      const long long e = min(i1, (long long)(tile + 1) * g.kb_per_tile);
      kb1 = kb0 + (int)(e - i);
      i = e;
      return true;
    }
    const int tiles_per_batch = g.m_blocks * g.n_blocks;
    while (t < g.num_tiles) {
      tile = t;
      t += nb;
      const int rem = tile % tiles_per_batch;
      const int n_blk = g.n_fast ? rem % g.n_blocks : rem / g.m_blocks;
      const int m_blk = g.n_fast ? rem / g.n_blocks : rem % g.m_blocks;
      if (tile_skipped(g, m_blk, n_blk, BN)) continue;
      k_range(g, m_blk, kb0, kb1);
      return true;
    }
    return false;
  }
};

template <int BN, bool A_MN, bool B_MN, bool PAIR, bool CE = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2, TcArgs g) {
  using Cfg = TcCfg<BN, PAIR>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int TM = PAIR ? 2 * BM : BM;           // rows of one (pair) tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sOut = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + Cfg::STAGE_OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;   // 0 = leader (issues the pair MMAs)

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], (PAIR ? 2 : 1) * EPI_WARPS * 32);   // both CTAs' epilogues release the leader's TMEM
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (g.tma_out) tma_prefetch(&tmC);
    if (g.act == 1) tma_prefetch(&tmC2);
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    else tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();      // barriers initialised cluster-wide, TMEM allocated in both CTAs
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int tiles_per_batch = g.m_blocks * g.n_blocks;
  pdl_entry();   // the prologue above overlaps the previous kernel's tail

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      // PAIR: both CTAs load their halves (A rows rank*128.., B rows rank*BN/2..)
      // and signal the leader's full barrier, which the leader arms for both.
      const uint32_t full_cl0 = PAIR ? mapa_shared(&full[0], 0) : 0;
      int stage = 0; uint32_t phase = 0;
      WorkIter it(g);
      int t, kb0, kb1;
      while (it.next<BN>(g, t, kb0, kb1)) {
        const int z = t / tiles_per_batch, rem = t % tiles_per_batch;
        const int n_blk = g.n_fast ? rem % g.n_blocks : rem / g.m_blocks;
        const int m_blk = g.n_fast ? rem / g.n_blocks : rem % g.m_blocks;
        const int arow = m_blk * TM + (int)rank * BM;
        const int brow = PAIR ? n_blk * BN + (int)rank * (BN / 2) : n_blk * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], (PAIR ? 2 : 1) * Cfg::STAGE_BYTES);
          uint8_t* a = sA + stage * Cfg::A_BYTES;
          uint8_t* b = sB + stage * Cfg::B_BYTES;
          if constexpr (PAIR) {
            const uint32_t fb = full_cl0 + stage * 8;
            if (!A_MN) {
              tma_load_3d_pair(a, &tmA, fb, kb * BK, arow, z);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_3d_pair(a + j * 8192, &tmA, fb, arow + 64 * j, kb * BK, z);
            }
            if (!B_MN) {
              tma_load_3d_pair(b, &tmB, fb, kb * BK, brow, z);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j) tma_load_3d_pair(b + j * 8192, &tmB, fb, brow + 64 * j, kb * BK, z);
            }
          } else {
            if (!A_MN) {
              tma_load_3d(a, &tmA, &full[stage], kb * BK, arow, z);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_3d(a + j * 8192, &tmA, &full[stage], arow + 64 * j, kb * BK, z);
            }
            if (!B_MN) {
              tma_load_3d(b, &tmB, &full[stage], kb * BK, brow, z);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_3d(b + j * 8192, &tmB, &full[stage], brow + 64 * j, kb * BK, z);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ------------------------------------------------ MMA issuer (the leader in PAIR mode)
      constexpr uint32_t idesc = idesc_bf16(TM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      WorkIter it(g);
      int t, kb0, kb1;
      while (it.next<BN>(g, t, kb0, kb1)) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart (SBO);
            //   the k-th 16-wide slice starts 32 B further into the row.
            // MN-major SW128: 64-element MN blocks 8 KB apart (LBO), 8-row
            //   K groups 1024 B apart (SBO); the k-th slice is 16 rows = 2 KB on.
            const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(b_addr + k * 32, 16, 1024);
            if constexpr (PAIR) umma_f16_pair(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else umma_f16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (PAIR) umma_commit_pair(&empty[stage], 0x3);   // frees the stage in both CTAs
          else umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR) umma_commit_pair(&tfull[acc], 0x3);
        else umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // -------------------------------------------------- epilogue
    const int quarter = warp % 4;            // TMEM lanes 32*quarter .. +31
    const int half = (warp - 2) / 4;         // the two warps of a quarter take alternate column boxes
    int acc = 0; uint32_t acc_phase = 0;
    uint8_t* stage_base = sOut + (warp - 2) * 4096;
    const uint32_t tempty_cl0 = PAIR ? mapa_shared(&tempty[0], 0) : 0;
    WorkIter it(g);
    int t, kb0, kb1;
    while (it.next<BN>(g, t, kb0, kb1)) {
      const int z = t / tiles_per_batch, rem = t % tiles_per_batch;
      const int n_blk = g.n_fast ? rem % g.n_blocks : rem / g.m_blocks;
      const int m_blk = g.n_fast ? rem / g.n_blocks : rem % g.m_blocks;
      const bool have_acc = kb1 > kb0;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row0 = m_blk * (PAIR ? 2 * BM : BM) + (int)rank * BM + quarter * 32;
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(quarter * 32) << 16);
      float ce_m = -INFINITY, ce_s = 0.f;   // CE: this lane's row over this warp's column boxes
      int ce_t = -1;                        // CE: label column relative to the tile, if in the tile
      if (CE && row0 + lane < g.M) {
        const int r = row0 + lane;
        ce_t = g.ce_lab[(long long)(r % g.ce_b) * g.ce_lab_ld + r / g.ce_b] - g.ce_v0 - n_blk * BN;
      }
      if (g.tma_out) {
        // TMEM -> registers -> 128B-swizzled staging box (32 rows x 128 B) -> TMA
        // store (bf16 / fp32) or TMA reduce-add (fp32 gradient accumulation).
        const int cw = g.c_fp32 ? 32 : 64;     // 128-byte rows: 32 fp32 or 64 bf16 columns per box
        for (int c0 = half * cw; c0 < BN; c0 += 2 * cw) {
          const int col0 = n_blk * BN + c0;
          if (col0 >= g.N) break;
          // this warp's previous box must have been read by its TMA store
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          uint8_t* buf = stage_base;
          const uint32_t rowaddr = smem_u32(buf) + lane * 128;
          if (g.c_fp32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float v[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = 4 * j + e;
                v[e] = have_acc ? __uint_as_float(r[c]) * g.alpha : 0.f;
                if (g.bias && col0 + c < g.N) v[e] += __bfloat162float(g.bias[col0 + c]);
              }
              st_shared_v4(rowaddr + ((j ^ (lane & 7)) << 4), __float_as_uint(v[0]), __float_as_uint(v[1]),
                           __float_as_uint(v[2]), __float_as_uint(v[3]));
            }
          } else {
            uint4 uq[8];
            if (g.act == 2) {   // all 8 loads in flight before any use
              const int row = row0 + lane;
              const __nv_bfloat16* U = g.aux + (long long)z * g.strideC + (long long)row * g.ldc + col0;
              const bool full = col0 + 64 <= g.N && row < g.M;
              if (full) {
#pragma unroll
                for (int chunk = 0; chunk < 8; ++chunk) uq[chunk] = __ldg(reinterpret_cast<const uint4*>(U) + chunk);
              } else {
#pragma unroll
                for (int chunk = 0; chunk < 8; ++chunk) {
                  uint32_t w[4] = {0, 0, 0, 0};
                  if (row < g.M)
                    for (int e = 0; e < 8; ++e)
                      if (col0 + 8 * chunk + e < g.N) {
                        const uint16_t hv = reinterpret_cast<const uint16_t*>(U)[8 * chunk + e];
                        w[e / 2] |= (uint32_t)hv << (16 * (e & 1));
                      }
                  uq[chunk] = make_uint4(w[0], w[1], w[2], w[3]);
                }
              }
            }
            float x[64];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(tbase + c0 + 32 * hf, r);
              tmem_ld_wait();
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                float a0 = have_acc ? __uint_as_float(r[c]) * g.alpha : 0.f;
                const int gc = col0 + 32 * hf + c;
                if (g.bias && gc < g.N) a0 += __bfloat162float(g.bias[gc]);
                x[32 * hf + c] = a0;
              }
            }
            if constexpr (CE) {
              // cross-entropy statistics of the unrounded logits (columns >= N excluded; the TMA
              // store clips them anyway) and the target logit, online over this warp's boxes
              float bm = -INFINITY;
#pragma unroll
              for (int e = 0; e < 64; ++e) {
                if (col0 + e >= g.N) x[e] = -INFINITY;
                bm = fmaxf(bm, x[e]);
                if (ce_t == c0 + e) g.ce_tgt[row0 + lane] = x[e];
              }
              if (bm > -INFINITY) {
                const float mn = fmaxf(ce_m, bm);
                float s = 0.f;
#pragma unroll
                for (int e = 0; e < 64; ++e) s += exp2f((x[e] - mn) * 1.4426950408889634f);
                ce_s = ce_s * exp2f((ce_m - mn) * 1.4426950408889634f) + s;
                ce_m = mn;
              }
            }
            if (g.act == 2) {
              // GeLU backward: x *= gelu'(U) for this lane's row (64 contiguous bf16 = 128 B,
              // loaded before the TMEM reads above so the latency overlaps them)
#pragma unroll
              for (int chunk = 0; chunk < 8; ++chunk) {
                const uint4 q = uq[chunk];
                const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  __nv_bfloat162 pr = *reinterpret_cast<const __nv_bfloat162*>(&qw[e]);
                  x[8 * chunk + 2 * e] *= dgelu_fast(__low2float(pr));
                  x[8 * chunk + 2 * e + 1] *= dgelu_fast(__high2float(pr));
                }
              }
            }
            // pass 0: x (the output, or the pre-activation when act); pass 1 (act): gelu(x)
            for (int pass = 0; pass < (g.act == 1 ? 2 : 1); ++pass) {
              if (pass == 1) {
                // the pre-activation box goes out first, then GeLU reuses the staging buffer
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  tma_store_3d(&tmC, buf, col0, row0, z);
                  bulk_commit();
                  bulk_wait_read<0>();
                }
                __syncwarp();
#pragma unroll
                for (int e = 0; e < 64; ++e) x[e] = gelu_fast(x[e]);
              }
#pragma unroll
              for (int chunk = 0; chunk < 8; ++chunk) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  __nv_bfloat162 pr = __floats2bfloat162_rn(x[8 * chunk + 2 * e], x[8 * chunk + 2 * e + 1]);
                  w[e] = *reinterpret_cast<uint32_t*>(&pr);
                  if (g.act == 2) {   // the column sum is of the stored (rounded) values
                    x[8 * chunk + 2 * e] = __low2float(pr);
                    x[8 * chunk + 2 * e + 1] = __high2float(pr);
                  }
                }
                st_shared_v4(rowaddr + ((chunk ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
              }
            }
            if (g.act == 2 && g.colsum) {
              // column sums of the 32 x 64 box: butterfly reduce-scatter over the warp
              // (halving the live columns each step), then 2 columns per lane -> fp32 atomics
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const bool hi = lane & 16;
                const float send = hi ? x[j] : x[j + 32], keep = hi ? x[j + 32] : x[j];
                x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
              }
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const bool hi = lane & 8;
                const float send = hi ? x[j] : x[j + 16], keep = hi ? x[j + 16] : x[j];
                x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const bool hi = lane & 4;
                const float send = hi ? x[j] : x[j + 8], keep = hi ? x[j + 8] : x[j];
                x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const bool hi = lane & 2;
                const float send = hi ? x[j] : x[j + 4], keep = hi ? x[j + 4] : x[j];
                x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
              }
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const bool hi = lane & 1;
                const float send = hi ? x[j] : x[j + 2], keep = hi ? x[j + 2] : x[j];
                x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
              }
              const int cl = 32 * ((lane >> 4) & 1) + 16 * ((lane >> 3) & 1) + 8 * ((lane >> 2) & 1) +
                             4 * ((lane >> 1) & 1) + 2 * (lane & 1);
#pragma unroll
              for (int j = 0; j < 2; ++j)
                if (col0 + cl + j < g.N) atomicAdd(g.colsum + col0 + cl + j, x[j]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (g.accumulate) tma_reduce_add_3d(&tmC, buf, col0, row0, z);
            else tma_store_3d(g.act == 1 ? &tmC2 : &tmC, buf, col0, row0, z);
            bulk_commit();
          }
        }
        if (CE && row0 + lane < g.M)
          g.ce_part[(long long)(row0 + lane) * (2 * g.n_blocks) + 2 * n_blk + half] = make_float2(ce_m, ce_s);
      } else {
        const int row = row0 + lane;
        const bool row_ok = row < g.M;
        for (int c0 = half * 32; c0 < BN; c0 += 64) {
          const int col0 = n_blk * BN + c0;
          if (col0 >= g.N) break;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + c0, r);
          tmem_ld_wait();
          if (!row_ok) continue;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = have_acc ? __uint_as_float(r[j]) * g.alpha : 0.f;
          const int ncols = min(32, g.N - col0);
          if (g.bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncols) v[j] += __bfloat162float(g.bias[col0 + j]);
          }
          const long long off = (long long)z * g.strideC + (long long)row * g.ldc + col0;
          if (g.c_fp32) {
            float* C = reinterpret_cast<float*>(g.C) + off;
            for (int j = 0; j < ncols; ++j) C[j] = g.accumulate ? C[j] + v[j] : v[j];
          } else {
            __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(g.C) + off;
            for (int j = 0; j < ncols; ++j) C[j] = __float2bfloat16_rn(v[j]);
          }
        }
      }
      tc_fence_before();
      if constexpr (PAIR) mbar_arrive_cluster(tempty_cl0 + acc * 8);   // the leader's barrier
      else mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();      // both CTAs done with the pair's TMEM before it is freed
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (PAIR) tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
    else tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// ----------------------------------------------------------- fp32 SIMT GEMM
constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

__global__ void __launch_bounds__(256)
simt_gemm_kernel(mp_gemm_desc g, int m_blocks, int n_blocks) {
  pdl_entry();
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int z = blockIdx.z;
  const int m_blk = blockIdx.x, n_blk = blockIdx.y;
  const int m0 = m_blk * SB_M, n0 = n_blk * SB_N;
  if (g.causal == 1 && n0 > m0 + SB_M - 1) return;
  int k0 = 0, k1 = g.K;
  if (g.causal == 2) k1 = min(g.K, (m0 / BM + 1) * BM);
  if (g.causal == 3) k0 = (m0 / BM) * BM;
  const float* A = reinterpret_cast<const float*>(g.A) + (long long)z * g.strideA;
  const float* B = reinterpret_cast<const float*>(g.B) + (long long)z * g.strideB;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int kk = k0; kk < k1; kk += SB_K) {
    for (int i = threadIdx.x; i < SB_K * SB_M; i += 256) {
      int kq = i / SB_M, mq = i % SB_M;          // mq fastest: coalesced for MN-major
      int m = m0 + mq, k = kk + kq;
      float va = 0.f;
      if (m < g.M && k < k1) va = g.a_major ? A[(long long)k * g.lda + m] : A[(long long)m * g.lda + k];
      As[kq][mq] = va;
      int n = n0 + mq;
      float vb = 0.f;
      if (n < g.N && k < k1) vb = g.b_major ? B[(long long)k * g.ldb + n] : B[(long long)n * g.ldb + k];
      Bs[kq][mq] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kq = 0; kq < SB_K; ++kq) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kq][ty * 4 + i]; b[i] = Bs[kq][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* C = reinterpret_cast<float*>(g.C) + (long long)z * g.strideC;
  const float* bias = reinterpret_cast<const float*>(g.bias);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j] * g.alpha + (bias ? bias[n] : 0.f);
      float* c = C + (long long)m * g.ldc + n;
      *c = g.accumulate ? *c + v : v;
    }
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D tensor map: dims (inner, outer, batch), 128B swizzle, box (128 B of inner, box_outer, 1).
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t batch,
              uint64_t ld_elems, uint64_t batch_stride_elems, uint32_t box_outer, int esize) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  if (batch <= 1) { batch = 1; batch_stride_elems = ld_elems * outer; }
  cuuint64_t dims[3] = {inner, outer, batch};
  cuuint64_t strides[2] = {ld_elems * esize, batch_stride_elems * esize};
  cuuint32_t box[3] = {(cuuint32_t)(128 / esize), box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int pick_bn(const mp_gemm_desc& g) {
  if (g.N <= 64) return 64;
  if (g.N <= 128) return 128;
  // prefer 256-wide tiles unless that leaves most SMs idle
  long long tiles256 = (long long)((g.M + BM - 1) / BM) * ((g.N + 255) / 256) * g.batch;
  if (tiles256 < num_sms() / 2) return 128;
  return 256;
}

template <int BN, bool A_MN, bool B_MN, bool PAIR, bool CE = false>
static cudaError_t launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                             const CUtensorMap& tc2, const TcArgs& a, int grid, cudaStream_t st) {
  using Cfg = TcCfg<BN, PAIR>;
  auto k = tc_gemm_kernel<BN, A_MN, B_MN, PAIR, CE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, k, ta, tb, tc, tc2, a);
  } else {
    pdl_launch(k, grid, GEMM_THREADS, Cfg::SMEM, st, ta, tb, tc, tc2, a);
    return cudaGetLastError();
  }
}

template <int BN, bool PAIR>
static cudaError_t dispatch_major(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                                  const CUtensorMap& tc2, const TcArgs& a, int grid, int am, int bm, cudaStream_t st) {
  if (!am && !bm) return launch_tc<BN, false, false, PAIR>(ta, tb, tc, tc2, a, grid, st);
  if (!am && bm) return launch_tc<BN, false, true, PAIR>(ta, tb, tc, tc2, a, grid, st);
  if (am && !bm) return launch_tc<BN, true, false, PAIR>(ta, tb, tc, tc2, a, grid, st);
  return launch_tc<BN, true, true, PAIR>(ta, tb, tc, tc2, a, grid, st);
}

// CTA budget of the next persistent GEMM launches (0 = every SM): lets a GEMM
// on a side stream leave SMs to a concurrent communication-bound kernel.
static int g_max_ctas = 0;
void gemm_set_max_ctas(int n) { g_max_ctas = n; }
static int sm_cap() { return g_max_ctas > 0 ? std::min(g_max_ctas, num_sms()) : num_sms(); }
static int tc_grid(const TcArgs& a) {
  if (a.pair) return a.stream_k ? 2 * (sm_cap() / 2) : 2 * std::max(1, std::min(a.num_tiles, sm_cap() / 2));
  if (a.stream_k) return sm_cap();
  return std::max(1, std::min(a.num_tiles, sm_cap()));
}
// Stream-K for an accumulate GEMM when whole-tile scheduling would leave the
// last wave less than ~90% full and every CTA still gets >= 8 k-blocks.
static bool want_stream_k(const TcArgs& a) {
  if (!a.accumulate || !a.tma_out || a.bias || a.causal) return false;
  const int G = a.pair ? sm_cap() / 2 : sm_cap();   // CTA pairs walk the work together
  if (a.num_tiles <= 0) return false;
  const long long waves = (a.num_tiles + G - 1) / G;
  const double fill = (double)a.num_tiles / (double)(waves * G);
  const long long iters = (long long)a.num_tiles * a.kb_per_tile;
  return fill < 0.9 && iters / G >= 8;
}

mp_status gemm_bf16(const mp_gemm_desc& g, cudaStream_t st, const GemmCe* ce = nullptr) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return set_err(MP_EINVAL, "gemm: empty shape");
  if (g.accumulate && !g.c_fp32) return set_err(MP_EINVAL, "gemm: accumulate needs fp32 C");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(g.A) || !al16(g.B) || (g.lda * 2) % 16 || (g.ldb * 2) % 16 || (g.strideA * 2) % 16 ||
      (g.strideB * 2) % 16)
    return set_err(MP_EINVAL, "gemm: TMA needs 16-byte aligned operands and strides");
  const int BN = pick_bn(g);
  TcArgs a;
  a.M = g.M; a.N = g.N; a.K = g.K; a.batch = g.batch;
  a.m_blocks = (g.M + BM - 1) / BM;
  a.n_blocks = (g.N + BN - 1) / BN;
  a.num_tiles = a.m_blocks * a.n_blocks * g.batch;
  a.C = g.C; a.ldc = g.ldc; a.strideC = g.strideC;
  a.bias = reinterpret_cast<const __nv_bfloat16*>(g.bias);
  a.c_fp32 = g.c_fp32; a.accumulate = g.accumulate; a.causal = g.causal; a.alpha = g.alpha;
  a.pair = 0;
  const int esz = g.c_fp32 ? 4 : 2;
  a.vec_ok = al16(g.C) && (g.ldc * esz) % 16 == 0 && (g.strideC * esz) % 16 == 0;
  CUtensorMap tc;
  memset(&tc, 0, sizeof(tc));
  // epilogue via TMA: C box = 32 rows x 128 bytes
  a.tma_out = a.vec_ok && make_map(&tc, g.C, g.N, g.M, g.batch, g.ldc, g.strideC, 32, esz);
  CUtensorMap tc2;
  memset(&tc2, 0, sizeof(tc2));
  a.act = g.act;
  a.aux = reinterpret_cast<const __nv_bfloat16*>(g.C2);
  a.colsum = g.colsum;
  a.ce_part = nullptr; a.ce_tgt = nullptr; a.ce_lab = nullptr;
  a.ce_lab_ld = 0; a.ce_b = 1; a.ce_v0 = 0;
  if (ce) {
    if (g.act || g.c_fp32 || g.accumulate || g.bias || g.causal || g.batch != 1 || !a.tma_out)
      return set_err(MP_EINVAL, "gemm: the cross-entropy epilogue needs a plain bf16 GEMM (16-byte aligned C)");
    a.act = 3;
    a.ce_part = ce->part; a.ce_tgt = ce->tgt; a.ce_lab = ce->lab;
    a.ce_lab_ld = ce->lab_ld; a.ce_b = ce->b; a.ce_v0 = ce->v0;
  } else if (g.act == 3) {
    return set_err(MP_EINVAL, "gemm: act 3 is internal (logit layer)");
  }
  if (g.act == 2) {
    if (g.c_fp32 || g.accumulate || g.bias || !a.tma_out || !g.C2 || g.causal)
      return set_err(MP_EINVAL, "gemm: act 2 needs bf16 C, the pre-activation C2, no bias / accumulate");
  } else if (g.act) {
    if (g.c_fp32 || g.accumulate || !a.tma_out || !al16(g.C2) ||
        !make_map(&tc2, g.C2, g.N, g.M, g.batch, g.ldc, g.strideC, 32, esz))
      return set_err(MP_EINVAL, "gemm: act needs bf16 C / C2, 16-byte aligned, no accumulate");
  }
  a.kb_per_tile = (g.K + BK - 1) / BK;
  // CTA pairs (cta_group::2, 256 x BN tiles): halves each SM's B-operand traffic
  // from L2.  GEMMs with >= 2 row blocks, BN >= 128, TMA epilogue, and >= 60
  // GFLOP: interleaved A/B timing (MP_GEMM_NO_PAIR on / off, round 1) had the pair
  // 3-23 % faster on the layer and logit GEMMs of >= 65 GFLOP and up to 14 %
  // slower on single-wave GEMMs below ~45 GFLOP.
  const bool no_pair = getenv("MP_GEMM_NO_PAIR") != nullptr;   // read per call (A/B timing)
  const double flop = 2.0 * g.M * (double)g.N * g.K * g.batch;
  if (!no_pair && !g.causal && BN >= 128 && a.m_blocks >= 2 && a.tma_out && (sm_cap() % 2) == 0 && flop >= 60e9) {
    a.pair = 1;
    a.m_blocks = (g.M + 2 * BM - 1) / (2 * BM);
    a.num_tiles = a.m_blocks * a.n_blocks * g.batch;
  }
  // Raster: by default consecutive tiles share the B panel (m fastest).  When A
  // is the large operand and B fits comfortably in L2 (e.g. the logit-layer
  // weight gradient dE = dlogits^T Z, A = 210 MB, B = 9 MB), walk n fastest so
  // every A panel is streamed from DRAM once instead of once per n-block.
  // More generally: in m-fast order every wave of concurrent tiles spans all m-blocks,
  // so A is streamed once per wave unless it stays L2-resident, while B is read once;
  // n-fast is the transpose.  Pick the order with the smaller estimated DRAM
  // operand traffic (an operand up to ~40 MB counts as L2-resident across waves).
  {
    const double a_bytes = 2.0 * g.M * (double)g.K * g.batch, b_bytes = 2.0 * g.N * (double)g.K * g.batch;
    const double conc = a.pair ? sm_cap() / 2 : sm_cap();   // tiles in flight (pair tiles are 256 rows)
    const double waves = std::max(1.0, std::ceil((double)a.num_tiles / std::max(1.0, conc)));
    const double l2 = 40e6;
    const double m_fast = (a_bytes > l2 ? a_bytes * std::min(waves, (double)a.n_blocks) : a_bytes) + b_bytes;
    const double n_fast = (b_bytes > l2 ? b_bytes * std::min(waves, (double)a.m_blocks) : b_bytes) + a_bytes;
    static const bool old_raster = getenv("MP_GEMM_RASTER_V1") != nullptr;   // A/B: round-1 rule
    if (old_raster)
      a.n_fast = (a.n_blocks > 1 && a_bytes > 2.0 * b_bytes && b_bytes < 32e6) ? 1 : 0;
    else
      a.n_fast = (a.n_blocks > 1 && n_fast < 0.95 * m_fast) ? 1 : 0;
  }
  a.stream_k = 0;
  a.sk_first = 0;
  static const bool no_sk = getenv("MP_GEMM_NO_STREAMK") != nullptr;
  a.stream_k = want_stream_k(a) && !no_sk;
  if (a.stream_k) {   // whole tiles for the full waves, stream-K only for the partial last wave
    static const bool sk_all = getenv("MP_GEMM_STREAMK_ALL") != nullptr;   // A/B: round-1 pure stream-K
    const int G = a.pair ? sm_cap() / 2 : sm_cap();
    a.sk_first = sk_all ? 0 : (a.num_tiles / G) * G;
  }
  CUtensorMap ta, tb;
  bool ok = g.a_major ? make_map(&ta, g.A, g.M, g.K, g.batch, g.lda, g.strideA, BK)
                      : make_map(&ta, g.A, g.K, g.M, g.batch, g.lda, g.strideA, BM);
  ok = ok && (g.b_major ? make_map(&tb, g.B, g.N, g.K, g.batch, g.ldb, g.strideB, BK)
                        : make_map(&tb, g.B, g.K, g.N, g.batch, g.ldb, g.strideB, a.pair ? BN / 2 : BN));
  if (!ok) return set_err(MP_ECUDA, "gemm: cuTensorMapEncodeTiled failed");
  const int grid = tc_grid(a);
  cudaError_t e;
  if (a.act == 3) {   // logit GEMM (both operands K-major) with the cross-entropy statistics epilogue
    if (g.a_major || g.b_major) return set_err(MP_EINVAL, "gemm: CE epilogue needs K-major operands");
    if (a.pair) e = BN == 128 ? launch_tc<128, false, false, true, true>(ta, tb, tc, tc2, a, grid, st)
                              : launch_tc<256, false, false, true, true>(ta, tb, tc, tc2, a, grid, st);
    else if (BN == 64) e = launch_tc<64, false, false, false, true>(ta, tb, tc, tc2, a, grid, st);
    else if (BN == 128) e = launch_tc<128, false, false, false, true>(ta, tb, tc, tc2, a, grid, st);
    else e = launch_tc<256, false, false, false, true>(ta, tb, tc, tc2, a, grid, st);
  } else if (a.pair) {
    if (BN == 128) e = dispatch_major<128, true>(ta, tb, tc, tc2, a, grid, g.a_major, g.b_major, st);
    else e = dispatch_major<256, true>(ta, tb, tc, tc2, a, grid, g.a_major, g.b_major, st);
  } else {
    if (BN == 64) e = dispatch_major<64, false>(ta, tb, tc, tc2, a, grid, g.a_major, g.b_major, st);
    else if (BN == 128) e = dispatch_major<128, false>(ta, tb, tc, tc2, a, grid, g.a_major, g.b_major, st);
    else e = dispatch_major<256, false>(ta, tb, tc, tc2, a, grid, g.a_major, g.b_major, st);
  }
  if (e != cudaSuccess) return set_err(MP_ECUDA, "gemm launch: %s", cudaGetErrorString(e));
  return MP_OK;
}

mp_status gemm_fp32(const mp_gemm_desc& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return set_err(MP_EINVAL, "gemm: empty shape");
  if (g.act) return set_err(MP_EUNSUPPORTED, "gemm: the fused GeLU epilogue is bf16-only");
  dim3 grid((g.M + SB_M - 1) / SB_M, (g.N + SB_N - 1) / SB_N, g.batch);
  pdl_launch(simt_gemm_kernel, grid, 256, 0, st, g, (int)grid.x, (int)grid.y);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MP_ECUDA, "simt gemm launch: %s", cudaGetErrorString(e));
  return MP_OK;
}

// ------------------------------------------------------ live GEMM profile
// Algorithmic FLOPs of one call: 2 M N K per batch for dense GEMMs; for the
// causal attention GEMMs only the defined (lower-triangular) part counts, the
// upper triangle being work the method avoids.
double gemm_algorithmic_flops(const mp_gemm_desc& g) {
  double rows = 0;
  if (g.causal == 0) return 2.0 * g.M * (double)g.N * g.K * g.batch;
  for (int i = 0; i < g.M; ++i) {
    if (g.causal == 1) rows += std::min(g.N, i + 1);
    else if (g.causal == 2) rows += std::min(g.K, i + 1);
    else rows += std::max(0, g.K - i);
  }
  return 2.0 * rows * (g.causal == 1 ? g.K : g.N) * g.batch;
}

// Logit GEMM with the cross-entropy statistics epilogue (act 3): n-blocks of the
// launch, so the caller can size ce_part ([M][2 n_blocks] float2).
int gemm_ce_nblocks(const mp_gemm_desc& g) {
  const int BN = pick_bn(g);
  return (g.N + BN - 1) / BN;
}

struct ProfRec { cudaEvent_t a, b; double flops; };
static bool g_prof = false;
static std::vector<ProfRec> g_recs;
static std::vector<cudaEvent_t> g_evpool;
static size_t g_evnext = 0;
static cudaEvent_t prof_event() {
  if (g_evnext == g_evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_evpool.push_back(e);
  }
  return g_evpool[g_evnext++];
}

mp_status gemm(mp_dtype dt, const mp_gemm_desc& g, cudaStream_t st, const GemmCe* ce) {
  if (dt != MP_BF16) { count_launch(); return ce ? set_err(MP_EINVAL, "gemm: CE epilogue is bf16") : gemm_fp32(g, st); }
  count_launch();
  if (!g_prof) return gemm_bf16(g, st, ce);
  ProfRec r{prof_event(), prof_event(), gemm_algorithmic_flops(g)};
  cudaEventRecord(r.a, st);
  mp_status s = gemm_bf16(g, st, ce);
  cudaEventRecord(r.b, st);
  g_recs.push_back(r);
  return s;
}

}  // namespace mp

extern "C" mp_status mp_op_gemm(mp_dtype dtype, const mp_gemm_desc* g, void* stream) {
  if (!g) return mp::set_err(MP_EINVAL, "null desc");
  MP_REQUIRE_DEVICE();
  return mp::gemm(dtype, *g, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" mp_status mp_profile_gemm(int enable) {
  mp::g_prof = enable != 0;
  mp::g_recs.clear();
  mp::g_evnext = 0;
  return MP_OK;
}

extern "C" mp_status mp_profile_gemm_read(double* flops, double* seconds, long long* launches) {
  if (!flops || !seconds || !launches) return mp::set_err(MP_EINVAL, "null arg");
  MP_CUDA(cudaDeviceSynchronize());
  double f = 0, t = 0;
  for (auto& r : mp::g_recs) {
    float ms = 0.f;
    MP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    f += r.flops;
    t += ms * 1e-3;
  }
  *flops = f; *seconds = t; *launches = (long long)mp::g_recs.size();
  return MP_OK;
}

extern "C" double mp_gemm_flops(const mp_gemm_desc* g) { return g ? mp::gemm_algorithmic_flops(*g) : 0.0; }

extern "C" mp_status mp_op_gemm_config(const mp_gemm_desc* g, int* out3) {
  if (!g || !out3) return mp::set_err(MP_EINVAL, "null arg");
  MP_REQUIRE_DEVICE();
  int BN = mp::pick_bn(*g);
  out3[0] = BN;
  out3[1] = BN == 256 ? mp::TcCfg<256>::STAGES : (BN == 128 ? mp::TcCfg<128>::STAGES : mp::TcCfg<64>::STAGES);
  long long tiles = (long long)((g->M + mp::BM - 1) / mp::BM) * ((g->N + BN - 1) / BN) * g->batch;
  out3[2] = (int)std::max(1LL, std::min<long long>(tiles, mp::num_sms()));
  return MP_OK;
}
