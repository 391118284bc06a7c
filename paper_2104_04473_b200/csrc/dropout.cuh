// Counter-based dropout masks (reading #6): Philox-4x32-10 keyed by
// the seed, with the counter holding the element's GLOBAL coordinates, so the
// mask of an element is independent of t, p, v, b, m and is regenerated
// (never stored) in the backward.
//   counter = (e / 4, lane_hi, n, stream), key = (seed_lo, seed_hi)
//   keep iff (word[e % 4] >> 8) < thresh, thresh = floor((1 - p) 2^24)
// hidden dropout: stream = layer*8 + {1 after proj, 2 after FC2}, lane_hi = 0,
//   n = global sequence index, e = position * h + feature
// attention dropout: stream = layer*8, lane_hi = global head, e = q * s + k
#pragma once
#include <cstdint>

namespace mp {

struct Dropout {
  unsigned long long seed = 0;
  uint32_t stream = 0;
  uint32_t thresh = 0;     // 0 = dropout off
  float scale = 1.f;       // 1 / (1 - p)
  int seq0 = 0;            // global index of the microbatch's first sequence
  int b = 1;               // sequences per microbatch (rows are i * b + beta)
  int head0 = 0;           // first global head of this TP rank (attention)
  int heads = 1;           // heads on this rank (attention: z = beta * heads + j)
  __host__ __device__ bool on() const { return thresh != 0; }
};

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

// 4-bit keep mask of elements 4q .. 4q+3 (bit e % 4)
__device__ __forceinline__ uint32_t keep4(const Dropout& d, unsigned long long q, uint32_t lane_hi, uint32_t n) {
  uint32_t c[4] = {(uint32_t)q, lane_hi, n, d.stream};
  philox4x32_10(c, (uint32_t)d.seed, (uint32_t)(d.seed >> 32));
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m |= ((c[i] >> 8) < d.thresh ? 1u : 0u) << i;
  return m;
}

}  // namespace mp
