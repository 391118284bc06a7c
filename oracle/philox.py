"""Philox-4x32-10 counter-based generator and the dropout masks derived from
it (oracle; test infrastructure only).

Dropout rates are not given by the paper (P:131, P:146, P:312 mention dropout
only); reading #6 keys every mask by global coordinates so that the
mask of an element does not depend on t, p, v, b or m:

  counter = (e // 4, lane_hi, n, layer * 8 + tensor), key = (seed_lo, seed_hi)
  one Philox call yields 4 words for the elements 4q .. 4q+3 (word e % 4)
  keep  iff  (word >> 8) < floor((1 - p) * 2^24)      (integer comparison)
  kept values are scaled by 1 / (1 - p)

  hidden dropout (tensor 1 after the projection, 2 after FC2): element
      (sequence n, position i, feature c) -> e = i * h + c, lane_hi = 0
  attention-probability dropout (tensor 0): (sequence n, global head g,
      query i, key k) -> e = i * s + k, lane_hi = g

Salmon et al., "Parallel random numbers: as easy as 1, 2, 3" (SC'11), define
Philox; the known-answer vectors pinned in tests/golden/philox_kat.json are
the Random123 distribution's for philox4x32_10.
"""
import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """ctr: 4 x uint32 arrays (broadcastable), key: 2 x uint32 -> 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) for x in ctr)
    k0, k1 = (np.asarray(x, dtype=np.uint64) for x in key)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK32, lo1, (hi0 ^ c3 ^ k1) & MASK32, lo0
    return [x.astype(np.uint32) for x in (c0, c1, c2, c3)]


def keep_threshold(p):
    """Words with (word >> 8) below this value are kept."""
    return int(np.floor((1.0 - p) * (1 << 24)))


def _words(e, lane_hi, n, stream, seed):
    e = np.asarray(e, dtype=np.uint64)
    q = e // 4
    ctr = (q & MASK32, np.full_like(q, lane_hi) , np.full_like(q, n), np.full_like(q, stream))
    key = (seed & MASK32, (seed >> 32) & MASK32)
    w = philox4x32_10(ctr, key)
    sel = (e % 4).astype(np.int64)
    return np.choose(sel, w)


def hidden_mask(seed, layer, tensor, n, s, h, p):
    """Multiplicative mask [s, h] (0 or 1/(1-p)) of sequence n."""
    e = np.arange(s * h, dtype=np.uint64)
    w = _words(e, 0, n, layer * 8 + tensor, seed)
    keep = (w >> 8) < keep_threshold(p)
    return (keep / (1.0 - p)).reshape(s, h)


def attn_mask(seed, layer, n, g, s, p):
    """Multiplicative mask [s, s] (0 or 1/(1-p)) of sequence n, global head g."""
    e = np.arange(s * s, dtype=np.uint64)
    w = _words(e, g, n, layer * 8 + 0, seed)
    keep = (w >> 8) < keep_threshold(p)
    return (keep / (1.0 - p)).reshape(s, s)


def layer_masks(seed, layer, seqs, s, h, a, p_attn, p_hidden):
    """oracle.layer mask dict for a microbatch of sequences `seqs` (global ids):
    attn [b, a, s, s], h1 / h2 [s, b, h]; None if both rates are 0."""
    if p_attn == 0 and p_hidden == 0:
        return None
    b = len(seqs)
    out = {}
    if p_attn > 0:
        out["attn"] = np.stack([np.stack([attn_mask(seed, layer, n, g, s, p_attn) for g in range(a)])
                                for n in seqs])
    if p_hidden > 0:
        out["h1"] = np.stack([hidden_mask(seed, layer, 1, n, s, h, p_hidden) for n in seqs], axis=1)
        out["h2"] = np.stack([hidden_mask(seed, layer, 2, n, s, h, p_hidden) for n in seqs], axis=1)
    return out
