"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method: it draws token ids and
random-init weights (numpy PCG64) in the unpartitioned "oracle layout", and
rounds them to the storage precision (bf16 round-to-nearest-even or fp32) so
that both sides consume bit-identical inputs.  Recipe (DESIGN.md Sec. Inputs):

  tokens   uniform over [0, V), int32 [B, s+1] (labels are tokens shifted by 1)
  weights  Megatron-style init: N(0, 0.02^2) for QKV / FC1 / embeddings,
           N(0, (0.02/sqrt(2l))^2) for the output projection and FC2,
           biases N(0, 0.02^2), LayerNorm gamma 1 + N(0, 0.1^2),
           beta N(0, 0.02^2).

Unpartitioned layout per layer (math orientation Y = X W):
  ln1_g, ln1_b [h]; w_qkv [h, 3h] columns head-major (head j owns columns
  [3 j hd, 3 (j+1) hd) = [q_j | k_j | v_j]); b_qkv [3h]; w_o [h, h] rows
  head-major; b_o [h]; ln2_g, ln2_b [h]; w_1 [h, 4h]; b_1 [4h];
  w_2 [4h, h]; b_2 [h].
Model: emb [V, h] (tied input/output embedding), pos [s, h], lnf_g, lnf_b [h].
"""
from dataclasses import dataclass

import numpy as np

LAYER_PARAMS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")
MODEL_PARAMS = ("emb", "pos", "lnf_g", "lnf_b")


@dataclass(frozen=True)
class ModelCfg:
    l: int
    h: int
    a: int
    s: int
    V: int

    @property
    def hd(self):
        return self.h // self.a


TINY = ModelCfg(l=4, h=64, a=4, s=32, V=512)
GPT_1_7B = ModelCfg(l=24, h=2304, a=24, s=2048, V=51200)
GPT_7_5B = ModelCfg(l=36, h=4096, a=32, s=2048, V=51200)
GPT_18_4B = ModelCfg(l=40, h=6144, a=48, s=2048, V=51200)
GPT_39_1B = ModelCfg(l=48, h=8192, a=64, s=2048, V=51200)
CONFIGS = {"tiny": TINY, "1.7B": GPT_1_7B, "7.5B": GPT_7_5B, "18.4B": GPT_18_4B, "39.1B": GPT_39_1B}


def layer_param_shapes(h):
    return {"ln1_g": (h,), "ln1_b": (h,), "w_qkv": (h, 3 * h), "b_qkv": (3 * h,),
            "w_o": (h, h), "b_o": (h,), "ln2_g": (h,), "ln2_b": (h,),
            "w_1": (h, 4 * h), "b_1": (4 * h,), "w_2": (4 * h, h), "b_2": (h,)}


def model_param_shapes(cfg):
    return {"emb": (cfg.V, cfg.h), "pos": (cfg.s, cfg.h), "lnf_g": (cfg.h,), "lnf_b": (cfg.h,)}


def round_bf16(x):
    """Round to the nearest bf16 (ties to even) and return fp64 values."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def to_bf16_bits(x):
    """bf16 bit patterns (uint16) of already-bf16-representable values."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def round_to(x, dtype):
    """Round fp64 values to the storage precision ('bf16' or 'fp32')."""
    if dtype == "bf16":
        return round_bf16(x)
    if dtype == "fp32":
        return np.asarray(x, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def _draw(rng, name, shape, l):
    if name.endswith("_g"):
        return 1.0 + 0.1 * rng.standard_normal(shape)
    if name in ("w_o", "w_2"):
        return (0.02 / np.sqrt(2.0 * l)) * rng.standard_normal(shape)
    return 0.02 * rng.standard_normal(shape)


def layer_weights(h, l_total, seed, layer, dtype="bf16"):
    """Random-init weights of one transformer layer, rounded to `dtype`."""
    rng = np.random.Generator(np.random.PCG64([seed, 1, layer]))
    return {k: round_to(_draw(rng, k, shp, l_total), dtype)
            for k, shp in layer_param_shapes(h).items()}


def _draw32(rng, name, shape, l):
    x = rng.standard_normal(shape, dtype=np.float32)
    if name.endswith("_g"):
        return 1.0 + 0.1 * x
    if name in ("w_o", "w_2"):
        return np.float32(0.02 / np.sqrt(2.0 * l)) * x
    return np.float32(0.02) * x


def layer_weights_fast(h, l_total, seed, layer):
    """Same recipe drawn directly in float32 (large benchmark models; the
    library rounds to its storage dtype).  Not used for parity tests."""
    rng = np.random.Generator(np.random.PCG64([seed, 1, layer]))
    return {k: _draw32(rng, k, shp, l_total) for k, shp in layer_param_shapes(h).items()}


def model_weights_fast(cfg, seed=42):
    """Model-level tensors (emb, pos, lnf_*) of the fast float32 recipe."""
    rng = np.random.Generator(np.random.PCG64([seed, 0]))
    return {k: _draw32(rng, k, shp, cfg.l) for k, shp in model_param_shapes(cfg).items()}


def model_weights(cfg, seed=42, dtype="bf16"):
    """All weights of a GPT model: {'layers': [dict per layer], 'emb', 'pos', 'lnf_g', 'lnf_b'}."""
    rng = np.random.Generator(np.random.PCG64([seed, 0]))
    out = {k: round_to(_draw(rng, k, shp, cfg.l), dtype) for k, shp in model_param_shapes(cfg).items()}
    out["layers"] = [layer_weights(cfg.h, cfg.l, seed, i, dtype) for i in range(cfg.l)]
    return out


def tokens(B, s, V, seed=1234):
    """Token ids int32 [B, s+1]; inputs x = tok[:, :s], labels y = tok[:, 1:]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, V, size=(B, s + 1), dtype=np.int64).astype(np.int32)


def activations(shape, seed, scale=1.0, dtype="bf16"):
    """A seeded activation / gradient tensor N(0, scale^2), rounded to `dtype`."""
    rng = np.random.Generator(np.random.PCG64([seed, 7]))
    return round_to(scale * rng.standard_normal(shape), dtype)
