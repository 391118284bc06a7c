"""Parity at the paper's widths on one GPU (SURVEY 8(c) parity tiers 2-3):

- one layer at each Table-1 width the BASELINE configs name -- 1.7B (hd=96)
  at b=1 and at the bench's b=2, and in fp32; 7.5B, 18.4B and 39.1B (hd=128),
  each with the fused flash attention core and with the paper's unfused
  scores-GEMM + softmax + P.V core;
- the head (final LN, tied logit layer, cross-entropy) at the paper's
  V = 51200, s = 2048 through mp_head_fwd_bwd;
- a depth-reduced paper-width model (l=2, h=2304, V=51200, m=2) through
  mp_run_batch: every gradient and the loss.

All against the fp64 oracle on the same generated inputs; tolerances are the
north_star's (normwise 2e-2 bf16, 1e-4 fp32).  The oracle side of each shape
is computed once per session (lru_cache) and shared by the fused / unfused
cases."""
import functools

import numpy as np
import pytest
import torch

import gen
from oracle import layer as L
from oracle import model as M
from paper_2104_04473_b200 import mp
from tests.gpu_util import TOL, dev, host, normwise

pytestmark = pytest.mark.gpu

WIDTHS = {"1.7B": (2304, 24, 24), "7.5B": (4096, 32, 36), "18.4B": (6144, 48, 40), "39.1B": (8192, 64, 48)}


@functools.lru_cache(maxsize=2)
def _layer_case(width, b, dtype):
    h, a, l = WIDTHS[width]
    W = gen.layer_weights(h, l, seed=31, layer=0, dtype=dtype)
    X = gen.activations((2048, b, h), 32, 1.0, dtype)
    dY = gen.activations((2048, b, h), 33, 1.0, dtype)
    Yr, cache = L.layer_fwd(X, W, a)
    dXr, gr = L.layer_bwd(dY, cache, W, a)
    del cache
    return W, X, dY, Yr, dXr, gr


def _run_layer(width, b, dtype, attn):
    h, a, _ = WIDTHS[width]
    W, X, dY, Yr, dXr, gr = _layer_case(width, b, dtype)
    c = mp.make_cfg(1, h, a, 2048, 51200, dtype=dtype, attn=attn)
    ctx = mp.Context(1, 1, 1, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
    try:
        for k, arr in W.items():
            ctx.set_weights(k, 0, arr)
        ctx.zero_grads()
        xd, yd = dev(X, dtype), dev(np.zeros_like(X), dtype)
        slot = ctx.layer_fwd(0, b, xd.data_ptr(), yd.data_ptr())
        dyd, dxd = dev(dY, dtype), dev(np.zeros_like(X), dtype)
        ctx.layer_bwd(0, b, slot, dyd.data_ptr(), dxd.data_ptr())
        torch.cuda.synchronize()
        tol = TOL[dtype]
        errs = {"Y": normwise(host(yd), Yr), "dX": normwise(host(dxd), dXr)}
        for k in W:
            errs[k] = normwise(ctx.get_grads(k, 0).reshape(gr[k].shape), gr[k])
        bad = {k: e for k, e in errs.items() if not e < tol}
        assert not bad, (width, b, dtype, attn, bad)
    finally:
        ctx.close()


@pytest.mark.parametrize("b", [1, 2])
@pytest.mark.parametrize("attn", ["fused", "unfused"])
def test_layer_1_7b_width(b, attn):
    """1.7B width (h=2304, a=24, hd=96) at b=1 and at the bench's b=2."""
    _run_layer("1.7B", b, "bf16", attn)


def test_layer_1_7b_width_fp32():
    """fp32 mode at the 1.7B width: normwise 1e-4 (north_star)."""
    _run_layer("1.7B", 1, "fp32", "unfused")


@pytest.mark.parametrize("width", ["7.5B", "18.4B", "39.1B"])
@pytest.mark.parametrize("attn", ["fused", "unfused"])
def test_layer_hd128_widths(width, attn):
    """hd = 128 widths: 7.5B (h=4096, a=32), 18.4B (h=6144, a=48), 39.1B
    (h=8192, a=64), s=2048, b=1 -- the GEMM shapes of the BASELINE configs'
    stages at t=1 (SURVEY 8 shape key)."""
    _run_layer(width, 1, "bf16", attn)


@pytest.mark.parametrize("b", [1, 2])
def test_head_paper_vocab(b):
    """Head at V=51200, s=2048, h=2304: the scaled loss, dX and
    the tied-embedding / final-LN gradients vs oracle.model.head_fwd_bwd."""
    h, s, V = 2304, 2048, 51200
    cfg = gen.ModelCfg(l=1, h=h, a=24, s=s, V=V)
    Wm = gen.model_weights(cfg, seed=41, dtype="bf16")
    X = gen.activations((s, b, h), 42, 1.0, "bf16")
    tok = gen.tokens(b, s, V, seed=43)                       # [b, s+1]; labels = tok[:, 1:]
    scale = 1.0 / (b * s)
    lr, dXr, demb, dg, db = M.head_fwd_bwd(X, tok[:, 1:], Wm, scale)
    c = mp.make_cfg(1, h, 24, s, V, dtype="bf16")
    ctx = mp.Context(1, 1, 1, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
    try:
        for name in ("emb", "pos", "lnf_g", "lnf_b"):
            ctx.set_weights(name, 0, Wm[name])
        ctx.zero_grads()
        xd, dxd = dev(X, "bf16"), dev(np.zeros_like(X), "bf16")
        dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
        loss = torch.zeros(1, dtype=torch.float32, device="cuda")
        ctx.head_fwd_bwd(b, xd.data_ptr(), dtok.data_ptr() + 4, s + 1, scale, dxd.data_ptr(), loss.data_ptr())
        torch.cuda.synchronize()
        tol = TOL["bf16"]
        assert abs(float(loss.item()) - lr) / abs(lr) < tol, (float(loss.item()), lr)
        assert normwise(host(dxd), dXr) < tol
        assert normwise(ctx.get_grads("emb", 0).reshape(demb.shape), demb) < tol
        assert normwise(ctx.get_grads("lnf_g", 0), dg) < tol
        assert normwise(ctx.get_grads("lnf_b", 0), db) < tol
    finally:
        ctx.close()


@pytest.mark.parametrize("sched,v", [("1f1b", 1), ("interleaved", 2)])
def test_run_batch_paper_width(sched, v):
    """Depth-reduced paper-width model (SURVEY 8(c) tier 3): l=2, h=2304, a=24,
    s=2048, V=51200, m=2 microbatches of b=1, fused attention, through
    mp_run_batch on one GPU: loss and every gradient vs the oracle's batch."""
    cfg = gen.ModelCfg(l=2, h=2304, a=24, s=2048, V=51200)
    m = 2
    W = _paper_model(cfg)
    tok = gen.tokens(m, cfg.s, cfg.V, seed=1234)
    lr, gr = _paper_batch(cfg, m)
    c = mp.make_cfg(cfg.l, cfg.h, cfg.a, cfg.s, cfg.V, dtype="bf16", attn="fused")
    ctx = mp.Context(1, 1, v, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
    try:
        for k, Wl in enumerate(W["layers"]):
            for name, arr in Wl.items():
                ctx.set_weights(name, k, arr)
        for name in ("emb", "pos", "lnf_g", "lnf_b"):
            ctx.set_weights(name, 0, W[name])
        loss, stats = ctx.run_batch(m, 1, m, sched, tok)
        tol = TOL["bf16"]
        assert abs(loss - lr) / abs(lr) < tol
        errs = {}
        for name in ("emb", "pos", "lnf_g", "lnf_b"):
            errs[name] = normwise(ctx.get_grads(name, 0).reshape(gr[name].shape), gr[name])
        for k in range(cfg.l):
            for name, ref in gr["layers"][k].items():
                errs[(k, name)] = normwise(ctx.get_grads(name, k).reshape(ref.shape), ref)
        bad = {k: e for k, e in errs.items() if not e < tol}
        assert not bad, bad
        assert stats["n_tasks"] == 2 * m * v
    finally:
        ctx.close()


@functools.lru_cache(maxsize=1)
def _paper_model(cfg):
    return gen.model_weights(cfg, seed=42, dtype="bf16")


@functools.lru_cache(maxsize=1)
def _paper_batch(cfg, m):
    tok = gen.tokens(m, cfg.s, cfg.V, seed=1234)
    return M.batch_fwd_bwd(_paper_model(cfg), tok, cfg.a, m)
