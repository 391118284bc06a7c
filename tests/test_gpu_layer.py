"""Parity of mp_layer_fwd / mp_layer_bwd and mp_run_batch (one GPU, t = p = 1)
with the fp64 oracle on the same generated inputs and random-init weights.
Tolerances (north_star): normwise 1e-4 in fp32 mode, 2e-2 in bf16 mode."""
import numpy as np
import pytest
import torch

import gen
from oracle import layer as L
from oracle import model as M
from paper_2104_04473_b200 import mp
from tests.gpu_util import TOL, dev, host, normwise

pytestmark = pytest.mark.gpu


def make_ctx(cfg_shape, dtype, t=1, p=1, v=1, l=None, attn="unfused"):
    c = mp.make_cfg(l or cfg_shape.l, cfg_shape.h, cfg_shape.a, cfg_shape.s, cfg_shape.V, dtype=dtype, attn=attn)
    return mp.Context(t, p, v, 1, c, 0, 1, 0, mp.mp_nccl_get_id())


def load_model(ctx, W):
    for k, Wl in enumerate(W["layers"]):
        for name, arr in Wl.items():
            ctx.set_weights(name, k, arr)
    for name in ("emb", "pos", "lnf_g", "lnf_b"):
        ctx.set_weights(name, 0, W[name])


LAYER_CASES = [
    ("tiny", gen.ModelCfg(l=1, h=64, a=4, s=32, V=512), 1),
    ("mid", gen.ModelCfg(l=1, h=256, a=4, s=256, V=512), 2),
    ("ragged", gen.ModelCfg(l=1, h=384, a=6, s=200, V=512), 1),
]


@pytest.mark.parametrize("dtype,attn", [("fp32", "unfused"), ("bf16", "unfused"), ("bf16", "fused")])
@pytest.mark.parametrize("name,shape,b", LAYER_CASES)
def test_layer_fwd_bwd(dtype, attn, name, shape, b):
    if shape.s % 8 and dtype == "bf16":
        pytest.skip("bf16 kernels need s % 8 == 0")
    if shape.s % 4 and dtype == "fp32":
        pytest.skip("fp32 kernels need s % 4 == 0")
    W = gen.layer_weights(shape.h, 4, seed=11, layer=0, dtype=dtype)
    X = gen.activations((shape.s, b, shape.h), 12, 1.0, dtype)
    dY = gen.activations((shape.s, b, shape.h), 13, 1.0, dtype)
    ctx = make_ctx(shape, dtype, attn=attn)
    try:
        for k, arr in W.items():
            ctx.set_weights(k, 0, arr)
        ctx.zero_grads()
        xd, yd = dev(X, dtype), dev(np.zeros_like(X), dtype)
        slot = ctx.layer_fwd(0, b, xd.data_ptr(), yd.data_ptr())
        dyd, dxd = dev(dY, dtype), dev(np.zeros_like(X), dtype)
        ctx.layer_bwd(0, b, slot, dyd.data_ptr(), dxd.data_ptr())
        torch.cuda.synchronize()
        Yr, cache = L.layer_fwd(X, W, shape.a)
        dXr, gr = L.layer_bwd(dY, cache, W, shape.a)
        tol = TOL[dtype]
        assert normwise(host(yd), Yr) < tol
        assert normwise(host(dxd), dXr) < tol
        for k in W:
            g = ctx.get_grads(k, 0).reshape(gr[k].shape)
            assert normwise(g, gr[k]) < tol, (k, normwise(g, gr[k]))
    finally:
        ctx.close()


@pytest.mark.parametrize("dtype,attn", [("bf16", "unfused"), ("bf16", "fused")])
def test_layer_paper_width_1_7b(dtype, attn):
    """One layer at the 1.7B config's width (h=2304, a=24, hd=96, s=2048, b=1)."""
    shape = gen.ModelCfg(l=1, h=2304, a=24, s=2048, V=51200)
    W = gen.layer_weights(shape.h, 24, seed=21, layer=0, dtype=dtype)
    X = gen.activations((shape.s, 1, shape.h), 22, 1.0, dtype)
    dY = gen.activations((shape.s, 1, shape.h), 23, 1.0, dtype)
    ctx = make_ctx(shape, dtype, attn=attn)
    try:
        for k, arr in W.items():
            ctx.set_weights(k, 0, arr)
        ctx.zero_grads()
        xd, yd = dev(X, dtype), dev(np.zeros_like(X), dtype)
        slot = ctx.layer_fwd(0, 1, xd.data_ptr(), yd.data_ptr())
        dxd = dev(np.zeros_like(X), dtype)
        dyd = dev(dY, dtype)
        ctx.layer_bwd(0, 1, slot, dyd.data_ptr(), dxd.data_ptr())
        torch.cuda.synchronize()
        Yr, cache = L.layer_fwd(X, W, shape.a)
        dXr, gr = L.layer_bwd(dY, cache, W, shape.a)
        assert normwise(host(yd), Yr) < TOL[dtype]
        assert normwise(host(dxd), dXr) < TOL[dtype]
        for k in W:
            g = ctx.get_grads(k, 0).reshape(gr[k].shape)
            assert normwise(g, gr[k]) < TOL[dtype], k
    finally:
        ctx.close()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("sched,v,m", [("gpipe", 1, 4), ("1f1b", 1, 4), ("interleaved", 2, 4), ("interleaved", 4, 2)])
def test_run_batch_single_gpu(dtype, sched, v, m):
    _run_batch_case(gen.TINY, dtype, sched, v, m, "unfused")


@pytest.mark.parametrize("sched,v,m", [("1f1b", 1, 4), ("interleaved", 2, 4)])
def test_run_batch_fused_attention(sched, v, m):
    """Same batch with the fused tcgen05 attention core (hd = 32 model)."""
    _run_batch_case(gen.ModelCfg(l=4, h=128, a=4, s=64, V=512), "bf16", sched, v, m, "fused")


def _run_batch_case(shape, dtype, sched, v, m, attn):
    """Tiny GPT (BASELINE config 0 shapes), whole batch through mp_run_batch on
    one GPU (p = 1, t = 1): loss and every gradient vs the oracle."""
    W = gen.model_weights(shape, seed=42, dtype=dtype)
    tok = gen.tokens(m, shape.s, shape.V, seed=1234)
    ctx = make_ctx(shape, dtype, v=v, attn=attn)
    try:
        load_model(ctx, W)
        loss, stats = ctx.run_batch(m, 1, m, sched, tok)
        lr, gr = M.batch_fwd_bwd(W, tok, shape.a, m)
        tol = TOL[dtype]
        assert abs(loss - lr) / abs(lr) < tol
        for name in ("emb", "pos", "lnf_g", "lnf_b"):
            g = ctx.get_grads(name, 0).reshape(gr[name].shape)
            assert normwise(g, gr[name]) < tol, name
        for k in range(shape.l):
            for name, ref in gr["layers"][k].items():
                g = ctx.get_grads(name, k).reshape(ref.shape)
                assert normwise(g, ref) < tol, (k, name, normwise(g, ref))
        assert stats["n_tasks"] == 2 * m * v
    finally:
        ctx.close()


def test_run_batch_adam_step():
    """One Adam step after the flush matches the oracle's Adam on the oracle's
    gradients (fp32 mode)."""
    shape = gen.TINY
    W = gen.model_weights(shape, seed=42, dtype="fp32")
    tok = gen.tokens(2, shape.s, shape.V, seed=99)
    c = mp.make_cfg(shape.l, shape.h, shape.a, shape.s, shape.V, dtype="fp32", lr=1e-3)
    ctx = mp.Context(1, 1, 1, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
    try:
        load_model(ctx, W)
        ctx.run_batch(2, 1, 2, "1f1b", tok, apply_optimizer=True)
        _, gr = M.batch_fwd_bwd(W, tok, shape.a, 2)
        for name in ("w_qkv", "b_1"):
            w1, _, _ = M.adam_step(W["layers"][1][name], gr["layers"][1][name], 0.0, 0.0, 1, 1e-3)
            got = ctx.get_weights(name, 1).reshape(w1.shape)
            assert np.max(np.abs(got - w1)) < 1e-5 + 1e-3 * 1e-2
    finally:
        ctx.close()


@pytest.mark.parametrize("dtype,attn", [("fp32", "unfused"), ("bf16", "unfused"), ("bf16", "fused")])
def test_layer_dropout(dtype, attn):
    """Attention-probability and hidden dropout (Philox masks keyed by global
    coordinates, reading #6) against the oracle with the same masks."""
    from oracle import philox as PH
    shape, b, pa, ph = gen.ModelCfg(l=1, h=256, a=4, s=256, V=512), 2, 0.1, 0.15
    W = gen.layer_weights(shape.h, 4, seed=61, layer=0, dtype=dtype)
    X = gen.activations((shape.s, b, shape.h), 62, 1.0, dtype)
    dY = gen.activations((shape.s, b, shape.h), 63, 1.0, dtype)
    c = mp.make_cfg(1, shape.h, shape.a, shape.s, shape.V, dtype=dtype, attn=attn, p_drop_attn=pa, p_drop_hidden=ph,
                    seed=777)
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
        masks = PH.layer_masks(777, 0, list(range(b)), shape.s, shape.h, shape.a, pa, ph)
        Yr, cache = L.layer_fwd(X, W, shape.a, masks)
        dXr, gr = L.layer_bwd(dY, cache, W, shape.a, masks)
        tol = TOL[dtype]
        assert normwise(host(yd), Yr) < tol
        assert normwise(host(dxd), dXr) < tol
        for k in W:
            g = ctx.get_grads(k, 0).reshape(gr[k].shape)
            assert normwise(g, gr[k]) < tol, (k, normwise(g, gr[k]))
    finally:
        ctx.close()


@pytest.mark.parametrize("dtype,attn,h", [("fp32", "unfused", 64), ("bf16", "unfused", 64), ("bf16", "fused", 128)])
def test_run_batch_dropout(dtype, attn, h):
    from oracle import philox as PH
    shape = gen.ModelCfg(l=4, h=h, a=4, s=32 if attn == "unfused" else 64, V=512)
    m, pa, ph = 4, 0.1, 0.1
    W = gen.model_weights(shape, seed=42, dtype=dtype)
    tok = gen.tokens(m, shape.s, shape.V, seed=1234)
    c = mp.make_cfg(shape.l, shape.h, shape.a, shape.s, shape.V, dtype=dtype, attn=attn, p_drop_attn=pa,
                    p_drop_hidden=ph, seed=99)
    ctx = mp.Context(1, 1, 2, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
    try:
        load_model(ctx, W)
        loss, _ = ctx.run_batch(m, 1, m, "interleaved", tok)
        masks = [[PH.layer_masks(99, k, [i], shape.s, shape.h, shape.a, pa, ph) for k in range(shape.l)]
                 for i in range(m)]
        lr, gr = M.batch_fwd_bwd(W, tok, shape.a, m, masks=masks)
        tol = TOL[dtype]
        assert abs(loss - lr) / abs(lr) < tol
        for k in range(shape.l):
            for name, ref in gr["layers"][k].items():
                g = ctx.get_grads(name, k).reshape(ref.shape)
                assert normwise(g, ref) < tol, (k, name, normwise(g, ref))
        for name in ("emb", "pos"):
            assert normwise(ctx.get_grads(name, 0).reshape(gr[name].shape), gr[name]) < tol, name
    finally:
        ctx.close()


@pytest.mark.parametrize("dtype,attn,h,pd", [("fp32", "unfused", 64, 0.0), ("bf16", "unfused", 64, 0.1),
                                             ("bf16", "fused", 128, 0.1)])
def test_run_batch_recompute(dtype, attn, h, pd):
    """Activation recomputation: same loss and gradients as the
    oracle (and bit-identical to the stashing run), FLOP count = Eq. (2)'s
    96-formula."""
    from oracle import formulas as F
    from oracle import philox as PH
    shape = gen.ModelCfg(l=4, h=h, a=4, s=32 if attn == "unfused" else 64, V=512)
    m = 4
    W = gen.model_weights(shape, seed=42, dtype=dtype)
    tok = gen.tokens(m, shape.s, shape.V, seed=1234)
    res = {}
    for rc in (0, 1):
        c = mp.make_cfg(shape.l, shape.h, shape.a, shape.s, shape.V, dtype=dtype, attn=attn, p_drop_attn=pd,
                        p_drop_hidden=pd, seed=99, recompute=bool(rc))
        ctx = mp.Context(1, 1, 2, 1, c, 0, 1, 0, mp.mp_nccl_get_id())
        try:
            load_model(ctx, W)
            loss, stats = ctx.run_batch(m, 1, m, "interleaved", tok)
            grads = {(name, k): ctx.get_grads(name, k) for k in range(shape.l) for name in W["layers"][k]}
            res[rc] = (loss, grads, stats)
        finally:
            ctx.close()
    masks = None
    if pd > 0:
        masks = [[PH.layer_masks(99, k, [i], shape.s, shape.h, shape.a, pd, pd) for k in range(shape.l)]
                 for i in range(m)]
    lr, gr = M.batch_fwd_bwd(W, tok, shape.a, m, masks=masks)
    loss, grads, stats = res[1]
    tol = TOL[dtype]
    assert abs(loss - lr) / abs(lr) < tol
    for (name, k), g in grads.items():
        ref = gr["layers"][k][name]
        assert normwise(g.reshape(ref.shape), ref) < tol, (k, name)
        # recomputation replays the same kernels on the same inputs (only the order of the
        # fp32 gradient reduce-adds may differ)
        assert normwise(g, res[0][1][(name, k)]) < 1e-5, (k, name)
    assert abs(res[1][0] - res[0][0]) <= 1e-6 * abs(res[0][0])
    assert stats["model_flops"] == float(F.flops(m, shape.s, shape.l, shape.h, shape.V, True))
    assert res[0][2]["model_flops"] == float(F.flops(m, shape.s, shape.l, shape.h, shape.V, False))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_set_weights_f64_matches_f32(dtype):
    """mp_set_weights_f64 (fp64 host data, rounded once to fp32) stores exactly what
    mp_set_weights stores for the same values rounded to fp32 on the host."""
    shape = gen.TINY
    W = gen.model_weights(shape, seed=7, dtype=dtype)
    ctx = make_ctx(shape, dtype)
    try:
        for name, arr in W["layers"][0].items():
            a64 = np.ascontiguousarray(arr, dtype=np.float64) * (1.0 + 1e-12)   # not representable in fp32
            st = mp._sym("mp_set_weights_f64")(ctx.ptr, name.encode(), 0, a64.ctypes.data)
            assert st == mp.MP_OK, mp.lib().mp_last_error()
            got64 = ctx.get_weights(name, 0).copy()
            ctx.set_weights(name, 0, a64.astype(np.float32))
            got32 = ctx.get_weights(name, 0)
            assert np.array_equal(got64, got32), name
    finally:
        ctx.close()
