"""Pins of oracle.layer: closed forms, special cases, finite differences and an
independent torch-autograd fp64 re-statement (test-only) of the same layer."""
import numpy as np
import pytest
import torch
import torch.nn.functional as TF

import gen
from oracle import layer as L


def _rand(shape, seed, scale=1.0):
    return scale * np.random.default_rng(seed).standard_normal(shape)


def test_gelu_closed_form():
    assert L.gelu(np.array(0.0)) == 0.0
    # 0.5 (1 + tanh(sqrt(2/pi) * 1.044715))
    assert abs(L.gelu(np.array(1.0)) - 0.8411919906082768) < 1e-15
    u = np.linspace(-6, 6, 101)
    ref = TF.gelu(torch.tensor(u), approximate="tanh").numpy()
    np.testing.assert_allclose(L.gelu(u), ref, rtol=1e-14, atol=1e-15)
    # large |u|: identity / zero
    assert abs(L.gelu(np.array(30.0)) - 30.0) < 1e-12 and abs(L.gelu(np.array(-30.0))) < 1e-12


def test_gelu_grad_central_difference():
    u = np.linspace(-5, 5, 41)
    eps = 1e-6
    fd = (L.gelu(u + eps) - L.gelu(u - eps)) / (2 * eps)
    np.testing.assert_allclose(L.gelu_grad(u), fd, rtol=1e-7, atol=1e-9)


def test_layernorm():
    x = _rand((5, 3, 16), 0)
    g, b = _rand(16, 1), _rand(16, 2)
    y, _ = L.ln_fwd(x, g, b)
    ref = TF.layer_norm(torch.tensor(x), (16,), torch.tensor(g), torch.tensor(b), eps=1e-5).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    # constant row -> beta exactly
    y0, _ = L.ln_fwd(np.full((1, 16), 3.25), g, b)
    np.testing.assert_array_equal(y0[0], b)


def test_causal_softmax():
    S = _rand((2, 7, 7), 3)
    P = L.causal_softmax(S)
    np.testing.assert_allclose(P.sum(-1), 1.0, rtol=0, atol=1e-15)
    assert np.all(P[..., 0, 1:] == 0) and np.all(P[..., 0, 0] == 1.0)
    assert np.all(np.triu(P[0], 1) == 0)


def test_attention_special_cases():
    s, b, a, hd = 6, 2, 3, 4
    QKV = _rand((s, b, 3 * a * hd), 4)
    C, _ = L.attention_fwd(QKV, a)
    Q4 = QKV.reshape(s, b, a, 3, hd)
    # token 0 attends only to itself: context = v_0
    np.testing.assert_allclose(C.reshape(s, b, a, hd)[0], Q4[0, :, :, 2], rtol=0, atol=1e-15)
    # s = 1: context = V
    C1, _ = L.attention_fwd(QKV[:1], a)
    np.testing.assert_allclose(C1.reshape(1, b, a, hd)[0], Q4[0, :, :, 2], atol=1e-15)
    # vs torch SDPA (is_causal) fp64, per (batch, head)
    q = torch.tensor(Q4[:, :, :, 0]).permute(1, 2, 0, 3)
    k = torch.tensor(Q4[:, :, :, 1]).permute(1, 2, 0, 3)
    v = torch.tensor(Q4[:, :, :, 2]).permute(1, 2, 0, 3)
    ref = TF.scaled_dot_product_attention(q, k, v, is_causal=True).permute(2, 0, 1, 3).numpy()
    np.testing.assert_allclose(C.reshape(s, b, a, hd), ref, rtol=1e-12, atol=1e-13)


def test_zero_weights_identity():
    h, a = 16, 2
    W = {k: np.zeros(s) for k, s in gen.layer_param_shapes(h).items()}
    W["ln1_g"] = _rand(h, 5)
    W["ln2_g"] = _rand(h, 6)
    X = _rand((5, 2, h), 7)
    Y, _ = L.layer_fwd(X, W, a)
    np.testing.assert_array_equal(Y, X)


def torch_layer(X, W, a, masks=None):
    """Independent statement of the layer with torch fp64 library ops."""
    s, b, h = X.shape
    hd = h // a
    A = TF.layer_norm(X, (h,), W["ln1_g"], W["ln1_b"], eps=1e-5)
    QKV = (A @ W["w_qkv"] + W["b_qkv"]).reshape(s, b, a, 3, hd)
    q, k, v = (QKV[:, :, :, i].permute(1, 2, 0, 3) for i in range(3))
    if masks is None:
        C = TF.scaled_dot_product_attention(q, k, v, is_causal=True)
    else:
        att = (q @ k.transpose(-1, -2)) / hd ** 0.5
        att = att.masked_fill(torch.ones(s, s, dtype=torch.bool).triu(1), float("-inf")).softmax(-1)
        C = (att * masks["attn"]) @ v
    C = C.permute(2, 0, 1, 3).reshape(s, b, h)
    z1 = C @ W["w_o"] + W["b_o"]
    X1 = X + (z1 if masks is None else z1 * masks["h1"])
    A2 = TF.layer_norm(X1, (h,), W["ln2_g"], W["ln2_b"], eps=1e-5)
    z2 = TF.gelu(A2 @ W["w_1"] + W["b_1"], approximate="tanh") @ W["w_2"] + W["b_2"]
    return X1 + (z2 if masks is None else z2 * masks["h2"])


def _masks(s, b, a, h, seed, p=0.3):
    rng = np.random.default_rng(seed)
    return {"attn": (rng.random((b, a, s, s)) >= p) / (1 - p),
            "h1": (rng.random((s, b, h)) >= p) / (1 - p),
            "h2": (rng.random((s, b, h)) >= p) / (1 - p)}


@pytest.mark.parametrize("with_masks", [False, True])
def test_layer_vs_torch_autograd(with_masks):
    s, b, h, a = 9, 2, 32, 4
    W = gen.layer_weights(h, 4, seed=3, layer=0, dtype="fp32")
    W = {k: v * (5.0 if k.startswith("w_") else 1.0) for k, v in W.items()}   # make it non-trivial
    X = _rand((s, b, h), 8)
    dY = _rand((s, b, h), 9)
    masks = _masks(s, b, a, h, 10) if with_masks else None
    Y, cache = L.layer_fwd(X, W, a, masks)
    dX, g = L.layer_bwd(dY, cache, W, a, masks)
    Xt = torch.tensor(X, requires_grad=True)
    Wt = {k: torch.tensor(v, requires_grad=True) for k, v in W.items()}
    Mt = None if masks is None else {k: torch.tensor(v) for k, v in masks.items()}
    Yt = torch_layer(Xt, Wt, a, Mt)
    (Yt * torch.tensor(dY)).sum().backward()
    np.testing.assert_allclose(Y, Yt.detach().numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-10, atol=1e-11)
    for k in W:
        np.testing.assert_allclose(g[k], Wt[k].grad.numpy(), rtol=1e-10, atol=1e-11, err_msg=k)


def test_layer_finite_differences():
    s, b, h, a = 5, 1, 16, 2
    W = gen.layer_weights(h, 2, seed=4, layer=1, dtype="fp32")
    W = {k: v * (4.0 if k.startswith("w_") else 1.0) for k, v in W.items()}
    X = _rand((s, b, h), 11)
    dY = _rand((s, b, h), 12)
    _, cache = L.layer_fwd(X, W, a)
    dX, g = L.layer_bwd(dY, cache, W, a)

    def f(X_, W_):
        return float((L.layer_fwd(X_, W_, a)[0] * dY).sum())
    eps = 1e-6
    rng = np.random.default_rng(0)
    for name in ("w_qkv", "b_qkv", "w_o", "w_1", "b_1", "w_2", "ln1_g", "ln2_b"):
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in W[name].shape)
            Wp = {k: v.copy() for k, v in W.items()}
            Wm = {k: v.copy() for k, v in W.items()}
            Wp[name][idx] += eps
            Wm[name][idx] -= eps
            fd = (f(X, Wp) - f(X, Wm)) / (2 * eps)
            assert abs(fd - g[name][idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, g[name][idx])
    for _ in range(5):
        idx = tuple(rng.integers(0, n) for n in X.shape)
        Xp, Xm = X.copy(), X.copy()
        Xp[idx] += eps
        Xm[idx] -= eps
        fd = (f(Xp, W) - f(Xm, W)) / (2 * eps)
        assert abs(fd - dX[idx]) <= 1e-6 * max(1.0, abs(fd))


@pytest.mark.parametrize("t", [1, 2, 4])
@pytest.mark.parametrize("with_masks", [False, True])
def test_tp_partition_equals_unpartitioned(t, with_masks):
    """c.2: the t-way partitioned layer (Megatron) equals the
    unpartitioned one; each rank's dW shard is the slice of the full dW;
    replicated parameters get identical gradients on every rank."""
    s, b, h, a = 8, 2, 32, 4
    W = gen.layer_weights(h, 4, seed=5, layer=2, dtype="fp32")
    X = _rand((s, b, h), 13)
    dY = _rand((s, b, h), 14)
    masks = _masks(s, b, a, h, 15) if with_masks else None
    Y, c = L.layer_fwd(X, W, a, masks)
    dX, g = L.layer_bwd(dY, c, W, a, masks)
    Yt, ct = L.layer_fwd_tp(X, W, a, t, masks)
    dXt, gr = L.layer_bwd_tp(dY, ct, W, a, t, masks)
    assert np.max(np.abs(Yt - Y)) <= 1e-12 * np.max(np.abs(Y))
    assert np.max(np.abs(dXt - dX)) <= 1e-12 * np.max(np.abs(dX))
    gu = L.unshard_grads(gr, h, t)
    for k in g:
        assert np.max(np.abs(gu[k] - g[k])) <= 1e-12 * max(1e-30, np.max(np.abs(g[k]))), k
    for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "b_o", "b_2"):
        for r in range(1, t):
            np.testing.assert_array_equal(gr[r][k], gr[0][k])
    for r in range(t):
        sh = L.shard_layer(g, h, t, r)
        for k in ("w_qkv", "b_qkv", "w_o", "w_1", "b_1", "w_2"):
            assert np.max(np.abs(gr[r][k] - sh[k])) <= 1e-12 * np.max(np.abs(g[k]))
