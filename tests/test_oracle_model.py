"""Pins of oracle.model: the ln V special case, an independent torch-autograd
statement of the whole model, microbatch-split invariance, pipeline-executed
== sequential for every schedule (strict optimizer semantics), Adam."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as TF

import gen
from oracle import model as M
from oracle import schedule as SC
from tests.test_oracle_layer import torch_layer

CFG = gen.ModelCfg(l=4, h=32, a=4, s=8, V=64)


def _weights(dtype="fp32", seed=42, cfg=CFG):
    return gen.model_weights(cfg, seed=seed, dtype=dtype)


def test_loss_is_lnV_when_final_ln_zero():
    """gamma_f = beta_f = 0 => logits = 0 => loss = ln V exactly."""
    cfg = gen.TINY
    W = _weights(cfg=cfg)
    W["lnf_g"][:] = 0
    W["lnf_b"][:] = 0
    tok = gen.tokens(4, cfg.s, cfg.V)
    loss, _ = M.batch_fwd_bwd(W, tok, cfg.a, 4)
    assert abs(loss - math.log(512)) < 1e-12
    assert abs(math.log(512) - 6.238324625039508) < 1e-15


def _torch_model_loss(W, tok, a):
    Wt = {k: torch.tensor(v, requires_grad=True) for k, v in W.items() if k != "layers"}
    Lt = [{k: torch.tensor(v, requires_grad=True) for k, v in Wl.items()} for Wl in W["layers"]]
    x = torch.tensor(tok[:, :-1], dtype=torch.long)
    y = torch.tensor(tok[:, 1:], dtype=torch.long)
    X = (Wt["emb"][x] + Wt["pos"][None]).transpose(0, 1)             # [s, b, h]
    for Wl in Lt:
        X = torch_layer(X, Wl, a)
    Z = TF.layer_norm(X, (X.shape[-1],), Wt["lnf_g"], Wt["lnf_b"], eps=1e-5)
    logits = Z @ Wt["emb"].T
    loss = TF.cross_entropy(logits.reshape(-1, logits.shape[-1]), y.T.reshape(-1), reduction="mean")
    loss.backward()
    return loss.item(), Wt, Lt


def test_model_vs_torch_autograd():
    W = _weights()
    for Wl in W["layers"]:
        for k in ("w_qkv", "w_1"):
            Wl[k] *= 5.0
    tok = gen.tokens(4, CFG.s, CFG.V, seed=5)
    loss, g = M.batch_fwd_bwd(W, tok, CFG.a, 2)
    lt, Wt, Lt = _torch_model_loss(W, tok, CFG.a)
    assert abs(loss - lt) <= 1e-12 * abs(lt)
    for k in ("emb", "pos", "lnf_g", "lnf_b"):
        np.testing.assert_allclose(g[k], Wt[k].grad.numpy(), rtol=1e-9, atol=1e-13, err_msg=k)
    for gl, tl in zip(g["layers"], Lt):
        for k in gl:
            np.testing.assert_allclose(gl[k], tl[k].grad.numpy(), rtol=1e-9, atol=1e-13, err_msg=k)


def test_microbatch_split_invariance():
    """Gradient accumulation over m microbatches == one big batch."""
    W = _weights()
    tok = gen.tokens(4, CFG.s, CFG.V, seed=6)
    l1, g1 = M.batch_fwd_bwd(W, tok, CFG.a, 1)
    l4, g4 = M.batch_fwd_bwd(W, tok, CFG.a, 4)
    assert abs(l1 - l4) <= 1e-13
    for k in ("emb", "pos"):
        np.testing.assert_allclose(g1[k], g4[k], rtol=1e-10, atol=1e-15)


@pytest.mark.parametrize("kind,p,v,m", [
    (SC.GPIPE, 2, 1, 4), (SC.ONE_F_ONE_B, 2, 1, 4), (SC.ONE_F_ONE_B, 4, 1, 4),
    (SC.INTERLEAVED, 2, 2, 4), (SC.INTERLEAVED, 2, 2, 2), (SC.INTERLEAVED, 4, 1, 4)])
def test_pipeline_executed_equals_sequential(kind, p, v, m):
    """c.4: running the batch in the schedule's task order reproduces the
    sequential loss and gradients (strict optimizer semantics)."""
    W = _weights()
    tok = gen.tokens(m, CFG.s, CFG.V, seed=7)
    ls, gs = M.batch_fwd_bwd(W, tok, CFG.a, m)
    lp, gp, executed = M.pipeline_fwd_bwd(W, tok, CFG.a, m, p, v, kind)
    assert abs(ls - lp) <= 1e-12 * abs(ls)
    for k in ("emb", "pos", "lnf_g", "lnf_b"):
        assert np.max(np.abs(gs[k] - gp[k])) <= 1e-12 * np.max(np.abs(gs[k])), k
    for a_, b_ in zip(gs["layers"], gp["layers"]):
        for k in a_:
            assert np.max(np.abs(a_[k] - b_[k])) <= 1e-12 * max(1e-300, np.max(np.abs(a_[k]))), k
    assert executed == SC.build_all(kind, p, m, v)


def test_adam_first_step_closed_form():
    """Step 1: m1hat = g, vhat = g^2 => w -= lr * g / (|g| + eps)."""
    rng = np.random.default_rng(0)
    w, g = rng.standard_normal(50), rng.standard_normal(50)
    w1, m1, m2 = M.adam_step(w, g, np.zeros(50), np.zeros(50), 1, 1e-3)
    np.testing.assert_allclose(w1, w - 1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12)
    np.testing.assert_allclose(m1, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(m2, 0.001 * g * g, rtol=1e-12)
