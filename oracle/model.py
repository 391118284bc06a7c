"""Plain fp64 GPT model, batch with gradient accumulation, pipeline-executed
batch, and Adam (oracle).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Model (readings #10-#14):
  X0 = E[x_0..s-1] + Epos             (tied word embedding, learned positions)
  X_{k+1} = layer_k(X_k)              (oracle.layer)
  Z = LN(X_l; g_f, b_f)               (final LayerNorm)
  logits = Z E^T                      (logit layer, 2BshV fwd FLOPs)
  loss = mean over all B*s tokens of logsumexp(logits_i) - logits_i[y_i]

A batch of B sequences is split into m microbatches of b sequences
(m = B/(b d), d = 1); gradients are summed over microbatches
(strict optimizer semantics: one optimizer step after the flush).
"""
import numpy as np

from . import layer as L
from .schedule import build_all, simulate, stage_map


# ---------------------------------------------------------------- embedding
def embed_fwd(tok, emb, pos):
    """tok int [b, s] -> X0 [s, b, h] = E[tok] + Epos."""
    return emb[tok.T] + pos[:, None, :]


def embed_bwd(dX0, tok, V):
    """Scatter-add of dX0 into dE rows; dpos = sum over the batch."""
    s, b, h = dX0.shape
    demb = np.zeros((V, h))
    np.add.at(demb, tok.T.reshape(-1), dX0.reshape(-1, h))
    return demb, dX0.sum(axis=1)


# --------------------------------------------------------------------- head
def head_fwd_bwd(X, labels, W, scale):
    """Final LN + tied logit layer + cross-entropy, forward and backward.

    labels int [b, s]; `scale` multiplies the summed token losses (1/(B s)
    for the batch mean).  Returns (scaled loss sum, dX, demb, dg_f, db_f).
    """
    s, b, h = X.shape
    Z, lnc = L.ln_fwd(X, W["lnf_g"], W["lnf_b"])
    logits = Z @ W["emb"].T                                   # [s, b, V]
    mx = logits.max(axis=-1, keepdims=True)
    lse = mx[..., 0] + np.log(np.exp(logits - mx).sum(axis=-1))
    y = labels.T                                              # [s, b]
    tgt = np.take_along_axis(logits, y[..., None], axis=-1)[..., 0]
    loss = scale * (lse - tgt).sum()
    dlogits = np.exp(logits - lse[..., None])
    np.put_along_axis(dlogits, y[..., None],
                      np.take_along_axis(dlogits, y[..., None], axis=-1) - 1.0, axis=-1)
    dlogits *= scale
    demb = dlogits.reshape(-1, dlogits.shape[-1]).T @ Z.reshape(-1, h)
    dZ = dlogits @ W["emb"]
    dX, dg, db = L.ln_bwd(dZ, lnc, W["lnf_g"])
    return loss, dX, demb, dg, db


def zero_grads(W):
    g = {k: np.zeros_like(W[k]) for k in ("emb", "pos", "lnf_g", "lnf_b")}
    g["layers"] = [{k: np.zeros_like(v) for k, v in Wl.items()} for Wl in W["layers"]]
    return g


def _acc(dst, src):
    for k, v in src.items():
        dst[k] += v


# ----------------------------------------------------------------- sequential
def microbatch_fwd_bwd(W, tok_mb, a, scale, grads, masks=None):
    """Forward + backward of one microbatch tok_mb int [b, s+1]; adds into grads.

    masks: optional per-layer list of dropout mask dicts (oracle.layer).
    Returns the scaled loss contribution.
    """
    x, y = tok_mb[:, :-1], tok_mb[:, 1:]
    V = W["emb"].shape[0]
    X = embed_fwd(x, W["emb"], W["pos"])
    caches = []
    for k, Wl in enumerate(W["layers"]):
        X, c = L.layer_fwd(X, Wl, a, None if masks is None else masks[k])
        caches.append(c)
    loss, dX, demb, dg, db = head_fwd_bwd(X, y, W, scale)
    grads["emb"] += demb
    grads["lnf_g"] += dg
    grads["lnf_b"] += db
    for k in reversed(range(len(W["layers"]))):
        dX, gl = L.layer_bwd(dX, caches[k], W["layers"][k], a, None if masks is None else masks[k])
        _acc(grads["layers"][k], gl)
    demb, dpos = embed_bwd(dX, x, V)
    grads["emb"] += demb
    grads["pos"] += dpos
    return loss


def batch_fwd_bwd(W, tokens, a, m, masks=None):
    """Whole batch tokens int [B, s+1] as m microbatches; returns (loss, grads).

    loss = mean over the B*s tokens (reading #13); grads summed over the
    microbatches in ascending order.
    """
    B, s1 = tokens.shape
    b = B // m
    scale = 1.0 / (B * (s1 - 1))
    grads = zero_grads(W)
    loss = 0.0
    for i in range(m):
        loss += microbatch_fwd_bwd(W, tokens[i * b:(i + 1) * b], a, scale, grads,
                                   None if masks is None else masks[i])
    return loss, grads


# ---------------------------------------------------------- pipeline-executed
def pipeline_fwd_bwd(W, tokens, a, m, p, v, kind, masks=None):
    """Run the batch in the exact per-device task order of `kind` (c.4).

    Tasks of all devices are executed in order of their simulated start time
    (unit durations; ties broken by device), each device consuming only its
    own stage's layers, activations received through explicit per-(mb,
    stage) buffers and a stash of per-layer caches for its backward.  Must
    equal batch_fwd_bwd (strict optimizer semantics).  Also checks
    that every microbatch's F precedes its B on every stage.
    Returns (loss, grads, executed) with executed = per-device task lists.
    """
    l = len(W["layers"])
    B, s1 = tokens.shape
    b = B // m
    scale = 1.0 / (B * (s1 - 1))
    V = W["emb"].shape[0]
    dev_of, chunk_of = stage_map(l, p, v)
    S = p * v
    layers_of_stage = [[k for k in range(l) if chunk_of[k] * p + dev_of[k] == sg] for sg in range(S)]
    orders = build_all(kind, p, m, v)
    sim = simulate(orders, p, v, 1, 2)
    events = sorted(((sim["start"][(r, t)], r, t) for r in range(p) for t in orders[r]))
    act, grd, stash, fdone = {}, {}, {}, set()
    grads = zero_grads(W)
    loss = 0.0
    executed = [[] for _ in range(p)]
    for _, r, (kind_, i, c) in events:
        sigma = c * p + r
        executed[r].append((kind_, i, c))
        tok = tokens[i * b:(i + 1) * b]
        if kind_ == "F":
            X = embed_fwd(tok[:, :-1], W["emb"], W["pos"]) if sigma == 0 else act.pop((i, sigma))
            cs = []
            for k in layers_of_stage[sigma]:
                X, cache = L.layer_fwd(X, W["layers"][k], a, None if masks is None else masks[i][k])
                cs.append(cache)
            stash[(i, sigma)] = cs
            fdone.add((i, sigma))
            if sigma == S - 1:
                lo, dX, demb, dg, db = head_fwd_bwd(X, tok[:, 1:], W, scale)
                loss += lo
                grads["emb"] += demb
                grads["lnf_g"] += dg
                grads["lnf_b"] += db
                grd[(i, sigma)] = dX
            else:
                act[(i, sigma + 1)] = X
        else:
            assert (i, sigma) in fdone, "backward before forward"
            dX = grd.pop((i, sigma))
            cs = stash.pop((i, sigma))
            for k, cache in zip(reversed(layers_of_stage[sigma]), reversed(cs)):
                dX, gl = L.layer_bwd(dX, cache, W["layers"][k], a, None if masks is None else masks[i][k])
                _acc(grads["layers"][k], gl)
            if sigma == 0:
                demb, dpos = embed_bwd(dX, tok[:, :-1], V)
                grads["emb"] += demb
                grads["pos"] += dpos
            else:
                grd[(i, sigma - 1)] = dX
    assert not stash and not act and not grd
    return loss, grads, executed


# ---------------------------------------------------------------------- Adam
ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.999, 1e-8


def adam_step(w, g, m1, m2, step, lr):
    """Plain Adam (reading #14: no weight decay, no clipping).

    m1 = b1 m1 + (1-b1) g; m2 = b2 m2 + (1-b2) g^2;
    w -= lr * (m1/(1-b1^step)) / (sqrt(m2/(1-b2^step)) + eps).
    Returns new (w, m1, m2).
    """
    m1 = ADAM_B1 * m1 + (1.0 - ADAM_B1) * g
    m2 = ADAM_B2 * m2 + (1.0 - ADAM_B2) * g * g
    mh = m1 / (1.0 - ADAM_B1 ** step)
    vh = m2 / (1.0 - ADAM_B2 ** step)
    return w - lr * mh / (np.sqrt(vh) + ADAM_EPS), m1, m2
