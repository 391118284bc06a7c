"""Plain fp64 GPT transformer layer, forward and hand-derived backward (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Architecture (with the readings of DESIGN.md Sec. Readings):
pre-LN GPT layer (reading #1), LayerNorm eps 1e-5 with biased variance
(reading #2), tanh-GeLU (reading #3), softmax scale 1/sqrt(hd)
(reading #4, "scale"), implicit causal mask k > i excluded (reading #5,
P:312), dropout as explicit multiplicative masks (reading #6), bias of the
row-parallel layers added once after the g reduction (reading #8).

  A   = LN(X; g1, b1)
  QKV = A W_qkv + b_qkv              split per head j into Q_j, K_j, V_j
  S_j = Q_j K_j^T / sqrt(hd),  S_j[i, k] = -inf for k > i
  P_j = softmax_row(S_j)  (x attention dropout mask)
  C   = concat_j (P_j V_j)
  X1  = X + drop(C W_o + b_o)
  A2  = LN(X1; g2, b2)
  U   = A2 W_1 + b_1,  H = gelu(U)
  Y   = X1 + drop(H W_2 + b_2)

Tensors are [s, b, h] (the paper's [s, b, a, h] layout).
The t-way partitioned layer (Megatron) is computed rank by rank
from sliced weights and joined by explicit sums for the g (forward) and f
(backward) operators.
"""
import numpy as np

LN_EPS = 1e-5
GELU_C = 0.7978845608028654   # sqrt(2/pi)
GELU_A = 0.044715


# ------------------------------------------------------------- primitives
def ln_fwd(x, g, b, eps=LN_EPS):
    """LayerNorm over the last axis with biased variance (reading #2)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * rstd
    return xhat * g + b, (xhat, rstd)


def ln_bwd(dy, cache, g):
    """Backward of ln_fwd: returns dx, dg, db (dg, db summed over rows)."""
    xhat, rstd = cache
    red = tuple(range(dy.ndim - 1))
    dg = (dy * xhat).sum(axis=red)
    db = dy.sum(axis=red)
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    return dx, dg, db


def gelu(u):
    """tanh-GeLU (reading #3): 0.5 u (1 + tanh(sqrt(2/pi)(u + 0.044715 u^3)))."""
    return 0.5 * u * (1.0 + np.tanh(GELU_C * (u + GELU_A * u ** 3)))


def gelu_grad(u):
    """d gelu / du of the tanh form."""
    th = np.tanh(GELU_C * (u + GELU_A * u ** 3))
    return 0.5 * (1.0 + th) + 0.5 * u * (1.0 - th * th) * GELU_C * (1.0 + 3.0 * GELU_A * u * u)


def causal_softmax(S):
    """Row softmax of S [..., s, s] with k > i excluded exactly (reading #5)."""
    s = S.shape[-1]
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)
    Sm = np.where(mask, -np.inf, S)
    Sm = Sm - Sm.max(axis=-1, keepdims=True)
    E = np.exp(Sm)
    return E / E.sum(axis=-1, keepdims=True)


def softmax_bwd(dP, P):
    """dS = P * (dP - rowsum(dP * P))."""
    return P * (dP - (dP * P).sum(axis=-1, keepdims=True))


# ------------------------------------------------------------ attention core
def attention_fwd(QKV, a, masks=None):
    """QKV [s, b, 3h] head-major -> context C [s, b, h].

    Loops over (batch, head) exactly as the strided batched GEMMs do.
    """
    s, b, h3 = QKV.shape
    h = h3 // 3
    hd = h // a
    scale = 1.0 / np.sqrt(hd)
    Q4 = QKV.reshape(s, b, a, 3, hd)
    C = np.zeros((s, b, a, hd))
    Ps = np.zeros((b, a, s, s))
    for bb in range(b):
        for j in range(a):
            Q, K, V = Q4[:, bb, j, 0], Q4[:, bb, j, 1], Q4[:, bb, j, 2]
            P = causal_softmax((Q @ K.T) * scale)
            Ps[bb, j] = P
            Pd = P if masks is None or "attn" not in masks else P * masks["attn"][bb, j]
            C[:, bb, j] = Pd @ V
    return C.reshape(s, b, h), Ps


def attention_bwd(dC, QKV, Ps, a, masks=None):
    """Backward of attention_fwd: dC [s, b, h] -> dQKV [s, b, 3h]."""
    s, b, h3 = QKV.shape
    h = h3 // 3
    hd = h // a
    scale = 1.0 / np.sqrt(hd)
    Q4 = QKV.reshape(s, b, a, 3, hd)
    dC4 = dC.reshape(s, b, a, hd)
    dQKV = np.zeros((s, b, a, 3, hd))
    for bb in range(b):
        for j in range(a):
            Q, K, V = Q4[:, bb, j, 0], Q4[:, bb, j, 1], Q4[:, bb, j, 2]
            P = Ps[bb, j]
            D = None if masks is None or "attn" not in masks else masks["attn"][bb, j]
            Pd = P if D is None else P * D
            dO = dC4[:, bb, j]
            dV = Pd.T @ dO
            dPd = dO @ V.T
            dP = dPd if D is None else dPd * D
            dS = softmax_bwd(dP, P) * scale
            dQKV[:, bb, j, 0] = dS @ K
            dQKV[:, bb, j, 1] = dS.T @ Q
            dQKV[:, bb, j, 2] = dV
    return dQKV.reshape(s, b, 3 * h)


def _mask(masks, key, x):
    return x if masks is None or key not in masks else x * masks[key]


# ----------------------------------------------------- unpartitioned layer
def layer_fwd(X, W, a, masks=None):
    """Forward of one layer (c.1); returns Y and the cache for layer_bwd."""
    A, ln1 = ln_fwd(X, W["ln1_g"], W["ln1_b"])
    QKV = A @ W["w_qkv"] + W["b_qkv"]
    C, Ps = attention_fwd(QKV, a, masks)
    X1 = X + _mask(masks, "h1", C @ W["w_o"] + W["b_o"])
    A2, ln2 = ln_fwd(X1, W["ln2_g"], W["ln2_b"])
    U = A2 @ W["w_1"] + W["b_1"]
    H = gelu(U)
    Y = X1 + _mask(masks, "h2", H @ W["w_2"] + W["b_2"])
    cache = dict(A=A, ln1=ln1, QKV=QKV, C=C, Ps=Ps, A2=A2, ln2=ln2, U=U, H=H)
    return Y, cache


def _sum_rows(x):
    return x.reshape(-1, x.shape[-1]).sum(axis=0)


def _wgrad(x, dy):
    return x.reshape(-1, x.shape[-1]).T @ dy.reshape(-1, dy.shape[-1])


def layer_bwd(dY, cache, W, a, masks=None):
    """Backward of layer_fwd: returns dX and the weight gradients dict."""
    g = {}
    dX1 = dY.copy()
    dZ2 = _mask(masks, "h2", dY)
    g["w_2"] = _wgrad(cache["H"], dZ2)
    g["b_2"] = _sum_rows(dZ2)
    dH = dZ2 @ W["w_2"].T
    dU = dH * gelu_grad(cache["U"])
    g["w_1"] = _wgrad(cache["A2"], dU)
    g["b_1"] = _sum_rows(dU)
    dA2 = dU @ W["w_1"].T
    dx, g["ln2_g"], g["ln2_b"] = ln_bwd(dA2, cache["ln2"], W["ln2_g"])
    dX1 = dX1 + dx
    dX = dX1.copy()
    dZ1 = _mask(masks, "h1", dX1)
    g["w_o"] = _wgrad(cache["C"], dZ1)
    g["b_o"] = _sum_rows(dZ1)
    dC = dZ1 @ W["w_o"].T
    dQKV = attention_bwd(dC, cache["QKV"], cache["Ps"], a, masks)
    g["w_qkv"] = _wgrad(cache["A"], dQKV)
    g["b_qkv"] = _sum_rows(dQKV)
    dA = dQKV @ W["w_qkv"].T
    dx, g["ln1_g"], g["ln1_b"] = ln_bwd(dA, cache["ln1"], W["ln1_g"])
    dX = dX + dx
    return dX, g


# ---------------------------------------------------- t-way partitioned layer
def shard_layer(W, h, t, r):
    """Rank r's shard (Megatron; reading #9).

    QKV columns of heads [r a/t, (r+1) a/t) (contiguous because the columns
    are head-major), W_o rows of the same heads; W_1 columns and W_2 rows
    [r 4h/t, (r+1) 4h/t); b_o, b_2 and the LayerNorm parameters replicated.
    """
    q0, q1 = r * 3 * h // t, (r + 1) * 3 * h // t
    o0, o1 = r * h // t, (r + 1) * h // t
    f0, f1 = r * 4 * h // t, (r + 1) * 4 * h // t
    return {"ln1_g": W["ln1_g"], "ln1_b": W["ln1_b"],
            "w_qkv": W["w_qkv"][:, q0:q1], "b_qkv": W["b_qkv"][q0:q1],
            "w_o": W["w_o"][o0:o1, :], "b_o": W["b_o"],
            "ln2_g": W["ln2_g"], "ln2_b": W["ln2_b"],
            "w_1": W["w_1"][:, f0:f1], "b_1": W["b_1"][f0:f1],
            "w_2": W["w_2"][f0:f1, :], "b_2": W["b_2"]}


def _head_masks(masks, a, t, r):
    if masks is None:
        return None
    out = dict(masks)
    if "attn" in masks:
        out["attn"] = masks["attn"][:, r * a // t:(r + 1) * a // t]
    return out


def layer_fwd_tp(X, W, a, t, masks=None):
    """t-way partitioned forward: per-rank partials joined by g = sum."""
    h = X.shape[-1]
    shards = [shard_layer(W, h, t, r) for r in range(t)]
    caches = [dict() for _ in range(t)]
    A, ln1 = ln_fwd(X, W["ln1_g"], W["ln1_b"])          # replicated on each rank
    part = []
    for r, Wr in enumerate(shards):                      # f: identity
        QKV = A @ Wr["w_qkv"] + Wr["b_qkv"]
        C, Ps = attention_fwd(QKV, a // t, _head_masks(masks, a, t, r))
        caches[r].update(QKV=QKV, C=C, Ps=Ps)
        part.append(C @ Wr["w_o"])
    Z = sum(part) + W["b_o"]                             # g: all-reduce, bias once
    X1 = X + _mask(masks, "h1", Z)
    A2, ln2 = ln_fwd(X1, W["ln2_g"], W["ln2_b"])
    part = []
    for r, Wr in enumerate(shards):
        U = A2 @ Wr["w_1"] + Wr["b_1"]
        H = gelu(U)
        caches[r].update(U=U, H=H)
        part.append(H @ Wr["w_2"])
    Y = X1 + _mask(masks, "h2", sum(part) + W["b_2"])
    return Y, dict(A=A, ln1=ln1, A2=A2, ln2=ln2, ranks=caches)


def layer_bwd_tp(dY, cache, W, a, t, masks=None):
    """t-way partitioned backward; returns dX and per-rank gradient dicts.

    f: the input gradients of the column-parallel GEMMs are summed
    over ranks.  Replicated parameters get identical gradients on every rank.
    """
    h = dY.shape[-1]
    shards = [shard_layer(W, h, t, r) for r in range(t)]
    gr = [dict() for _ in range(t)]
    dZ2 = _mask(masks, "h2", dY)
    dA2_parts = []
    for r, Wr in enumerate(shards):
        c = cache["ranks"][r]
        gr[r]["w_2"] = _wgrad(c["H"], dZ2)
        gr[r]["b_2"] = _sum_rows(dZ2)
        dU = (dZ2 @ Wr["w_2"].T) * gelu_grad(c["U"])
        gr[r]["w_1"] = _wgrad(cache["A2"], dU)
        gr[r]["b_1"] = _sum_rows(dU)
        dA2_parts.append(dU @ Wr["w_1"].T)
    dA2 = sum(dA2_parts)                                  # f: all-reduce
    dx, dg, db = ln_bwd(dA2, cache["ln2"], W["ln2_g"])
    dX1 = dY + dx
    dZ1 = _mask(masks, "h1", dX1)
    dA_parts = []
    for r, Wr in enumerate(shards):
        c = cache["ranks"][r]
        gr[r]["ln2_g"], gr[r]["ln2_b"] = dg, db
        gr[r]["w_o"] = _wgrad(c["C"], dZ1)
        gr[r]["b_o"] = _sum_rows(dZ1)
        dC = dZ1 @ Wr["w_o"].T
        dQKV = attention_bwd(dC, c["QKV"], c["Ps"], a // t, _head_masks(masks, a, t, r))
        gr[r]["w_qkv"] = _wgrad(cache["A"], dQKV)
        gr[r]["b_qkv"] = _sum_rows(dQKV)
        dA_parts.append(dQKV @ Wr["w_qkv"].T)
    dA = sum(dA_parts)                                    # f: all-reduce
    dx, dg, db = ln_bwd(dA, cache["ln1"], W["ln1_g"])
    for r in range(t):
        gr[r]["ln1_g"], gr[r]["ln1_b"] = dg, db
    return dX1 + dx, gr


def unshard_grads(gr, h, t):
    """Reassemble per-rank gradients into the unpartitioned layout."""
    out = {}
    for k in gr[0]:
        if k in ("w_qkv", "w_1"):
            out[k] = np.concatenate([g[k] for g in gr], axis=1)
        elif k in ("b_qkv", "b_1"):
            out[k] = np.concatenate([g[k] for g in gr], axis=0)
        elif k in ("w_o", "w_2"):
            out[k] = np.concatenate([g[k] for g in gr], axis=0)
        else:
            out[k] = gr[0][k]
    return out
