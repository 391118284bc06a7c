"""Closed-form counts from the paper (oracle; test infrastructure only).

P:342-346 Eq. (1)  P = 12 l h^2 (1 + 13/(12h) + (V+s)/(12 l h))
P:347-352 Eq. (2)  F = 96 B s l h^2 (1 + s/(6h) + V/(16 l h))
P:570-580 Appendix: per-layer forward 24Bsh^2 + 4Bs^2h; backward = 2x forward;
          recomputation adds one forward; logit layer 2BshV fwd + 4BshV bwd.
P:193-197 Sec. 3.2: pipeline P2P bsh per microbatch per boundary; TP
          8bsh(t-1)/t per layer per device per microbatch.
P:307     Sec. 4.1: scatter/gather reduces the boundary volume to bsh/t.
P:120     interleaving multiplies P2P communication by v.
P:358-362 Eq. (3) end-to-end training time ~ 8TP/(nX).

All integer results are exact Python ints; FLOP results are exact Fractions
where the paper's formula has fractional factors.
"""
from fractions import Fraction


def param_count(l, h, s, V):
    """Eq. (1) as the exact integer 12lh^2 + 13lh + (V+s)h.

    12 l h^2 (1 + 13/(12h) + (V+s)/(12lh)) = 12lh^2 + 13lh + (V+s)h.
    """
    return 12 * l * h * h + 13 * l * h + (V + s) * h


def param_count_eq1(l, h, s, V):
    """Eq. (1) evaluated literally in exact rationals."""
    l, h, s, V = (Fraction(x) for x in (l, h, s, V))
    return 12 * l * h ** 2 * (1 + Fraction(13, 12) / h + (V + s) / (12 * l * h))


def param_count_bruteforce(l, h, s, V):
    """Sum of the individual tensors of one GPT model (P:128-173 architecture).

    Per layer: QKV weight 3h^2 + bias 3h; output projection h^2 + h;
    FC1 4h^2 + 4h; FC2 4h^2 + h; two LayerNorms 2*(h + h).
    Model: word embedding V*h (tied with the logit layer, counted once),
    learned positions s*h.  The final LayerNorm (2h) is NOT part of Eq. (1);
    callers that count it add 2h themselves.
    """
    per_layer = (3 * h * h + 3 * h) + (h * h + h) + (4 * h * h + 4 * h) + (4 * h * h + h) + 4 * h
    return l * per_layer + V * h + s * h


def layer_fwd_flops(B, s, h):
    """Appendix: one transformer layer forward = 24Bsh^2 + 4Bs^2h.

    QKV 6Bsh^2, scores 2Bs^2h, attention over values 2Bs^2h, projection
    2Bsh^2, MLP 16Bsh^2.
    """
    return 6 * B * s * h * h + 2 * B * s * s * h + 2 * B * s * s * h + 2 * B * s * h * h + 16 * B * s * h * h


def flops_appendix(B, s, l, h, V, recompute=True):
    """Sum of the Appendix terms.

    With recomputation each layer costs 4x its forward (fwd + 2x bwd + refwd);
    without, 3x (the 72-variant).  Logit layer: 2BshV fwd + 4BshV bwd.
    """
    mult = 4 if recompute else 3
    return mult * l * layer_fwd_flops(B, s, h) + 6 * B * s * h * V


def flops(B, s, l, h, V, recompute=True):
    """Eq. (2) literally, in exact rationals.

    recompute=False gives the 72 B s l h^2 (1 + s/(6h)) + 6BshV variant
    (the paper's formula assumes recomputation).
    """
    B, s, l, h, V = (Fraction(x) for x in (B, s, l, h, V))
    if recompute:
        return 96 * B * s * l * h ** 2 * (1 + s / (6 * h) + V / (16 * l * h))
    return 72 * B * s * l * h ** 2 * (1 + s / (6 * h)) + 6 * B * s * h * V


def train_time_seconds(T_tokens, P, n, X):
    """Eq. (3): end-to-end training time ~ 8TP/(nX) seconds."""
    return 8 * T_tokens * P / (n * X)


def p2p_elems_per_microbatch(b, s, h, t=1, scatter_gather=False):
    """bsh per pair of consecutive stages per microbatch per direction;
    P:307 -- bsh/t with the scatter/gather optimisation."""
    return Fraction(b * s * h, t) if scatter_gather else b * s * h


def tp_elems_per_layer(b, s, h, t):
    """8bsh(t-1)/t per layer per device per microbatch (ring)."""
    return Fraction(8 * b * s * h * (t - 1), t)


def p2p_boundaries_per_microbatch(p, v):
    """interleaving multiplies P2P communication by v.

    A microbatch's activations cross p*v - 1 stage boundaries forward (stages
    sigma -> sigma + 1 for sigma < p*v - 1), the same number backward.  Only
    boundaries between different devices cost a transfer; with p > 1 every
    boundary sigma -> sigma+1 changes device, so the count is p*v - 1
    (vs p - 1 without interleaving).
    """
    return p * v - 1 if p > 1 else 0
