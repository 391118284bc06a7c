"""Pins of oracle.formulas against what the paper fixes (CPU only)."""
import json
import math
import os
from fractions import Fraction

import pytest

from oracle import formulas as F

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TABLE1_SHAPES = [  # (h, a, l) of the BASELINE.json configs (Table-1 rows 1, 3, 4, 5)
    (2304, 24, 24), (4096, 32, 36), (6144, 48, 40), (8192, 64, 48)]
V, S = 51200, 2048


@pytest.mark.parametrize("h,a,l", TABLE1_SHAPES + [(64, 4, 4), (12288, 96, 96)])
def test_eq1_exact_identity(h, a, l):
    """Eq. (1) == brute-force sum of tensors == literal rational form."""
    s, Vv = (32, 512) if h == 64 else (S, V)
    assert F.param_count(l, h, s, Vv) == F.param_count_bruteforce(l, h, s, Vv)
    assert F.param_count_eq1(l, h, s, Vv) == F.param_count(l, h, s, Vv)


def test_eq1_quoted_sizes():
    """Sizes the paper's text quotes with their shapes (tests/golden)."""
    cases = json.load(open(os.path.join(GOLD, "paper_quoted_sizes.json")))["cases"]
    for c in cases:
        full = F.param_count(c["l"], c["h"], S, V)
        nonemb = 12 * c["l"] * c["h"] ** 2 + 13 * c["l"] * c["h"]
        x = (full if c["kind"] == "all" else nonemb) / 1e9
        q = c["quoted_billion"]
        if c["round"] == "nearest_int":
            assert round(x) == q, c
        elif c["round"] == "floor_int":
            assert math.floor(x) == q, c
        else:
            assert round(x, 1) == q, c


def test_baseline_model_sizes():
    """The BASELINE config names (1.7B, 7.5B, 18.4B, 39.1B) follow from Eq. (1)."""
    names = [1.7, 7.5, 18.4, 39.1]
    for (h, a, l), name in zip(TABLE1_SHAPES, names):
        p = F.param_count(l, h, S, V) / 1e9
        assert abs(p - name) < 0.06, (h, p)


@pytest.mark.parametrize("h,a,l", TABLE1_SHAPES + [(64, 4, 4)])
@pytest.mark.parametrize("recompute", [True, False])
def test_eq2_equals_appendix_sum(h, a, l, recompute):
    """Eq. (2) is exactly the sum of the Appendix terms."""
    s, Vv = (32, 512) if h == 64 else (S, V)
    for B in (1, 4, 1536):
        assert F.flops(B, s, l, h, Vv, recompute) == F.flops_appendix(B, s, l, h, Vv, recompute)


def test_eq2_unit_case_and_linearity():
    """B=s=l=h=V=1: 96(1 + 1/6 + 1/16) = 118; F is linear in B."""
    assert F.flops(1, 1, 1, 1, 1) == 118
    assert F.flops(7, 2048, 40, 6144, V) == 7 * F.flops(1, 2048, 40, 6144, V)
    # recomputation adds exactly one layer forward
    d = F.flops(3, S, 40, 6144, V, True) - F.flops(3, S, 40, 6144, V, False)
    assert d == 40 * F.layer_fwd_flops(3, S, 6144)


def test_layer_flops_terms():
    """24Bsh^2 + 4Bs^2h per layer forward."""
    B, s, h = 2, 2048, 6144
    assert F.layer_fwd_flops(B, s, h) == 24 * B * s * h * h + 4 * B * s * s * h


def test_training_time_quotes():
    """Eq. (3): 34 days (GPT-3) and 84 days (1T)."""
    d = json.load(open(os.path.join(GOLD, "paper_schedule_examples.json")))["training_time"]
    for c in d:
        days = F.train_time_seconds(c["T"], c["P"], c["n"], c["X"]) / 86400
        assert abs(days - c["quoted_days"]) <= 1.0, (c, days)


def test_comm_volumes():
    """P:197 8bsh(t-1)/t per layer; bsh P2P; P:307 bsh/t; P:120 v-times more."""
    b, s, h = 1, 2048, 6144
    assert F.tp_elems_per_layer(b, s, h, 1) == 0
    assert F.tp_elems_per_layer(b, s, h, 8) == Fraction(8 * b * s * h * 7, 8)
    assert F.p2p_elems_per_microbatch(b, s, h) == b * s * h
    assert F.p2p_elems_per_microbatch(b, s, h, 8, True) * 8 == b * s * h
    # interleaving: boundaries per microbatch grow from p-1 to pv-1, i.e.
    # total P2P volume ~ v times larger for p >> 1
    assert F.p2p_boundaries_per_microbatch(4, 1) == 3
    assert F.p2p_boundaries_per_microbatch(4, 2) == 7
    assert F.p2p_boundaries_per_microbatch(1, 1) == 0
