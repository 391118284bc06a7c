"""Pins of oracle.schedule against the paper's closed forms and brute force."""
import json
import os
from fractions import Fraction

import pytest

from oracle import schedule as SC

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RATIOS = [(1, 2), (1, 1), (3, 7), (5, 3)]


def test_stage_map_paper_example():
    """16 layers, p=4, v=2 -> device 1 has layers 1,2,9,10."""
    g = json.load(open(os.path.join(GOLD, "paper_schedule_examples.json")))
    for key in ("stage_map", "noninterleaved_stage_map"):
        ex = g[key]
        dev, _ = SC.stage_map(ex["l"], ex["p"], ex["v"])
        for d1, layers in ex["device_layers_1based"].items():
            got = [k + 1 for k in range(ex["l"]) if dev[k] == int(d1) - 1]
            assert got == layers


def test_stage_map_divisibility():
    with pytest.raises(SC.ScheduleError):
        SC.stage_map(10, 4, 1)
    with pytest.raises(SC.ScheduleError):
        SC.stage_map(8, 2, 3)


def test_spec_examples():
    """S:331-333 examples (0-based ids here)."""
    assert SC.build_schedule(SC.ONE_F_ONE_B, 1, 4, 1, 0) == [
        (k, i, 0) for i in range(4) for k in ("F", "B")]
    assert SC.build_schedule(SC.GPIPE, 2, 2, 1, 0) == [("F", 0, 0), ("F", 1, 0), ("B", 0, 0), ("B", 1, 0)]
    o = SC.build_schedule(SC.ONE_F_ONE_B, 4, 8, 1, 0)
    first_b = next(k for k, t in enumerate(o) if t[0] == "B")
    # p-r-1 = 3 warm-up forwards, then the steady-state forward, then the first B
    assert [t[0] for t in o[:first_b]] == ["F"] * 4


def test_interleaved_requires_m_multiple_of_p():
    """m must be an integer multiple of p."""
    with pytest.raises(SC.ScheduleError):
        SC.build_schedule(SC.INTERLEAVED, 4, 6, 2, 0)
    with pytest.raises(SC.ScheduleError):
        SC.build_schedule(SC.ONE_F_ONE_B, 4, 8, 2, 0)


@pytest.mark.parametrize("kind", [SC.GPIPE, SC.ONE_F_ONE_B])
def test_bubble_noninterleaved_exact(kind):
    """(p-1)/m exactly, any t_f, t_b."""
    for p in range(1, 9):
        for m in range(1, 33):
            for tf, tb in RATIOS:
                orders = SC.build_all(kind, p, m, 1)
                sim = SC.simulate(orders, p, 1, tf, tb)
                assert SC.bubble_fraction(sim, m, tf, tb) == Fraction(p - 1, m)
                assert not SC.validate(orders, sim, p, 1, m)


def test_bubble_interleaved_exact():
    """(p-1)/(v m) exactly for p<=8, v<=6, m<=32 multiples of p."""
    for p in range(1, 9):
        for v in range(1, 7):
            for m in range(p, 33, p):
                for tf, tb in RATIOS[::2]:
                    orders = SC.build_all(SC.INTERLEAVED, p, m, v)
                    sim = SC.simulate(orders, p, v, tf, tb)
                    assert SC.bubble_fraction(sim, m, tf, tb) == Fraction(p - 1, v * m), (p, m, v)


def test_interleaved_validity_and_channels():
    """Each microbatch's F precedes its B on every stage; every directed
    channel's send order equals the receiver's consume order (FIFO-safe)."""
    for p in range(1, 7):
        for v in range(1, 5):
            for m in range(p, 4 * p + 1, p):
                orders = SC.build_all(SC.INTERLEAVED, p, m, v)
                for o in orders:
                    assert len(o) == 2 * m * v
                    assert sorted(o) == sorted({t for t in o})
                sim = SC.simulate(orders, p, v, 1, 2)
                assert not SC.validate(orders, sim, p, v, m)
                for ch, (snd, rcv) in SC.channel_orders(orders, p, v).items():
                    assert snd == rcv, (p, m, v, ch)


def test_inflight_bounds():
    """GPipe stashes m; 1F1B at most p - r; interleaved device 0
    holds v p + p - 1 chunk activations (derived)."""
    assert SC.peak_inflight(SC.build_all(SC.GPIPE, 2, 8, 1)) == [8, 8]
    for p in range(1, 9):
        for m in range(1, 20):
            pk = SC.peak_inflight(SC.build_all(SC.ONE_F_ONE_B, p, m, 1))
            assert pk == [min(p - r, m) for r in range(p)]
    assert SC.peak_inflight(SC.build_all(SC.INTERLEAVED, 4, 8, 2)) == [11, 9, 7, 5]


def test_gpipe_and_1f1b_same_span():
    """'The time spent in the bubble is the same for this new schedule'."""
    for p in range(1, 6):
        for m in range(1, 10):
            a = SC.simulate(SC.build_all(SC.GPIPE, p, m, 1), p, 1, 1, 2)["span"]
            b = SC.simulate(SC.build_all(SC.ONE_F_ONE_B, p, m, 1), p, 1, 1, 2)["span"]
            assert a == b


@pytest.mark.parametrize("p,m,v", [(2, 2, 1), (2, 2, 2), (3, 3, 1)])
def test_brute_force_minimum(p, m, v):
    """Over every deadlock-free per-device order, the minimum bubble equals the
    closed form, and the constructed schedule attains it."""
    best, n, dead = SC.brute_force_min_bubble(p, m, v, 1, 2)
    assert n > dead > 0
    assert best == Fraction(p - 1, v * m)
    kind = SC.INTERLEAVED if v > 1 else SC.ONE_F_ONE_B
    sim = SC.simulate(SC.build_all(kind, p, m, v), p, v, 1, 2)
    assert SC.bubble_fraction(sim, m, 1, 2) == best


def test_round_robin_reading_is_wrong():
    """Per-microbatch round-robin over chunks (one literal reading of S:379)
    either deadlocks or loses the 1/v bubble: evidence for the group-of-p
    reading (reading #15)."""
    def rr(p, m, v, r):
        F_ = [("F", i, c) for i in range(m) for c in range(v)]
        B_ = [("B", i, c) for i in range(m) for c in reversed(range(v))]
        warm = min(2 * (p - r - 1) + (v - 1) * p, m * v)
        o = F_[:warm]
        for k in range(m * v - warm):
            o += [F_[warm + k], B_[k]]
        return o + B_[m * v - warm:]
    p, m, v = 2, 4, 2
    try:
        sim = SC.simulate([rr(p, m, v, r) for r in range(p)], p, v, 1, 2)
        assert SC.bubble_fraction(sim, m, 1, 2) > Fraction(p - 1, v * m)
    except SC.DeadlockError:
        pass
