"""CPU tests of bench.py's host-side bookkeeping: the ideal-pipeline replay used
next to the measured bubble must reproduce the paper's closed forms when every
stage has the same task durations (P:105 (p-1)/m for 1F1B, P:118 (p-1)/(v m)
for the interleaved schedule), and must show the last-stage imbalance when the
last stage is slower.  The replay reports (end_r - busy_r) / busy_r per rank
from t = 0; the pipeline's span ends with stage 0's last backward, so the
paper's bubble is the maximum over ranks (stage 0), as in the bench line."""
from fractions import Fraction

import pytest

import bench


@pytest.mark.parametrize("p,m", [(2, 4), (4, 8), (4, 16), (8, 16)])
@pytest.mark.parametrize("tf,tb", [(1.0, 2.0), (3.0, 7.0)])
def test_replay_1f1b_closed_form(p, m, tf, tb):
    rp = bench.replay_bubble(p, m, 1, "1f1b", [tf] * p, [tb] * p)
    assert rp is not None
    assert abs(max(rp) - float(Fraction(p - 1, m))) < 1e-9
    assert abs(rp[0] - max(rp)) < 1e-12


@pytest.mark.parametrize("p,m,v", [(2, 4, 2), (4, 8, 2), (4, 16, 3), (2, 8, 6)])
def test_replay_interleaved_closed_form(p, m, v):
    rp = bench.replay_bubble(p, m, v, "interleaved", [1.0] * p, [2.0] * p)
    assert rp is not None
    assert abs(max(rp) - float(Fraction(p - 1, v * m))) < 1e-9
    assert abs(rp[0] - max(rp)) < 1e-12


def test_replay_last_stage_imbalance():
    # a slower last stage (logit layer + loss) raises the pipeline bubble above (p-1)/m
    p, m = 4, 8
    rp = bench.replay_bubble(p, m, 1, "1f1b", [1.0] * (p - 1) + [1.4], [2.0] * p)
    assert max(rp) > (p - 1) / m + 0.01


def test_workload_config_names_layout():
    import argparse
    import gen
    a = argparse.Namespace(model="1.7B", gpus=4, p=1, d=2, t=0, v=1, sched="", B=16, b=2, attn="fused",
                           recompute=True)
    c = bench.workload_config(a, gen.CONFIGS["1.7B"])
    assert c["parallelism"] == "t2p1v1d2" and c["m"] == 4 and c["d"] == 2 and c["recompute"]
    assert c["flop_formula"].startswith("Eq. (2) with recomputation")


@pytest.mark.parametrize("p,m,v", [(2, 8, 1), (4, 8, 1), (4, 16, 2), (2, 8, 3)])
def test_paper_bubble_of_an_ideal_pipeline_is_the_closed_form(p, m, v):
    """Feeding bench.paper_bubble the per-device spans and busy times of an ideal
    pipeline (the oracle's exact event simulation, equal stages) gives exactly
    (p-1)/m or (p-1)/(v m) on every device: every device idles the
    same total (p-1)(t_f+t_b)/v, split between warm-up and cool-down."""
    from oracle import schedule as SC
    kind = "interleaved" if v > 1 else "1f1b"
    tf, tb = 1, 2
    orders = SC.build_all(kind, p, m, v)
    sim = SC.simulate(orders, p, v, tf, tb)
    spans = [float(max(e for (r, _), e in sim["end"].items() if r == dev)) for dev in range(p)]
    busy = [float(m * (tf + tb))] * p
    mean_b, max_b = bench.paper_bubble(spans, busy)
    f = (p - 1) / (v * m)
    assert abs(mean_b - f) < 1e-12 and abs(max_b - f) < 1e-12


def test_paper_bubble_counts_the_tail_idle():
    # rank 1 ends early (its last task at 90 of a 100-long pipeline): its bubble includes the tail
    mean_b, max_b = bench.paper_bubble([100.0, 90.0], [80.0, 80.0])
    assert abs(max_b - 0.25) < 1e-12 and abs(mean_b - 0.25) < 1e-12
