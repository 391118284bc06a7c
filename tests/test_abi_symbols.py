"""The C-ABI library loads on a CPU-only machine and exports every function
include/*.h declares; host-only entry points agree with the oracle."""
import ctypes
import glob
import os
import re

import pytest

from paper_2104_04473_b200 import mp
from oracle import formulas as F
from oracle import schedule as SC

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(mp_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = mp.lib()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the binding covers every declared entry point
    assert not [n for n in names if n not in mp.SIGNATURES], [n for n in names if n not in mp.SIGNATURES]


def test_flops_and_params_match_oracle():
    for (l, h, a, s, V) in [(24, 2304, 24, 2048, 51200), (40, 6144, 48, 2048, 51200), (4, 64, 4, 32, 512)]:
        assert mp.mp_param_count(l, h, s, V) == F.param_count(l, h, s, V)
        for B in (1, 64):
            for rc in (True, False):
                assert mp.mp_flops(B, s, l, h, V, rc) == float(F.flops(B, s, l, h, V, rc))


@pytest.mark.parametrize("kind", ["gpipe", "1f1b", "interleaved"])
def test_schedule_bit_exact(kind):
    for p in range(1, 9):
        for v in ([1] if kind != "interleaved" else [1, 2, 3, 4, 6]):
            for m in range(p if kind == "interleaved" else 1, 33, p if kind == "interleaved" else 1):
                for r in range(p):
                    assert mp.mp_get_schedule(p, m, v, kind, r) == SC.build_schedule(kind, p, m, v, r)


def test_schedule_errors():
    with pytest.raises(mp.MPError) as e:
        mp.mp_get_schedule(4, 6, 2, "interleaved", 0)
    assert e.value.status == mp.MP_ESCHED
    with pytest.raises(mp.MPError) as e:
        mp.mp_get_schedule(4, 8, 2, "1f1b", 0)
    assert e.value.status == mp.MP_ESCHED


def test_stage_map_bit_exact():
    for l in (4, 16, 24, 36, 40, 48):
        for p in (1, 2, 4, 8):
            for v in (1, 2, 3, 4, 6):
                if l % (p * v):
                    with pytest.raises(mp.MPError):
                        mp.mp_get_stage_map(l, p, v)
                    continue
                assert mp.mp_get_stage_map(l, p, v) == tuple(SC.stage_map(l, p, v)) or \
                    list(mp.mp_get_stage_map(l, p, v)) == list(SC.stage_map(l, p, v))


def test_validate():
    cfg = mp.make_cfg(40, 6144, 48, 2048, 51200)
    assert mp.mp_validate(cfg, 2, 4, 2, 1, 64, 1, "interleaved") == mp.MP_OK
    assert mp.mp_validate(cfg, 5, 1, 1, 1) == mp.MP_EDIV          # a % t
    assert mp.mp_validate(cfg, 2, 3, 1, 1) == mp.MP_EDIV          # l % (p v)
    assert mp.mp_validate(cfg, 2, 4, 2, 1, 38, 1, "interleaved") == mp.MP_ESCHED   # m % p
    assert mp.mp_validate(cfg, 2, 4, 1, 2) == mp.MP_OK             # d > 1
    assert mp.mp_validate(cfg, 2, 4, 1, 2, 64, 1, "1f1b") == mp.MP_OK
    assert mp.mp_validate(cfg, 2, 4, 1, 2, 66, 2, "1f1b") == mp.MP_EDIV   # B % (b d)


def test_compute_call_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = mp.GemmDesc()
    d.M = d.N = d.K = d.batch = 1
    with pytest.raises(mp.MPError) as e:
        mp.mp_op_gemm("bf16", d)
    assert e.value.status == mp.MP_ECUDA


@pytest.mark.parametrize("kind", ["gpipe", "1f1b", "interleaved"])
@pytest.mark.parametrize("p,v", [(2, 1), (4, 1), (2, 2), (4, 2), (2, 3), (3, 2)])
@pytest.mark.parametrize("tf,tb", [(1, 2), (3, 7)])
def test_bubble_replay_matches_oracle_simulator(kind, p, v, tf, tb):
    """mp_bubble_replay (the library's host-side replay the bench reports) against the
    oracle's exact-rational event simulator of the same orders:
    every device's idle share agrees, and device 0 attains the closed form."""
    if kind != "interleaved" and v != 1:
        pytest.skip("v > 1 only for the interleaved schedule")
    for m in (p, 2 * p, 4 * p):
        orders = SC.build_all(kind, p, m, v)
        sim = SC.simulate(orders, p, v, tf, tb)
        busy = m * (tf + tb)
        ends = [max(e for (r, _), e in sim["end"].items() if r == dev) for dev in range(p)]
        ref = [float((ends[r] - busy) / busy) for r in range(p)]
        got = mp.mp_bubble_replay(p, m, v, kind, [tf / v] * p, [tb / v] * p)
        assert max(abs(a - b) for a, b in zip(got, ref)) < 1e-12, (got, ref)
        assert abs(got[0] - float(SC.bubble_formula(kind, p, m, v))) < 1e-12
