"""The built library is Blackwell-native (CPU check of the sm_100a SASS): the GEMM
and fused-attention kernels issue tcgen05 MMAs (UTCHMMA) fed by TMA (UTMALDG) with
TMEM accumulators (LDTM), the NVLS consumers use multimem reduce-loads (LDGMC), and
no kernel falls back to the legacy mma.sync tensor-core path (HMMA)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sass():
    lib = os.path.join(ROOT, "paper_2104_04473_b200", "lib", "libmp.so")
    if not os.path.exists(lib) or not shutil.which("cuobjdump"):
        pytest.skip("library or cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        s = line.strip()
        if s.startswith("Function : "):
            cur = s.split("Function : ", 1)[1]
            funcs[cur] = []
        elif cur is not None and "/*" in s:
            funcs[cur].append(s)
    return funcs


def ops(lines):
    found = []
    for s in lines:
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", s)
        if m:
            found.append(m.group(1))
    return found


def test_sm100a_only(sass):
    assert sass, "no SASS in the library"


@pytest.mark.parametrize("kernel", ["tc_gemm_kernel", "flash_fwd_kernel", "flash_bwd_kernel", "flash_fwd_pair_kernel"])
def test_tensor_kernels_use_tcgen05_tma_tmem(sass, kernel):
    fs = [f for f in sass if kernel in f]
    assert fs, f"{kernel} not found"
    for f in fs:
        o = ops(sass[f])
        assert any(x.startswith("UTCHMMA") for x in o), f
        assert any(x.startswith("UTMALDG") for x in o), f
        assert any(x.startswith("LDTM") for x in o), f


def test_no_legacy_mma(sass):
    bad = [f for f, lines in sass.items() if any(x.startswith("HMMA") for x in ops(lines))]
    assert not bad, bad


def test_nvls_consumers_reduce_load(sass):
    o = [x for f, lines in sass.items() if "bias_add_residual_kernel" in f or "ln_fwd_kernel" in f for x in ops(lines)]
    assert any(x.startswith("LDGMC") for x in o)
