"""Parity of the GEMM engine (tcgen05 bf16 / SIMT fp32) with the oracle's plain
GEMM definition, through the C ABI (mp_op_gemm)."""
import numpy as np
import pytest
import torch

import gen
from oracle.gemm import gemm_ref
from paper_2104_04473_b200 import mp
from tests.gpu_util import dev, host, normwise

pytestmark = pytest.mark.gpu


def _operand(rows_m, K, major, z, seed, dtype):
    """Logical [z, rows_m, K] operand stored K-major ([z, rows, K]) or MN-major ([z, K, rows])."""
    x = gen.activations((z, rows_m, K), seed, 1.0, dtype)
    stored = x if major == 0 else np.ascontiguousarray(np.swapaxes(x, 1, 2))
    return x, stored


def run_gemm(M, N, K, z, am, bm, dtype="bf16", c_fp32=False, bias=False, accumulate=False, causal=0,
             alpha=1.0, seed=0):
    A, As = _operand(M, K, am, z, seed, dtype)
    Bt, Bs = _operand(N, K, bm, z, seed + 1, dtype)       # Bt[z, n, k] = B(k, n)
    dA, dB = dev(As, dtype), dev(Bs, dtype)
    out_dt = torch.float32 if (c_fp32 or dtype == "fp32") else torch.bfloat16
    C0 = gen.activations((z, M, N), seed + 2, 1.0, "fp32") if accumulate else np.zeros((z, M, N))
    dC = torch.tensor(C0, dtype=torch.float32).cuda().to(out_dt).contiguous()
    bvec = gen.activations((N,), seed + 3, 1.0, dtype) if bias else None
    dbias = dev(bvec, dtype) if bias else None
    d = mp.GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, z
    d.a_major, d.b_major = am, bm
    d.A, d.lda, d.strideA = dA.data_ptr(), (K if am == 0 else M), M * K
    d.B, d.ldb, d.strideB = dB.data_ptr(), (K if bm == 0 else N), N * K
    d.C, d.ldc, d.strideC = dC.data_ptr(), N, M * N
    d.bias = dbias.data_ptr() if bias else None
    d.c_fp32 = int(out_dt == torch.float32)
    d.accumulate = int(accumulate)
    d.causal = causal
    d.alpha = alpha
    mp.mp_op_gemm(dtype, d)
    torch.cuda.synchronize()
    Bm = np.swapaxes(Bt, 1, 2)
    blk = (np.arange(M)[:, None] // 128) * 128
    kk = np.arange(K)[None, :]
    if causal == 2:       # reduction limited to k < 128 (floor(m/128) + 1)
        A = A * (kk < blk + 128)[None]
    if causal == 3:       # reduction limited to k >= 128 floor(m/128)
        A = A * (kk >= blk)[None]
    ref = gemm_ref(A, Bm, alpha, bvec) + (C0 if accumulate else 0)
    got = host(dC)
    if causal == 1:
        rows = np.arange(M)[:, None] // 128
        cols = np.arange(N)[None, :]
        keep = cols <= rows * 128 + 127
        ref = np.where(keep[None], ref, 0.0)
        got = np.where(keep[None], got, 0.0)
    return got, ref


@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,z", [(256, 384, 320, 1), (200, 136, 72, 2), (128, 64, 64, 1),
                                     (384, 512, 256, 1), (96, 1000, 136, 1), (2048, 2304, 576, 1)])
def test_gemm_bf16_majors(am, bm, M, N, K, z):
    got, ref = run_gemm(M, N, K, z, am, bm)
    assert normwise(got, ref) < 1e-2


@pytest.mark.parametrize("opts", [dict(c_fp32=True), dict(c_fp32=True, accumulate=True), dict(bias=True),
                                  dict(alpha=0.125, c_fp32=True)])
def test_gemm_bf16_epilogues(opts):
    got, ref = run_gemm(304, 520, 200, 1, 1, 1, **opts)
    tol = 1e-4 if opts.get("c_fp32") else 1e-2
    assert normwise(got, ref) < tol


@pytest.mark.parametrize("causal,am,bm", [(1, 0, 0), (2, 0, 1), (3, 1, 1)])
@pytest.mark.parametrize("s,hd", [(384, 64), (640, 96), (32, 16)])
def test_gemm_bf16_causal(causal, am, bm, s, hd):
    if causal == 1:
        got, ref = run_gemm(s, s, hd, 3, am, bm, causal=1)
    else:
        got, ref = run_gemm(s, hd, s, 3, am, bm, causal=causal, c_fp32=True)
    assert normwise(got, ref) < 1e-2


@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("causal", [0, 1, 2, 3])
def test_gemm_fp32(am, bm, causal):
    if causal in (2, 3):
        got, ref = run_gemm(200, 72, 200, 2, am, bm, dtype="fp32", causal=causal, bias=True)
    else:
        got, ref = run_gemm(200, 136, 72, 2, am, bm, dtype="fp32", causal=causal, bias=True, accumulate=True)
    assert normwise(got, ref) < 1e-5
