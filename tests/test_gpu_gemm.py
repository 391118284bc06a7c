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
        # only the causal part j <= i is defined (P:312 implicit causal mask)
        keep = np.arange(N)[None, :] <= np.arange(M)[:, None]
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


@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(512, 64, 32), (64, 512, 16), (256, 256, 8), (32, 96, 64), (512, 64, 48)])
def test_gemm_bf16_short_k(am, bm, M, N, K):
    """Reductions shorter than one 64-wide k-block (TMA zero-fills the rest):
    the dE = dlogits^T Z GEMM of the tiny model has K = T = 32."""
    got, ref = run_gemm(M, N, K, 1, am, bm, c_fp32=True)
    assert normwise(got, ref) < 1e-4


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("s,b,heads,hd", [(256, 2, 4, 64), (128, 3, 2, 96), (32, 1, 2, 16), (256, 1, 4, 64)])
def test_gemm_attention_layout(dtype, s, b, heads, hd):
    """Scores S = Q K^T and context P V straight from the [s, b, heads, 3, hd]
    QKV layout (strided batched over b*heads, no transposes)."""
    QKV = gen.activations((s, b, heads, 3, hd), 31, 1.0, dtype)
    q = dev(QKV, dtype)
    z = b * heads
    ldq = b * heads * 3 * hd
    S = torch.zeros((z, s, s), dtype=torch.float32, device="cuda")
    d = mp.GemmDesc()
    d.M, d.N, d.K, d.batch = s, s, hd, z
    d.A, d.lda, d.strideA = q.data_ptr(), ldq, 3 * hd
    d.B, d.ldb, d.strideB = q.data_ptr() + hd * q.element_size(), ldq, 3 * hd
    d.C, d.ldc, d.strideC = S.data_ptr(), s, s * s
    d.c_fp32, d.alpha = 1, 1.0
    mp.mp_op_gemm(dtype, d)
    P = gen.activations((z, s, s), 32, 1.0, dtype)
    Pd = dev(P, dtype)
    ctx = torch.zeros((s, b, heads, hd), dtype=torch.float32, device="cuda")
    e = mp.GemmDesc()
    e.M, e.N, e.K, e.batch = s, hd, s, z
    e.A, e.lda, e.strideA = Pd.data_ptr(), s, s * s
    e.B, e.ldb, e.strideB = q.data_ptr() + 2 * hd * q.element_size(), ldq, 3 * hd
    e.b_major = 1
    e.C, e.ldc, e.strideC = ctx.data_ptr(), b * heads * hd, hd
    e.c_fp32, e.alpha = 1, 1.0
    mp.mp_op_gemm(dtype, e)
    torch.cuda.synchronize()
    Q4 = QKV
    for bb in range(b):
        for j in range(heads):
            zz = bb * heads + j
            Sr = Q4[:, bb, j, 0] @ Q4[:, bb, j, 1].T
            assert normwise(host(S[zz]), Sr) < 1e-4, (bb, j)
            Cr = P[zz] @ Q4[:, bb, j, 2]
            assert normwise(host(ctx[:, bb, j]), Cr) < 1e-4, (bb, j)


@pytest.mark.parametrize("am,bm", [(1, 1), (0, 1)])
@pytest.mark.parametrize("M,N,K", [(2304, 2304, 2048), (1000, 1304, 2048), (768, 2304, 4096)])
def test_gemm_bf16_stream_k_accumulate(am, bm, M, N, K):
    """Weight-gradient-shaped accumulate GEMMs whose tile count leaves the last
    wave mostly empty: the (tile, k-block) iterations are split evenly across
    the SMs and partial tiles are reduce-added into the fp32 accumulator."""
    got, ref = run_gemm(M, N, K, 1, am, bm, c_fp32=True, accumulate=True)
    assert normwise(got, ref) < 1e-4


@pytest.mark.parametrize("M,N,K", [(2048, 2304, 576), (304, 520, 200), (96, 1000, 136)])
def test_gemm_bf16_gelu_epilogue(M, N, K):
    """act = 1: one GEMM writes the biased pre-activation U = A B + bias and
    H = gelu(U) (the FC1 + bias-GeLU of the MLP block, a14 + a15)."""
    from oracle.layer import gelu
    A = gen.activations((1, M, K), 7, 1.0, "bf16")
    Bt = gen.activations((1, N, K), 8, 1.0, "bf16")
    bvec = gen.activations((N,), 9, 1.0, "bf16")
    dA, dB, db = dev(A, "bf16"), dev(Bt, "bf16"), dev(bvec, "bf16")
    U = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    H = torch.zeros_like(U)
    d = mp.GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, 1
    d.A, d.lda, d.strideA = dA.data_ptr(), K, M * K
    d.B, d.ldb, d.strideB = dB.data_ptr(), K, N * K
    d.C, d.ldc, d.strideC = U.data_ptr(), N, M * N
    d.bias = db.data_ptr()
    d.alpha = 1.0
    d.act = 1
    d.C2 = H.data_ptr()
    mp.mp_op_gemm("bf16", d)
    torch.cuda.synchronize()
    ref_u = gemm_ref(A, np.swapaxes(Bt, 1, 2), 1.0, bvec)[0]
    assert normwise(host(U), ref_u) < 1e-2
    assert normwise(host(H), gelu(ref_u)) < 1e-2


@pytest.mark.parametrize("M,N,K,colsum", [(2048, 9216, 2304, True), (2048, 1152, 2304, True), (304, 520, 200, True),
                                          (96, 1000, 136, False)])
def test_gemm_bf16_dgelu_epilogue(M, N, K, colsum):
    """act = 2: the FC2 dgrad GEMM writes dU = (dY W) * gelu'(U) and adds the
    column sums of dU (the FC1 bias gradient) into an fp32 accumulator (a17).
    Shapes include the 1.7B t=1 / t=8 MLP widths (CTA-pair kernel) and ragged
    M, N."""
    from oracle.layer import gelu_grad
    A = gen.activations((1, M, K), 17, 1.0, "bf16")
    Bt = gen.activations((1, N, K), 18, 1.0, "bf16")
    Uh = gen.activations((M, N), 19, 1.0, "bf16")
    dA, dB, dU_in = dev(A, "bf16"), dev(Bt, "bf16"), dev(Uh, "bf16")
    out = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
    acc0 = gen.activations((N,), 20, 1.0, "fp32")
    db = dev(acc0, "fp32")
    d = mp.GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, 1
    d.A, d.lda, d.strideA = dA.data_ptr(), K, M * K
    d.B, d.ldb, d.strideB = dB.data_ptr(), K, N * K
    d.C, d.ldc, d.strideC = out.data_ptr(), N, M * N
    d.alpha = 1.0
    d.act = 2
    d.C2 = dU_in.data_ptr()
    d.colsum = db.data_ptr() if colsum else None
    mp.mp_op_gemm("bf16", d)
    torch.cuda.synchronize()
    ref = gemm_ref(A, np.swapaxes(Bt, 1, 2), 1.0, None)[0] * gelu_grad(Uh)
    got = host(out)
    assert normwise(got, ref) < 1e-2
    if colsum:
        # the sum of the stored values, accumulated onto the previous contents
        assert normwise(host(db) - acc0, got.astype(np.float64).sum(axis=0)) < 1e-4
        assert normwise(host(db) - acc0, ref.sum(axis=0)) < 1e-2
    else:
        assert np.array_equal(host(db), acc0.astype(np.float32).astype(np.float64))


def test_gemm_gelu_epilogue_rejects_fp32():
    d = mp.GemmDesc()
    d.M = d.N = d.K = 64
    d.batch = 1
    d.act = 1
    with pytest.raises(mp.MPError):
        mp.mp_op_gemm("fp32", d)


@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 1)])
def test_gemm_bf16_cta_pair(am, bm):
    """>= 60 GFLOP GEMMs run on CTA pairs (tcgen05.mma.cta_group::2, 256-row
    tiles, each CTA loading half of B); ragged M and N included."""
    got, ref = run_gemm(2048 + 136, 6912 - 64, 2304, 1, am, bm)
    assert normwise(got, ref) < 1e-2


@pytest.mark.parametrize("am,bm", [(1, 1), (0, 1)])
def test_gemm_bf16_cta_pair_stream_k_accumulate(am, bm):
    """Weight-gradient GEMMs >= 60 GFLOP: CTA pairs walking stream-K ranges,
    partial tiles reduce-added into the fp32 accumulator."""
    got, ref = run_gemm(6912, 2304, 2048, 1, am, bm, c_fp32=True, accumulate=True)
    assert normwise(got, ref) < 1e-4
