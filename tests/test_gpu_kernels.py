"""Parity of the memory-bound kernels with the oracle's primitives, through
the C ABI (mp_op_*), on seeded inputs, bf16 and fp32."""
import numpy as np
import pytest
import torch

import gen
from oracle import layer as L
from paper_2104_04473_b200 import mp
from tests.gpu_util import TOL, dev, host, normwise

pytestmark = pytest.mark.gpu
DT = ["bf16", "fp32"]


def f32(n):
    return torch.zeros(n, dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("R,h", [(32, 64), (300, 2304), (64, 8192 // 2), (4096, 2304), (333, 6144), (40, 8192), (7, 16384)])
def test_layernorm_fwd_bwd(dtype, R, h):
    if h // (8 if dtype == "bf16" else 4) > 1024:
        pytest.skip("row kernels are limited to h / vector width <= 1024")
    x = gen.activations((R, h), 1, 1.0, dtype)
    g = gen.round_to(1 + 0.1 * np.random.default_rng(0).standard_normal(h), dtype)
    b = gen.activations((h,), 2, 0.1, dtype)
    dy = gen.activations((R, h), 3, 1.0, dtype)
    dres = gen.activations((R, h), 4, 1.0, dtype)
    dx_, y_ = dev(np.zeros((R, h)), dtype), dev(np.zeros((R, h)), dtype)
    mu, rs = f32(R), f32(R)
    xd, gd, bd, dyd, dresd = (dev(a, dtype) for a in (x, g, b, dy, dres))   # keep device buffers alive
    mp.call("mp_op_layernorm_fwd", dtype, xd.data_ptr(), gd.data_ptr(), bd.data_ptr(), y_.data_ptr(),
            mu.data_ptr(), rs.data_ptr(), R, h, 1e-5, None)
    yr, cache = L.ln_fwd(x, g, b)
    torch.cuda.synchronize()
    assert normwise(host(y_), yr) < TOL[dtype] / 4
    dg, db = f32(h), f32(h)
    mp.call("mp_op_layernorm_bwd", dtype, dyd.data_ptr(), xd.data_ptr(), gd.data_ptr(), mu.data_ptr(),
            rs.data_ptr(), dresd.data_ptr(), dx_.data_ptr(), dg.data_ptr(), db.data_ptr(), R, h, None)
    torch.cuda.synchronize()
    dxr, dgr, dbr = L.ln_bwd(dy, cache, g)
    assert normwise(host(dx_), dxr + dres) < TOL[dtype] / 4
    assert normwise(host(dg), dgr) < TOL[dtype] / 4
    assert normwise(host(db), dbr) < TOL[dtype] / 4
    # the one-pass variant that also takes the two bias gradients around LN2 (b2 = colsum of the
    # residual input dres, bo = colsum of the stored dx); accumulators start non-zero (+=)
    acc0 = gen.activations((4, h), 11, 1.0, "fp32")
    acc = dev(acc0, "fp32")
    dx2 = dev(np.zeros((R, h)), dtype)
    mp.call("mp_op_layernorm_bwd_sums", dtype, dyd.data_ptr(), xd.data_ptr(), gd.data_ptr(), mu.data_ptr(),
            rs.data_ptr(), dresd.data_ptr(), dx2.data_ptr(), acc[0].data_ptr(), acc[1].data_ptr(),
            acc[2].data_ptr(), acc[3].data_ptr(), R, h, None)
    torch.cuda.synchronize()
    got = host(acc)
    assert np.array_equal(host(dx2), host(dx_))            # same dx, bit for bit
    assert normwise(got[0] - acc0[0], dgr) < TOL[dtype] / 4
    assert normwise(got[1] - acc0[1], dbr) < TOL[dtype] / 4
    assert normwise(got[2] - acc0[2], dres.sum(0)) < TOL[dtype] / 4
    assert normwise(got[3] - acc0[3], host(dx2).sum(0)) < TOL[dtype] / 4
    assert normwise(got[3] - acc0[3], (dxr + dres).sum(0)) < TOL[dtype]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("z,s", [(3, 32), (2, 384), (1, 2048), (2, 136)])
def test_softmax_causal(dtype, z, s):
    S = gen.activations((z, s, s), 5, 3.0, dtype)
    hd = 64
    scale = 1 / np.sqrt(hd)
    buf = dev(S, dtype)
    mp.call("mp_op_softmax_causal_fwd", dtype, buf.data_ptr(), z, s, float(scale), None)
    torch.cuda.synchronize()
    P = host(buf)
    Pr = L.causal_softmax(S * scale)
    i = np.arange(s)[:, None]
    j = np.arange(s)[None, :]
    kend = np.minimum(s, (i // 128 + 1) * 128)
    written = j < kend
    assert normwise(np.where(written, P, 0), Pr) < TOL[dtype] / 4
    assert np.all(P[:, (j > i) & written] == 0)
    # backward
    dP = gen.activations((z, s, s), 6, 1.0, dtype)
    Pd = gen.round_to(Pr, dtype)          # the kernel consumes the stored P
    dbuf = dev(dP, dtype)
    Pdd = dev(Pd, dtype)
    mp.call("mp_op_softmax_causal_bwd", dtype, dbuf.data_ptr(), Pdd.data_ptr(), z, s, float(scale), None)
    torch.cuda.synchronize()
    dS = host(dbuf)
    dSr = L.softmax_bwd(np.where(j <= i, dP, 0), Pd) * scale
    assert normwise(np.where(written, dS, 0), dSr) < TOL[dtype] / 4
    assert np.all(dS[:, (j > i) & written] == 0)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("R,N", [(32, 128), (2048, 4608), (100, 1000)])
def test_bias_gelu(dtype, R, N):
    y = gen.activations((R, N), 7, 1.5, dtype)
    b = gen.activations((N,), 8, 0.5, dtype)
    out = dev(np.zeros((R, N)), dtype)
    yd, bd = dev(y, dtype), dev(b, dtype)
    mp.call("mp_op_bias_gelu_fwd", dtype, yd.data_ptr(), bd.data_ptr(), out.data_ptr(), R, N, None)
    dh = gen.activations((R, N), 9, 1.0, dtype)
    du = dev(dh, dtype)
    db = f32(N)
    mp.call("mp_op_bias_gelu_bwd", dtype, du.data_ptr(), yd.data_ptr(), bd.data_ptr(), du.data_ptr(), db.data_ptr(),
            R, N, None)
    torch.cuda.synchronize()
    assert normwise(host(out), L.gelu(y + b)) < TOL[dtype] / 4
    dur = dh * L.gelu_grad(y + b)
    assert normwise(host(du), dur) < TOL[dtype] / 4
    assert normwise(host(db), dur.sum(0)) < TOL[dtype] / 4
