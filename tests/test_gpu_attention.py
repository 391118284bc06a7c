"""Parity of the fused causal attention core (tcgen05 flash kernel) with the
oracle's attention (scores, causal softmax, P V in fp64), through the C ABI."""
import numpy as np
import pytest
import torch

import gen
from oracle import layer as L
from paper_2104_04473_b200 import mp
from tests.gpu_util import dev, host, normwise

pytestmark = pytest.mark.gpu


# forward kernel: "auto" = the library's choice; "pair" forces the query-tile-pair forward
# (two ping-ponging softmax warpgroups, P in TMEM), "single" the one-tile forward
KERNELS = {"auto": None, "pair": "1", "single": "0"}


@pytest.fixture(params=list(KERNELS))
def fwd_kernel(request, monkeypatch):
    if KERNELS[request.param] is not None:
        monkeypatch.setenv("MP_FA_FWD_PAIR", KERNELS[request.param])
    return request.param


@pytest.mark.parametrize("s,b,heads,hd", [(128, 1, 1, 64), (256, 1, 2, 128), (384, 2, 3, 96), (200, 1, 2, 64),
                                          (2048, 1, 4, 128), (1000, 2, 2, 96), (32, 1, 2, 32), (640, 1, 2, 96)])
def test_flash_fwd(s, b, heads, hd, fwd_kernel):
    QKV = gen.activations((s, b, heads, 3, hd), 41, 1.0, "bf16")
    q = dev(QKV.reshape(s, b, -1), "bf16")
    ctx = torch.zeros((s, b, heads * hd), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((b * heads, s), dtype=torch.float32, device="cuda")
    mp.call("mp_op_flash_attn_fwd", q.data_ptr(), ctx.data_ptr(), lse.data_ptr(), s, b, heads, hd, None)
    torch.cuda.synchronize()
    C, Ps = L.attention_fwd(QKV.reshape(s, b, -1), heads)
    assert normwise(host(ctx), C) < 2e-2
    # base-2 log-sum-exp of the scaled scores
    Q4 = QKV
    for bb in range(b):
        for j in range(heads):
            S = Q4[:, bb, j, 0] @ Q4[:, bb, j, 1].T / np.sqrt(hd)
            S = np.where(np.triu(np.ones((s, s), bool), 1), -np.inf, S)
            mx = S.max(-1)
            l2 = (mx + np.log(np.exp(S - mx[:, None]).sum(-1))) / np.log(2)
            got = host(lse[bb * heads + j])
            assert np.max(np.abs(got - l2)) < 2e-2 * max(1.0, np.max(np.abs(l2)))


@pytest.mark.parametrize("s,b,heads,hd", [(128, 1, 1, 64), (256, 1, 2, 128), (384, 2, 3, 96), (200, 1, 2, 64),
                                          (2048, 1, 2, 128), (1000, 2, 2, 96), (32, 1, 2, 32)])
def test_flash_bwd(s, b, heads, hd, fwd_kernel):
    QKV = gen.activations((s, b, heads, 3, hd), 51, 1.0, "bf16")
    dC = gen.activations((s, b, heads * hd), 52, 1.0, "bf16")
    q = dev(QKV.reshape(s, b, -1), "bf16")
    dc = dev(dC, "bf16")
    ctx = torch.zeros((s, b, heads * hd), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((b * heads, s), dtype=torch.float32, device="cuda")
    mp.call("mp_op_flash_attn_fwd", q.data_ptr(), ctx.data_ptr(), lse.data_ptr(), s, b, heads, hd, None)
    dq = torch.zeros_like(q)
    ws = torch.zeros(mp.raw("mp_op_flash_attn_bwd_ws_floats", s, b, heads, hd), dtype=torch.float32, device="cuda")
    mp.call("mp_op_flash_attn_bwd", q.data_ptr(), ctx.data_ptr(), dc.data_ptr(), lse.data_ptr(), dq.data_ptr(),
            ws.data_ptr(), s, b, heads, hd, None)
    torch.cuda.synchronize()
    C, Ps = L.attention_fwd(QKV.reshape(s, b, -1), heads)
    dref = L.attention_bwd(dC, QKV.reshape(s, b, -1), Ps, heads).reshape(s, b, heads, 3, hd)
    got = host(dq).reshape(s, b, heads, 3, hd)
    for part, name in enumerate("QKV"):
        assert normwise(got[..., part, :], dref[..., part, :]) < 2e-2, name
