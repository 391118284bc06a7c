"""Per-iteration timeline of the flash kernels from the in-kernel %globaltimer
stamps of CTA 0 (MP_FA_TRACE), 1.7B b=2 shape.

    MP_FA_TRACE=1 python tools/fa_trace.py [--fwd]

Backward (CTA 0 = kv tile 0, all 16 query tiles): 0 loads issued (producer),
1 S/dP products issued (MMA), 2 dV/dK/dQ products issued, 3 S/dP ready
(compute), 4 P/dS written, 5 dQ ready, 6 dQ staged.
Forward (CTA 0 = the last query tile, 16 kv tiles): 0 K issued, 1 V issued,
2 S product issued, 3 P.V issued, 4 S read, 5 max / rescale done, 6 P written.
Printed relative to the first event, in ns.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04473_b200 import mp  # noqa: E402


def main():
    s, b, heads, hd = 2048, 2, 24, 96
    lib = mp.lib()
    q = (0.5 * torch.randn(s, b, heads * 3 * hd, device="cuda")).to(torch.bfloat16)
    dc = torch.randn(s, b, heads * hd, device="cuda").to(torch.bfloat16)
    ctx = torch.zeros(s, b, heads * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(b * heads, s, device="cuda")
    dq = torch.zeros_like(q)
    ws = torch.zeros(mp.raw("mp_op_flash_attn_bwd_ws_floats", s, b, heads, hd), device="cuda")
    mp.call("mp_op_flash_attn_fwd", q.data_ptr(), ctx.data_ptr(), lse.data_ptr(), s, b, heads, hd, None)
    fwd = "--fwd" in sys.argv
    for _ in range(3):
        if fwd:
            mp.call("mp_op_flash_attn_fwd", q.data_ptr(), ctx.data_ptr(), lse.data_ptr(), s, b, heads, hd, None)
            continue
        mp.call("mp_op_flash_attn_bwd", q.data_ptr(), ctx.data_ptr(), dc.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                ws.data_ptr(), s, b, heads, hd, None)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 512)()
    lib.mp_debug_fa_trace(buf)
    t = np.array(buf[:], dtype=np.int64).reshape(8, 64)
    t0 = t[t > 0].min()
    rows = []
    for j in range(64):
        if t[0, j] == 0 and t[3, j] == 0:
            continue
        rows.append([int(t[e, j] - t0) if t[e, j] else None for e in range(7)])
    print(json.dumps({"events_ns": rows}))
    it = [r[6] for r in rows if r[6] is not None]
    print(json.dumps({"per_iteration_ns": [b_ - a_ for a_, b_ in zip(it, it[1:])]}))


if __name__ == "__main__":
    main()
