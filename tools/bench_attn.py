"""Time the fused attention kernels through the C ABI with CUDA events.

    python tools/bench_attn.py [--reps 20] [--ab]

Shapes (s = 2048): the per-rank attention of the BASELINE configs --
1.7B b=2 t=1 (48 heads x hd 96), 1.7B b=2 t=2 (24 x 96), 18.4B b=1 t=2
(24 x 128), 39.1B b=1 t=2 (32 x 128).  Reports fwd and bwd (incl. the D /
dQ-convert helpers) in us and TFLOP/s of causal-algorithmic work:
fwd 2 products, bwd 5 products, each 2 hd s(s+1)/2 per head.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04473_b200 import mp  # noqa: E402


def timeit(fn, reps):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):   # back-to-back launches between two events: host overhead overlaps the GPU work
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    mp.lib()
    shapes = [("1.7B b2 t1", 2048, 2, 24, 96), ("1.7B b2 t2", 2048, 2, 12, 96), ("18.4B b1 t2", 2048, 1, 24, 128),
              ("39.1B b1 t2", 2048, 1, 32, 128)]
    for name, s, b, heads, hd in shapes:
        q = (0.5 * torch.randn(s, b, heads * 3 * hd, device="cuda")).to(torch.bfloat16)
        dc = torch.randn(s, b, heads * hd, device="cuda").to(torch.bfloat16)
        ctx = torch.zeros(s, b, heads * hd, device="cuda", dtype=torch.bfloat16)
        lse = torch.zeros(b * heads, s, device="cuda")
        dq = torch.zeros_like(q)
        ws = torch.zeros(mp.raw("mp_op_flash_attn_bwd_ws_floats", s, b, heads, hd), device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        fwd = lambda: mp.call("mp_op_flash_attn_fwd", q.data_ptr(), ctx.data_ptr(), lse.data_ptr(), s, b, heads, hd, st)
        bwd = lambda: mp.call("mp_op_flash_attn_bwd", q.data_ptr(), ctx.data_ptr(), dc.data_ptr(), lse.data_ptr(),
                              dq.data_ptr(), ws.data_ptr(), s, b, heads, hd, st)
        fwd()
        prod = 2.0 * hd * s * (s + 1) / 2 * b * heads
        tf = timeit(fwd, args.reps)
        tb = timeit(bwd, args.reps)
        rec = {"shape": name, "s": s, "b": b, "heads": heads, "hd": hd, "fwd_us": round(tf, 1),
               "fwd_tflops": round(2 * prod / tf / 1e6, 1), "bwd_us": round(tb, 1),
               "bwd_tflops": round(5 * prod / tb / 1e6, 1)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
