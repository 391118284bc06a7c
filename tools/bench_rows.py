"""Time the LayerNorm row kernels through the C ABI (mp_op_*) with CUDA events.

    python tools/bench_rows.py [--reps 50]

Shapes: the per-layer LayerNorm shapes of the BASELINE configs at b=2
(R = s*b = 4096 rows; h = 2304, 4096, 6144, 8192).  Two timings per kernel:
"warm" = back-to-back launches (inputs L2-resident, as in the layer step where
the producer GEMM has just written them), "cold" = a 512 MB buffer is written
between launches (L2 flushed), only the kernel inside the events.  GB/s =
algorithmic bytes (each tensor read / written once) / time, against the
measured HBM copy bandwidth in MEASURED_PEAKS.json.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04473_b200 import mp  # noqa: E402


def timeit(fn, reps, flush=None):
    """Median kernel time in us.  Warm: `reps` back-to-back launches between two events
    (host launch overhead overlaps the GPU work).  Cold: a 512 MB write before each
    launch, only the launch inside the events."""
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(3):
        fn()
    if flush is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            a.record(st)
            for _ in range(reps):
                fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / reps)
        return min(ts)
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--R", type=int, default=4096)
    ap.add_argument("--widths", default="2304,4096,6144,8192")
    args = ap.parse_args()
    mp.lib()
    peak = None
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = json.load(open(pk)).get("hbm_gbs")
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    R = args.R
    out = []
    for h in [int(x) for x in args.widths.split(",")]:
        bf = torch.bfloat16
        x, dy, dres, y, r = (torch.randn(R, h, device="cuda", dtype=bf) for _ in range(5))
        x1, o, dx = (torch.empty(R, h, device="cuda", dtype=bf) for _ in range(3))
        g = (1 + 0.1 * torch.randn(h, device="cuda")).to(bf)
        b = (0.1 * torch.randn(h, device="cuda")).to(bf)
        mu, rs = (torch.empty(R, device="cuda") for _ in range(2))
        acc = torch.zeros(4, h, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        E = 2 * R * h
        kernels = {
            "ln_fwd": (lambda: mp.call("mp_op_layernorm_fwd", "bf16", x.data_ptr(), g.data_ptr(), b.data_ptr(),
                                       o.data_ptr(), mu.data_ptr(), rs.data_ptr(), R, h, 1e-5, st), 2 * E + 8 * R),
            "bda_ln_fwd": (lambda: mp.call("mp_op_bda_layernorm_fwd", "bf16", y.data_ptr(), b.data_ptr(), r.data_ptr(),
                                           x1.data_ptr(), g.data_ptr(), b.data_ptr(), o.data_ptr(), mu.data_ptr(),
                                           rs.data_ptr(), R, h, 1e-5, st), 4 * E + 8 * R),
            "ln_bwd": (lambda: mp.call("mp_op_layernorm_bwd", "bf16", dy.data_ptr(), x.data_ptr(), g.data_ptr(),
                                       mu.data_ptr(), rs.data_ptr(), dres.data_ptr(), dx.data_ptr(),
                                       acc[0].data_ptr(), acc[1].data_ptr(), R, h, st),
                       4 * E + 8 * R),
            "ln_bwd_sums": (lambda: mp.call("mp_op_layernorm_bwd_sums", "bf16", dy.data_ptr(), x.data_ptr(),
                                            g.data_ptr(), mu.data_ptr(), rs.data_ptr(), dres.data_ptr(),
                                            dx.data_ptr(), acc[0].data_ptr(), acc[1].data_ptr(), acc[2].data_ptr(),
                                            acc[3].data_ptr(), R, h, st), 4 * E + 8 * R),
            "colsum": (lambda: mp.call("mp_op_colsum_accum", "bf16", dy.data_ptr(), acc[0].data_ptr(), R, h, st),
                       E),
        }
        mp.call("mp_op_layernorm_fwd", "bf16", x.data_ptr(), g.data_ptr(), b.data_ptr(), o.data_ptr(),
                mu.data_ptr(), rs.data_ptr(), R, h, 1e-5, st)
        for variant in ["current"]:
            for name, (fn, nbytes) in kernels.items():
                warm = timeit(fn, args.reps)
                cold = timeit(fn, args.reps, flush)
                rec = {"kernel": name, "variant": variant, "R": R, "h": h, "bytes": nbytes, "warm_us": round(warm, 2),
                       "cold_us": round(cold, 2), "warm_gbs": round(nbytes / warm / 1e3, 1),
                       "cold_gbs": round(nbytes / cold / 1e3, 1)}
                if peak:
                    rec["cold_frac"] = round(nbytes / cold / 1e3 / peak, 3)
                out.append(rec)
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
