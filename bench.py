"""Benchmark of the PTD-P hot path on B200: one full GPT training iteration
(forward + backward of every layer under tensor / pipeline parallelism,
flush, tied-embedding all-reduce, Adam) through the C ABI, reported as model
TFLOP/s by the paper's formula (Eq. (2)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Default workload (BASELINE.json configs[1], "GPT 1.7B, t=1..8, p=1"): GPT-1.7B
(h=2304, a=24, l=24, s=2048, V=51200), tensor parallel t = N, p = 1, global
batch B = 16 sequences of microbatch b = 2 (m = 8, 1F1B), bf16 storage with
fp32 accumulation, synthetic tokens and random-init weights.  Every step's
working set (3.3 GB of bf16 weights alone) exceeds the 126 MB L2, so no L2
flush is needed between steps.

FLOP accounting: without activation recomputation the honest per-iteration
count is the 72-variant of Eq. (2), 72 B s l h^2 (1 + s/6h) + 6 B s h V
(reading #18); `value` uses it.  The 96-formula number is
reported beside it for reference.  `value` is the paper's metric, model
TFLOP/s PER GPU (F / (N t_step)); `aggregate_tflops` is the whole-job sum.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

_JSON_FD = None


def redirect_stdout():
    """stdout carries exactly one JSON line: library chatter (e.g. NCCL's version
    banner printed from C) is sent to stderr, the JSON goes to the saved stdout.
    Called from main() only, so importing this module has no side effects."""
    global _JSON_FD
    if _JSON_FD is None:
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj):
    sys.stdout.flush()
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "model TFLOP/s/GPU (paper FLOP formula), % of bf16 peak, at 1/2/4/8 GPUs"
DATASHEET_BF16 = 2250.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--tp-comm", dest="tp_comm", default="auto", choices=["auto", "nccl", "nvls"],
                    help="transport of the layer all-reduces (auto: NVLS fused when available)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="1.7B", help="tiny | 1.7B | 7.5B | 18.4B | 39.1B")
    ap.add_argument("--tp", dest="t", type=int, default=0, help="tensor parallel size (default: N / p)")
    ap.add_argument("--pp", dest="p", type=int, default=1, help="pipeline parallel size")
    ap.add_argument("--vp", dest="v", type=int, default=1, help="model chunks per device (interleaved)")
    ap.add_argument("--dp", dest="d", type=int, default=1, help="data-parallel replicas (P:85-89)")
    ap.add_argument("--recompute", action="store_true",
                    help="activation recomputation (P:268-272); FLOPs then follow Eq. (2)'s 96-formula")
    ap.add_argument("--layers", type=int, default=0, help="override l (depth-reduced proxy; reported)")
    ap.add_argument("--vocab", type=int, default=0,
                    help="override V (e.g. 512: a negligible head, so the pipeline stages are balanced as the "
                         "bubble formula assumes, P:104-118; reported in config)")
    ap.add_argument("--bubble-batches", dest="bubble_batches", type=int, default=10,
                    help="p > 1: extra batches run after the timed region with per-task events; the bubble "
                         "is reported as the median over them (SURVEY 8(d): >= 10)")
    ap.add_argument("--B", type=int, default=16, help="global batch (sequences)")
    ap.add_argument("--b", type=int, default=2,
                    help="microbatch size (default 2: the best of the b in {1, 2, 4} sweep at 1.7B on 1xB200, "
                         "the paper's own tuning knob, P:259-266, P:492)")
    ap.add_argument("--sched", default="", help="gpipe | 1f1b | interleaved (default: 1f1b, interleaved if v > 1)")
    ap.add_argument("--attn", default="fused", choices=["fused", "unfused"],
                    help="attention core: fused tcgen05 flash kernel (default) or the paper's unfused "
                         "scores GEMM + softmax + P.V GEMM")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return {"bf16_burst": float(d["bf16_tflops"]), "bf16_sustained": float(d["bf16_tflops_sustained"]),
                "hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        return {"bf16_burst": 1590.0, "bf16_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "B200_PROFILING.md fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, util, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                util.append(float(f[4]))
            except ValueError:
                continue
            for nm, val in zip(names, f[6:10]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s, u in zip(sm, util) if u >= 50] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    return world, rank, local


def cpu_oracle_layer(cfg, reps=1):
    """The fp64 oracle (as it stands) on one unpartitioned layer fwd+bwd at the
    workload's width, b = 1, s = cfg.s: FLOPs 3 (24 s h^2 + 4 s^2 h)."""
    import threadpoolctl
    import gen
    from oracle import layer as L
    h, a, s = cfg.h, cfg.a, cfg.s
    W = gen.layer_weights(h, cfg.l, seed=5, layer=0, dtype="bf16")
    X = gen.activations((s, 1, h), 6, 1.0, "bf16")
    dY = gen.activations((s, 1, h), 7, 1e-3, "bf16")
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 runs this alone)
    with threadpoolctl.threadpool_limits(limits=os.cpu_count() or 1):
        t0 = time.perf_counter()
        for _ in range(reps):
            _, cache = L.layer_fwd(X, W, a)
            L.layer_bwd(dY, cache, W, a)
        dt = time.perf_counter() - t0
        info = threadpoolctl.threadpool_info()
    flops = reps * 3 * (24 * s * h * h + 4 * s * s * h)
    threads = max([i.get("num_threads", 1) for i in info] or [1])
    return flops, dt, threads


def run_reference(args, cfg, world, rank):
    """--impl reference: the oracle timed on the host cores, on this arm's
    metric; each step = one unpartitioned layer fwd+bwd of the workload."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_oracle_layer(cfg)
    tot_f, tot_t, threads = 0.0, 0.0, 1
    for _ in range(args.steps):
        f, t, threads = cpu_oracle_layer(cfg)
        tot_f += f
        tot_t += t
    val = tot_f / tot_t / 1e12
    sample = f"one unpartitioned GPT-{args.model} layer fwd+bwd (b=1, s={cfg.s}, h={cfg.h}) per step, fp64 numpy"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": dict(workload_config(args, cfg),
                          workload=f"one unpartitioned GPT-{args.model}-width layer fwd+bwd, b=1, s={cfg.s}, "
                                   f"fp64 numpy oracle on the host cores (a bounded sample of the iteration)"),
           "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def replay_bubble(p, m, v, sched, tf, tb):
    """Ideal-pipeline replay of the library's own static task orders with this run's
    measured per-rank mean task durations and zero communication (mp_bubble_replay,
    host-only C ABI): the bubble the schedule itself implies once stage imbalance
    (embedding on the first stage, logit layer + loss on the last) is accounted for.
    Returns the per-rank idle share (span_r - busy_r) / busy_r, span from t = 0, or
    None if the replay cannot run."""
    from paper_2104_04473_b200 import mp
    try:
        return mp.mp_bubble_replay(p, m, v, sched, tf, tb)
    except mp.MPError:
        return None


def paper_bubble(spans, busy):
    """The paper's pipeline bubble of one batch from per-rank measurements:
    every rank idles from the batch start to its first task and from its last task to
    the end of the whole pipeline, so bubble_r = (max_r' span_r' - busy_r) / busy_r,
    with span_r = the rank's last task end from the common batch start (all ranks start
    at a barrier) and busy_r = its summed task durations.  Returns (mean, max) over the
    ranks with busy_r > 0."""
    total = max(spans)
    vals = [(total - b) / b for b in busy if b > 0]
    return float(np.mean(vals)), float(np.max(vals))


def bubble_report(stats_list, world, p, v, m, sched, d=1):
    """Per-rank pipeline idle share (span_r - busy_r) / busy_r of each measured batch,
    max over ranks, median over the batches, next to the closed form (p-1)/m or
    (p-1)/(v m), and the ideal-pipeline replay of the library's own
    static task orders with this run's measured per-stage task durations (zero
    communication; captures stage imbalance such as the last stage's head)."""
    stats_list = [st for st in stats_list if st]
    if not stats_list:
        return None
    keys = ("bubble_measured", "pipeline_seconds", "busy_seconds", "t_fwd_task", "t_bwd_task", "iter_seconds")
    batches = []   # [batch][rank][key]
    for st in stats_list:
        vals = [st[k] for k in keys]
        if world > 1:
            import torch
            import torch.distributed as dist
            t = torch.tensor(vals, dtype=torch.float64, device="cuda")
            g = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(g, t)
            batches.append([x.tolist() for x in g])
        else:
            batches.append([vals])
    per_batch = [max(r[0] for r in pr) for pr in batches]
    med = float(np.median(per_batch))
    # the paper's definition: a device idles from the batch start to its first
    # task AND from its last task to the end of the whole pipeline, so the bubble of rank r is
    # (global pipeline span - busy_r) / busy_r with the span = the longest rank's (all ranks
    # start at a barrier); the per-rank-local value above stops at the rank's own last task
    paper_mean, paper_max = [], []
    for pr in batches:
        mean_b, max_b = paper_bubble([r[1] for r in pr], [r[2] for r in pr])
        paper_mean.append(mean_b)
        paper_max.append(max_b)
    mid = batches[int(np.argsort(per_batch)[len(per_batch) // 2])]
    per_rank = [[float(np.median([pr[r][k] for pr in batches])) for k in range(len(keys))]
                for r in range(len(batches[0]))]
    st = stats_list[-1]
    rep = {"formula": st["bubble_formula"], "schedule": sched, "p": p, "v": v, "m": m,
           "batches": len(batches),
           "paper_definition_mean_over_ranks": float(np.median(paper_mean)),
           "paper_definition_max_over_ranks": float(np.median(paper_max)),
           "paper_definition_rel_error_vs_formula": (float(np.median(paper_mean)) - st["bubble_formula"]) /
           st["bubble_formula"] if st["bubble_formula"] else None,
           "measured_max_over_ranks": med,
           "measured_max_over_ranks_per_batch": [round(x, 5) for x in per_batch],
           "measured_per_rank_median_batch": [round(r[0], 5) for r in mid],
           "rel_error_vs_formula": (med - st["bubble_formula"]) / st["bubble_formula"] if st["bubble_formula"] else None,
           "peak_inflight_rank0": st["peak_inflight"],
           "t_fwd_task_s": [round(r[3], 6) for r in per_rank], "t_bwd_task_s": [round(r[4], 6) for r in per_rank],
           "flush_and_optimizer_s": max(r[5] - r[1] for r in per_rank),
           "how": "per-task CUDA events on the compute stream; measured_*: bubble_r = (last task end - batch "
                  "start - sum of task durations) / sum of task durations (rank-local span), max over ranks; "
                  "paper_definition_*: (longest rank's span - busy_r) / busy_r, i.e. warm-up AND cool-down "
                  "idle of every rank (P:104-105), mean / max over ranks; medians over the batches"}
    if p > 1:
        # pipeline stage r = the ranks with pp = r in replica 0, rank = (dp p + pp) t + tp
        # (TP ranks of a stage behave alike: use the max)
        t = world // (p * d)
        tf = [max(per_rank[r * t + k][3] for k in range(t)) for r in range(p)]
        tb = [max(per_rank[r * t + k][4] for k in range(t)) for r in range(p)]
        rp = replay_bubble(p, m, v, sched, tf, tb)
        if rp:
            rep["replay_per_stage"] = [round(x, 5) for x in rp]
            rep["replay_note"] = ("same static orders, measured per-stage task durations, zero communication; "
                                  "measured - replay = communication / launch stalls")
    return rep


def comm_calibration(cfg, b, t, p, d, world, m, t_step):
    """NVLink roofline of the TP communication (t > 1, p = d = 1 so the TP group is the
    world): one layer's g / f payload (s*b*h bf16) all-reduced by NCCL over the TP group,
    CUDA events, after warm-up.  busbw = algbw * 2(t-1)/t against the 900 GB/s per-direction
    NVLink 5 peak.  The library's default NVLS path fuses the reduction into the consuming
    LayerNorm / residual kernel, so this is the calibration of the paper's transport and an
    upper bound of the communication share (4 reductions per layer per microbatch)."""
    if t <= 1 or p != 1 or d != 1 or world != t:
        return None
    import torch
    import torch.distributed as dist
    n = cfg.s * b * cfg.h
    x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / reps
    from paper_2104_04473_b200 import launch
    sec = launch.max_over_ranks(sec, world, "cuda")
    algbw = 2.0 * n / sec / 1e9
    busbw = algbw * 2.0 * (t - 1) / t
    per_step = 4 * cfg.l * m
    return {"payload_bytes": 2 * n, "nccl_allreduce_us": sec * 1e6, "algbw_gbs": algbw, "busbw_gbs": busbw,
            "nvlink_peak_gbs": 900.0, "frac": busbw / 900.0, "reductions_per_step": per_step,
            "nccl_share_of_step_upper_bound": per_step * sec / t_step,
            "how": "torch NCCL all_reduce of one layer payload (s*b*h bf16) on the TP group, 20 reps after 5 "
                   "warm-up, CUDA events, max over ranks; busbw = algbw*2(t-1)/t vs 900 GB/s NVLink 5 per "
                   "direction; share = reductions * time / step (the NVLS default fuses them into consumers)"}


def workload_config(args, cfg):
    t = args.t or max(1, args.gpus // (args.p * args.d))
    sched = args.sched or ("interleaved" if args.v > 1 else "1f1b")
    return {"workload": f"GPT-{args.model} full training iteration (fwd+bwd all layers, flush, Adam)",
            "model": f"GPT-{args.model}", "l": cfg.l, "h": cfg.h, "a": cfg.a, "seq_len": cfg.s, "V": cfg.V,
            "global_batch": args.B, "micro_batch": args.b, "m": args.B // (args.b * args.d), "t": t, "p": args.p,
            "v": args.v, "d": args.d, "schedule": sched,
            "parallelism": f"t{t}p{args.p}v{args.v}" + (f"d{args.d}" if args.d > 1 else ""),
            "attention": {"fused": "fused tcgen05 flash kernel (scores never materialised)",
                          "unfused": "paper: strided-batched scores GEMM + fused causal softmax + P.V GEMM"}[args.attn],
            "l2": "working set > 126 MB L2 every step (weights alone exceed it); no flush",
            "recompute": bool(args.recompute),
            "flop_formula": ("Eq. (2) with recomputation: 96Bslh^2(1+s/6h+V/16lh)" if args.recompute else
                             "Eq. (2) 72-variant (no recomputation): 72Bslh^2(1+s/6h)+6BshV")}


def main():
    redirect_stdout()
    # Enough hardware work queues that a stream's wait on a pipeline-channel flag
    # (cuStreamWaitValue32, p2p.cu) never blocks unrelated streams' work through a
    # shared queue.  Must be set before CUDA initialises (mp.py sets it too).
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    args = parse()
    import gen
    cfg = gen.CONFIGS[args.model]
    if args.layers or args.vocab:
        cfg = gen.ModelCfg(l=args.layers or cfg.l, h=cfg.h, a=cfg.a, s=cfg.s, V=args.vocab or cfg.V)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_2104_04473_b200 import mp
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    d = args.d
    t = args.t or max(1, world // (args.p * d))
    p, v = args.p, args.v
    sched = args.sched or ("interleaved" if v > 1 else "1f1b")
    B, b = args.B, args.b
    m = B // (b * d)
    # ---- context (NCCL id from rank 0, broadcast by the launcher)
    from paper_2104_04473_b200 import launch
    nid = launch.share_bytes(mp.mp_nccl_get_id() if rank == 0 else None, rank, world)
    c = mp.make_cfg(cfg.l, cfg.h, cfg.a, cfg.s, cfg.V, dtype="bf16", lr=1e-5, attn=args.attn, tp_comm=args.tp_comm,
                    recompute=args.recompute)
    ctx = mp.Context(t, p, v, d, c, rank, world, local, nid)
    # ---- random-init weights (only the owned shards are kept)
    dev_of, _ = mp.mp_get_stage_map(cfg.l, p, v)
    pp = (rank // t) % p
    for k in range(cfg.l):
        if dev_of[k] != pp:
            continue
        for name, arr in gen.layer_weights_fast(cfg.h, cfg.l, 42, k).items():
            ctx.set_weights(name, k, arr)
    for name, arr in gen.model_weights_fast(cfg, 42).items():
        ctx.set_weights(name, 0, arr)
    tok = gen.tokens(B, cfg.s, cfg.V, seed=1234)
    d_tok = torch.tensor(tok, dtype=torch.int32, device="cuda")
    d_loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream())
    F = mp.mp_flops(B, cfg.s, cfg.l, cfg.h, cfg.V, args.recompute)
    F96 = mp.mp_flops(B, cfg.s, cfg.l, cfg.h, cfg.V, True)
    # ---- warm-up (also yields the bubble statistics of one batch)
    wstats = None
    for i in range(args.warmup):
        wstats = ctx.run_batch_dev(B, b, m, sched, d_tok.data_ptr(), d_loss.data_ptr(), apply_optimizer=True,
                                   stats=(i == args.warmup - 1))
    torch.cuda.synchronize()
    # ---- timed region: K back-to-back iterations, CUDA events on the compute stream
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = mp.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0, e1 = ev[0], ev[-1]
    e0.record(stream)
    for k in range(args.steps):
        ctx.run_batch_dev(B, b, m, sched, d_tok.data_ptr(), d_loss.data_ptr(), apply_optimizer=True)
        ev[k + 1].record(stream)
    torch.cuda.synchronize()
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    launches = mp.launch_count() - l0
    # GEMM roofline: the same iterations again with every GEMM launch bracketed by CUDA
    # events on its stream (kept out of the timed region above: ~2 events per launch
    # perturb the step by a few per cent)
    mp.profile_gemm(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        ctx.run_batch_dev(B, b, m, sched, d_tok.data_ptr(), d_loss.data_ptr(), apply_optimizer=True)
    p1.record(stream)
    g_flops, g_sec, g_n = mp.profile_gemm_read()
    mp.profile_gemm(False)
    prof_ms = p0.elapsed_time(p1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t_step = ms / 1e3 / args.steps
    t_step = launch.max_over_ranks(t_step, world, "cuda")
    loss_val = float(d_loss.item())
    # ---- end to end through the public API: pinned host tokens in, loss out, every step
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(tok).pin_memory()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.run_batch(B, b, m, sched, pinned.data_ptr(), apply_optimizer=True, stats=False)
        torch.cuda.synchronize()
        w = (time.perf_counter() - w0) / args.steps
        w = launch.max_over_ranks(w, world, "cuda")
        e2e = {"value": F / w / 1e12 / world, "unit": "TFLOP/s (per GPU)", "h2d_bytes_per_step": int(tok.nbytes),
               "d2h_bytes_per_step": 4, "ms_per_step": 1e3 * w,
               "how": "mp_run_batch with pinned host tokens (H2D inside) and the loss read back every step; "
                      "wall clock with device sync, max over ranks"}
    # ---- pipeline bubble over several batches (per-task CUDA events; outside the timed region)
    bstats = []
    if p > 1:
        for _ in range(max(0, args.bubble_batches)):
            bstats.append(ctx.run_batch_dev(B, b, m, sched, d_tok.data_ptr(), d_loss.data_ptr(),
                                            apply_optimizer=True, stats=True))
    pk = peaks()
    agg = F / t_step / 1e12
    per_gpu = agg / world
    achieved = g_flops / g_sec / 1e12 if g_sec > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.model)
        except Exception:
            traffic = None
    out = {
        "metric": METRIC, "value": per_gpu, "unit": "TFLOP/s per GPU", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random-init weights)",
        "config": dict(workload_config(args, cfg), tp_comm=ctx.tp_comm_mode() if t > 1 else "none (t=1)"),
        "per_gpu_tflops": per_gpu, "aggregate_tflops": agg,
        "pct_of_bf16_peak": {"measured_burst_1683": 100 * per_gpu / pk["bf16_burst"],
                             "measured_sustained": 100 * per_gpu / pk["bf16_sustained"],
                             "datasheet_2250": 100 * per_gpu / DATASHEET_BF16},
        "model_flops_per_step": F, "eq2_96_formula_tflops_per_gpu": F96 / t_step / 1e12 / world,
        "loss": loss_val,
        "roofline": {"kernel": "tcgen05 GEMM engine (all bf16 GEMM launches of the step)", "bound": "tensor",
                     "achieved": achieved, "peak": pk["bf16_sustained"], "unit": "TFLOP/s",
                     "frac": achieved / pk["bf16_sustained"], "traffic": traffic,
                     "peak_source": pk["source"] + ", sustained (kernels timed inside a long step)",
                     "gemm_share_of_step": g_sec / max(1e-12, prof_ms / 1e3), "gemm_launches": g_n,
                     "how": "CUDA events around every GEMM launch on its stream, over --steps iterations "
                            "run right after the timed region"},
        "gpu_launches": int(launches),
        "step_ms_rank0": [round(x, 3) for x in step_ms],
        "clocks": clk,
        "bubble": bubble_report(bstats or [wstats], world, p, v, m, sched, d),
    }
    if world > 1:
        out["comm"] = comm_calibration(cfg, b, t, p, d, world, m, t_step)
        if out["comm"] is not None and ctx.tp_comm_mode() == "nvls":
            # the default path: the same payload through the library's fused NVLS reduction
            sec = ctx.tp_reduce_probe(b, 20)
            from paper_2104_04473_b200 import launch
            sec = launch.max_over_ranks(sec, world, "cuda")
            payload = 2.0 * cfg.s * b * cfg.h
            busbw = payload / sec / 1e9 * 2.0 * (t - 1) / t
            out["comm"]["nvls"] = {
                "us_per_reduction": sec * 1e6, "busbw_gbs": busbw, "nvlink_peak_gbs": 900.0, "frac": busbw / 900.0,
                "shot": "two" if t >= 4 else "one",
                "share_of_step_upper_bound": 4 * cfg.l * m * sec / t_step,
                "how": "mp_tp_reduce_probe: next symmetric buffer, NVLS barrier (one-shot) or slab reduce-load + "
                       "multicast store + barrier (two-shot), then the consuming bias-residual kernel reading the "
                       "t-way sum of s*b*h bf16; CUDA events, 20 reps after 3, max over ranks; busbw convention "
                       "of NCCL (payload * 2(t-1)/t / time) vs 900 GB/s NVLink 5 per direction"}
    if e2e:
        out["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        f, dt, threads = cpu_oracle_layer(cfg, reps=1)
        out["cpu_baseline"] = {"value": f / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                               "seconds": dt, "host_cpus": os.cpu_count(),
                               "sample": f"one unpartitioned GPT-{args.model} layer fwd+bwd (b=1, s={cfg.s}), "
                                         f"fp64 numpy oracle, {f:.3g} FLOP"}
    if rank == 0:
        emit(out)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
