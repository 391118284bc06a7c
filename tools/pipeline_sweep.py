"""Pipeline-bubble sweep: bench.py under torchrun for a list of (model, t, p, v, m)
layouts, each with >= 10 measured batches (bench --bubble-batches), one JSON
line per run appended to the output file.

    python tools/pipeline_sweep.py OUT.jsonl SET [--steps K]

SET:
  balanced  GPT-1.7B width (h=2304, l=24) with V=512 (negligible head, so the
            stages are balanced as (p-1)/(v m) assumes), t=1,
            p in {2, 4}, v in {1, 2, 3}, m in {8, 16}, b=1.
  balanced_b2  the same layouts at b=2 (twice the work per task).
  w391      39.1B width (h=8192, a=64), l=24, t=2 x p=2, m=16, b=1,
            v in {1, 2, 3, 6}, full V=51200 head (BASELINE configs[4] sweep).
  w391v6    only the v=6 point of w391.
Each run is wrapped in `timeout`; a failed run records its exit code.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def runs(which):
    if which == "balanced":
        for p in (2, 4):
            for v in (1, 2, 3):
                for m in (8, 16):
                    yield dict(model="1.7B", t=1, p=p, v=v, m=m, b=1, vocab=512, layers=24)
    elif which == "balanced_b2":
        for p in (2, 4):
            for v in (1, 2, 3):
                for m in (8, 16):
                    yield dict(model="1.7B", t=1, p=p, v=v, m=m, b=2, vocab=512, layers=24)
    elif which in ("w391", "w391v6"):
        for v in ((1, 2, 3, 6) if which == "w391" else (6,)):
            yield dict(model="39.1B", t=2, p=2, v=v, m=16, b=1, vocab=0, layers=24)
    else:
        raise SystemExit(f"unknown set {which}")


def main():
    out, which = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 10
    port = 29600
    for r in runs(which):
        n = r["t"] * r["p"]
        port += 1
        cmd = ["timeout", "900", sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
               os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--model", r["model"], "--tp", str(r["t"]),
               "--pp", str(r["p"]), "--vp", str(r["v"]), "--B", str(r["m"] * r["b"]), "--b", str(r["b"]),
               "--layers", str(r["layers"]), "--steps", str(steps), "--warmup", "3", "--bubble-batches", "10",
               "--no-cpu-baseline", "--no-e2e"]
        if r["vocab"]:
            cmd += ["--vocab", str(r["vocab"])]
        p = subprocess.run(cmd, capture_output=True, text=True)
        line = None
        for ln in p.stdout.splitlines():
            if ln.startswith("{"):
                line = ln
        rec = {"run": r, "rc": p.returncode}
        if line:
            rec["bench"] = json.loads(line)
        else:
            rec["stderr_tail"] = p.stderr[-3000:]
        with open(out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        b = rec.get("bench", {}).get("bubble") or {}
        print(json.dumps({"run": r, "rc": p.returncode, "tflops": rec.get("bench", {}).get("value"),
                          "bubble": b.get("measured_max_over_ranks"), "formula": b.get("formula"),
                          "replay": b.get("replay_per_stage")}), flush=True)


if __name__ == "__main__":
    main()
