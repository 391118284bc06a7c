"""Scatter/gather ablation of the pipeline P2P inside one NVLink box.

    torchrun --nproc-per-node 4 tools/scatter_gather_probe.py [OUT.json]

Layout t = 2, p = 2: ranks {0, 1} = stage 0 (TP group), {2, 3} = stage 1.  The
paper's optimisation sends 1/t of the (replicated) stage-boundary activation
from each TP rank and all-gathers it over NVLink on the receiving stage,
instead of every TP rank sending the whole tensor.  Both variants are timed
with CUDA events over NCCL on the GPT-18.4B / 39.1B boundary payloads
(s b h bf16, b = 1), max over ranks, median of 20 repetitions.
"""
import json
import os
import sys

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 4
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    t = 2
    tp = rank % t
    stage = rank // t
    peer = (1 - stage) * t + tp                       # same TP index on the other stage
    recv_group = [dist.new_group([0, 1]), dist.new_group([2, 3])]
    res = {}
    for name, h in (("18.4B", 6144), ("39.1B", 8192)):
        n = 2048 * h
        full = torch.ones(n, dtype=torch.bfloat16, device="cuda")
        part = torch.empty(n // t, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(n, dtype=torch.bfloat16, device="cuda")

        def plain():
            if stage == 0:
                dist.send(full, peer)
            else:
                dist.recv(out, peer)

        def scatter_gather():
            if stage == 0:
                dist.send(full[tp * (n // t):(tp + 1) * (n // t)].contiguous(), peer)
            else:
                dist.recv(part, peer)
                dist.all_gather_into_tensor(out, part, group=recv_group[1])
            if stage == 0:   # keep the stage-0 ranks in the same collective sequence as stage 1
                pass

        for vname, fn in (("plain", plain), ("scatter_gather", scatter_gather)):
            ts = []
            for it in range(25):
                dist.barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                if it >= 5:
                    ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            med = torch.tensor([ts[len(ts) // 2]], device="cuda")
            dist.all_reduce(med, op=dist.ReduceOp.MAX)
            res[f"{name}_{vname}_us"] = round(float(med), 1)
        res[f"{name}_bytes"] = 2 * n
    if rank == 0:
        res["note"] = ("max over ranks of the median per-transfer time; plain = every TP rank sends the whole "
                       "s b h boundary tensor to its peer; scatter_gather = 1/t each + all-gather on the receiver")
        print(json.dumps(res))
        if len(sys.argv) > 1:
            json.dump(res, open(sys.argv[1], "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
