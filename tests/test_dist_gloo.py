"""N > 1 host-side logic on CPU with the gloo backend (world_size 2 and 4):
id broadcast, max-over-ranks timing, grid coordinates, and the pipeline
channel protocol of the stage runtime executed by real concurrent processes
(each rank owns only its stages and exchanges activations / gradients in the
exact order the C++ runtime enqueues them: sends are asynchronous FIFO
pushes, receives block at consume time).  The math inside each stage is the
oracle's (test infrastructure); the result must equal the sequential oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp_

import gen
from oracle import layer as L
from oracle import model as M
from oracle import schedule as SC
from paper_2104_04473_b200 import launch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_plumbing(rank, world, port, q):
    _init(rank, world, port)
    blob = launch.share_bytes(b"id-from-rank-0" if rank == 0 else None, rank, world)
    mx = launch.max_over_ranks(float(rank + 1), world)
    q.put((rank, blob, mx, launch.tp_pp_of(rank, 2, world // 2)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_plumbing(world):
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_plumbing, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
    assert all(b == b"id-from-rank-0" for _, b, _, _ in out)
    assert all(m == float(world) for _, _, m, _ in out)
    assert [tpp for *_, tpp in out] == [(r % 2, (r // 2) % (world // 2), 0) for r in range(world)]


def _worker_pipeline(rank, p, v, m, kind, port, q):
    """Rank `rank` = device r of a p-stage pipeline (t = 1)."""
    _init(rank, p, port)
    cfg = gen.ModelCfg(l=2 * p * v, h=16, a=2, s=8, V=32)
    W = gen.model_weights(cfg, seed=3, dtype="fp32")
    tok = gen.tokens(m, cfg.s, cfg.V, seed=4)
    scale = 1.0 / (m * cfg.s)
    dev_of, chunk_of = SC.stage_map(cfg.l, p, v)
    S = p * v
    layers = {sg: [k for k in range(cfg.l) if chunk_of[k] * p + dev_of[k] == sg] for sg in range(S)}
    nxt, prv = (rank + 1) % p, (rank - 1) % p
    grads = M.zero_grads(W)
    stash, pending, loss = {}, [], 0.0
    shape = (cfg.s, 1, cfg.h)
    for kind_, i, c in SC.build_schedule(kind, p, m, v, rank):
        sigma = c * p + rank
        tk = tok[i:i + 1]
        if kind_ == "F":
            if sigma == 0:
                X = M.embed_fwd(tk[:, :-1], W["emb"], W["pos"])
            else:
                buf = torch.empty(shape, dtype=torch.float64)
                dist.recv(buf, src=prv, tag=0)                  # activation channel, FIFO
                X = buf.numpy()
            cs = []
            for k in layers[sigma]:
                X, cache = L.layer_fwd(X, W["layers"][k], cfg.a)
                cs.append(cache)
            stash[(i, sigma)] = cs
            if sigma == S - 1:
                lo, dX, demb, dg, db = M.head_fwd_bwd(X, tk[:, 1:], W, scale)
                loss += lo
                grads["emb"] += demb
                grads["lnf_g"] += dg
                grads["lnf_b"] += db
                stash[("g", i)] = dX
            else:
                pending.append(dist.isend(torch.from_numpy(np.ascontiguousarray(X)), dst=nxt, tag=0))
        else:
            if sigma == S - 1:
                dX = stash.pop(("g", i))
            else:
                buf = torch.empty(shape, dtype=torch.float64)
                dist.recv(buf, src=nxt, tag=1)                  # gradient channel, FIFO
                dX = buf.numpy()
            for k, cache in zip(reversed(layers[sigma]), reversed(stash.pop((i, sigma)))):
                dX, gl = L.layer_bwd(dX, cache, W["layers"][k], cfg.a)
                for name, val in gl.items():
                    grads["layers"][k][name] += val
            if sigma == 0:
                demb, dpos = M.embed_bwd(dX, tk[:, :-1], cfg.V)
                grads["emb"] += demb
                grads["pos"] += dpos
            else:
                pending.append(dist.isend(torch.from_numpy(np.ascontiguousarray(dX)), dst=prv, tag=1))
    for h in pending:
        h.wait()
    # flush: tied embedding gradient and loss summed over ranks (t = 1)
    ge = torch.from_numpy(grads["emb"])
    dist.all_reduce(ge)
    lt = torch.tensor([loss], dtype=torch.float64)
    dist.all_reduce(lt)
    mine = {k: grads["layers"][k] for k in range(cfg.l) if dev_of[k] == rank}
    q.put((rank, float(lt.item()), ge.numpy(), mine))
    dist.destroy_process_group()


@pytest.mark.parametrize("p,v,m,kind", [(2, 1, 4, SC.ONE_F_ONE_B), (2, 2, 4, SC.INTERLEAVED),
                                        (2, 1, 3, SC.GPIPE), (4, 2, 4, SC.INTERLEAVED), (4, 1, 6, SC.ONE_F_ONE_B)])
def test_pipeline_channels_gloo(p, v, m, kind):
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_pipeline, args=(r, p, v, m, kind, port, q)) for r in range(p)]
    for pr in ps:
        pr.start()
    res = sorted((q.get(timeout=240) for _ in range(p)), key=lambda x: x[0])
    for pr in ps:
        pr.join(60)
    cfg = gen.ModelCfg(l=2 * p * v, h=16, a=2, s=8, V=32)
    W = gen.model_weights(cfg, seed=3, dtype="fp32")
    tok = gen.tokens(m, cfg.s, cfg.V, seed=4)
    loss, g = M.batch_fwd_bwd(W, tok, cfg.a, m)
    for _, lo, ge, mine in res:
        assert abs(lo - loss) <= 1e-12 * abs(loss)
        assert np.max(np.abs(ge - g["emb"])) <= 1e-12 * np.max(np.abs(g["emb"]))
        for k, gl in mine.items():
            for name, val in gl.items():
                assert np.max(np.abs(val - g["layers"][k][name])) <= 1e-12 * max(1e-300, np.max(np.abs(val))), (k, name)


def _worker_dp(rank, world, port, q):
    """Data-parallel replica `rank` (t = p = 1, d = world): the runtime's
    convention -- replica dp trains on rows [dp B/d, (dp+1) B/d), scales its
    loss by 1/(B s) of the GLOBAL batch and the flush sums the replicas'
    gradients -- must reproduce the whole-batch gradient."""
    _init(rank, world, port)
    shape = gen.TINY
    W = gen.model_weights(shape, seed=42, dtype="fp32")
    m = 2
    tok = gen.tokens(m * world, shape.s, shape.V, seed=1234)
    dp = launch.tp_pp_of(rank, 1, 1)[2]
    mine = tok[dp * m:(dp + 1) * m]
    loss, g = M.batch_fwd_bwd(W, mine, shape.a, m)          # mean over this replica's m*s tokens
    flat = np.concatenate([g["emb"].ravel()] + [v.ravel() for Wl in g["layers"] for v in Wl.values()])
    t_ = torch.tensor(np.append(flat, loss) / world, dtype=torch.float64)   # -> 1/(B s) of the global batch
    dist.all_reduce(t_)
    q.put((rank, t_.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_data_parallel_gradient_sum(world):
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_dp, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(world)), key=lambda x: x[0])
    for p in ps:
        p.join(60)
    shape = gen.TINY
    W = gen.model_weights(shape, seed=42, dtype="fp32")
    tok = gen.tokens(2 * world, shape.s, shape.V, seed=1234)
    loss, g = M.batch_fwd_bwd(W, tok, shape.a, 2 * world)
    ref = np.append(np.concatenate([g["emb"].ravel()] + [v.ravel() for Wl in g["layers"] for v in Wl.values()]), loss)
    for _, got in out:
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15 * np.abs(ref).max())
