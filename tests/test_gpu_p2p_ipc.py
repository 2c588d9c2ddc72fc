"""Peer-memory exchange across PROCESSES (CUDA IPC handles exchanged over a gloo
process group, epoch flags released / acquired at system scope), with two rank
processes sharing the one GPU of the test box: outputs and EF bit-identical to the
W-rank oracle.  (On a multi-GPU box the same calls go over NVLink.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layers():
    sizes = [(1, 1), (127, 1), (129, 1), (77, 0), (4097, 1), (300, 1), (12800, 1)]
    out, off = [], 0
    for n, c in sizes:
        out.append(W.Layer(off, n, 0, 0, c))
        off += n
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2210_17357_b200 import lgreco
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers = _layers()
        ctx = lg = None
        ctx = lgreco.Context(layers, lgreco.QSGD, W.QSGD_BITS, seed=99, rank=rank, world=world)
        blobs = [None] * world
        dist.all_gather_object(blobs, ctx.p2p_export())
        ctx.p2p_open(blobs)
        dist.barrier()
        g, e = W.gaussian_outliers(layers, seed=W.rank_seed(13, rank))
        gd = torch.from_numpy(g).cuda()
        ed = torch.from_numpy(e).cuda()
        out = torch.empty_like(gd)
        # plan agreement over peer memory: each rank proposes a plan, rank 0's is used
        prop = [(2 if rank == 0 else 5) if l.compress else -1 for l in layers]
        d_choice = torch.tensor(prop, dtype=torch.int32, device="cuda")
        ctx.plan_broadcast(d_choice)
        ctx.compress_allreduce_dev(d_choice, gd, ed, out, 4)
        torch.cuda.synchronize()
        ctx.check()
        q.put((rank, out.cpu().numpy().tobytes(), ed.cpu().numpy().tobytes()))
        dist.barrier()  # peers' windows stay mapped until everyone is done
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_p2p_exchange_two_processes(ref):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, e2 = q.get(timeout=300)
        res[r] = (out, e2)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    layers = _layers()
    lbits = [W.QSGD_BITS[2] if l.compress else 0 for l in layers]
    gs, es = zip(*[W.gaussian_outliers(layers, seed=W.rank_seed(13, r)) for r in range(world)])
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, list(gs), list(es), B=128, seed=99, step=4)
    for r in range(world):
        assert res[r][0] == out_ref.tobytes()
        assert res[r][1] == es_ref[r].tobytes()
