"""World-size-2 CPU (gloo) coverage of the N > 1 host path: plan agreement (rank 0's
plan is broadcast), identical byte-balanced shard bounds from the C-ABI host layout on
every rank, and the exchange choreography (all-to-all of stage-1 shards, owner
reduce, all-gather of stage-2 shards) reproducing the single-process W-rank result
bit for bit.  The per-record arithmetic here is the oracle's (no GPU in this
container); the GPU kernels for the same steps are parity-tested in test_gpu_qsgd.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_17357_b200 import workloads as W


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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ref
        from paper_2210_17357_b200 import lgreco
        bits = W.QSGD_BITS
        layers = _layers()
        seed, step, B = 11, 3, 128
        # plan agreement: every rank proposes a different plan, rank 0's wins
        rng = np.random.default_rng(100 + rank)
        choice = torch.tensor([int(rng.integers(0, len(bits))) if l.compress else -1 for l in layers],
                              dtype=torch.int32)
        dist.broadcast(choice, src=0)
        choice = choice.tolist()
        lbits = [bits[c] if l.compress else 0 for c, l in zip(choice, layers)]
        S, rb, bb = lgreco.plan_layout(layers, lgreco.QSGD, bits, choice, world, qbucket=B)
        allb = [None] * world
        dist.all_gather_object(allb, (S, rb, bb))
        assert all(x == allb[0] for x in allb)
        rb_ref, bb_ref = ref.shard_bounds(layers, lbits, B, world)
        assert list(rb) == list(rb_ref) and list(bb) == list(bb_ref)
        # stage 1 on this rank
        g, e = W.gaussian_outliers(layers, seed=W.rank_seed(7, rank))
        pay1, e2, _ = ref.qsgd_pack(layers, lbits, g, e, B=B, seed=seed, rank=rank, step=step)
        # all-to-all of shards: shard j -> rank j (equal-size transport buffers, padded)
        mx = max(bb[j + 1] - bb[j] for j in range(world))
        send = torch.zeros(world, mx, dtype=torch.uint8)
        for j in range(world):
            send[j, :bb[j + 1] - bb[j]] = torch.from_numpy(pay1[bb[j]:bb[j + 1]].copy())
        recv = torch.zeros(world, mx, dtype=torch.uint8)
        reqs = []
        for j in range(world):
            if j == rank:
                recv[j] = send[j]
            else:
                reqs.append(dist.isend(send[j].contiguous(), dst=j))
                reqs.append(dist.irecv(recv[j], src=j))
        for r in reqs:
            r.wait()
        mine = bb[rank + 1] - bb[rank]
        recv_c = recv[:, :mine].contiguous().numpy().reshape(-1)
        pay2 = np.zeros(S, np.uint8)
        ref.qsgd_reduce_shard(layers, lbits, B, seed, step, world, recv_c, rb[rank], rb[rank + 1], bb[rank], mine,
                              pay2)
        # all-gather of stage-2 shards
        mine_t = torch.zeros(mx, dtype=torch.uint8)
        mine_t[:mine] = torch.from_numpy(pay2[bb[rank]:bb[rank + 1]].copy())
        gath = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gath, mine_t)
        full = np.zeros(S, np.uint8)
        for j in range(world):
            full[bb[j]:bb[j + 1]] = gath[j][:bb[j + 1] - bb[j]].numpy()
        out = ref.qsgd_unpack(layers, lbits, full, W.total_numel(layers), B=B)
        q.put((rank, choice, out.tobytes(), e2.tobytes(), full.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_qsgd_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, choice, out, e2, full = q.get(timeout=240)
        res[r] = (choice, out, e2, full)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import ref
    layers = _layers()
    choice = res[0][0]
    assert all(res[r][0] == choice for r in res)
    lbits = [W.QSGD_BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    gs, es = zip(*[W.gaussian_outliers(layers, seed=W.rank_seed(7, r)) for r in range(world)])
    out_ref, es_ref, _, p2_ref = ref.qsgd_allreduce(layers, lbits, list(gs), list(es), B=128, seed=11, step=3)
    for r in range(world):
        assert res[r][1] == out_ref.tobytes()          # identical on every rank, = W-rank oracle
        assert res[r][2] == es_ref[r].tobytes()
        assert res[r][3] == p2_ref.tobytes()
