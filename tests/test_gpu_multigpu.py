"""Multi-GPU exchange: W = 2, 4, 8 rank
processes, one per GPU, NCCL process group -- QSGD over peer memory (CUDA IPC over
NVLink, epoch flags) and over NCCL (grouped send/recv all-to-all + all-gather), TopK
(NCCL all-gather + ordered sparse sum), PowerSGD (two NCCL all-reduces, two steps with
the warm start) and the plan agreement (every rank proposes its own plan; rank 0's
wins).  Every rank's output and EF are checked against the W-rank oracle: bit-exact for
QSGD and TopK, 1e-5 normwise for PowerSGD.  Skipped below 2 GPUs (the test box has
one; the driver's 8-GPU runs collect it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2210_17357_b200 import workloads as W

# LG_MULTI_ONE_DEVICE=1 (harness check on a one-GPU box): every rank on cuda:0 with a
# gloo group; only the peer-memory mode runs (NCCL refuses two ranks on one device)
ONE_DEV = os.environ.get("LG_MULTI_ONE_DEVICE") == "1"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ONE_DEV and (not torch.cuda.is_available() or torch.cuda.device_count() < 2),
                                 reason="needs >= 2 GPUs")]

PPM = [1000, 10000, 100000, 1000000]
RANKS = [1, 2, 4, 8]
SEED = 99


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _vec_layers():
    sizes = [(1, 1), (127, 1), (129, 1), (77, 0), (4097, 1), (300, 1), (12800, 1), (65536, 1)]
    out, off = [], 0
    for n, c in sizes:
        out.append(W.Layer(off, n, 0, 0, c))
        off += n
    return out


def _mat_layers():
    shapes = [(40, 30, 1), (0, 17, 0), (64, 200, 1), (130, 70, 1), (257, 96, 1)]
    out, off = [], 0
    for m, k, c in shapes:
        n = m * k if m else k
        out.append(W.Layer(off, n, m, k if m else 0, c))
        off += n
    return out


def _inputs(fam, layers, rank, step):
    if fam == "topk":
        return W.heavy_tailed(layers, seed=W.rank_seed(31 + 7 * step, rank), sparse_rows_layer=None)
    if fam == "psgd":
        return W.low_rank_plus_noise(layers, seed=W.rank_seed(41 + 7 * step, rank), with_ef=True)
    return W.gaussian_outliers(layers, seed=W.rank_seed(13 + 7 * step, rank))


def _worker(rank, world, port, fam, mode, q):
    import torch.distributed as dist
    from paper_2210_17357_b200 import lgreco
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0 if ONE_DEV else rank)
    torch.cuda.set_device(dev)
    if ONE_DEV:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        layers = _mat_layers() if fam == "psgd" else _vec_layers()
        family, params = {"qsgd": (lgreco.QSGD, W.QSGD_BITS), "topk": (lgreco.TOPK, PPM),
                          "psgd": (lgreco.POWERSGD, RANKS)}[fam]
        if mode.startswith("p2p"):
            ctx = lgreco.Context(layers, family, params, seed=SEED, rank=rank, world=world)
            blobs = [None] * world
            dist.all_gather_object(blobs, ctx.p2p_export())
            ctx.p2p_open(blobs)
        else:
            obj = [lgreco.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx = lgreco.Context(layers, family, params, seed=SEED, rank=rank, world=world, nccl_id=obj[0])
        dist.barrier()
        _, e0 = _inputs(fam, layers, rank, 0)
        ed = torch.from_numpy(e0).to(dev)
        res = []
        for step in range(2):
            g, _ = _inputs(fam, layers, rank, step)
            gd = torch.from_numpy(g).to(dev)
            out = torch.empty_like(gd)
            # every rank proposes its own plan; the plan agreement makes rank 0's the plan
            prop = [((step + 2 * rank + li) % len(params)) if l.compress else -1 for li, l in enumerate(layers)]
            d_choice = torch.tensor(prop, dtype=torch.int32, device=dev)
            ctx.plan_broadcast(d_choice)
            errn = None
            if fam == "qsgd" and mode.endswith("_pc"):
                # the pipelined schedule's per-step call: profile of this rank's x + the
                # compressed exchange with the plan in force
                err = torch.empty(len(layers), len(params), dtype=torch.float64, device=dev)
                bits = torch.empty(len(layers), len(params), dtype=torch.int64, device=dev)
                ctx.profile_compress(d_choice, gd, ed, out, step, err, bits)
                errn = err.cpu().numpy()
            elif fam == "qsgd":
                ctx.compress_allreduce_dev(d_choice, gd, ed, out, step)
            else:
                ctx.compress_allreduce(d_choice.cpu().tolist(), gd, ed, out, step)
            torch.cuda.synchronize(dev)
            ctx.check()
            res.append((d_choice.cpu().numpy(), out.cpu().numpy(), ed.cpu().numpy(), errn))
        ctx.close()
        q.put((rank, res, None))
    except Exception as ex:  # reported to the parent
        q.put((rank, None, repr(ex)))
    finally:
        dist.destroy_process_group()


def _run(world, fam, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fam, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, res, err = q.get(timeout=600)
        assert err is None, (r, err)
        got[r] = res
    for p in procs:
        p.join(timeout=120)
    return got


def _worlds(mode="nccl"):
    if ONE_DEV:
        return [2, 4] if mode == "p2p" else []
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    return [w for w in (2, 4, 8) if w <= n]


@pytest.mark.parametrize("mode", ["p2p", "nccl", "p2p_pc", "nccl_pc"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_qsgd_exchange_multi_gpu(ref, world, mode):
    """mode p2p_pc: the per-step call of the pipelined schedule (lgreco_profile_compress)
    -- every rank's profile of its own x as well (rankfield = rank, R3)."""
    if world not in _worlds(mode.replace("_pc", "")):
        pytest.skip(f"needs {world} GPUs")
    got = _run(world, "qsgd", mode)
    layers = _vec_layers()
    es = [_inputs("qsgd", layers, w, 0)[1] for w in range(world)]
    for step in range(2):
        plan0 = [((step + li) % len(W.QSGD_BITS)) if l.compress else -1 for li, l in enumerate(layers)]
        gs = [_inputs("qsgd", layers, w, step)[0] for w in range(world)]
        lbits = [W.QSGD_BITS[c] if c >= 0 else 0 for c in plan0]
        if mode.endswith("_pc"):
            for w in range(world):
                rerr, _ = ref.qsgd_profile(layers, gs[w], es[w], W.QSGD_BITS, seed=SEED, rank=w, step=step)
                gerr = got[w][step][3]
                assert np.all((rerr == 0) == (gerr == 0))
                assert (np.abs(gerr - rerr) / np.maximum(rerr, 1e-300)).max() <= 1e-5, (w, step)
        out_ref, es, _, _ = ref.qsgd_allreduce(layers, lbits, gs, es, seed=SEED, step=step)
        for w in range(world):
            choice, out, ef, _ = got[w][step]
            assert list(choice) == plan0
            assert np.array_equal(out.view(np.uint32), out_ref.view(np.uint32)), (w, step)
            assert np.array_equal(ef.view(np.uint32), es[w].view(np.uint32)), (w, step)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_topk_exchange_multi_gpu(ref, world):
    if world not in _worlds():
        pytest.skip(f"needs {world} GPUs")
    got = _run(world, "topk", "nccl")
    layers = _vec_layers()
    es = [_inputs("topk", layers, w, 0)[1] for w in range(world)]
    for step in range(2):
        plan0 = [((step + li) % len(PPM)) if l.compress else -1 for li, l in enumerate(layers)]
        gs = [_inputs("topk", layers, w, step)[0] for w in range(world)]
        lppm = [PPM[c] if c >= 0 else 0 for c in plan0]
        out_ref, es, _ = ref.topk_allreduce(layers, lppm, gs, es)
        for w in range(world):
            choice, out, ef, _ = got[w][step]
            assert list(choice) == plan0
            assert np.array_equal(out.view(np.uint32), out_ref.view(np.uint32)), (w, step)
            assert np.array_equal(ef.view(np.uint32), es[w].view(np.uint32)), (w, step)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_psgd_exchange_multi_gpu(ref, world):
    if world not in _worlds():
        pytest.skip(f"needs {world} GPUs")
    got = _run(world, "psgd", "nccl")
    layers = _mat_layers()
    es = [_inputs("psgd", layers, w, 0)[1] for w in range(world)]
    Qs, last = {}, {}
    for step in range(2):
        plan0 = [((step + li) % len(RANKS)) if l.compress else -1 for li, l in enumerate(layers)]
        lrank = [RANKS[c] if c >= 0 else 0 for c in plan0]
        for l, ly in enumerate(layers):  # warm start re-initialised when a layer's rank changes (R12)
            r = lrank[l]
            if r and ly.rows and not ref.psgd_lossless(ly.rows, ly.cols, r):
                if last.get(l) != r:
                    Qs[l] = ref.psgd_init_q(SEED, l, step, ly.cols, r)
            else:
                Qs.pop(l, None)
            last[l] = r
        gs = [_inputs("psgd", layers, w, step)[0] for w in range(world)]
        out_ref, es, _ = ref.psgd_allreduce(layers, lrank, gs, es, Qs)
        for w in range(world):
            choice, out, ef, _ = got[w][step]
            assert list(choice) == plan0
            for l, ly in enumerate(layers):
                sl = slice(ly.offset, ly.offset + ly.numel)
                if l in Qs:
                    assert _rel(out[sl], out_ref[sl]) <= 1e-5, (w, step, l)
                    assert _rel(ef[sl], es[w][sl]) <= 1e-5, (w, step, l)
                else:
                    assert np.array_equal(out[sl].view(np.uint32), out_ref[sl].view(np.uint32)), (w, step, l)
