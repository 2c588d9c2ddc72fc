"""NEXT-4 mixed-family compression: one context per family on the same
layer table, a joint (family, parameter) plan, per-layer dispatch with CHOICE_SKIP.
Every layer's output and EF must equal its own family's oracle (QSGD / TopK bitwise,
PowerSGD 1e-5 normwise); the joint table and its solve equal the oracle's."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu

BITS, PPM, RANKS = [2, 4, 8], [10000, 100000], [1, 4]
SEED = 21


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    return lgreco


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _layers():
    shapes = [(40, 30, 1), (0, 17, 0), (64, 200, 1), (130, 70, 1), (0, 999, 1), (257, 96, 1), (33, 33, 1)]
    out, off = [], 0
    for m, k, c in shapes:
        n = m * k if m else k
        out.append(W.Layer(off, n, m, k if m else 0, c))
        off += n
    return out


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / max(np.linalg.norm(b), 1e-300)


def _oracle(ref, layers, fam, par, g, e, step):
    """Compose the families' oracles: layer l's out / EF from the oracle of fam[l]."""
    L = len(layers)
    lbits = [BITS[par[l]] if fam[l] == 0 and layers[l].compress else 0 for l in range(L)]
    oq, eq, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e.copy()], seed=SEED, step=step)
    lppm = [PPM[par[l]] if fam[l] == 1 else (1000000 if layers[l].compress else 0) for l in range(L)]
    ot, et, _ = ref.topk_allreduce(layers, lppm, [g], [e.copy()])
    lrank = [RANKS[par[l]] if fam[l] == 2 else 0 for l in range(L)]
    Qs = {}
    for l, ly in enumerate(layers):
        r = lrank[l]
        if r and ly.rows and not ref.psgd_lossless(ly.rows, ly.cols, r):
            Qs[l] = ref.psgd_init_q(SEED, l, step, ly.cols, r)
    op, ep, _ = ref.psgd_allreduce(layers, lrank, [g], [e.copy()], Qs)
    return (oq, eq[0]), (ot, et[0]), (op, ep[0]), Qs


@pytest.mark.parametrize("mode", ["fixed", "solved"])
def test_hybrid_plan_dispatch(lg, ref, mode):
    from paper_2210_17357_b200.hybrid import Hybrid
    layers = _layers()
    L = len(layers)
    g, e = W.low_rank_plus_noise(layers, seed=3, with_ef=True)
    h = Hybrid(layers, [(lg.QSGD, BITS), (lg.TOPK, PPM), (lg.POWERSGD, RANKS)], seed=SEED, default_family=0,
               default_idx=1)
    gd, ed = _dev(g), _dev(e)
    err, bits = h.profile(gd, ed, 0)
    # the joint table is the families' tables side by side
    ks = [len(BITS), len(PPM), len(RANKS)]
    eq, bq = ref.qsgd_profile(layers, g, e, BITS, seed=SEED, step=0)
    assert np.array_equal(bits.cpu().numpy()[:, :ks[0]], bq)
    if mode == "fixed":  # every family owns some layers
        fam = [0, 0, 1, 2, 1, 0, 2]
        par = [1, 0, 1, 1, 0, 2, 0]
        cols = [(h.col0[f] + p) if layers[l].compress else -1 for l, (f, p) in enumerate(zip(fam, par))]
        choice = torch.tensor(cols, dtype=torch.int32, device="cuda")
    else:
        comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device="cuda")
        choice, info = h.solve(err, bits, comp)
        dflt = np.full(L, h.default_col, np.int32)
        st, c_ref, _ = ref.solve(err.cpu().numpy(), bits.cpu().numpy(), dflt, comp.cpu().numpy(), D=10000)
        assert list(choice.cpu().numpy()) == list(c_ref)
        cols = list(c_ref)
        fam, par = [], []
        for c in cols:
            f = 0 if c < 0 else max(i for i in range(3) if c >= h.col0[i])
            fam.append(f)
            par.append(0 if c < 0 else c - h.col0[f])
    out = torch.empty_like(gd)
    h.compress_allreduce(choice, gd, ed, out, 0)
    h.check()
    (oq, eqs), (ot, ets), (op, eps), Qs = _oracle(ref, layers, fam, par, g, e, 0)
    o, ef = out.cpu().numpy(), ed.cpu().numpy()
    for l, ly in enumerate(layers):
        sl = slice(ly.offset, ly.offset + ly.numel)
        if not ly.compress:
            assert np.array_equal(o[sl].view(np.uint32), oq[sl].view(np.uint32)) and not ef[sl].any()
        elif fam[l] == 0:
            assert np.array_equal(o[sl].view(np.uint32), oq[sl].view(np.uint32)), l
            assert np.array_equal(ef[sl].view(np.uint32), eqs[sl].view(np.uint32)), l
        elif fam[l] == 1:
            assert np.array_equal(o[sl].view(np.uint32), ot[sl].view(np.uint32)), l
            assert np.array_equal(ef[sl].view(np.uint32), ets[sl].view(np.uint32)), l
        else:
            assert _rel(o[sl], op[sl]) <= 1e-5, l
            assert _rel(ef[sl], eps[sl]) <= 1e-5, l
    h.close()


@pytest.mark.parametrize("Wn", [2, 3])
def test_hybrid_exchange_simulated_ranks(lg, ref, Wn):
    """NEXT-4 at W > 1 (R24): each family's exchange carries only its own layers -- a
    CHOICE_SKIP layer has no QSGD records and no TopK pairs, its output and EF are left
    untouched -- and every own layer's mean gradient and EF equal the family's W-rank
    oracle.  W ranks simulated through the stage entry points (QSGD: pack per rank,
    byte-balanced shards of the ctx's own payload, owner reduce, decode; TopK: pack per
    rank, all-gather as a concatenation, combine)."""
    from paper_2210_17357_b200.hybrid import Hybrid
    layers = _layers()
    L = len(layers)
    fam = [0, 0, 1, 2, 1, 0, 2]
    par = [1, 0, 1, 1, 0, 2, 0]
    h = Hybrid(layers, [(lg.QSGD, BITS), (lg.TOPK, PPM), (lg.POWERSGD, RANKS)], seed=SEED)
    cols = [(h.col0[f] + p) if layers[l].compress else -1 for l, (f, p) in enumerate(zip(fam, par))]
    per = lg.hybrid_split(torch.tensor(cols, dtype=torch.int32, device="cuda"), h.Ks)
    chq, cht = per[0].cpu().tolist(), per[1].cpu().tolist()
    assert lg.CHOICE_SKIP in chq and lg.CHOICE_SKIP in cht
    gs, es = [], []
    for w in range(Wn):
        g, e = W.low_rank_plus_noise(layers, seed=30 + w, with_ef=True)
        gs.append(g)
        es.append(e)
    step = 4
    # the families' oracles (other families' layers given any valid parameter: a layer's
    # exchange result does not depend on the others')
    lbits = [BITS[par[l]] if fam[l] == 0 and layers[l].compress else (2 if layers[l].compress else 0)
             for l in range(L)]
    oq, eq, _, _ = ref.qsgd_allreduce(layers, lbits, gs, [e.copy() for e in es], seed=SEED, step=step)
    lppm = [PPM[par[l]] if fam[l] == 1 else (1000000 if layers[l].compress else 0) for l in range(L)]
    ot, et, _ = ref.topk_allreduce(layers, lppm, gs, [e.copy() for e in es])
    sentinel = 7.0
    # ---- QSGD family
    ctx = h.ctxs[0]
    S = ctx.payload_bytes(chq)
    rb, bb = ctx.shard_bounds(chq, Wn)
    pays, eds = [], []
    for w in range(Wn):
        pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
        ed = _dev(es[w])
        ctx.qsgd_pack(chq, _dev(gs[w]), ed, pay, None, w, step)
        pays.append(pay)
        eds.append(ed)
    stage2 = torch.zeros(S, dtype=torch.uint8, device="cuda")
    for j in range(Wn):
        nbytes = bb[j + 1] - bb[j]
        recv = torch.cat([pays[w][bb[j]:bb[j + 1]] for w in range(Wn)]) if nbytes else \
            torch.zeros(1, dtype=torch.uint8, device="cuda")
        ctx.qsgd_reduce(chq, Wn, rb[j], rb[j + 1], recv.contiguous(), stage2, step)
    outq = torch.full((len(gs[0]),), sentinel, dtype=torch.float32, device="cuda")
    ctx.qsgd_unpack(chq, stage2, outq)
    # ---- TopK family
    ctx = h.ctxs[1]
    St = ctx.payload_bytes(cht)
    tp, ets = [], []
    for w in range(Wn):
        pay = torch.zeros(St, dtype=torch.uint8, device="cuda")
        ed = _dev(es[w])
        ctx.topk_pack(cht, _dev(gs[w]), ed, pay, None)
        tp.append(pay)
        ets.append(ed)
    outt = torch.full((len(gs[0]),), sentinel, dtype=torch.float32, device="cuda")
    ctx.topk_combine(cht, Wn, torch.cat(tp).contiguous(), outt)
    torch.cuda.synchronize()
    h.check()
    o_q, o_t = outq.cpu().numpy(), outt.cpu().numpy()
    for l, ly in enumerate(layers):
        sl = slice(ly.offset, ly.offset + ly.numel)
        # QSGD ctx: family 0's layers (and the lossless ones) exchanged, the rest untouched
        if chq[l] == lg.CHOICE_SKIP:
            assert np.all(o_q[sl] == sentinel), l
            for w in range(Wn):
                assert np.array_equal(eds[w].cpu().numpy()[sl].view(np.uint32), es[w][sl].view(np.uint32)), l
        else:
            assert np.array_equal(o_q[sl].view(np.uint32), oq[sl].view(np.uint32)), l
            for w in range(Wn):
                assert np.array_equal(eds[w].cpu().numpy()[sl].view(np.uint32), eq[w][sl].view(np.uint32)), l
        if cht[l] == lg.CHOICE_SKIP:
            assert np.all(o_t[sl] == sentinel), l
            for w in range(Wn):
                assert np.array_equal(ets[w].cpu().numpy()[sl].view(np.uint32), es[w][sl].view(np.uint32)), l
        elif fam[l] == 1:
            assert np.array_equal(o_t[sl].view(np.uint32), ot[sl].view(np.uint32)), l
            for w in range(Wn):
                assert np.array_equal(ets[w].cpu().numpy()[sl].view(np.uint32), et[w][sl].view(np.uint32)), l
    h.close()
