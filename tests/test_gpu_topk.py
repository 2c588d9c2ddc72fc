"""GPU parity for the TopK rows (a3 profile, a8 select + EF, a9-a10 exchange) vs the
oracle: bit-exact pairs / EF / outputs, 1e-5 relative error norms."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu

PPM = [1000, 5000, 10000, 50000, 100000, 250000, 1000000]


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    return lgreco


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _layers():
    sizes = [(1, 1), (7, 1), (300, 1), (77, 0), (4096, 1), (20001, 1), (50, 0), (70000, 1), (3, 1)]
    out, off = [], 0
    for n, c in sizes:
        out.append(W.Layer(off, n, 0, 0, c))
        off += n
    return out


def _data(layers, seed):
    g, e = W.heavy_tailed(layers, seed=seed, sparse_rows_layer=None)
    rng = np.random.default_rng(seed)
    # ties and zeros: a run of equal magnitudes with both signs, a block of zeros
    l = layers[4]
    g[l.offset:l.offset + 600] = np.where(rng.random(600) < 0.5, 0.125, -0.125).astype(np.float32)
    e[l.offset:l.offset + 600] = 0.0
    l = layers[5]
    g[l.offset:l.offset + 15000] = 0.0
    e[l.offset:l.offset + 15000] = 0.0
    return g, e


@pytest.mark.parametrize("seed", [0, 1])
def test_profile_parity(lg, ref, seed):
    layers = _layers()
    g, e = _data(layers, seed)
    ctx = lg.Context(layers, lg.TOPK, PPM)
    L, K = len(layers), len(PPM)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), _dev(e), 0, err, bits)
    rerr, rbits = ref.topk_profile(layers, g, e, PPM)
    assert np.array_equal(bits.cpu().numpy(), rbits)
    ge = err.cpu().numpy()
    assert np.all((rerr == 0) == (ge == 0))
    rel = np.abs(ge - rerr) / np.maximum(rerr, 1e-300)
    assert rel.max() <= 1e-5, rel.max()


def test_profile_paper_mode_and_row_sparse(lg, ref):
    # paper mode (EF = NULL), a row-sparse "embedding" matrix (90% zero rows)
    layers = [W.Layer(0, 2000 * 64, 2000, 64, 1), W.Layer(128000, 512, 0, 0, 0), W.Layer(128512, 64 * 300, 64, 300, 1)]
    g, _ = W.heavy_tailed(layers, seed=4, with_ef=False, sparse_rows_layer=0)
    ppm = [1000 * i for i in range(1, 101)]  # 0.1% .. 10% (C3 candidate set)
    ctx = lg.Context(layers, lg.TOPK, ppm)
    err = torch.empty(3, 100, dtype=torch.float64, device="cuda")
    bits = torch.empty(3, 100, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), None, 0, err, bits)
    rerr, rbits = ref.topk_profile(layers, g, None, ppm)
    assert np.array_equal(bits.cpu().numpy(), rbits)
    ge = err.cpu().numpy()
    rel = np.abs(ge - rerr) / np.maximum(rerr, 1e-300)
    assert rel.max() <= 1e-5


@pytest.mark.parametrize("seed", [0, 3])
def test_pack_parity(lg, ref, seed):
    layers = _layers()
    g, e = _data(layers, seed)
    rng = np.random.default_rng(seed)
    choice = [int(rng.integers(0, len(PPM))) if l.compress else -1 for l in layers]
    lppm = [PPM[c] if l.compress else 0 for c, l in zip(choice, layers)]
    ctx = lg.Context(layers, lg.TOPK, PPM)
    S = ctx.payload_bytes(choice)
    pay_ref, e_ref = ref.topk_pack(layers, lppm, g, e)
    assert S == pay_ref.size
    gd, ed = _dev(g), _dev(e)
    pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(gd)
    ctx.topk_pack(choice, gd, ed, pay, out)
    torch.cuda.synchronize()
    assert np.array_equal(pay.cpu().numpy(), pay_ref)
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), e_ref.view(np.uint32))
    out_ref, _, _ = ref.topk_allreduce(layers, lppm, [g], [e])
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))
    ctx.check()


@pytest.mark.parametrize("Wn", [1, 2, 4, 8])
def test_exchange_simulated_ranks(lg, ref, Wn):
    layers = _layers()
    rng = np.random.default_rng(10 + Wn)
    choice = [int(rng.integers(0, len(PPM))) if l.compress else -1 for l in layers]
    lppm = [PPM[c] if l.compress else 0 for c, l in zip(choice, layers)]
    gs, es = [], []
    for w in range(Wn):
        g, e = _data(layers, 50 + w)
        gs.append(g)
        es.append(e)
    out_ref, es_ref, pays_ref = ref.topk_allreduce(layers, lppm, gs, es)
    ctx = lg.Context(layers, lg.TOPK, PPM)
    S = ctx.payload_bytes(choice)
    pays = []
    for w in range(Wn):
        pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
        ed = _dev(es[w])
        ctx.topk_pack(choice, _dev(gs[w]), ed, pay, None)
        assert np.array_equal(pay.cpu().numpy(), pays_ref[w])
        assert np.array_equal(ed.cpu().numpy().view(np.uint32), es_ref[w].view(np.uint32))
        pays.append(pay)
    gathered = torch.cat(pays).contiguous()
    out = torch.empty(len(gs[0]), dtype=torch.float32, device="cuda")
    ctx.topk_combine(choice, Wn, gathered, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))


def test_compress_allreduce_w1_and_nonfinite(lg, ref):
    layers = _layers()
    g, e = _data(layers, 7)
    choice = [2 if l.compress else -1 for l in layers]
    lppm = [PPM[2] if l.compress else 0 for l in layers]
    ctx = lg.Context(layers, lg.TOPK, PPM)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, ed, out, 0)
    out_ref, es_ref, _ = ref.topk_allreduce(layers, lppm, [g], [e])
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), es_ref[0].view(np.uint32))
    g[layers[4].offset + 5] = np.inf
    ctx.compress_allreduce(choice, _dev(g), _dev(e), out, 0)
    with pytest.raises(lg.LGrecoError):
        ctx.check()


def test_c3_sampled_full_size(lg, ref):
    """C3 (Transformer-XL, 191.9M fp32) at full size in the bench launch configuration;
    the oracle checks a sample of layers (the others are profiled but not compared)."""
    layers = W.config_layers("C3")
    g, e = W.heavy_tailed(layers, seed=W.rank_seed(0x5EED, 0))
    ppm = W.TOPK_PPM_C3
    ctx = lg.Context(layers, lg.TOPK, ppm)
    L, K = len(layers), len(ppm)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    gd, ed = _dev(g), _dev(e)
    ctx.profile(gd, ed, 0, err, bits)
    ge, gb = err.cpu().numpy(), bits.cpu().numpy()
    sample = [i for i, l in enumerate(layers) if l.compress][1:7] + [len(layers) - 1]
    sub = [W.Layer(l.offset, l.numel, l.rows, l.cols, l.compress if i in sample else 0) for i, l in enumerate(layers)]
    rerr, rbits = ref.topk_profile(sub, g, e, ppm)
    for i in sample:
        assert np.array_equal(gb[i], rbits[i])
        assert (np.abs(ge[i] - rerr[i]) / np.maximum(rerr[i], 1e-300)).max() <= 1e-5
    # compress with the default 1% and compare the sampled layers' EF bitwise
    choice = [ppm.index(10000) if l.compress else -1 for l in layers]
    out = torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, ed, out, 0)
    lppm = [10000 if l.compress else 0 for l in sub]
    out_ref, es_ref, _ = ref.topk_allreduce(sub, lppm, [g], [e])
    oc, ec = out.cpu().numpy(), ed.cpu().numpy()
    for i in sample:
        l = layers[i]
        sl = slice(l.offset, l.offset + l.numel)
        assert np.array_equal(oc[sl].view(np.uint32), out_ref[sl].view(np.uint32))
        assert np.array_equal(ec[sl].view(np.uint32), es_ref[0][sl].view(np.uint32))


def test_compress_allreduce_dev_matches_host_path(lg):
    layers = _layers()
    g, e = _data(layers, 21)
    choice = [3 if l.compress else -1 for l in layers]
    ctx = lg.Context(layers, lg.TOPK, PPM)
    gd = _dev(g)
    e1, e2 = _dev(e), _dev(e)
    o1, o2 = torch.empty_like(gd), torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, e1, o1, 0)
    ctx.compress_allreduce_dev(torch.tensor(choice, dtype=torch.int32, device="cuda"), gd, e2, o2, 0)
    assert torch.equal(o1.view(torch.int32), o2.view(torch.int32)) and torch.equal(e1.view(torch.int32), e2.view(torch.int32))


@pytest.mark.parametrize("seed", [0, 1])
def test_compress_reuses_profile_thresholds(lg, ref, seed):
    """A compress of the same x right after the profile (same g / e pointers and step)
    takes the profile's per-layer thresholds instead of selecting again: outputs and EF
    bit-identical to a compress without a preceding profile and to the oracle, with the
    tie-heavy layers (600 equal magnitudes, 15000 zeros) where only some ties are kept."""
    layers = _layers()
    g, e = _data(layers, seed)
    L, K = len(layers), len(PPM)
    rng = np.random.default_rng(40 + seed)
    choice = [int(rng.integers(0, K)) if l.compress else -1 for l in layers]
    lppm = [PPM[c] if l.compress else 0 for c, l in zip(choice, layers)]
    out_ref, es_ref, _ = ref.topk_allreduce(layers, lppm, [g], [e])
    res = []
    for with_profile in (True, False):
        ctx = lg.Context(layers, lg.TOPK, PPM)
        gd, ed = _dev(g), _dev(e)
        if with_profile:
            err = torch.empty(L, K, dtype=torch.float64, device="cuda")
            bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
            ctx.profile(gd, ed, 5, err, bits)
        out = torch.empty_like(gd)
        ctx.compress_allreduce_dev(torch.tensor(choice, dtype=torch.int32, device="cuda"), gd, ed, out, 5)
        ctx.check()
        res.append((out.cpu().numpy(), ed.cpu().numpy()))
        ctx.close()
    for out, ef in res:
        assert np.array_equal(out.view(np.uint32), out_ref.view(np.uint32))
        assert np.array_equal(ef.view(np.uint32), es_ref[0].view(np.uint32))


def test_no_payload_compress_after_payload_compress(lg, ref):
    """A W = 1 compress without payload skips the count / scan of layers keeping every
    tie at T or none (their chunk offsets are not needed); its write pass must not read
    the offsets a preceding payload-writing call left behind (regression: the last tie of
    a layer was dropped in the hybrid test).  Continuous layers have ties = r = 1."""
    layers = _layers()
    L, K = len(layers), len(PPM)
    ctx = lg.Context(layers, lg.TOPK, PPM)
    for it, seed in enumerate((31, 32, 33)):
        g, e = W.heavy_tailed(layers, seed=seed, sparse_rows_layer=None)
        rng = np.random.default_rng(seed)
        choice = [int(rng.integers(0, K)) if l.compress else -1 for l in layers]
        lppm = [PPM[c] if l.compress else 0 for c, l in zip(choice, layers)]
        gd = _dev(g)
        # payload-writing pack first (fills the chunk offsets), on a copy of the EF
        S = ctx.payload_bytes(choice)
        pay = torch.zeros(max(S, 16), dtype=torch.uint8, device="cuda")
        ctx.topk_pack(choice, gd, _dev(e), pay, None)
        ed = _dev(e)
        out = torch.empty_like(gd)
        ctx.compress_allreduce_dev(torch.tensor(choice, dtype=torch.int32, device="cuda"), gd, ed, out, 100 + it)
        ctx.check()
        out_ref, es_ref, _ = ref.topk_allreduce(layers, lppm, [g], [e])
        assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32)), it
        assert np.array_equal(ed.cpu().numpy().view(np.uint32), es_ref[0].view(np.uint32)), it
    ctx.close()
