"""GPU parity of the fused per-step pass lgreco_profile_compress (K1 with K5's compress
folded in, include/lgreco.h): err / bits against the oracle's profile (1e-5, bits
exact), out and the new EF bitwise against the oracle's compress of the same x with
the plan in force, and bitwise against the library's own two-call definition.  Then the
pipelined chain of the paper's schedule: the plan that compresses
step t is the one solved from the profile of step t - lag, checked step by step against
the oracle chain (oracle profile -> oracle solve -> oracle compress)."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu

BITS = W.QSGD_BITS


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    assert torch.cuda.is_available()
    return lgreco


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _edge_layers():
    sizes = [(1, 1), (3, 1), (127, 1), (128, 1), (129, 1), (1000, 1), (4097, 1), (77, 0), (12800, 1), (5, 1),
             (513, 1), (2048, 0), (65536 + 3, 1)]
    out, off = [], 0
    for n, c in sizes:
        out.append(W.Layer(off, n, 0, 0, c))
        off += n
    return out


def _edge_data(layers, seed):
    g, e = W.gaussian_outliers(layers, seed=seed)
    l = layers[5]
    g[l.offset:l.offset + l.numel] = 0.5
    e[l.offset:l.offset + l.numel] = 0.0
    l = layers[1]
    g[l.offset:l.offset + l.numel] = 0.0
    e[l.offset:l.offset + l.numel] = -0.0
    g[layers[8].offset] = -0.0
    e[layers[8].offset] = -0.0
    g[layers[8].offset + 7] = -0.0
    e[layers[8].offset + 7] = 0.0
    return g, e


def _check_profile(err, bits, ref_err, ref_bits):
    assert np.array_equal(bits.cpu().numpy(), ref_bits)
    ge = err.cpu().numpy()
    assert np.all((ref_err == 0) == (ge == 0))
    rel = np.abs(ge - ref_err) / np.maximum(ref_err, 1e-300)
    assert rel.max() <= 1e-5, rel.max()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("cfg", ["C1", "edge", "C4"])
def test_profile_compress_parity(lg, ref, cfg):
    layers = W.config_layers(cfg) if cfg != "edge" else _edge_layers()
    g, e = W.gaussian_outliers(layers, seed=31) if cfg != "edge" else _edge_data(layers, 31)
    rng = np.random.default_rng(4)
    choice = [int(rng.integers(0, len(BITS))) if l.compress else -1 for l in layers]
    lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    seed, step = 0x77AB, 5
    L, K = len(layers), len(BITS)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=seed)
    gd, ed = _dev(g), _dev(e)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    out = torch.empty_like(gd)
    dch = torch.tensor(choice, dtype=torch.int32, device="cuda")
    ctx.profile_compress(dch, gd, ed, out, step, err, bits)
    ctx.check()
    ref_err, ref_bits = ref.qsgd_profile(layers, g, e, BITS, seed=seed, step=step)
    _check_profile(err, bits, ref_err, ref_bits)
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=seed, step=step)
    assert np.array_equal(_u32(out), out_ref.view(np.uint32))
    assert np.array_equal(_u32(ed), es_ref[0].view(np.uint32))
    # the library's own two-call definition gives the same bytes (err bitwise too)
    ed2, out2 = _dev(e), torch.empty_like(gd)
    err2, bits2 = torch.empty_like(err), torch.empty_like(bits)
    ctx.profile(gd, ed2, step, err2, bits2)
    ctx.compress_allreduce_dev(dch, gd, ed2, out2, step)
    assert torch.equal(err.view(torch.int64), err2.view(torch.int64)) and torch.equal(bits, bits2)
    assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
    assert torch.equal(ed.view(torch.int32), ed2.view(torch.int32))
    ctx.close()


def test_profile_compress_skip_and_bad_choice(lg, ref):
    """LGRECO_CHOICE_SKIP leaves a layer's output and EF untouched (lossless layers too);
    a choice outside [0, K) is reported as EINVAL and candidate 0 is used (K5's rule)."""
    layers = _edge_layers()
    g, e = _edge_data(layers, 9)
    L, K = len(layers), len(BITS)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=3)
    comp = [i for i, l in enumerate(layers) if l.compress]
    raw = [i for i, l in enumerate(layers) if not l.compress]
    choice = [3 if l.compress else -1 for l in layers]
    choice[comp[2]] = lg.CHOICE_SKIP
    choice[comp[-1]] = lg.CHOICE_SKIP
    choice[raw[0]] = lg.CHOICE_SKIP
    gd, ed = _dev(g), _dev(e)
    out = torch.full_like(gd, 7.0)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile_compress(torch.tensor(choice, dtype=torch.int32, device="cuda"), gd, ed, out, 1, err, bits)
    ctx.check()
    o, en = out.cpu().numpy(), ed.cpu().numpy()
    lbits = [BITS[3] if l.compress else 0 for l in layers]
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=3, step=1)
    for i, l in enumerate(layers):
        s = slice(l.offset, l.offset + l.numel)
        if choice[i] == lg.CHOICE_SKIP:
            assert np.all(o[s] == 7.0) and np.array_equal(en[s].view(np.uint32), e[s].view(np.uint32))
        else:
            assert np.array_equal(o[s].view(np.uint32), out_ref[s].view(np.uint32))
            assert np.array_equal(en[s].view(np.uint32), es_ref[0][s].view(np.uint32))
    ref_err, ref_bits = ref.qsgd_profile(layers, g, e, BITS, seed=3, step=1)
    _check_profile(err, bits, ref_err, ref_bits)
    bad = [0 if l.compress else -1 for l in layers]
    bad[comp[1]] = K
    ctx.profile_compress(torch.tensor(bad, dtype=torch.int32, device="cuda"), gd, ed, out, 2, err, bits)
    with pytest.raises(lg.LGrecoError) as ei:
        ctx.check()
    assert ei.value.status == lg.EINVAL
    ctx.close()


def test_profile_compress_nonfinite(lg):
    layers = W.config_layers("C1")[:4]
    g, e = W.gaussian_outliers(layers, seed=2)
    g[layers[2].offset + 300] = np.inf
    ctx = lg.Context(layers, lg.QSGD, BITS)
    L, K = len(layers), len(BITS)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile_compress(torch.zeros(L, dtype=torch.int32, device="cuda"), gd, ed, out, 0, err, bits)
    with pytest.raises(lg.LGrecoError) as ei:
        ctx.check()
    assert ei.value.status == lg.ENONFINITE
    ctx.close()


@pytest.mark.parametrize("cfg,lag", [("C1", 1), ("C1", 2), ("C4", 2)])
def test_pipelined_chain_matches_oracle(lg, ref, cfg, lag):
    """The paper's schedule with a re-solve every step: step t compresses with the plan
    solved from the profile of step t - lag (the defaults before that), the solve of
    step t - 1 running beside the fused pass of step t when lag = 2
    (LGRECO_PC_CONCURRENT, the bench's configuration).  Every step's plan, output and EF
    equal the oracle chain's."""
    layers = W.config_layers(cfg)
    L, K = len(layers), len(BITS)
    seed = 0x5EED
    nsteps = 4
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=seed)
    dflt = [BITS.index(4)] * L
    comp = torch.tensor([1 if l.compress else 0 for l in layers], dtype=torch.int32, device="cuda")
    ddef = torch.tensor(dflt, dtype=torch.int32, device="cuda")
    plans = [torch.tensor(dflt, dtype=torch.int32, device="cuda") for _ in range(lag + 1)]
    tabs = [(torch.empty(L, K, dtype=torch.float64, device="cuda"), torch.empty(L, K, dtype=torch.int64, device="cuda"))
            for _ in range(2)]  # (the concurrent pass writes one pair while the solve reads the other)
    ws = torch.empty(lg.solve_workspace_bytes(L, K, 10000), dtype=torch.uint8, device="cuda")
    info = torch.empty(64, dtype=torch.uint8, device="cuda")
    g0, e0 = W.gaussian_outliers(layers, seed=11)
    ed = _dev(e0)
    e_ref = e0.copy()
    ref_plans = [list(dflt)] * lag
    grads = []
    outs = []
    used = []
    for t in range(nsteps):
        g = (g0 * (1.0 + 0.25 * t)).astype(np.float32)
        grads.append(g)
        gd = _dev(g)
        out = torch.empty_like(gd)
        use = plans[t % (lag + 1)]
        used.append(use.clone())  # (the plan buffer is reused lag + 1 steps later)
        err, bits = tabs[t % 2]
        ctx.profile_compress(use, gd, ed, out, t, err, bits, concurrent=(lag == 2 and t > 0))
        nxt = plans[(t + lag) % (lag + 1)]
        lg.solve(err, bits, ddef, comp, flags=lg.SOLVE_NARROW if lag == 2 else 0, choice=nxt, info=info,
                 workspace=ws)
        outs.append((out.clone(), ed.clone()))
    torch.cuda.synchronize()
    ctx.check()
    for t in range(nsteps):
        g = grads[t]
        plan = ref_plans[t]
        assert [c for c, l in zip(used[t].cpu().tolist(), layers) if l.compress] == \
            [c for c, l in zip(plan, layers) if l.compress], t
        lbits = [BITS[c] if l.compress else 0 for c, l in zip(plan, layers)]
        rerr, rbits = ref.qsgd_profile(layers, g, e_ref, BITS, seed=seed, step=t)
        _, rch, _ = ref.solve(rerr, rbits, dflt, [1 if l.compress else 0 for l in layers])
        out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e_ref], seed=seed, step=t)
        o, en = outs[t]
        assert np.array_equal(_u32(o), out_ref.view(np.uint32)), t
        assert np.array_equal(_u32(en), es_ref[0].view(np.uint32)), t
        e_ref = es_ref[0]
        ref_plans.append([int(c) for c in rch])
    ctx.close()


@pytest.mark.parametrize("Wn", [2, 3, 4])
def test_profile_compress_p2p_simulated_ranks(lg, ref, Wn):
    """W > 1 over peer memory: the fused pass packs every stage-1 record (R7) in K1's lane
    layout straight into its owner's window, then the peer-memory exchange runs -- W rank
    contexts on W streams of the one GPU (peers set in-process); every rank's output and
    EF bit-identical to the W-rank oracle, every rank's profile of its own x = the
    oracle's (rankfield = rank)."""
    layers = _edge_layers()
    seed, step = 91, 6
    L, K = len(layers), len(BITS)
    ctxs = [lg.Context(layers, lg.QSGD, BITS, seed=seed, rank=w, world=Wn) for w in range(Wn)]
    loc = [c.p2p_local() for c in ctxs]
    for c in ctxs:
        c.p2p_set_peers([p[0] for p in loc], [p[1] for p in loc], [p[2] for p in loc])
    gs, es = zip(*[_edge_data(layers, 700 + w) for w in range(Wn)])
    rng = np.random.default_rng(Wn + 5)
    choice = [int(rng.integers(0, K)) if l.compress else -1 for l in layers]
    lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, list(gs), list(es), seed=seed, step=step)
    streams = [torch.cuda.Stream() for _ in range(Wn)]
    gds, eds = [_dev(g) for g in gs], [_dev(e) for e in es]
    outs = [torch.empty(len(gs[0]), dtype=torch.float32, device="cuda") for _ in range(Wn)]
    dch = [torch.tensor(choice, dtype=torch.int32, device="cuda") for _ in range(Wn)]
    errs = [torch.empty(L, K, dtype=torch.float64, device="cuda") for _ in range(Wn)]
    bits = [torch.empty(L, K, dtype=torch.int64, device="cuda") for _ in range(Wn)]
    torch.cuda.synchronize()
    for w in range(Wn):
        ctxs[w].profile_compress(dch[w], gds[w], eds[w], outs[w], step, errs[w], bits[w], stream=streams[w])
    torch.cuda.synchronize()
    for w in range(Wn):
        assert np.array_equal(_u32(outs[w]), out_ref.view(np.uint32)), w
        assert np.array_equal(_u32(eds[w]), es_ref[w].view(np.uint32)), w
        rerr, rbits = ref.qsgd_profile(layers, gs[w], es[w], BITS, seed=seed, rank=w, step=step)
        _check_profile(errs[w], bits[w], rerr, rbits)
    for c in ctxs:
        c.check()
        c.close()


def test_profile_compress_without_ef(lg, ref):
    """d_ef = NULL (no error feedback: x = g, the EF is neither read nor written): the fused
    pass equals the two-call definition and the oracle with a zero EF."""
    layers = _edge_layers()
    g, _ = _edge_data(layers, 44)
    L, K = len(layers), len(BITS)
    choice = [3 if l.compress else -1 for l in layers]
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=8)
    gd = _dev(g)
    dch = torch.tensor(choice, dtype=torch.int32, device="cuda")
    out, out2 = torch.empty_like(gd), torch.empty_like(gd)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    err2, bits2 = torch.empty_like(err), torch.empty_like(bits)
    ctx.profile_compress(dch, gd, None, out, 2, err, bits)
    ctx.profile(gd, None, 2, err2, bits2)
    ctx.compress_allreduce_dev(dch, gd, None, out2, 2)
    ctx.check()
    assert torch.equal(out.view(torch.int32), out2.view(torch.int32))
    assert torch.equal(err.view(torch.int64), err2.view(torch.int64)) and torch.equal(bits, bits2)
    lbits = [BITS[3] if l.compress else 0 for l in layers]
    zero = np.zeros_like(g)
    out_ref, _, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [zero], seed=8, step=2)
    assert np.array_equal(_u32(out), out_ref.view(np.uint32))
    rerr, rbits = ref.qsgd_profile(layers, g, None, BITS, seed=8, step=2)
    _check_profile(err, bits, rerr, rbits)
    ctx.close()
