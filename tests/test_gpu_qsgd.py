"""GPU parity: the CUDA QSGD path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Bit-exact for payload bytes, codes, EF and exchange outputs; 1e-5
relative for the fp64 error norms (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu

BITS = W.QSGD_BITS  # 2..8


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    assert torch.cuda.is_available()
    return lgreco


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _edge_layers():
    """Ragged sizes, misaligned offsets, a lossless layer, constant/zero layers."""
    sizes = [(1, 1), (3, 1), (127, 1), (128, 1), (129, 1), (1000, 1), (4097, 1), (77, 0), (12800, 1), (5, 1)]
    out, off = [], 0
    for n, c in sizes:
        out.append(W.Layer(off, n, 0, 0, c))
        off += n
    return out


def _edge_data(layers, seed):
    g, e = W.gaussian_outliers(layers, seed=seed)
    # constant layer, all-zero layer, on-grid layer, -0.0 entries
    l = layers[5]
    g[l.offset:l.offset + l.numel] = 0.5
    e[l.offset:l.offset + l.numel] = 0.0
    l = layers[1]
    g[l.offset:l.offset + l.numel] = 0.0
    e[l.offset:l.offset + l.numel] = -0.0
    g[layers[8].offset] = -0.0
    e[layers[8].offset] = -0.0
    return g, e


def test_philox_matches_kat(lg, ref):
    ctr = torch.tensor([[0, 0, 0, 0], [0xffffffff] * 4, [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344]],
                       dtype=torch.int64).to(torch.int32).cuda()
    keys = [(0, 0), (0xffffffff, 0xffffffff), (0xa4093822, 0x299f31d0)]
    for i, (k0, k1) in enumerate(keys):
        out = lg.debug_philox(ctr[i:i + 1].contiguous(), k0, k1).cpu().numpy().view(np.uint32)
        c = [int(v) & 0xffffffff for v in ctr[i].cpu().numpy().view(np.uint32)]
        assert tuple(out.ravel()) == ref.philox(c, (k0, k1))


@pytest.mark.parametrize("cfg,B,with_ef", [("C1", 128, True), ("C1", 128, False), ("edge", 128, True),
                                           ("edge", 256, True)])
def test_profile_parity(lg, ref, cfg, B, with_ef):
    layers = W.config_layers("C1") if cfg == "C1" else _edge_layers()
    g, e = (W.gaussian_outliers(layers, seed=3) if cfg == "C1" else _edge_data(layers, 3))
    if not with_ef:
        e = None
    seed, step, rank = 0x1234ABCD5678, 7, 0
    ctx = lg.Context(layers, lg.QSGD, BITS, qbucket=B, seed=seed)
    L, K = len(layers), len(BITS)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), None if e is None else _dev(e), step, err, bits)
    ref_err, ref_bits = ref.qsgd_profile(layers, g, e, BITS, B=B, seed=seed, rank=rank, step=step)
    assert np.array_equal(bits.cpu().numpy(), ref_bits)
    ge = err.cpu().numpy()
    rel = np.abs(ge - ref_err) / np.maximum(ref_err, 1e-300)
    assert np.all((ref_err == 0) == (ge == 0))
    assert rel.max() <= 1e-5, rel.max()


def _choice_for(layers, rng):
    return [int(rng.integers(0, len(BITS))) if l.compress else -1 for l in layers]


@pytest.mark.parametrize("cfg,B", [("C1", 128), ("edge", 128), ("edge", 256)])
def test_pack_parity(lg, ref, cfg, B):
    layers = W.config_layers("C1") if cfg == "C1" else _edge_layers()
    g, e = (W.gaussian_outliers(layers, seed=5) if cfg == "C1" else _edge_data(layers, 5))
    rng = np.random.default_rng(1)
    choice = _choice_for(layers, rng)
    lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    seed, step, rank = 99, 3, 2
    ctx = lg.Context(layers, lg.QSGD, BITS, qbucket=B, seed=seed)
    S = ctx.payload_bytes(choice)
    pay_ref, e_ref, dec_ref = ref.qsgd_pack(layers, lbits, g, e, B=B, seed=seed, rank=rank, step=step, want_dec=True)
    assert S == pay_ref.size
    gd, ed = _dev(g), _dev(e)
    pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
    dec = torch.empty_like(gd)
    ctx.qsgd_pack(choice, gd, ed, pay, dec, rank, step)
    torch.cuda.synchronize()
    assert np.array_equal(pay.cpu().numpy(), pay_ref)
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), e_ref.view(np.uint32))
    assert np.array_equal(dec.cpu().numpy().view(np.uint32), dec_ref.view(np.uint32))
    out = torch.empty_like(gd)
    ctx.qsgd_unpack(choice, pay, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), dec_ref.view(np.uint32))
    ctx.check()


@pytest.mark.parametrize("Wn", [1, 2, 3, 4, 8])
def test_exchange_parity_simulated_ranks(lg, ref, Wn):
    """W ranks simulated on one GPU through the stage entry points: pack per rank,
    byte-balanced shards (all-to-all as copies), owner reduce, all-gather, decode."""
    layers = _edge_layers()
    rng = np.random.default_rng(Wn)
    choice = _choice_for(layers, rng)
    lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    seed, step, B = 4242, 11, 128
    gs, es = [], []
    for w in range(Wn):
        g, e = _edge_data(layers, 100 + w)
        gs.append(g)
        es.append(e)
    out_ref, es_ref, p1_ref, p2_ref = ref.qsgd_allreduce(layers, lbits, gs, es, B=B, seed=seed, step=step)
    ctx = lg.Context(layers, lg.QSGD, BITS, qbucket=B, seed=seed)
    S = ctx.payload_bytes(choice)
    rb, bb = ctx.shard_bounds(choice, Wn)
    rb_ref, bb_ref = ref.shard_bounds(layers, lbits, B, Wn)
    assert list(rb) == list(rb_ref) and list(bb) == list(bb_ref)
    pays, eds = [], []
    for w in range(Wn):
        pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
        ed = _dev(es[w])
        ctx.qsgd_pack(choice, _dev(gs[w]), ed, pay, None, w, step)
        pays.append(pay)
        eds.append(ed)
    for w in range(Wn):
        assert np.array_equal(pays[w].cpu().numpy(), p1_ref[w])
        assert np.array_equal(eds[w].cpu().numpy().view(np.uint32), es_ref[w].view(np.uint32))
    out = torch.empty(len(gs[0]), dtype=torch.float32, device="cuda")
    if Wn == 1:
        ctx.qsgd_unpack(choice, pays[0], out)
    else:
        stage2 = torch.zeros(S, dtype=torch.uint8, device="cuda")
        for j in range(Wn):
            nbytes = bb[j + 1] - bb[j]
            recv = torch.cat([pays[w][bb[j]:bb[j + 1]] for w in range(Wn)]) if nbytes else \
                torch.zeros(1, dtype=torch.uint8, device="cuda")
            ctx.qsgd_reduce(choice, Wn, rb[j], rb[j + 1], recv.contiguous(), stage2, step)
        torch.cuda.synchronize()
        assert np.array_equal(stage2.cpu().numpy(), p2_ref)
        ctx.qsgd_unpack(choice, stage2, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))


def test_compress_allreduce_w1(lg, ref):
    layers = W.config_layers("C1")
    g, e = W.gaussian_outliers(layers, seed=8)
    choice = _choice_for(layers, np.random.default_rng(8))
    lbits = [BITS[c] for c in choice]
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=5)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, ed, out, 2)
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=5, step=2)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), es_ref[0].view(np.uint32))


def test_nonfinite_flag(lg):
    layers = W.config_layers("C1")[:3]
    g, e = W.gaussian_outliers(layers, seed=1)
    g[5] = np.nan
    ctx = lg.Context(layers, lg.QSGD, BITS)
    out = torch.empty(len(g), dtype=torch.float32, device="cuda")
    ctx.compress_allreduce([2, 2, 2], _dev(g), _dev(e), out, 0)
    with pytest.raises(lg.LGrecoError) as ei:
        ctx.check()
    assert ei.value.status == lg.ENONFINITE
    ctx.check()  # flag cleared


def test_c4_full_size(lg, ref):
    """C4 (ResNet-50, 25.6M fp32) at full size in the launch configuration bench.py
    times: profile err/bits vs the oracle on every layer, pack + EF + decode bitwise."""
    layers = W.config_layers("C4")
    g, e = W.gaussian_outliers(layers, seed=W.rank_seed(0x5EED, 0))
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=0x5EED)
    L, K = len(layers), len(BITS)
    gd, ed = _dev(g), _dev(e)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(gd, ed, 0, err, bits)
    ref_err, ref_bits = ref.qsgd_profile(layers, g, e, BITS, seed=0x5EED, step=0)
    assert np.array_equal(bits.cpu().numpy(), ref_bits)
    ge = err.cpu().numpy()
    assert (np.abs(ge - ref_err) / np.maximum(ref_err, 1e-300)).max() <= 1e-5
    choice = [BITS.index(4) if l.compress else -1 for l in layers]
    out = torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, ed, out, 0)
    lbits = [4 if l.compress else 0 for l in layers]
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=0x5EED, step=0)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), out_ref.view(np.uint32))
    assert np.array_equal(ed.cpu().numpy().view(np.uint32), es_ref[0].view(np.uint32))


def test_compress_allreduce_dev_matches_host_path(lg):
    """The device-plan entry point (no host round trip at W = 1) gives the same bytes."""
    layers = W.config_layers("C1")
    g, e = W.gaussian_outliers(layers, seed=12)
    choice = [int(c) for c in np.random.default_rng(12).integers(0, len(BITS), len(layers))]
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=5)
    gd = _dev(g)
    e1, e2 = _dev(e), _dev(e)
    o1, o2 = torch.empty_like(gd), torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, e1, o1, 3)
    ctx.compress_allreduce_dev(torch.tensor(choice, dtype=torch.int32, device="cuda"), gd, e2, o2, 3)
    assert torch.equal(o1.view(torch.int32), o2.view(torch.int32)) and torch.equal(e1.view(torch.int32), e2.view(torch.int32))


def test_compress_allreduce_dev_bad_choice(lg):
    """A device choice outside [0, K) on a compressed layer is reported by ctx_check as
    EINVAL (the kernel uses candidate 0 there); a valid one afterwards checks clean."""
    layers = W.config_layers("C1")
    g, e = W.gaussian_outliers(layers, seed=13)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=5)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    comp = [i for i, l in enumerate(layers) if l.compress]
    bad = [0] * len(layers)
    bad[comp[0]] = len(BITS)
    ctx.compress_allreduce_dev(torch.tensor(bad, dtype=torch.int32, device="cuda"), gd, ed, out, 1)
    with pytest.raises(lg.LGrecoError) as ei:
        ctx.check()
    assert ei.value.status == lg.EINVAL
    ctx.compress_allreduce_dev(torch.zeros(len(layers), dtype=torch.int32, device="cuda"), gd, ed, out, 2)
    ctx.check()


def _adversarial_buckets(seed=21):
    """One-bucket layers (128 elements, 16-byte aligned offsets: the K1 fast path) whose
    codes are easy to get wrong, so that ONE wrong stochastic-rounding decision moves the
    layer's error by far more than the 1e-5 tolerance:
      - large offset, tiny range (x = 1000 + N(0, 1e-3)): t = x - mn exact, dec rounds coarsely;
      - on-grid values of one candidate (v exactly integral, frac = 0);
      - ranges r with fl32(r * fl32(s/r)) > s for some s: the maximum element gives v > s,
        so the clamp min(., s) decides (R6);
      - a near-subnormal range (inv = s/range overflows: constant-bucket rule, R5);
      - repeated maxima/minima and exact zeros."""
    rng = np.random.default_rng(seed)
    f32 = np.float32
    blocks = []
    for _ in range(12):
        blocks.append((f32(1000.0) + rng.normal(0, 1e-3, 128).astype(f32)).astype(f32))
    for b in BITS:
        s = f32(2 ** b - 1)
        unit = f32(rng.uniform(1e-4, 1e-1))
        mn = f32(rng.normal(0, 1))
        k = rng.integers(0, int(s) + 1, 128).astype(f32)
        k[0], k[1] = 0, s
        blocks.append((mn + k * unit).astype(f32))
    found = 0
    while found < 16:
        r = f32(rng.uniform(1e-3, 10.0))
        hit = [b for b in BITS if f32(r * f32(f32(2 ** b - 1) / r)) > f32(2 ** b - 1)]
        if not hit:
            continue
        x = (rng.uniform(0, 1, 128) * r).astype(f32)
        x[:6] = r
        x[6] = f32(0.0)
        if found % 2:
            x = -x  # mn = -r: t = x - mn
        blocks.append(x.astype(f32))
        found += 1
    tiny = np.zeros(128, f32)
    tiny[::3] = f32(1e-44)
    blocks.append(tiny)
    blocks.append(np.concatenate([np.full(64, f32(-2.5)), np.full(64, f32(3.0))]).astype(f32))
    g = np.concatenate(blocks).astype(f32)
    layers = [W.Layer(128 * i, 128, 0, 0, 1) for i in range(len(blocks))]
    return layers, g


def _dev_shifted(a):
    """Device copy whose data pointer is 4 bytes past a 16-byte boundary (the K1
    bulk-copy path must fall back to masked direct loads)."""
    buf = torch.empty(a.size + 1, dtype=torch.float32, device="cuda")
    v = buf[1:]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


@pytest.mark.parametrize("with_ef,shifted", [(False, False), (True, False), (True, True)])
def test_profile_parity_adversarial_buckets(lg, ref, with_ef, shifted):
    """Per-bucket exactness of the fused profile's codes (fast path) against the oracle."""
    layers, g = _adversarial_buckets()
    e = None
    if with_ef:
        e = np.zeros_like(g)  # x = g + 0: exercises the EF add without moving the values
    seed, step = 0xC0FFEE, 11
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=seed)
    L, K = len(layers), len(BITS)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    mk = _dev_shifted if shifted else _dev
    ctx.profile(mk(g), None if e is None else mk(e), step, err, bits)
    ref_err, ref_bits = ref.qsgd_profile(layers, g, e, BITS, seed=seed, step=step)
    assert np.array_equal(bits.cpu().numpy(), ref_bits)
    ge = err.cpu().numpy()
    assert np.all((ref_err == 0) == (ge == 0))
    rel = np.abs(ge - ref_err) / np.maximum(ref_err, 1e-300)
    assert rel.max() <= 1e-5, (rel.max(), np.unravel_index(rel.argmax(), rel.shape))


def test_misaligned_buffers_rejected(lg):
    """Compress entry points need 16-byte aligned g / e / out (EINVAL, no launch); the
    QSGD profile accepts them (masked loads, covered by the adversarial test)."""
    layers = W.config_layers("C1")[:3]
    N = W.total_numel(layers)
    g, e = W.gaussian_outliers(layers, seed=2)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=1)
    gs, es = _dev_shifted(g), _dev_shifted(e)
    out = torch.empty(N, dtype=torch.float32, device="cuda")
    with pytest.raises(lg.LGrecoError) as ex:
        ctx.compress_allreduce([2] * len(layers), gs, es, out, 0)
    assert ex.value.status == lg.EINVAL
    ctx.check()
    ctx.close()


def test_c5_sampled_full_size(lg, ref):
    """C5 (GPT-2-medium-like, 354.8M fp32, 292 tensors) at full size in the bench launch
    configuration (every >= 2-D tensor compressed): the profile rows of sampled layers
    -- the 50257x1024 token embedding, first / middle / last blocks and a ragged-size
    vector -- against the oracle, which recomputes only those layers (the others are
    marked lossless on its side; global bucket numbering is unchanged, R3)."""
    layers = W.config_layers("C5")
    N = W.total_numel(layers)
    comp_idx = [i for i, l in enumerate(layers) if l.compress]
    big = max(comp_idx, key=lambda i: layers[i].numel)
    sample = sorted({big, comp_idx[1], comp_idx[len(comp_idx) // 2], comp_idx[-1]})
    rng = np.random.default_rng(55)
    g = np.zeros(N, np.float32)
    e = np.zeros(N, np.float32)
    for i in sample:
        l = layers[i]
        s = 10.0 ** rng.uniform(-4, -1)
        g[l.offset:l.offset + l.numel] = (rng.standard_normal(l.numel) * s).astype(np.float32)
        e[l.offset:l.offset + l.numel] = (rng.standard_normal(l.numel) * 0.1 * s).astype(np.float32)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=0x5EED)
    L, K = len(layers), len(BITS)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), _dev(e), 3, err, bits)
    sub = [W.Layer(l.offset, l.numel, l.rows, l.cols, 1 if i in sample else 0) for i, l in enumerate(layers)]
    ref_err, ref_bits = ref.qsgd_profile(sub, g, e, BITS, seed=0x5EED, step=3)
    ge, gb = err.cpu().numpy(), bits.cpu().numpy()
    for i in sample:
        assert np.array_equal(gb[i], ref_bits[i])
        assert (np.abs(ge[i] - ref_err[i]) / np.maximum(ref_err[i], 1e-300)).max() <= 1e-5, i
    ctx.close()


def test_device_chain_without_sync_matches_synced(lg):
    """profile -> solve -> compress_allreduce_dev chained on one stream with no host
    synchronisation (the PDL-launched kernels wait in-kernel for their producers) gives
    bitwise the same plans, EF and outputs over several steps as the same calls with a
    device synchronisation after each."""
    layers = W.config_layers("C4")
    g, e = W.gaussian_outliers(layers, seed=21)
    L, K = len(layers), len(BITS)
    comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device="cuda")
    dflt = torch.full((L,), BITS.index(4), dtype=torch.int32, device="cuda")

    def run(sync):
        ctx = lg.Context(layers, lg.QSGD, BITS, seed=9)
        gd, ed = _dev(g), _dev(e)
        out = torch.empty_like(gd)
        err = torch.empty(L, K, dtype=torch.float64, device="cuda")
        bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
        ch = torch.empty(L, dtype=torch.int32, device="cuda")
        info = torch.empty(48, dtype=torch.uint8, device="cuda")
        ws = torch.empty(lg.solve_workspace_bytes(L, K, 10000), dtype=torch.uint8, device="cuda")
        outs = []
        for s in range(4):
            ctx.profile(gd, ed, s, err, bits)
            if sync: torch.cuda.synchronize()
            lg.solve(err, bits, dflt, comp, D=10000, choice=ch, info=info, workspace=ws)
            if sync: torch.cuda.synchronize()
            ctx.compress_allreduce_dev(ch, gd, ed, out, s)
            if sync: torch.cuda.synchronize()
            outs.append((ch.clone(), out.clone()))
        torch.cuda.synchronize()
        ctx.check()
        ctx.close()
        return outs, ed

    a, ea = run(False)
    b, eb = run(True)
    for (c1, o1), (c2, o2) in zip(a, b):
        assert torch.equal(c1, c2)
        assert torch.equal(o1.view(torch.int32), o2.view(torch.int32))
    assert torch.equal(ea.view(torch.int32), eb.view(torch.int32))


def test_layer_norms(lg):
    """NEXT-4 helper: per-layer L2 norms of g + e (fp64) vs numpy on the same fp32 x."""
    layers = W.config_layers("C1")
    g, e = W.gaussian_outliers(layers, seed=4)
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=1)
    nrm = torch.empty(len(layers), dtype=torch.float64, device="cuda")
    ctx.layer_norms(_dev(g), _dev(e), nrm)
    x = (g + e).astype(np.float32).astype(np.float64)
    ref_n = np.array([np.sqrt(np.sum(x[l.offset:l.offset + l.numel] ** 2)) for l in layers])
    assert np.allclose(nrm.cpu().numpy(), ref_n, rtol=1e-12)
    ctx.close()


def test_hybrid_qsgd_topk_plan(lg, ref):
    """NEXT-4 hybrid: QSGD and TopK profiles of the same layers side by side in one DP
    table (device), solved on the GPU = the oracle's plan on the same table."""
    from paper_2210_17357_b200 import objectives as O
    layers = W.config_layers("C1")
    g, e = W.gaussian_outliers(layers, seed=6)
    L = len(layers)
    ppm = [1000, 10000, 100000]
    cq = lg.Context(layers, lg.QSGD, BITS, seed=2)
    ct = lg.Context(layers, lg.TOPK, ppm, seed=2)
    gd, ed = _dev(g), _dev(e)
    eq = torch.empty(L, len(BITS), dtype=torch.float64, device="cuda")
    bq = torch.empty(L, len(BITS), dtype=torch.int64, device="cuda")
    et = torch.empty(L, len(ppm), dtype=torch.float64, device="cuda")
    bt = torch.empty(L, len(ppm), dtype=torch.int64, device="cuda")
    cq.profile(gd, ed, 0, eq, bq)
    ct.profile(gd, ed, 0, et, bt)
    err, bits, cols = O.hybrid_table([eq, et], [bq, bt])
    dflt = torch.full((L,), BITS.index(4), dtype=torch.int32, device="cuda")
    choice, info = lg.solve(err, bits, dflt, None, D=10000)
    st, c_ref, i_ref = ref.solve(err.cpu().numpy(), bits.cpu().numpy(), dflt.cpu().numpy(), None, D=10000)
    assert list(choice.cpu().numpy()) == list(c_ref)
    fams = {cols[c][0] for c in c_ref}
    assert fams <= {0, 1}
    cq.close()
    ct.close()


@pytest.mark.parametrize("Wn", [2, 3, 4, 8])
def test_p2p_exchange_simulated_ranks(lg, ref, Wn):
    """Peer-memory exchange (no NCCL): W rank contexts in one process, each given the
    others' device buffers (lgreco_p2p_set_peers); stage 1 (pack straight into the
    owners' windows + epoch release) on every rank, then stage 2 (acquire, owner reduce,
    push to every peer), then stage 3 (acquire, decode) -- two steps with a plan change:
    outputs, EF and every rank's stage-2 payload bit-identical to the W-rank oracle."""
    layers = _edge_layers()
    seed, B = 4242, 128
    ctxs = [lg.Context(layers, lg.QSGD, BITS, qbucket=B, seed=seed, rank=w, world=Wn) for w in range(Wn)]
    loc = [c.p2p_local() for c in ctxs]
    for c in ctxs:
        c.p2p_set_peers([p[0] for p in loc], [p[1] for p in loc], [p[2] for p in loc])
    gs, es = [], []
    for w in range(Wn):
        g, e = _edge_data(layers, 300 + w)
        gs.append(g)
        es.append(e)
    eds = [_dev(e) for e in es]
    es_cur = [e.copy() for e in es]
    for step, cs in ((5, Wn), (6, Wn + 7)):
        choice = _choice_for(layers, np.random.default_rng(cs))
        lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
        out_ref, es_ref, _, p2_ref = ref.qsgd_allreduce(layers, lbits, gs, es_cur, B=B, seed=seed, step=step)
        outs = [torch.empty(len(gs[0]), dtype=torch.float32, device="cuda") for _ in range(Wn)]
        gds = [_dev(g) for g in gs]
        for stage in (1, 2, 3):
            for w in range(Wn):
                ctxs[w].p2p_stage(choice, gds[w], eds[w], outs[w], step, stage)
        torch.cuda.synchronize()
        for w in range(Wn):
            assert np.array_equal(outs[w].cpu().numpy().view(np.uint32), out_ref.view(np.uint32)), (step, w)
            assert np.array_equal(eds[w].cpu().numpy().view(np.uint32), es_ref[w].view(np.uint32)), (step, w)
        es_cur = [e.copy() for e in es_ref]
    # plan agreement over peer memory: every rank proposes its own plan, rank 0's wins
    props = [torch.tensor(_choice_for(layers, np.random.default_rng(50 + w)), dtype=torch.int32, device="cuda")
             for w in range(Wn)]
    want = props[0].clone()
    for w in range(Wn):  # rank 0 pushes first (one process: launch order = dependency order)
        ctxs[w].plan_broadcast(props[w])
    torch.cuda.synchronize()
    for w in range(Wn):
        assert torch.equal(props[w], want)
    for c in ctxs:
        c.check()
        c.close()


@pytest.mark.parametrize("Wn", [2, 4])
def test_p2p_device_plan_simulated_ranks(lg, ref, Wn):
    """The W > 1 peer-memory step with the plan laid out on the device (no host round
    trip): W rank contexts on W streams of the one GPU, each running the whole step
    (layout, pack into the owners' windows, epoch waits, reduce, push, decode) via
    compress_allreduce_dev -- outputs and EF bit-identical to the W-rank oracle."""
    layers = _edge_layers()
    seed, B, step = 77, 128, 9
    ctxs = [lg.Context(layers, lg.QSGD, BITS, qbucket=B, seed=seed, rank=w, world=Wn) for w in range(Wn)]
    loc = [c.p2p_local() for c in ctxs]
    for c in ctxs:
        c.p2p_set_peers([p[0] for p in loc], [p[1] for p in loc], [p[2] for p in loc])
    gs, es = zip(*[_edge_data(layers, 500 + w) for w in range(Wn)])
    choice = _choice_for(layers, np.random.default_rng(Wn + 40))
    lbits = [BITS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    out_ref, es_ref, _, _ = ref.qsgd_allreduce(layers, lbits, list(gs), list(es), B=B, seed=seed, step=step)
    streams = [torch.cuda.Stream() for _ in range(Wn)]
    gds, eds = [_dev(g) for g in gs], [_dev(e) for e in es]
    outs = [torch.empty(len(gs[0]), dtype=torch.float32, device="cuda") for _ in range(Wn)]
    dch = [torch.tensor(choice, dtype=torch.int32, device="cuda") for _ in range(Wn)]
    torch.cuda.synchronize()
    for w in range(Wn):
        ctxs[w].compress_allreduce_dev(dch[w], gds[w], eds[w], outs[w], step, stream=streams[w])
    torch.cuda.synchronize()
    for w in range(Wn):
        assert np.array_equal(outs[w].cpu().numpy().view(np.uint32), out_ref.view(np.uint32)), w
        assert np.array_equal(eds[w].cpu().numpy().view(np.uint32), es_ref[w].view(np.uint32)), w
    for c in ctxs:
        c.check()
        c.close()


@pytest.mark.parametrize("case", ["A", "B"])
def test_golden_packed_record_gpu(lg, case):
    """K5's record bytes equal the hand-derived R7 records (tests/golden/qsgd_record.txt)."""
    from goldens import golden_record_cases
    bits, x, words = {cs: (b, x, w) for cs, b, x, w in golden_record_cases()}[case]
    layers = [W.Layer(0, 128, 0, 0, 1)]
    ctx = lg.Context(layers, lg.QSGD, BITS, seed=3)
    choice = [BITS.index(bits)]
    S = ctx.payload_bytes(choice)
    assert S == 4 * words.size
    pay = torch.zeros(S, dtype=torch.uint8, device="cuda")
    dec = torch.empty(128, dtype=torch.float32, device="cuda")
    ef = torch.zeros(128, dtype=torch.float32, device="cuda")
    ctx.qsgd_pack(choice, _dev(x), ef, pay, dec, 0, 5)
    assert np.array_equal(pay.cpu().numpy().view(np.uint32), words)
    assert np.array_equal(dec.cpu().numpy(), x)
    ctx.close()


@pytest.mark.parametrize("n,shift", [(0, 0), (1, 0), (3, 1), (1000, 0), (4099, 2), (4099, 1), (25557032, 0)])
def test_accumulate_parity(lg, ref, n, shift):
    """Row a1 / K0: G += g bitwise equal to the oracle over several steps, for ragged
    sizes, shared and differing misalignments (scalar head / scalar path)."""
    rng = np.random.default_rng(n + shift)
    G0 = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    Gd = torch.zeros(n + 4, dtype=torch.float32, device="cuda")
    Gv = Gd[shift:shift + n]
    Gv.copy_(_dev(G0))
    want = G0
    for t in range(3):
        g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 0)).astype(np.float32)
        gd = torch.zeros(n + 4, dtype=torch.float32, device="cuda")
        gsh = shift if t != 1 else (shift + 1) % 4  # step 1: different alignment -> scalar path
        gv = gd[gsh:gsh + n]
        gv.copy_(_dev(g))
        lg.accumulate(Gv, gv)
        want = ref.accumulate(want, g)
    torch.cuda.synchronize()
    assert np.array_equal(Gv.cpu().numpy().view(np.uint32), want.view(np.uint32))
