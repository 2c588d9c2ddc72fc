"""GPU parity for the PowerSGD rows (a4 profile, a8-a10 compress + two all-reduces)
vs the fp64 oracle: 1e-5 relative on error norms, normwise 1e-5 on reconstructions,
EF and the warm-start factors (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    return lgreco


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _layers():
    shapes = [(40, 30, 1), (0, 17, 0), (64, 200, 1), (6, 5, 1), (130, 70, 1), (0, 33, 1), (257, 96, 1)]
    out, off = [], 0
    for m, k, c in shapes:
        n = m * k if m else k
        out.append(W.Layer(off, n, m, k if m else 0, c))
        off += n
    return out


RANKS = [1, 2, 4, 8]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("with_ef", [True, False])
def test_profile_parity(lg, ref, with_ef):
    layers = _layers()
    g, e = W.low_rank_plus_noise(layers, seed=2, with_ef=True)
    if not with_ef:
        e = None
    ctx = lg.Context(layers, lg.POWERSGD, RANKS, power_steps=5, seed=77)
    L, K = len(layers), len(RANKS)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), None if e is None else _dev(e), 3, err, bits)
    rerr, rbits = ref.psgd_profile(layers, g, e, RANKS, steps=5, seed=77, step=3)
    assert np.array_equal(bits.cpu().numpy(), rbits)
    ge = err.cpu().numpy()
    assert np.all((rerr == 0) == (ge == 0))
    rel = np.abs(ge - rerr) / np.maximum(rerr, 1e-300)
    assert rel.max() <= 1e-5, rel.max()


def test_profile_exact_low_rank(lg, ref):
    # exactly rank-2 matrix: err -> 0 at r >= 2 (direct fp64 fallback)
    rng = np.random.default_rng(0)
    M = (rng.standard_normal((50, 2)) @ rng.standard_normal((2, 40))).astype(np.float32)
    layers = [W.Layer(0, 2000, 50, 40, 1)]
    ctx = lg.Context(layers, lg.POWERSGD, RANKS, seed=1)
    err = torch.empty(1, 4, dtype=torch.float64, device="cuda")
    bits = torch.empty(1, 4, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(M.ravel()), None, 0, err, bits)
    rerr, _ = ref.psgd_profile(layers, M.ravel(), None, RANKS, seed=1, step=0)
    nM = np.linalg.norm(M.astype(np.float64))
    ge = err.cpu().numpy()[0]
    assert abs(ge[0] - rerr[0, 0]) <= 1e-5 * rerr[0, 0]
    assert np.all(np.abs(ge[1:] - rerr[0, 1:]) <= 1e-5 * nM)


def test_c2_full_size_profile(lg, ref):
    """C2 (ResNet-18 CIFAR-10, 11.2M fp32) at full size, ranks {1,2,4,8,16}."""
    layers = W.config_layers("C2")
    g, _ = W.low_rank_plus_noise(layers, seed=W.rank_seed(0x5EED, 0))
    ctx = lg.Context(layers, lg.POWERSGD, W.PSGD_RANKS_C2, seed=0x5EED)
    L, K = len(layers), len(W.PSGD_RANKS_C2)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile(_dev(g), None, 0, err, bits)
    rerr, rbits = ref.psgd_profile(layers, g, None, W.PSGD_RANKS_C2, seed=0x5EED, step=0)
    assert np.array_equal(bits.cpu().numpy(), rbits)
    ge = err.cpu().numpy()
    assert (np.abs(ge - rerr) / np.maximum(rerr, 1e-300)).max() <= 1e-5


def _slots(ref, layers, ranks):
    """P / Q slot offsets of the ctx factor areas (include/lgreco.h lgreco_psgd_factors)."""
    po, qo, p, q = {}, {}, 0, 0
    for l, ly in enumerate(layers):
        if ly.compress and ly.rows > 0:
            rmax = max([r for r in ranks if not ref.psgd_lossless(ly.rows, ly.cols, r)], default=0)
            po[l], qo[l] = p, q
            p += ly.rows * rmax
            q += ly.cols * rmax
    return po, qo


def _check_factors(ctx, ref, layers, lrank, Ps_ref, Qs_ref, ranks):
    """Phat and the warm-start Q of the ctx vs the oracle's (R12), 1e-5 normwise per layer."""
    Psz, Qsz = ctx.psgd_sizes()
    Ph = torch.zeros(max(Psz, 1), dtype=torch.float32, device="cuda")
    Qw = torch.zeros(max(Qsz, 1), dtype=torch.float32, device="cuda")
    ctx.psgd_factors(Ph, Qw)
    Ph, Qw = Ph.cpu().numpy(), Qw.cpu().numpy()
    po, qo = _slots(ref, layers, ranks)
    n = 0
    for l, P_ref in Ps_ref.items():
        m, k, r = layers[l].rows, layers[l].cols, lrank[l]
        P = Ph[po[l]:po[l] + m * r].reshape(r, m).T
        Q = Qw[qo[l]:qo[l] + k * r].reshape(r, k).T
        assert _rel(P, P_ref) <= 1e-5, (l, _rel(P, P_ref))
        assert _rel(Q, Qs_ref[l]) <= 1e-5, (l, _rel(Q, Qs_ref[l]))
        n += 1
    return n


def _choice(layers, rng):
    return [int(rng.integers(0, len(RANKS))) if l.compress else -1 for l in layers]


@pytest.mark.parametrize("Wn", [1, 2, 3])
def test_compress_simulated_ranks_two_steps(lg, ref, Wn):
    layers = _layers()
    N = W.total_numel(layers)
    rng = np.random.default_rng(Wn)
    choice = _choice(layers, rng)
    lrank = [RANKS[c] if l.compress else 0 for c, l in zip(choice, layers)]
    seed = 5
    ctx = lg.Context(layers, lg.POWERSGD, RANKS, seed=seed)
    Psz, Qsz = ctx.psgd_sizes()
    # oracle warm-start state initialised like the ctx (stream 2 at the first step)
    Qs = {}
    for l, ly in enumerate(layers):
        r = lrank[l]
        if r and ly.compress and ly.rows and not ref.psgd_lossless(ly.rows, ly.cols, r):
            Qs[l] = ref.psgd_init_q(seed, l, 0, ly.cols, r)
    es_ref = [W.low_rank_plus_noise(layers, seed=30 + w, with_ef=True)[1] for w in range(Wn)]
    es_gpu = [_dev(x) for x in es_ref]
    S = ctx.payload_bytes(choice)
    for step in range(2):
        gs = [W.low_rank_plus_noise(layers, seed=100 * step + w)[0] for w in range(Wn)]
        gd = [_dev(x) for x in gs]
        out_ref, es_ref, Ps = ref.psgd_allreduce(layers, lrank, gs, es_ref, Qs)
        Pw = [torch.zeros(max(Psz, 1), dtype=torch.float32, device="cuda") for _ in range(Wn)]
        for w in range(Wn):
            ctx.psgd_p(choice, gd[w], es_gpu[w], Pw[w], step)
        Psum = Pw[0].clone()
        for w in range(1, Wn):
            Psum += Pw[w]
        Qw = [torch.zeros(max(Qsz, 1), dtype=torch.float32, device="cuda") for _ in range(Wn)]
        for w in range(Wn):
            ctx.psgd_q(choice, gd[w], es_gpu[w], Psum, Wn, Qw[w])
        Qsum = Qw[0].clone()
        for w in range(1, Wn):
            Qsum += Qw[w]
        outs = []
        pays = []
        for w in range(Wn):
            out = torch.zeros(N, dtype=torch.float32, device="cuda")
            ctx.psgd_out(choice, gd[w], es_gpu[w], Qsum, Wn, out)
            pay = torch.zeros(max(S, 1), dtype=torch.uint8, device="cuda")
            ctx.psgd_raw_pack(choice, gd[w], es_gpu[w], pay, None)
            pays.append(pay[:S] if S else pay)
            outs.append(out)
        if S:
            ctx.psgd_raw_combine(choice, Wn, torch.cat(pays).contiguous(), outs[0])
        assert _check_factors(ctx, ref, layers, lrank, Ps, Qs, RANKS) == len(Qs)
        o = outs[0].cpu().numpy()
        for l, ly in enumerate(layers):
            sl = slice(ly.offset, ly.offset + ly.numel)
            if l in Qs:
                assert _rel(o[sl], out_ref[sl]) <= 1e-5
                for w in range(Wn):
                    assert _rel(es_gpu[w].cpu().numpy()[sl], es_ref[w][sl]) <= 1e-5
            else:
                assert np.array_equal(o[sl].view(np.uint32), out_ref[sl].view(np.uint32))
                for w in range(Wn):
                    assert not es_gpu[w].cpu().numpy()[sl].any()


def test_compress_allreduce_w1(lg, ref):
    layers = _layers()
    choice = [1 if l.compress else -1 for l in layers]
    lrank = [RANKS[1] if l.compress else 0 for l in layers]
    g, e = W.low_rank_plus_noise(layers, seed=9, with_ef=True)
    ctx = lg.Context(layers, lg.POWERSGD, RANKS, seed=3)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    ctx.compress_allreduce(choice, gd, ed, out, 4)
    Qs = {l: ref.psgd_init_q(3, l, 4, ly.cols, 2) for l, ly in enumerate(layers)
          if ly.compress and ly.rows and not ref.psgd_lossless(ly.rows, ly.cols, 2)}
    out_ref, es_ref, Ps = ref.psgd_allreduce(layers, lrank, [g], [e], Qs)
    assert _rel(out.cpu().numpy(), out_ref) <= 1e-5
    assert _rel(ed.cpu().numpy(), es_ref[0]) <= 1e-5
    assert _check_factors(ctx, ref, layers, lrank, Ps, Qs, RANKS) == len(Qs) > 0
    ctx.check()


@pytest.mark.parametrize("cfg", ["C2", "tall", "special"])
def test_profile_svd_parity(lg, ref, cfg):
    """NEXT-2: errors of every candidate rank from the singular values (fp64 Gram of the
    smaller side + the library's own eigensolver: Householder tridiagonalisation, Sturm
    bisection) vs the oracle's LAPACK SVD; bits identical.  "special": a zero matrix, an
    exactly rank-3 one, repeated singular values, a 2 x k and a 3 x 3-view matrix."""
    if cfg == "special":
        shapes = [(64, 96), (80, 50), (120, 40), (2, 300), (3, 3), (200, 130)]
        layers, off = [], 0
        for m, k in shapes:
            layers.append(W.Layer(off, m * k, m, k, 1))
            off += m * k
        rng = np.random.default_rng(12)
        g = np.zeros(off, np.float32)
        ly = layers[1]  # exactly rank 3
        g[ly.offset:ly.offset + ly.numel] = (rng.standard_normal((80, 3)) @ rng.standard_normal((3, 50))).astype(
            np.float32).ravel()
        ly = layers[2]  # singular values 5, 5, 5, 1, 1, 0.1 ...
        U, _ = np.linalg.qr(rng.standard_normal((120, 40)))
        V, _ = np.linalg.qr(rng.standard_normal((40, 40)))
        sv = np.array([5, 5, 5, 1, 1] + [0.1] * 35)
        g[ly.offset:ly.offset + ly.numel] = ((U * sv) @ V.T).astype(np.float32).ravel()
        for ly in layers[3:]:
            g[ly.offset:ly.offset + ly.numel] = rng.standard_normal(ly.numel).astype(np.float32)
        e = None
    elif cfg == "C2":
        layers = W.config_layers("C2")
        g, _ = W.low_rank_plus_noise(layers, seed=8)
        e = (np.random.default_rng(8).standard_normal(g.size) * 1e-4).astype(np.float32)
    else:  # m > k (Gram of the columns), a wide one, a vector, an uncompressed matrix
        shapes = [(3000, 40, 1), (40, 700, 1), (1, 333, 0), (300, 200, 0), (257, 129, 1)]
        layers, off = [], 0
        for m, k, c in shapes:
            layers.append(W.Layer(off, m * k, m, k, c) if m > 1 else W.Layer(off, k, 0, 0, c))
            off += m * k
        rng = np.random.default_rng(9)
        g = np.zeros(off, np.float32)
        for l in layers:
            if l.rows > 0:
                A = rng.standard_normal((l.rows, 8)) @ rng.standard_normal((8, l.cols))
                g[l.offset:l.offset + l.numel] = (A + 0.1 * rng.standard_normal((l.rows, l.cols))).astype(np.float32).ravel()
        e = (rng.standard_normal(off) * 1e-3).astype(np.float32)
    ranks = W.PSGD_RANKS_C2
    ctx = lg.Context(layers, lg.POWERSGD, ranks, seed=3)
    L, K = len(layers), len(ranks)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    ctx.profile_svd(_dev(g), None if e is None else _dev(e), err, bits)
    r_err, r_bits = ref.psgd_svd_profile(layers, g, e, ranks)
    assert np.array_equal(bits.cpu().numpy(), r_bits)
    ge = err.cpu().numpy()
    if cfg == "special":  # (exact zeros: the eigenvalues of a rank-deficient Gram are only ~eps ||G||)
        scale = np.array([[np.linalg.norm(g[l.offset:l.offset + l.numel])] * K for l in layers])
        assert (np.abs(ge - r_err) <= 1e-6 * np.maximum(r_err, 1e-300) + 1e-6 * scale).all(), (ge, r_err)
    else:
        assert np.all((r_err == 0) == (ge == 0))
        assert (np.abs(ge - r_err) / np.maximum(r_err, 1e-300)).max() <= 1e-6
    ctx.close()


def test_profile_method_selector(lg, ref):
    """NEXT-2 selector: AUTO keeps the power method where the rank
    range is small against the matrix (C2: r_max 16 on up to 512 x 4608) and takes the
    singular values where it is large against the smaller side (a 3000 x 40 matrix with
    ranks up to 16 and a 40 x 700 one: n = 40); lgreco_profile then returns exactly what
    the chosen method's own entry returns, and the SVD result matches the oracle's SVD."""
    layers = W.config_layers("C2")
    ctx = lg.Context(layers, lg.POWERSGD, W.PSGD_RANKS_C2, seed=3)
    assert ctx.psgd_method() == lg.PSGD_POWER
    ctx.set_psgd_method(lg.PSGD_AUTO)
    assert ctx.psgd_method() == lg.PSGD_POWER
    ctx.close()
    shapes = [(3000, 40), (40, 700)]
    tall, off = [], 0
    for m, k in shapes:
        tall.append(W.Layer(off, m * k, m, k, 1))
        off += m * k
    rng = np.random.default_rng(4)
    g = rng.standard_normal(off).astype(np.float32)
    ranks = [1, 2, 4, 8, 16]
    ctx = lg.Context(tall, lg.POWERSGD, ranks, seed=3)
    ctx.set_psgd_method(lg.PSGD_AUTO)
    assert ctx.psgd_method() == lg.PSGD_SVD
    L, K = len(tall), len(ranks)
    e1 = torch.empty(L, K, dtype=torch.float64, device="cuda")
    b1 = torch.empty(L, K, dtype=torch.int64, device="cuda")
    e2, b2 = torch.empty_like(e1), torch.empty_like(b1)
    gd = _dev(g)
    ctx.profile(gd, None, 0, e1, b1)
    ctx.profile_svd(gd, None, e2, b2)
    assert torch.equal(e1, e2) and torch.equal(b1, b2)
    r_err, _ = ref.psgd_svd_profile(tall, g, None, ranks)
    assert (np.abs(e1.cpu().numpy() - r_err) / np.maximum(r_err, 1e-300)).max() <= 1e-6
    with pytest.raises(lg.LGrecoError):
        ctx.set_psgd_method(7)
    ctx.close()
