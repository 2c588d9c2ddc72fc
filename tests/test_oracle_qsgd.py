"""Pins for the oracle's Philox generator and QSGD-style quantiser / exchange.

Each test checks the oracle against something other than itself: published
known-answer vectors, values derived by hand (tests/golden/), closed forms,
invariants, Monte-Carlo unbiasedness, or ratios printed in PAPER.md Tables 1-2.
"""
import os

import numpy as np
import pytest

from paper_2210_17357_b200 import workloads as W
from goldens import golden_record_cases

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#", 1)[0].strip()
        if line:
            rows.append(line.split())
    return rows


def test_philox_kat(ref):
    for r in _read("philox_kat.txt"):
        vals = [int(v, 16) for v in r if v != "->"]
        ctr, key, out = vals[:4], vals[4:6], vals[6:10]
        assert ref.philox(ctr, key) == tuple(out)


def test_golden_chain(ref):
    d = {r[0]: r[1:] for r in _read("qsgd_chain.txt")}
    u = ref.bucket_uniforms(0, 0, 0, 0, 0, 128, 4)
    want_u = np.array([int(v) for v in d["u_words"]], np.float64) / 2 ** 24
    assert np.array_equal(u.astype(np.float64), want_u)
    x = np.array([float(v) for v in d["x"]], np.float32)
    st, q, dec, mn, unit = ref.quantize_bucket(x, int(d["bits"][0]), u)
    assert st == 0
    assert list(q) == [int(v) for v in d["q"]]
    assert np.float32(unit).view(np.uint32) == int(d["unit"][0], 16)
    assert list(dec.view(np.uint32)) == [int(v, 16) for v in d["dec"]]


def test_uniform_counter_layout(ref):
    # element p of bucket gb uses ctr=(gb*B/4 + p/4, rank, step, stream), word p%4 (R3)
    seed, rank, step, stream, gb, B = 0x1234_5678_9ABC, 3, 77, 0, 5, 256
    u = ref.bucket_uniforms(seed, rank, step, stream, gb, B, B)
    for p in (0, 1, 5, 130, 255):
        ctr = (gb * B // 4 + p // 4, rank, step, stream)
        key = (seed & 0xFFFFFFFF, seed >> 32)
        w = ref.philox(ctr, key)[p % 4]
        assert u[p] == np.float32((w >> 8) / 2 ** 24)


def _rand_bucket(rng, n=128):
    return (rng.standard_t(3, n) * 1e-2).astype(np.float32)


@pytest.mark.parametrize("bits", [1, 2, 4, 8, 16])
def test_on_grid_identity(ref, bits):
    # values on the quantisation grid mn + q*unit reproduce themselves
    s = 2 ** bits - 1
    rng = np.random.default_rng(bits)
    q = rng.integers(0, s + 1, 128)
    q[0], q[1] = 0, s
    x = (q.astype(np.float32) * np.float32(1.0)).astype(np.float32)  # mn=0, range=s, unit=1
    u = rng.random(128).astype(np.float32)
    st, qq, dec, mn, unit = ref.quantize_bucket(x, bits, u)
    assert st == 0 and unit == 1.0 and mn == 0.0
    assert np.array_equal(qq, q.astype(np.uint32))
    assert np.array_equal(dec, x)


def test_zeros_and_constant(ref):
    u = np.full(128, 0.5, np.float32)
    for val in (0.0, 1.5, -3.25):
        x = np.full(128, val, np.float32)
        st, q, dec, mn, unit = ref.quantize_bucket(x, 4, u)
        assert st == 0 and not q.any() and np.array_equal(dec, x) and unit == 0.0


def test_nonfinite_rejected(ref):
    u = np.zeros(4, np.float32)
    for bad in (np.inf, -np.inf, np.nan):
        st, *_ = ref.quantize_bucket(np.array([0, 1, bad, 2], np.float32), 4, u)
        assert st == ref.REF_ENONFINITE
    # range overflow: mx - mn = +inf
    st, *_ = ref.quantize_bucket(np.array([-3e38, 3e38], np.float32), 4, u[:2])
    assert st == ref.REF_ENONFINITE


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_error_bounded_by_unit(ref, bits):
    rng = np.random.default_rng(10 + bits)
    for _ in range(20):
        x = _rand_bucket(rng)
        u = rng.random(128).astype(np.float32)
        st, q, dec, mn, unit = ref.quantize_bucket(x, bits, u)
        assert st == 0
        assert q.max() <= 2 ** bits - 1
        assert np.all(np.abs(x.astype(np.float64) - dec) <= unit * (1 + 1e-6))


@pytest.mark.parametrize("bits", [2, 4])
def test_unbiased_and_closed_form_mse(ref, bits):
    # E[dec] = x and E[(x-dec)^2] = unit^2 f (1-f) for stochastic rounding
    rng = np.random.default_rng(7)
    x = _rand_bucket(rng)
    T = 20000
    U = rng.random((T, 128)).astype(np.float32)
    decs = np.empty((T, 128), np.float64)
    for t in range(T):
        st, q, dec, mn, unit = ref.quantize_bucket(x, bits, U[t])
        decs[t] = dec
    mean = decs.mean(0)
    se = decs.std(0, ddof=1) / np.sqrt(T)
    det = se == 0  # bucket min/max elements are deterministic: dec = mn + q*unit,
    # exact for the min, within the rounding of unit = fl(range/s) for the max
    rng_ = float(x.max()) - float(x.min())
    assert np.all(np.abs(decs[:, det] - x[det]) <= 4 * np.spacing(np.float32(rng_)))
    z = np.abs(mean[~det] - x[~det]) / se[~det]
    assert z.max() < 5.0  # 128 simultaneous comparisons
    # closed form of the per-element MSE
    s = 2 ** bits - 1
    from fractions import Fraction as F
    inv = _rd32(F(s) / F(float(np.float32(x.max() - x.min()))))  # R5: RD(s / range)
    v = (x - x.min()).astype(np.float32).astype(np.float64) * np.float64(inv)  # exact (R6)
    f = v - np.floor(v)
    mse_cf = (unit ** 2 * f * (1 - f)).sum()
    mse_mc = ((decs - x) ** 2).sum(1).mean()
    assert abs(mse_mc - mse_cf) / mse_cf < 0.03


def _rn32(r):
    """Round a Fraction to the nearest float32, ties to even (no double rounding)."""
    from fractions import Fraction as F
    c = np.float32(float(r))
    cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
    best = min(abs(F(float(v)) - r) for v in cands)
    ties = [v for v in cands if abs(F(float(v)) - r) == best]
    return ties[0] if len(ties) == 1 else [v for v in ties if (v.view(np.uint32) & 1) == 0][0]


def _rd32(r):
    """Round a positive Fraction down to a float32 (the largest float32 <= r)."""
    from fractions import Fraction as F
    c = np.float32(float(r))
    while F(float(c)) > r:
        c = np.nextafter(c, np.float32(0))
    while np.isfinite(np.nextafter(c, np.float32(np.inf))) and F(float(np.nextafter(c, np.float32(np.inf)))) <= r:
        c = np.nextafter(c, np.float32(np.inf))
    return c


def test_code_is_exact_rational_rounding(ref):
    """R6 against exact rational arithmetic (fractions.Fraction, not the oracle's
    doubles): q = floor(v) + [u < frac(v)] with v = fl(x - mn) * RD(s / range) taken
    exactly (v <= s: no clamp), dec = fl(fma(q, unit, mn)).  Inputs are chosen so that u
    lands on, just below and just above frac(v)."""
    from fractions import Fraction as F
    rng = np.random.default_rng(11)
    for trial in range(40):
        bits = int(rng.integers(1, 9))
        s = 2 ** bits - 1
        x = rng.standard_normal(128).astype(np.float32) * np.float32(10.0 ** rng.integers(-6, 4))
        mn, mx = np.float32(x.min()), np.float32(x.max())
        rngv = np.float32(mx - mn)
        inv = _rd32(F(s) / F(float(rngv)))  # R5: the largest float <= s / range
        t = (x - mn).astype(np.float32)
        vq = [F(float(ti)) * F(float(inv)) for ti in t]
        assert max(vq) <= s  # so the code never needs the clamp
        fr = [v - (v.numerator // v.denominator) for v in vq]
        u = rng.random(128).astype(np.float32)
        for i in range(0, 128, 3):  # u at frac(v) rounded to float and its neighbours
            k = (i // 3) % 3
            ui = np.float32(float(fr[i]))
            u[i] = [ui, np.nextafter(ui, np.float32(0)), np.nextafter(ui, np.float32(1))][k]
            u[i] = min(u[i], np.float32(1 - 2 ** -24))
        st, q, dec, mn_o, unit = ref.quantize_bucket(x, bits, u)
        assert st == 0 and mn_o == mn
        for i in range(128):
            fl = vq[i].numerator // vq[i].denominator
            qe = min(fl + (1 if F(float(u[i])) < fr[i] else 0), s)
            assert q[i] == qe, (trial, i, bits)
            de = _rn32(F(qe) * F(float(unit)) + F(float(mn)))  # one rounding of the exact fma
            assert dec[i] == de


def test_pow2_scale_invariance(ref):
    # scaling x by 2^k leaves codes unchanged and scales dec exactly (R4 sum-vs-mean)
    rng = np.random.default_rng(3)
    x = _rand_bucket(rng)
    u = rng.random(128).astype(np.float32)
    _, q1, d1, _, _ = ref.quantize_bucket(x, 4, u)
    _, q2, d2, _, _ = ref.quantize_bucket(x * np.float32(8.0), 4, u)
    assert np.array_equal(q1, q2) and np.array_equal(d1 * np.float32(8.0), d2)


def _small_layers():
    sizes = [1, 127, 128, 129, 300, 1024, 1500]
    out, off = [], 0
    for n in sizes:
        out.append(W.Layer(off, n, 0, 0, 1))
        off += n
    out.append(W.Layer(off, 77, 0, 0, 0))  # lossless layer
    return out


def test_bits_formula_and_profile_consistency(ref):
    # bits = ceil(n/B)*(B*b+64); err(l, b) equals ||x - dec|| of the actual pack (R6:
    # common random numbers between profile and compress)
    layers = _small_layers()
    g, e = W.gaussian_outliers(layers, seed=1)
    cand = [2, 3, 4, 8]
    err, bits = ref.qsgd_profile(layers, g, e, cand, B=128, seed=9, rank=0, step=4)
    x = ((g + e) + np.float32(0)).astype(np.float32)
    for j, b in enumerate(cand):
        lbits = [b if l.compress else 0 for l in layers]
        pay, e2, dec = ref.qsgd_pack(layers, lbits, g, e, B=128, seed=9, rank=0, step=4, want_dec=True)
        for li, l in enumerate(layers):
            sl = slice(l.offset, l.offset + l.numel)
            if l.compress:
                assert bits[li, j] == -(-l.numel // 128) * (128 * b + 64)
                d = x[sl].astype(np.float64) - dec[sl].astype(np.float64)
                assert abs(err[li, j] - np.sqrt((d * d).sum())) <= 1e-12 * max(1e-30, err[li, j])
            else:
                assert bits[li, j] == 32 * l.numel and err[li, j] == 0.0


def test_pack_unpack_roundtrip_and_ef(ref):
    layers = _small_layers()
    g, e = W.gaussian_outliers(layers, seed=2)
    lbits = [3, 5, 4, 2, 7, 8, 1, 0]
    pay, e2, dec = ref.qsgd_pack(layers, lbits, g, e, B=128, seed=1, rank=2, step=3, want_dec=True)
    S, _, _ = ref.layout(layers, lbits, 128)
    assert pay.size == S
    out = ref.qsgd_unpack(layers, lbits, pay, len(g), B=128)
    assert np.array_equal(out.view(np.uint32), dec.view(np.uint32))
    x = ((g + e) + np.float32(0)).astype(np.float32)
    # EF: dec + e' == x up to half an ulp of e' (e' = fl(x - dec) is rounded once)
    back = dec.astype(np.float64) + e2.astype(np.float64)
    assert np.all(np.abs(back - x) <= 0.5 * np.spacing(np.abs(e2)).astype(np.float64))
    # lossless layer: raw, e' = 0
    ll = layers[-1]
    sl = slice(ll.offset, ll.offset + ll.numel)
    assert np.array_equal(dec[sl], x[sl]) and not e2[sl].any()


def test_bucket_size_multiple(ref):
    layers = _small_layers()
    g, e = W.gaussian_outliers(layers, seed=4)
    lbits = [4] * 7 + [0]
    pay, _, dec = ref.qsgd_pack(layers, lbits, g, e, B=256, want_dec=True)
    out = ref.qsgd_unpack(layers, lbits, pay, len(g), B=256)
    assert np.array_equal(out, dec)


def test_ef_conserves_gradient_sum(ref):
    # sum_t g_t = sum_t dec_t + e_T - e_0 (EF conservation, SURVEY.md §8(c) EF pin)
    layers = _small_layers()
    lbits = [2] * 7 + [0]
    N = W.total_numel(layers)
    e = np.zeros(N, np.float32)
    gs, decs = np.zeros(N), np.zeros(N)
    for t in range(12):
        g, _ = W.gaussian_outliers(layers, seed=100 + t, with_ef=False)
        _, e, dec = ref.qsgd_pack(layers, lbits, g, e, seed=5, step=t, want_dec=True)
        gs += g
        decs += dec
    scale = np.abs(gs).max()
    assert np.abs(gs - (decs + e)).max() <= 1e-5 * scale


def test_exchange_w1_and_lossless_mean(ref):
    layers = _small_layers()
    g, e = W.gaussian_outliers(layers, seed=6)
    lbits = [4] * 7 + [0]
    out, es, p1, p2 = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=3, step=1)
    pay, e2, dec = ref.qsgd_pack(layers, lbits, g, e, seed=3, rank=0, step=1, want_dec=True)
    assert np.array_equal(out, dec) and np.array_equal(es[0], e2) and np.array_equal(p1[0], pay)
    # all layers lossless -> exact rank-ordered fp32 mean
    ll = [W.Layer(l.offset, l.numel, 0, 0, 0) for l in layers]
    gr = [W.gaussian_outliers(layers, seed=20 + w, with_ef=False)[0] for w in range(4)]
    out, *_ = ref.qsgd_allreduce(ll, [0] * len(ll), gr, None)
    s = gr[0].copy()
    for w in range(1, 4):
        s = (s + gr[w]).astype(np.float32)
    assert np.array_equal(out, (s * np.float32(0.25)).astype(np.float32))


def test_exchange_unbiased(ref):
    # E[out] = mean_w x_w over the stochastic rounding (two unbiased stages)
    layers = [W.Layer(0, 256, 0, 0, 1)]
    rng = np.random.default_rng(11)
    gr = [(rng.standard_normal(256) * 0.01).astype(np.float32) for _ in range(4)]
    acc = np.zeros(256)
    T = 1500
    for s in range(T):
        out, *_ = ref.qsgd_allreduce(layers, [2], gr, None, seed=1000 + s, step=0)
        acc += out
    mean = acc / T
    target = np.mean(np.stack(gr).astype(np.float64), 0)
    spread = np.abs(np.stack(gr)).max() * 2 / 3  # ~unit at 2 bits
    assert np.abs(mean - target).max() < 5 * spread / np.sqrt(T)


def test_shard_bounds(ref):
    layers = W.config_layers("C2")
    lbits = [4 if l.compress else 0 for l in layers]
    S, bs, bo = ref.layout(layers, lbits, 128)
    R = int(bs[-1])
    for Wn in (1, 2, 3, 4, 8):
        rb, bb = ref.shard_bounds(layers, lbits, 128, Wn)
        assert rb[0] == 0 and rb[-1] == R and bb[0] == 0 and bb[-1] == S
        assert np.all(np.diff(rb) >= 0)
        for j in range(1, Wn):
            assert bb[j] >= j * S // Wn and bb[j] - j * S // Wn < 4 * 128 + 1


@pytest.mark.parametrize("name,paper", [("C4", 7.7), ("C2", 7.8), ("C3", 7.8), ("TLM", 7.8)])
def test_quant_ratio_pin(ref, name, paper):
    # PAPER.md:400,419 (Tables 1-2) uniform 4-bit ratio 7.7-7.8, reproduced at bucket
    # 1024 with 1-D tensors raw (R5); at the config's bucket 128 it is ~7.0-7.1
    layers = W.config_layers(name)
    N = W.total_numel(layers)
    lbits = [4 if l.compress else 0 for l in layers]
    S1024, _, _ = ref.layout(layers, lbits, 1024)
    S128, _, _ = ref.layout(layers, lbits, 128)
    assert abs(32 * N / (8 * S1024) - paper) < 0.1
    assert 7.0 < 32 * N / (8 * S128) < 7.15


@pytest.mark.parametrize("case", ["A", "B"])
def test_golden_packed_record(ref, case):
    """R7 byte layout against records derived by hand (tests/golden/qsgd_record.txt): a
    transposed (element, bit) or (lane, slot) mapping, a swapped metadata pair or missing
    16-byte padding fails here -- the pack->unpack round trip alone cannot see them."""
    c = {cs: (b, x, w) for cs, b, x, w in golden_record_cases()}[case]
    bits, x, words = c
    layers = [W.Layer(0, 128, 0, 0, 1)]
    for step in (0, 7):  # on-grid: the code does not depend on the uniforms
        pay, e2, dec = ref.qsgd_pack(layers, [bits], x, np.zeros(128, np.float32), seed=3, step=step, want_dec=True)
        assert pay.size == 4 * words.size
        assert np.array_equal(pay.view(np.uint32), words)
        assert np.array_equal(dec, x)
        assert not e2.any()


def test_accumulate_exact_sums(ref):
    """Row a1: G += g is one fp32 add per element.  On a dyadic grid (multiples of 2^-10,
    |partial sums| < 2^13) every add is exact, so after T steps G equals the integer
    closed form sum_t g_t exactly; off-grid, one step equals the correctly rounded sum
    (fp64 sum of two floats is exact, then one rounding to fp32)."""
    rng = np.random.default_rng(0)
    n, T = 1001, 9
    gs = [(rng.integers(-2 ** 12, 2 ** 12, n) / 1024.0).astype(np.float32) for _ in range(T)]
    G = np.zeros(n, np.float32)
    for g in gs:
        G = ref.accumulate(G, g)
    want = sum(g.astype(np.float64) for g in gs)
    assert np.array_equal(G.astype(np.float64), want)
    a = (rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8, n)).astype(np.float32)
    b = (rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8, n)).astype(np.float32)
    got = ref.accumulate(a, b)
    assert np.array_equal(got, (a.astype(np.float64) + b.astype(np.float64)).astype(np.float32))
    assert np.array_equal(ref.accumulate(a, np.zeros(n, np.float32)), a)


def test_openmp_build_identical(ref):
    """The oracle's OpenMP build (bench.py cpu_baseline / reference arm: layer loops on
    all host cores) returns exactly what the single-thread build returns: profile,
    compress + EF and the W-rank exchange, bit for bit."""
    layers = _small_layers()
    rng = np.random.default_rng(5)
    N = sum(l.numel for l in layers)
    gs = [rng.standard_normal(N).astype(np.float32) * 1e-2 for _ in range(2)]
    es = [rng.standard_normal(N).astype(np.float32) * 1e-3 for _ in range(2)]
    lb = [W.QSGD_BITS[i % 7] if l.compress else 0 for i, l in enumerate(layers)]
    outs = []
    for omp in (False, True):
        ref.use_openmp(omp)
        try:
            p = ref.qsgd_profile(layers, gs[0], es[0], W.QSGD_BITS, seed=3, step=1)
            r = ref.qsgd_allreduce(layers, lb, gs, [e.copy() for e in es], seed=3, step=1)
        finally:
            ref.use_openmp(False)
        outs.append((p, r))
    (p0, r0), (p1, r1) = outs
    assert np.array_equal(p0[0], p1[0]) and np.array_equal(p0[1], p1[1])
    assert np.array_equal(r0[0].view(np.uint32), r1[0].view(np.uint32))
    for a, b in zip(r0[1], r1[1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(r0[3], r1[3])
