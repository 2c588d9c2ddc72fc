"""Weighted objective: the oracle's
Algorithm 1 on the weighted cost table, pinned against brute force and the
scale-invariance of the argmin; bucket assignment and the least-squares fit of T(b)
against closed forms."""
import itertools

import numpy as np

from paper_2210_17357_b200 import objectives as O
from paper_2210_17357_b200 import workloads as W

from test_oracle_dp import _disc


def _brute_weighted(err, bits, w, dflt, D):
    L, K = err.shape
    emax = sum(err[l, dflt[l]] for l in range(L))
    best = None
    for a in itertools.product(range(K), repeat=L):
        ds = [_disc(err[l, a[l]], D, emax) for l in range(L)]
        if any(d is None for d in ds) or sum(ds) > D:
            continue
        c = sum(int(bits[l, a[l]]) * int(w[l]) for l in range(L))
        if best is None or c < best:
            best = c
    return best


def test_weighted_solve_matches_brute_force(ref):
    rng = np.random.default_rng(5)
    for _ in range(150):
        L, K = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        D = int(rng.choice([10, 100, 1000]))
        err = np.sort(rng.uniform(0, 1, (L, K)), 1)[:, ::-1].copy()
        bits = np.sort(rng.integers(1, 1000, (L, K)), 1).astype(np.int64)
        w = rng.integers(1, 9, L).astype(np.int64)
        dflt = rng.integers(0, K, L).astype(np.int32)
        st, ch, info = ref.solve(err, bits * w[:, None], dflt, None, D=D)
        assert st == 0
        best = _brute_weighted(err, bits, w, dflt, D)
        got = sum(int(bits[l, ch[l]]) * int(w[l]) for l in range(L))
        dcost = sum(int(bits[l, dflt[l]]) * int(w[l]) for l in range(L))
        # Algorithm 1 returns the optimum of the discretised problem, or the defaults when
        # the optimum does not beat them (R20)
        if info.used_default:
            assert got == dcost
        else:
            assert best is not None and got == best <= dcost


def test_constant_weight_leaves_the_plan_unchanged(ref):
    rng = np.random.default_rng(6)
    for _ in range(60):
        L, K = int(rng.integers(2, 40)), int(rng.integers(2, 9))
        err = np.sort(rng.uniform(0, 1, (L, K)), 1)[:, ::-1].copy()
        bits = np.sort(rng.integers(64, 10 ** 6, (L, K)), 1).astype(np.int64)
        dflt = np.full(L, K // 2, np.int32)
        _, c1, i1 = ref.solve(err, bits, dflt, None, D=1000)
        _, c3, i3 = ref.solve(err, bits * 3, dflt, None, D=1000)
        assert list(c1) == list(c3) and i3.total_bits == 3 * i1.total_bits


def test_ddp_buckets_closed_form():
    # 6 layers of 0.5 MiB each (fp32): the first bucket (1 MiB cap) takes the last two,
    # the next (25 MiB) the remaining four
    layers = [W.Layer(i * 131072, 131072, 0, 0, 1) for i in range(6)]
    assert O.ddp_buckets(layers) == [1, 1, 1, 1, 0, 0]
    assert list(O.bucket_priority_weights(layers)) == [2, 2, 2, 2, 1, 1]
    # DDP appends a tensor before checking the cap: a layer larger than the cap joins the
    # open bucket and closes it; the next layer starts a new one
    big = [W.Layer(0, 16, 0, 0, 1), W.Layer(16, 10 * 2 ** 20, 0, 0, 1), W.Layer(10 * 2 ** 20 + 16, 16, 0, 0, 1)]
    assert O.ddp_buckets(big, bucket_bytes=2 ** 20) == [1, 0, 0]


def test_fit_bucket_time_recovers_coefficients():
    rng = np.random.default_rng(7)
    T = np.array([3e-9, 1e-9, 5e-10, 2e-9])
    sizes = rng.uniform(1e6, 1e8, (200, 4))
    times = sizes @ T + 4e-5
    Tf, c = O.fit_bucket_time(sizes, times)
    assert np.allclose(Tf, T, rtol=1e-8) and abs(c - 4e-5) < 1e-9
    w = O.time_weights([W.Layer(0, 1, 0, 0, 1)] * 4, Tf, buckets=[0, 1, 2, 3], scale=600)
    assert list(w) == [600, 200, 100, 400]


def test_accordion_defaults_rule():
    prev = [1.0, 1.0, 2.0, 0.5]
    cur = [1.6, 1.2, 0.9, 0.5]
    # |dn| / n: 0.6, 0.2, 0.55, 0  -> critical, calm, critical, calm (eta = 0.5)
    assert list(O.accordion_defaults(prev, cur, low_idx=4, high_idx=1, eta=0.5)) == [4, 1, 4, 1]


def test_hybrid_table_picks_across_families(ref):
    """Two families side by side: the DP optimum over the hybrid table is the brute-force
    optimum over per-layer (family, parameter) choices."""
    rng = np.random.default_rng(8)
    for _ in range(60):
        L = int(rng.integers(1, 5))
        e1 = np.sort(rng.uniform(0, 1, (L, 2)), 1)[:, ::-1].copy()
        b1 = np.sort(rng.integers(1, 500, (L, 2)), 1).astype(np.int64)
        e2 = np.sort(rng.uniform(0, 1, (L, 2)), 1)[:, ::-1].copy()
        b2 = np.sort(rng.integers(1, 500, (L, 2)), 1).astype(np.int64)
        err, bits, cols = O.hybrid_table([e1, e2], [b1, b2])
        assert err.shape == (L, 4) and cols == [(0, 0), (0, 1), (1, 0), (1, 1)]
        dflt = np.full(L, 1, np.int32)  # family 0, second candidate
        st, ch, info = ref.solve(err, bits, dflt, None, D=100)
        best = _brute_weighted(err, bits, np.ones(L, np.int64), dflt, 100)
        got = sum(int(bits[l, ch[l]]) for l in range(L))
        if info.used_default:
            assert got == sum(int(bits[l, 1]) for l in range(L))
        else:
            assert got == best


def test_r_squared_of_the_bucket_time_fit():
    """bucket_timer.r_squared: 1 on exactly linear samples, lower with noise, and the
    least-squares fit (objectives.fit_bucket_time) recovers per-byte coefficients from
    samples shaped like the timer's (bytes per bucket, total sync time)."""
    import numpy as np
    from paper_2210_17357_b200 import objectives as O
    from paper_2210_17357_b200.bucket_timer import r_squared
    rng = np.random.default_rng(3)
    sizes = rng.uniform(1e5, 7e6, (40, 5))
    T = np.array([1.8e-8, 2.0e-8, 1.9e-8, 2.1e-8, 1.7e-8])
    y = sizes @ T + 3e-5
    Tf, c = O.fit_bucket_time(sizes, y)
    assert np.allclose(Tf, T, rtol=1e-9) and abs(c - 3e-5) < 1e-12
    assert abs(r_squared(sizes, y, Tf, c) - 1.0) < 1e-12
    yn = y + rng.normal(0, 2e-5, y.shape)
    Tn, cn = O.fit_bucket_time(sizes, yn)
    r2 = r_squared(sizes, yn, Tn, cn)
    assert 0.5 < r2 < 1.0
    assert np.all(np.abs(Tn - T) / T < 0.5)
