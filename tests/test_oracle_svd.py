"""Pins for the oracle's SVD-based low-rank errors (NEXT-2): a matrix
with prescribed singular values (closed form), Eckart-Young optimality against the
oracle's power method (and the paper's "5 power steps" closeness), the lossless rule."""
import numpy as np

from paper_2210_17357_b200 import workloads as W


def _layer_set(shapes):
    out, off = [], 0
    for m, k, c in shapes:
        out.append(W.Layer(off, m * k, m, k, c) if m > 1 else W.Layer(off, k, 0, 0, c))
        off += m * k
    return out


def test_prescribed_singular_values(ref):
    rng = np.random.default_rng(3)
    m, k = 60, 45
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    V, _ = np.linalg.qr(rng.standard_normal((k, k)))
    s = np.sort(rng.uniform(0.1, 2.0, k))[::-1]
    M = (U[:, :k] * s) @ V.T
    g = M.astype(np.float32).ravel()
    layers = _layer_set([(m, k, 1)])
    ranks = [1, 2, 5, 10, 20]
    err, bits = ref.psgd_svd_profile(layers, g, None, ranks)
    # the fp32 rounding of M perturbs sigma_i by ~1e-7 |M|
    for j, r in enumerate(ranks):
        assert abs(err[0, j] - np.sqrt(np.sum(s[r:] ** 2))) <= 1e-5 * np.sqrt(np.sum(s ** 2))
        assert bits[0, j] == 32 * r * (m + k)


def test_optimal_vs_power_method(ref):
    rng = np.random.default_rng(4)
    shapes = [(64, 96, 1), (1, 50, 0), (120, 30, 1), (8, 8, 1)]
    layers = _layer_set(shapes)
    N = sum(m * k for m, k, _ in shapes)
    g = np.zeros(N, np.float32)
    for ly in layers:
        if ly.rows > 0:
            m, k = ly.rows, ly.cols
            A = rng.standard_normal((m, 6)) @ rng.standard_normal((6, k)) * np.linspace(3, 1, 6)[:6].sum()
            g[ly.offset:ly.offset + ly.numel] = (A + 0.05 * rng.standard_normal((m, k))).astype(np.float32).ravel()
    e = (rng.standard_normal(N) * 1e-3).astype(np.float32)
    ranks = [1, 2, 4, 8]
    es, bs = ref.psgd_svd_profile(layers, g, e, ranks)
    ep, bp = ref.psgd_profile(layers, g, e, ranks)
    assert np.array_equal(bs, bp)  # same size rule (R11)
    assert np.all(es <= ep * (1 + 1e-9) + 1e-12)  # Eckart-Young: SVD error is optimal
    lossy = bs != 32 * np.array([l.numel for l in layers])[:, None]
    assert np.all(ep[lossy] <= 1.05 * es[lossy])  # 5 power steps are close
    assert np.all(es[~lossy] == 0)
