"""Pins for the oracle's PowerSGD power iteration, profile, ratios and exchange."""
import numpy as np
import pytest

from paper_2210_17357_b200 import workloads as W


def test_spec_examples(ref):
    # rank-1 input -> error 0; I2 with r=1 -> error 1.0
    M = np.array([[1, 2], [2, 4]], np.float64)
    Q0 = ref.psgd_init_q(0, 0, 0, 2, 1)
    P, Q = ref.psgd_power(M, Q0, 5)
    assert ref.psgd_err(M, P, Q) < 1e-12
    I2 = np.eye(2)
    P, Q = ref.psgd_power(I2, Q0, 5)
    assert abs(ref.psgd_err(I2, P, Q) - 1.0) < 1e-12


def _lowrank(m, k, seed, noise=0.1, rank=8):
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((m, rank))
    V = rng.standard_normal((k, rank))
    S = (U / np.arange(1, rank + 1)) @ V.T
    N = rng.standard_normal((m, k))
    return S + noise * np.linalg.norm(S) / np.linalg.norm(N) * N


def test_eckart_young_and_near_optimal(ref):
    # Eckart-Young: err >= sqrt(sum_{i>r} sigma_i^2) (LAPACK SVD, independent);
    # with a spectral gap 5 power steps come within 5% of it (PAPER.md:699
    # "applying only 5 power steps is enough")
    for seed, (m, k) in enumerate([(8, 6), (40, 30), (64, 200)]):
        rng = np.random.default_rng(seed)
        for r in (1, 2, 4):
            U, _ = np.linalg.qr(rng.standard_normal((m, min(m, k))))
            V, _ = np.linalg.qr(rng.standard_normal((k, min(m, k))))
            sig = np.where(np.arange(min(m, k)) < r, 1.0, 0.3) * rng.uniform(0.5, 1.0, min(m, k))
            M = (U * sig) @ V.T
            sv = np.linalg.svd(M, compute_uv=False)
            Q0 = ref.psgd_init_q(7, seed, 0, k, r)
            P, Q = ref.psgd_power(M, Q0, 5)
            e = ref.psgd_err(M, P, Q)
            opt = np.sqrt((sv[r:] ** 2).sum())
            assert e >= opt * (1 - 1e-12)
            assert e <= 1.05 * opt + 1e-12
            # and on the gap-free low-rank-plus-noise recipe the bound still holds
            M2 = _lowrank(m, k, seed)
            P, Q = ref.psgd_power(M2, Q0, 5)
            assert ref.psgd_err(M2, P, Q) >= np.sqrt((np.linalg.svd(M2, compute_uv=False)[r:] ** 2).sum()) * (1 - 1e-12)


def test_orthonormal_and_identity(ref):
    # MGS output is orthonormal; err^2 = ||M||^2 - sum_j ||q_j||^2 for orthonormal P
    M = _lowrank(50, 37, 3)
    Q0 = ref.psgd_init_q(1, 2, 3, 37, 6)
    P, Q = ref.psgd_power(M, Q0, 3)
    assert np.abs(P.T @ P - np.eye(6)).max() < 1e-12
    e = ref.psgd_err(M, P, Q)
    assert abs(e ** 2 - ((M ** 2).sum() - (Q ** 2).sum())) < 1e-10 * (M ** 2).sum()
    # an independent Gram-Schmidt: numpy QR gives the same column space and signs up to +-1
    Pm = ref.mgs(M @ Q0)
    Qr, _ = np.linalg.qr(M @ Q0)
    assert np.abs(np.abs(np.sum(Pm * Qr, 0)) - 1).max() < 1e-10


def test_zero_column_stays_zero(ref):
    P = np.zeros((5, 3))
    P[:, 0] = [1, 2, 3, 4, 5]
    P[:, 2] = P[:, 0] * 2  # dependent -> zero after projection
    Ph = ref.mgs(P)
    assert np.allclose(np.linalg.norm(Ph[:, 0]), 1) and not Ph[:, 1].any()
    assert np.linalg.norm(Ph[:, 2]) < 1e-12 or np.isclose(np.linalg.norm(Ph[:, 2]), 1)


def test_rank_prefix_consistency(ref):
    # a run at r_max contains every smaller-rank run as its first r columns
    # (Q0 is column-major-indexed, MGS is column sequential; R11)
    M = _lowrank(60, 45, 9)
    Qmax = ref.psgd_init_q(3, 1, 2, 45, 8)
    Pm, Qm = ref.psgd_power(M, Qmax, 5)
    for r in (1, 3, 5):
        Qr0 = ref.psgd_init_q(3, 1, 2, 45, r)
        assert np.array_equal(Qr0, Qmax[:, :r])
        P, Q = ref.psgd_power(M, Qr0, 5)
        assert np.abs(P - Pm[:, :r]).max() < 1e-13 and np.abs(Q - Qm[:, :r]).max() < 1e-12


def test_profile_lossless_rule_and_bits(ref):
    # r (m+k) >= m k -> sent raw: err 0, bits 32 n; else bits 32 r (m+k)
    layers = [W.Layer(0, 8 * 6, 8, 6, 1), W.Layer(48, 30, 0, 0, 0), W.Layer(78, 40 * 30, 40, 30, 1)]
    g, _ = W.low_rank_plus_noise(layers, seed=1)
    err, bits = ref.psgd_profile(layers, g, None, [1, 2, 4, 8], steps=5)
    assert list(bits[0]) == [32 * 1 * 14, 32 * 2 * 14, 32 * 48, 32 * 48]
    assert err[0, 2] == 0 and err[0, 3] == 0
    assert list(bits[1]) == [32 * 30] * 4 and not err[1].any()
    assert list(bits[2]) == [32 * r * 70 for r in (1, 2, 4, 8)]
    assert np.all(np.diff(err[2]) < 0)


@pytest.mark.parametrize("shape,r,paper", [("rn18c100", 4, 72.2), ("C4", 4, 66.5), ("C3", 32, 14.1),
                                           ("TLM", 32, 15.0)])
def test_psgd_ratio_pin(ref, shape, r, paper):
    # PAPER.md:404 (Table 1: 72.2, 66.5), :562 (Table 4 TXL r32: 14.1), :423 (Table 2 TLM: 15.0)
    layers = W.layer_table(W.resnet18_cifar(100)) if shape == "rn18c100" else W.config_layers(shape)
    N = W.total_numel(layers)
    bits = 0
    for l in layers:
        if l.compress and l.rows > 0 and not ref.psgd_lossless(l.rows, l.cols, r):
            bits += 32 * r * (l.rows + l.cols)
        else:
            bits += 32 * l.numel
    assert abs(32 * N / bits - paper) < 0.05


def test_exchange_w1_and_mean(ref):
    layers = [W.Layer(0, 30 * 20, 30, 20, 1), W.Layer(600, 10, 0, 0, 0), W.Layer(610, 16 * 40, 16, 40, 1)]
    N = W.total_numel(layers)
    gr, er = [], []
    for w in range(3):
        g, e = W.low_rank_plus_noise(layers, seed=10 + w, with_ef=True)
        gr.append(g)
        er.append(e)
    lrank = [3, 0, 2]
    Qs = {0: ref.psgd_init_q(5, 0, 0, 20, 3), 2: ref.psgd_init_q(5, 2, 0, 40, 2)}
    Q00 = {k: v.copy() for k, v in Qs.items()}
    out, es, Ps = ref.psgd_allreduce(layers, lrank, gr, er, Qs)
    # independent numpy restatement of one PowerSGD step (Vogels et al. 2019)
    xs = [((gr[w] + er[w]) + np.float32(0)).astype(np.float32) for w in range(3)]
    for l, ly in ((0, layers[0]), (2, layers[2])):
        Ms = [x[ly.offset:ly.offset + ly.numel].astype(np.float64).reshape(ly.rows, ly.cols) for x in xs]
        Pb = sum(M @ Q00[l] for M in Ms) / 3
        Ph, _ = np.linalg.qr(Pb)
        Ph *= np.sign(np.sum(Ph * Ps[l], 0))
        assert np.abs(Ph - Ps[l]).max() < 1e-10
        Qb = sum(M.T @ Ph for M in Ms) / 3
        assert np.abs(Qb - Qs[l]).max() < 1e-10 * np.abs(Qb).max()
        rec = (Ph @ Qb.T).astype(np.float32).reshape(-1)
        assert np.abs(out[ly.offset:ly.offset + ly.numel] - rec).max() <= 1e-6 * np.abs(rec).max()
        for w in range(3):
            assert np.array_equal(es[w][ly.offset:ly.offset + ly.numel],
                                  (xs[w][ly.offset:ly.offset + ly.numel] - out[ly.offset:ly.offset + ly.numel]))
    s = (xs[0][600:610] + xs[1][600:610]).astype(np.float32)
    s = (s + xs[2][600:610]).astype(np.float32)
    assert np.array_equal(out[600:610], (s * np.float32(1 / 3)).astype(np.float32))


def test_rank_deficient(ref):
    # exactly rank-2 M (in fp64): the extra power-iteration columns are dependent and
    # dropped, err_r = 0 for r >= 2; the fp32-rounded rank-2 matrix has a
    # tiny noise spectrum and err_r follows Eckart-Young (LAPACK) closely, including the
    # nearly dependent columns for r > 2 (the reorthogonalisation sweep keeps P orthonormal)
    rng = np.random.default_rng(0)
    A, B = rng.standard_normal((50, 2)), rng.standard_normal((2, 40))
    M = A @ B
    for r in (2, 4, 8):
        P, Q = ref.psgd_power(M, ref.psgd_init_q(1, 0, 0, 40, r), 5)
        assert ref.psgd_err(M, P, Q) <= 1e-12 * np.linalg.norm(M)
    M32 = M.astype(np.float32).astype(np.float64)
    sv = np.linalg.svd(M32, compute_uv=False)
    for r in (2, 4, 8):
        P, Q = ref.psgd_power(M32, ref.psgd_init_q(1, 0, 0, 40, r), 5)
        assert np.abs(P.T @ P - np.diag((np.linalg.norm(P, axis=0) > 0).astype(float))).max() < 1e-12
        assert ref.psgd_err(M32, P, Q) <= 2.0 * np.sqrt((sv[r:] ** 2).sum())
