"""Pins for the oracle's TopK sparsifier, its profile and its exchange."""
import itertools

import numpy as np
import pytest

from paper_2210_17357_b200 import workloads as W


def test_spec_example(ref):
    # [3,-1,0.5,2], density 0.5 (k=2) -> [3,0,0,2], error sqrt(1.25)
    layers = [W.Layer(0, 4, 0, 0, 1)]
    g = np.array([3, -1, 0.5, 2], np.float32)
    assert ref.topk_k(4, 500000) == 2
    err, bits = ref.topk_profile(layers, g, None, [500000])
    assert abs(err[0, 0] - np.sqrt(1.25)) < 1e-15 and bits[0, 0] == 128
    pay, e2 = ref.topk_pack(layers, [500000], g, np.zeros(4, np.float32))
    pairs = pay.view(np.uint32).reshape(-1, 2)
    assert list(pairs[:, 0]) == [0, 3]
    assert list(pairs[:, 1].view(np.float32)) == [3.0, 2.0]
    assert list(e2) == [0.0, -1.0, 0.5, 0.0]


def test_k_rule(ref):
    # k = max(1, ceil(density*n)), density in ppm, integer arithmetic
    assert ref.topk_k(1000, 1000) == 1
    assert ref.topk_k(1001, 1000) == 2
    assert ref.topk_k(10, 1) == 1
    assert ref.topk_k(7, 1000000) == 7
    assert ref.topk_k(137080320, 1000) == 137081


def test_exhaustive_k_sparse_optimum(ref):
    # err equals the minimum l2 error over all k-sparse approximations
    rng = np.random.default_rng(0)
    for trial in range(30):
        n = int(rng.integers(1, 11))
        x = rng.standard_normal(n).astype(np.float32)
        if trial % 3 == 0:  # force ties
            x[rng.integers(0, n, n // 2)] = x[0]
        k = int(rng.integers(1, n + 1))
        ppm = k * 1000000 // n
        assert ref.topk_k(n, ppm) == k
        best = min(sum(float(x[i]) ** 2 for i in range(n) if i not in S)
                   for S in itertools.combinations(range(n), k))
        err, _ = ref.topk_profile([W.Layer(0, n, 0, 0, 1)], x, None, [ppm])
        assert abs(err[0, 0] - np.sqrt(best)) <= 1e-12
        idx = ref.topk_select(x, k)
        # selection: k largest |x|, ties to the lower index
        order = sorted(range(n), key=lambda i: (-abs(float(x[i])), i))[:k]
        assert list(idx) == sorted(order)


def test_sort_based_error(ref):
    # err = sqrt(sum of the n-k smallest squares), a textbook sort check
    layers = W.config_layers("C1")[:6]
    g, e = W.heavy_tailed(layers, seed=3)
    ppm = [1000, 10000, 100000, 500000, 1000000]
    err, bits = ref.topk_profile(layers, g, e, ppm)
    x = ((g + e) + np.float32(0)).astype(np.float32)
    for li, l in enumerate(layers):
        sq = np.sort(x[l.offset:l.offset + l.numel].astype(np.float64) ** 2)
        for j, p in enumerate(ppm):
            k = ref.topk_k(l.numel, p)
            assert abs(err[li, j] - np.sqrt(sq[:l.numel - k].sum())) <= 1e-9 * max(err[li, j], 1e-300)
            assert bits[li, j] == 64 * k
        assert err[li, -1] == 0.0  # density 100% -> identity


def test_ef_exact_and_idempotent(ref):
    layers = W.config_layers("C1")[:5] + []
    g, e = W.heavy_tailed(layers, seed=5)
    lppm = [10000, 50000, 1000, 1000000, 300000]
    pay, e2 = ref.topk_pack(layers, lppm, g, e)
    x = ((g + e) + np.float32(0)).astype(np.float32)
    S, bo = ref.topk_layout(layers, lppm)
    dec = np.zeros_like(x)
    for li, l in enumerate(layers):
        k = ref.topk_k(l.numel, lppm[li])
        pr = pay[bo[li]:bo[li] + 8 * k].view(np.uint32).reshape(-1, 2)
        assert np.all(np.diff(pr[:, 0].astype(np.int64)) > 0)
        dec[l.offset + pr[:, 0]] = pr[:, 1].view(np.float32)
    # x == dec + e' bitwise (kept entries moved, the rest untouched)
    assert np.array_equal(np.where(dec != 0, dec, e2), x)
    assert np.all((dec == 0) | (e2 == 0))
    # idempotence: compressing the decoded vector reproduces it
    pay2, e3 = ref.topk_pack(layers, lppm, dec, np.zeros_like(dec))
    assert np.array_equal(pay2, pay) and not e3.any()


def test_exchange(ref):
    layers = W.config_layers("C1")[:4]
    N = W.total_numel(layers)
    lppm = [20000, 100000, 5000, 0]
    layers = layers[:3] + [W.Layer(layers[3].offset, layers[3].numel, 0, 0, 0)]
    gr, er = [], []
    for w in range(4):
        g, e = W.heavy_tailed(layers, seed=40 + w)
        gr.append(g)
        er.append(e)
    out, es, pays = ref.topk_allreduce(layers, lppm, gr, er)
    # reconstruct independently: dense decode of each rank, ordered fp32 sum
    acc = np.zeros(N, np.float32)
    S, bo = ref.topk_layout(layers, lppm)
    for w in range(4):
        p = pays[w]
        for li, l in enumerate(layers[:3]):
            k = ref.topk_k(l.numel, lppm[li])
            pr = p[bo[li]:bo[li] + 8 * k].view(np.uint32).reshape(-1, 2)
            acc[l.offset + pr[:, 0]] = (acc[l.offset + pr[:, 0]] + pr[:, 1].view(np.float32) * np.float32(0.25)).astype(np.float32)
    ll = layers[3]
    sl = slice(ll.offset, ll.offset + ll.numel)
    xs = [((gr[w] + er[w]) + np.float32(0)).astype(np.float32) for w in range(4)]
    s = xs[0][sl].copy()
    for w in range(1, 4):
        s = (s + xs[w][sl]).astype(np.float32)
    acc[sl] = s * np.float32(0.25)
    assert np.array_equal(out, acc)
    # W=1: out == local dec
    out1, es1, p1 = ref.topk_allreduce(layers, lppm, gr[:1], er[:1])
    assert np.array_equal(np.where(out1 != 0, out1, es1[0]), xs[0])


@pytest.mark.parametrize("shape,ppm,paper", [("rn18c100", 10000, 48.1), ("C4", 10000, 45.6),
                                             ("C3", 100000, 4.9), ("TLM", 100000, 4.9)])
def test_topk_ratio_pin(ref, shape, ppm, paper):
    # PAPER.md:402 (Table 1 TopK 1%: 48.1 / 45.6), :421 (Table 2 TopK 10%: 4.9);
    # 64 bits per kept entry, 1-D tensors raw (R8)
    layers = W.layer_table(W.resnet18_cifar(100)) if shape == "rn18c100" else W.config_layers(shape)
    N = W.total_numel(layers)
    bits = sum(64 * ref.topk_k(l.numel, ppm) if l.compress else 32 * l.numel for l in layers)
    assert abs(32 * N / bits - paper) / paper < 0.02  # printed to 1 decimal; 10% caps at 5.0
