"""GPU parity of K4 (Algorithm 1 on device) vs the oracle: identical tables in,
bit-exact choices and summary out."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lg():
    from paper_2210_17357_b200 import lgreco
    return lgreco


def _run(lg, err, bits, dflt, compress, D, flags):
    e = torch.from_numpy(np.array(err, dtype=np.float64, order="C", copy=True)).cuda()
    b = torch.from_numpy(np.array(bits, dtype=np.int64, order="C", copy=True)).cuda()
    d = torch.from_numpy(np.asarray(dflt, np.int32)).cuda()
    c = None if compress is None else torch.from_numpy(np.asarray(compress, np.int32)).cuda()
    choice, info = lg.solve(e, b, d, c, D=D, flags=flags)
    torch.cuda.synchronize()
    return choice.cpu().numpy(), lg.read_info(info)


def _table(rng, L, K, zero_frac=0.0):
    err = np.sort(rng.uniform(0, 1, (L, K)) * rng.uniform(0.01, 10, (L, 1)), 1)[:, ::-1].copy()
    if zero_frac:
        err[rng.random((L, K)) < zero_frac] = 0.0
    bits = np.sort(rng.integers(64, 10 ** 7, (L, K)), 1).astype(np.int64)
    return err, bits


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 4, 7, 8, 9])
def test_random_tables(lg, ref, flags):
    """flags bit 2 (LGRECO_SOLVE_SINGLE_CTA) selects the one-CTA kernel, otherwise the
    8-CTA cluster kernel runs (K <= 16): both must reproduce the oracle exactly."""
    rng = np.random.default_rng(flags)
    for trial in range(40):
        L = int(rng.integers(1, 30))
        K = int(rng.integers(1, 9))
        D = int(rng.choice([1, 7, 100, 1000, 10000]))
        err, bits = _table(rng, L, K, zero_frac=0.2 if trial % 4 == 0 else 0.0)
        dflt = rng.integers(0, K, L).astype(np.int32)
        comp = (rng.random(L) < 0.8).astype(np.int32) if trial % 3 == 0 else None
        st, c_ref, i_ref = ref.solve(err, bits, dflt, comp, D=D, flags=flags & 3)
        c_gpu, i_gpu = _run(lg, err, bits, dflt, comp, D, flags)
        assert st == 0 and i_gpu.status == 0
        assert list(c_gpu) == list(c_ref)
        assert (i_gpu.total_bits, i_gpu.default_bits, i_gpu.used_default, i_gpu.n_active) == \
            (i_ref.total_bits, i_ref.default_bits, i_ref.used_default, i_ref.n_active)
        assert i_gpu.emax == i_ref.emax and i_gpu.total_err == i_ref.total_err


@pytest.mark.parametrize("cfg,K,flags", [("C4", 7, 0), ("C4", 7, 8), ("C3", 100, 0), ("C5", 100, 0), ("C5", 49, 0),
                                         ("C5", 7, 8)])
def test_model_sized_tables(lg, ref, cfg, K, flags):
    """flags 8 = LGRECO_SOLVE_NARROW (8-CTA clusters, the pipelined bench's solve)."""
    layers = W.config_layers(cfg)
    L = len(layers)
    rng = np.random.default_rng(K + L)
    err, bits = _table(rng, L, K)
    comp = np.array([l.compress for l in layers], np.int32)
    dflt = np.full(L, K // 3, np.int32)
    st, c_ref, i_ref = ref.solve(err, bits, dflt, comp, D=10000)
    c_gpu, i_gpu = _run(lg, err, bits, dflt, comp, 10000, flags)
    assert list(c_gpu) == list(c_ref) and i_gpu.total_bits == i_ref.total_bits
    assert i_gpu.total_bits <= i_gpu.default_bits


def test_nonfinite_table(lg):
    err = np.array([[1.0, np.inf], [0.5, 0.2]])
    bits = np.array([[1, 2], [1, 2]], np.int64)
    c, info = _run(lg, err, bits, [0, 0], None, 100, 0)
    assert info.status == lg.ENONFINITE


def test_worked_example(lg):
    err = np.array([[0.0, 1.0, 2.0], [0.0, 2.0, 5.0]])
    bits = np.array([[100, 60, 20], [120, 100, 40]], np.int64)
    c, info = _run(lg, err, bits, [1, 1], None, 300, 0)
    assert list(c) == [2, 0] and info.total_bits == 140


@pytest.mark.parametrize("single", [False, True])
@pytest.mark.parametrize("K", [1, 3, 5, 7, 8, 12, 16, 17, 33, 100])
def test_narrow_keys_ties_and_bands(lg, ref, K, single):
    """Small costs (32-bit keys: the K <= 16 unrolled path, the grouped K > 16 path),
    quantised errors so that many (layer, candidate) pairs tie in both disc and cost
    (tie-breaks R19), and a few inadmissible candidates (disc > D, R17) so that the
    reachable band is ragged."""
    rng = np.random.default_rng(100 + K)
    for D in (100, 5000, 10000, 12000):
        L = int(rng.integers(20, 160))
        err = np.sort(rng.integers(0, 6, (L, K)).astype(np.float64) * rng.choice([0.5, 1.0, 2.0], (L, 1)), 1)[:, ::-1]
        err = err.copy()  # a fresh C-ordered array (the reversed view has negative strides)
        err[rng.random((L, K)) < 0.03] = 1e6  # disc > D -> skipped
        bits = np.sort(rng.integers(1, 40, (L, K)), 1).astype(np.int64) * 64
        dflt = np.full(L, K - 1, np.int32)  # the default must stay admissible
        err[:, K - 1] = np.minimum(err[:, K - 1], 1.0)
        comp = (rng.random(L) < 0.85).astype(np.int32)
        st, c_ref, i_ref = ref.solve(err, bits, dflt, comp, D=D)
        c_gpu, i_gpu = _run(lg, err, bits, dflt, comp, D, 4 if single else 0)
        assert st == 0 and i_gpu.status == 0
        assert list(c_gpu) == list(c_ref), (K, D)
        assert (i_gpu.total_bits, i_gpu.used_default) == (i_ref.total_bits, i_ref.used_default)
        assert i_gpu.emax == i_ref.emax and i_gpu.total_err == i_ref.total_err


def test_weighted_costs_and_solve(lg, ref):
    """NEXT-1: the device product bits * w is exact (-1 on
    overflow or a negative input), and the solve on it reproduces the oracle's weighted
    plan (C4-sized table, DDP bucket-priority weights)."""
    from paper_2210_17357_b200 import objectives as O
    layers = W.config_layers("C4")
    L, K = len(layers), 7
    rng = np.random.default_rng(77)
    err, bits = _table(rng, L, K)
    w = O.bucket_priority_weights(layers)
    b_d = torch.from_numpy(bits).cuda()
    w_d = torch.from_numpy(w).cuda()
    wb = lg.weight_costs(b_d, w_d).cpu().numpy()
    assert np.array_equal(wb, bits * w[:, None])
    # overflow and negative inputs -> -1
    big = torch.tensor([[2 ** 62, 5], [-3, 7]], dtype=torch.int64, device="cuda")
    ww = torch.tensor([4, -1], dtype=torch.int64, device="cuda")
    assert lg.weight_costs(big, ww).cpu().tolist() == [[-1, 20], [-1, -1]]
    comp = np.array([l.compress for l in layers], np.int32)
    dflt = np.full(L, 2, np.int32)
    st, c_ref, i_ref = ref.solve(err, bits * w[:, None], dflt, comp, D=10000)
    c_gpu, i_gpu = _run(lg, err, wb, dflt, comp, 10000, 0)
    assert list(c_gpu) == list(c_ref) and i_gpu.total_bits == i_ref.total_bits


@pytest.mark.parametrize("groups", ["2", "1"])
def test_layer_groups_bit_exact(lg, ref, groups, monkeypatch):
    """The two-group solve (k_solve_cl on two clusters + k_solve_join, forced for every
    table size with LGRECO_DP_GROUPS=2) reproduces the oracle's plan exactly: random and
    tie-heavy tables (many optimal plans, so |E2| > 1 and the lexicographic walk of the
    top group decides), 1..80 layers (split points at the edges: La = 0, 1, 2), all
    layers inactive, D from 1 to 10000."""
    monkeypatch.setenv("LGRECO_DP_GROUPS", groups)
    rng = np.random.default_rng(7 + int(groups))
    n_multi = 0
    for trial in range(120):
        L = int(rng.integers(1, 81))
        K = int(rng.integers(1, 17))
        D = int(rng.choice([1, 7, 100, 1000, 10000]))
        if trial % 2:
            err = rng.integers(0, 4, (L, K)).astype(np.float64) * rng.choice([0.5, 1.0], (L, 1))
            bits = rng.integers(1, 4, (L, K)).astype(np.int64) * 64
        else:
            err, bits = _table(rng, L, K, zero_frac=0.1)
        dflt = rng.integers(0, K, L).astype(np.int32)
        comp = (rng.random(L) < rng.choice([0.0, 0.5, 1.0])).astype(np.int32) if trial % 5 == 0 else None
        st, c_ref, i_ref = ref.solve(err, bits, dflt, comp, D=D)
        c_gpu, i_gpu = _run(lg, err, bits, dflt, comp, D, 0)
        assert st == 0 and i_gpu.status == 0
        assert list(c_gpu) == list(c_ref), (trial, L, K, D)
        assert (i_gpu.total_bits, i_gpu.default_bits, i_gpu.used_default, i_gpu.n_active) == \
            (i_ref.total_bits, i_ref.default_bits, i_ref.used_default, i_ref.n_active)
        assert i_gpu.emax == i_ref.emax and i_gpu.total_err == i_ref.total_err
        n_multi += trial % 2
    assert n_multi > 0


def test_solve_host_mode(lg, ref):
    """lgreco_solve with HOST tables and outputs (SURVEY 8(b)'s host mode): staged through
    device scratch around the same kernels; the plan and summary equal the oracle's, and
    mixing host and device pointers is refused."""
    layers = W.config_layers("C4")
    L, K = len(layers), 7
    rng = np.random.default_rng(5)
    err, bits = _table(rng, L, K)
    comp = np.array([l.compress for l in layers], np.int32)
    dflt = np.full(L, 2, np.int32)
    st, c_ref, i_ref = ref.solve(err, bits, dflt, comp, D=10000)
    ch, inf = lg.solve_host(err, bits, dflt, comp)
    assert list(ch) == list(c_ref) and inf.total_bits == i_ref.total_bits and inf.emax == i_ref.emax
    ch2, _ = lg.solve_host(err, bits, dflt, None, D=1000, flags=4)
    st2, c_ref2, _ = ref.solve(err, bits, dflt, None, D=1000)
    assert list(ch2) == list(c_ref2)
    import ctypes as C
    e_d = torch.from_numpy(err).cuda()
    b_h = np.ascontiguousarray(bits)
    d_h = np.ascontiguousarray(dflt)
    out_h = np.empty(L, np.int32)
    info = lg.SolveInfo()
    rc = lg.lib().lgreco_solve(e_d.data_ptr(), b_h.ctypes.data, L, K, d_h.ctypes.data, None, 10000, 0,
                               out_h.ctypes.data, C.addressof(info), None, 0, None)
    assert rc == lg.EINVAL
