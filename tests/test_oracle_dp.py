"""Pins for the oracle's Algorithm 1: brute force, worked
example, invariants, discretisation examples, fallbacks."""
import itertools
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _disc(err, D, emax, floor=False):
    if emax == 0:
        return 0 if err == 0 else None
    q = (err * D) / emax
    r = math.floor(q) if floor else math.ceil(q)
    return None if r > D else int(r)


def _brute(err, bits, dflt, D, floor=False):
    """Exhaustive optimum of the discretised problem."""
    L, K = err.shape
    emax = sum(err[l, dflt[l]] for l in range(L))
    best = None
    for a in itertools.product(range(K), repeat=L):
        ds = [_disc(err[l, a[l]], D, emax, floor) for l in range(L)]
        if any(d is None for d in ds) or sum(ds) > D:
            continue
        c = sum(int(bits[l, a[l]]) for l in range(L))
        if best is None or c < best:
            best = c
    return best, emax


def test_worked_example(ref):
    rows = [l.split("#")[0].split() for l in open(os.path.join(GOLD, "dp_worked_example.txt"))]
    rows = [r for r in rows if r]
    err = np.array([[float(v) for v in r[1:]] for r in rows if r[0] == "err"])
    bits = np.array([[int(v) for v in r[1:]] for r in rows if r[0] == "bits"])
    d = {r[0]: r[1:] for r in rows if r[0] not in ("err", "bits")}
    for flags in (0, ref.DISC_FLOOR):
        st, choice, info = ref.solve(err, bits, [int(v) for v in d["default"]], D=int(d["D"][0]), flags=flags)
        assert st == 0
        assert list(choice) == [int(v) for v in d["choice"]]
        assert info.total_bits == int(d["total_bits"][0]) and info.emax == 3.0
        assert info.used_default == 0 and info.total_err == 2.0


def test_discretisation_examples(ref):
    # Emax=3, D=300 -> 1.0 maps to 100; 0.004 maps to 0 (floor) / 1 (ceil).
    # Observed through the solver: a layer whose cheap candidate has error 0.004.
    err = np.array([[0.004, 0.0], [3.0 - 0.004, 3.0 - 0.004]])
    err[0, 1] = 0.0
    bits = np.array([[10, 20], [5, 5]])
    # layer 0 default = 1 (err 0), layer 1 default 0 -> Emax = 2.996; ceil makes 0.004 cost 1 bin
    st, choice, info = ref.solve(err, bits, [1, 0], D=300)
    assert st == 0
    # with ceil, the cheap candidate needs disc(0.004)=1 extra bin beyond disc(2.996)=300 -> infeasible
    assert list(choice) == [1, 0]
    st, choice, info = ref.solve(err, bits, [1, 0], D=300, flags=ref.DISC_FLOOR)
    # floor: 0 bins -> picked, but raw error 3.0 > Emax 2.996 -> R20 fallback to defaults
    assert list(choice) == [1, 0] and info.used_default == 1
    assert _disc(1.0, 300, 3.0) == 100 and _disc(0.004, 300, 3.0, True) == 0 and _disc(0.004, 300, 3.0) == 1


def test_floor_can_exceed_uniform_error_ceil_cannot(ref):
    # 2 layers, err {1.19 cheap, 1.0 default}, D=10 -> floor picks both
    # cheap ones (raw 2.38 > Emax 2.0); the R20 check restores the defaults.
    err = np.array([[1.19, 1.0], [1.19, 1.0]])
    bits = np.array([[1, 2], [1, 2]])
    st, c, info = ref.solve(err, bits, [1, 1], D=10, flags=ref.DISC_FLOOR)
    assert list(c) == [1, 1] and info.used_default == 1
    st, c, info = ref.solve(err, bits, [1, 1], D=10)
    assert info.total_err <= info.emax


@pytest.mark.parametrize("floor", [False, True])
def test_brute_force_random(ref, floor):
    rng = np.random.default_rng(123 + floor)
    for trial in range(150):
        L = int(rng.integers(1, 6))
        K = int(rng.integers(1, 5))
        D = int(rng.integers(1, 200))
        err = np.sort(rng.uniform(0, 3, (L, K)), 1)[:, ::-1].copy()
        if trial % 5 == 0:
            err[rng.random((L, K)) < 0.3] = 0.0
        bits = np.sort(rng.integers(1, 100, (L, K)), 1)
        if trial % 7 == 0:
            bits = rng.integers(1, 100, (L, K))
        dflt = rng.integers(0, K, L)
        best, emax = _brute(err, bits, dflt, D, floor)
        st, choice, info = ref.solve(err, bits, dflt, D=D, flags=ref.DISC_FLOOR if floor else 0)
        assert st == 0
        default_bits = sum(int(bits[l, dflt[l]]) for l in range(L))
        if info.used_default:
            # either nothing feasible, the optimum is worse than the defaults, or (floor) raw
            # error above Emax
            assert list(choice) == list(dflt)
            assert best is None or best >= default_bits or floor or \
                sum(err[l, choice[l]] for l in range(L)) <= emax
        else:
            assert info.total_bits == best
            ds = [_disc(err[l, choice[l]], D, emax, floor) for l in range(L)]
            assert sum(ds) <= D
        # invariants: never worse than defaults; ceil mode never above Emax in raw error
        assert info.total_bits <= default_bits
        if not floor:
            assert sum(err[l, choice[l]] for l in range(L)) <= emax


def test_single_candidate_and_zero_emax(ref):
    err = np.array([[0.5], [0.2], [0.0]])
    bits = np.array([[7], [9], [1]])
    st, c, info = ref.solve(err, bits, [0, 0, 0], D=100)
    assert list(c) == [0, 0, 0] and info.total_bits == 17
    # Emax = 0 (lossless defaults) -> only zero-error candidates
    err = np.array([[0.3, 0.0], [0.1, 0.0]])
    bits = np.array([[1, 32], [1, 32]])
    st, c, info = ref.solve(err, bits, [1, 1], D=100)
    assert list(c) == [1, 1] and info.emax == 0.0


def test_inactive_layers_and_errors(ref):
    err = np.array([[1.0, 0.5], [9.0, 9.0], [2.0, 1.0]])
    bits = np.array([[1, 2], [100, 100], [3, 4]])
    st, c, info = ref.solve(err, bits, [1, 0, 1], compress=[1, 0, 1], D=1000)
    assert st == 0 and c[1] == -1 and info.n_active == 2
    bad = err.copy()
    bad[0, 0] = np.nan
    st, c, info = ref.solve(bad, bits, [1, 0, 1], D=1000)
    assert st == ref.REF_ENONFINITE
    st, *_ = ref.solve(err, bits, [1, 0, 1], D=0)
    assert st == ref.REF_EINVAL


def test_literal_init_differs(ref):
    # Alg.1 line 10 literally *assigns* DP[1][Errors[1][c]] = Costs[1][c],
    # so a later, costlier candidate with the same bin overwrites a cheaper one.  The min-update
    # reading agrees with brute force where the literal one does not.
    err = np.array([[1.0, 1.0], [0.0, 0.0]])
    bits = np.array([[10, 50], [60, 70]])
    st, c, info = ref.solve(err, bits, [0, 0], D=10)
    assert info.total_bits == 70 == _brute(err, bits, [0, 0], 10)[0]
    # literal: DP1[10] = 50 (overwritten) -> best 110
    assert 50 + 60 == 110


def test_monotone_in_budget(ref):
    # a larger error budget (more bins at the same step) never increases the optimum
    rng = np.random.default_rng(5)
    for _ in range(30):
        L, K = 4, 3
        err = np.sort(rng.uniform(0, 2, (L, K)), 1)[:, ::-1].copy()
        bits = np.sort(rng.integers(1, 50, (L, K)), 1)
        dflt = np.full(L, 1)
        b1, emax = _brute(err, bits, dflt, 100)
        # doubling D with doubled Emax keeps the step and doubles the budget
        b2 = None
        for a in itertools.product(range(K), repeat=L):
            ds = [math.ceil(err[l, a[l]] * 100 / emax) for l in range(L)]
            if sum(ds) <= 200:
                c = sum(int(bits[l, a[l]]) for l in range(L))
                b2 = c if b2 is None or c < b2 else b2
        assert b1 is None or b2 <= b1
