"""ctypes wrapper around oracle/liblgreco_ref.so (the CPU oracle).

TEST INFRASTRUCTURE ONLY: importable by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never by the product package.
Shares nothing with paper_2210_17357_b200/ except the seeded input generators.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lgreco_ref.c")
_LIB = os.path.join(_HERE, "liblgreco_ref.so")
# the same source built with -fopenmp: layers of the QSGD profile / pack / unpack on all
# host cores (a timing baseline for bench.py's cpu_baseline; identical results)
_LIB_OMP = os.path.join(_HERE, "liblgreco_ref_omp.so")

REF_OK, REF_EINVAL, REF_ENONFINITE, REF_EINFEASIBLE, REF_ENOMEM = 0, -1, -2, -3, -6
METRIC_SQ, DISC_FLOOR = 1, 2


def build(force: bool = False, omp: bool = False) -> str:
    out = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC"] +
                              (["-fopenmp"] if omp else []) + ["-shared", "-o", out, _SRC, "-lm"])
    return out


class Layer(C.Structure):
    _fields_ = [("offset", C.c_int64), ("numel", C.c_int64), ("rows", C.c_int32),
                ("cols", C.c_int32), ("compress", C.c_int32)]


class SolveInfo(C.Structure):
    _fields_ = [("emax", C.c_double), ("total_err", C.c_double), ("total_bits", C.c_int64),
                ("default_bits", C.c_int64), ("used_default", C.c_int32), ("n_active", C.c_int32)]


_lib = None
_use_omp = False


def use_openmp(on: bool) -> None:
    """Switch the oracle to its OpenMP build (same source, layers in parallel) or back."""
    global _lib, _use_omp
    if on != _use_omp:
        _use_omp, _lib = on, None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build(omp=_use_omp))
        _lib.ref_uniform.restype = C.c_float
        _lib.ref_layout.restype = C.c_int64
        _lib.ref_topk_k.restype = C.c_int64
        _lib.ref_topk_layout.restype = C.c_int64
        _lib.ref_psgd_err.restype = C.c_double
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _layers(layers):
    arr = (Layer * max(1, len(layers)))()
    for i, l in enumerate(layers):
        arr[i] = Layer(l.offset, l.numel, l.rows, l.cols, l.compress)
    return arr


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _f32(x):
    return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _check(st, what):
    if st != REF_OK:
        raise RuntimeError(f"oracle {what} failed: status {st}")


# -------------------------------------------------------------------- Philox
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().ref_philox4x32_10(c, k, o)
    return tuple(o)


def bucket_uniforms(seed, rankfield, step, stream, gb, B, nvalid):
    u = np.zeros(nvalid, np.float32)
    lib().ref_bucket_uniforms(C.c_uint64(seed), C.c_uint32(rankfield), C.c_uint64(step),
                              C.c_uint32(stream), C.c_int64(gb), C.c_int32(B), C.c_int32(nvalid), _p(u))
    return u


# ------------------------------------------------------------- accumulation
def accumulate(G, g):
    """Row a1: returns a copy of G with g added (fp32, one add each)."""
    out = _f32(G).copy()
    lib().ref_accumulate(_p(out), _p(_f32(g)), C.c_int64(out.size))
    return out


# ----------------------------------------------------------------- quantiser
def quantize_bucket(x, bits, u):
    x = _f32(x)
    u = _f32(u)
    n = x.size
    q = np.zeros(n, np.uint32)
    dec = np.zeros(n, np.float32)
    mn = C.c_float()
    unit = C.c_float()
    st = lib().ref_quantize_bucket(_p(x), C.c_int32(n), C.c_int32(bits), _p(u), _p(q), _p(dec),
                                   C.byref(mn), C.byref(unit))
    return st, q, dec, mn.value, unit.value


def layout(layers, lbits, B):
    L = len(layers)
    bs = np.zeros(L + 1, np.int64)
    bo = np.zeros(L + 1, np.int64)
    S = lib().ref_layout(_layers(layers), C.c_int32(L), _p(_i32(lbits)), C.c_int32(B), _p(bs), _p(bo))
    return int(S), bs, bo


def qsgd_profile(layers, g, e, cand_bits, B=128, seed=0, rank=0, step=0):
    L, K = len(layers), len(cand_bits)
    err = np.zeros((L, K), np.float64)
    bits = np.zeros((L, K), np.int64)
    st = lib().ref_qsgd_profile(_layers(layers), C.c_int32(L), _p(_f32(g)), _p(_f32(e)),
                                _p(_i32(cand_bits)), C.c_int32(K), C.c_int32(B), C.c_uint64(seed),
                                C.c_uint32(rank), C.c_uint64(step), _p(err), _p(bits))
    _check(st, "qsgd_profile")
    return err, bits


def qsgd_pack(layers, lbits, g, e, B=128, seed=0, rank=0, step=0, want_dec=False):
    """Returns (payload u8, e' (copy) or None, dec or None)."""
    S, _, _ = layout(layers, lbits, B)
    pay = np.zeros(max(S, 1), np.uint8)
    e2 = None if e is None else _f32(e).copy()
    n = len(g)
    dec = np.zeros(n, np.float32) if want_dec else None
    st = lib().ref_qsgd_pack(_layers(layers), C.c_int32(len(layers)), _p(_i32(lbits)), C.c_int32(B),
                             C.c_uint64(seed), C.c_uint32(rank), C.c_uint64(step), _p(_f32(g)), _p(e2),
                             _p(pay), _p(dec))
    _check(st, "qsgd_pack")
    return pay[:S], e2, dec


def qsgd_unpack(layers, lbits, payload, N, B=128):
    out = np.zeros(N, np.float32)
    pay = np.ascontiguousarray(payload, dtype=np.uint8)
    st = lib().ref_qsgd_unpack(_layers(layers), C.c_int32(len(layers)), _p(_i32(lbits)), C.c_int32(B),
                               _p(pay), _p(out))
    _check(st, "qsgd_unpack")
    return out


def shard_bounds(layers, lbits, B, W):
    rb = np.zeros(W + 1, np.int64)
    bb = np.zeros(W + 1, np.int64)
    lib().ref_shard_bounds(_layers(layers), C.c_int32(len(layers)), _p(_i32(lbits)), C.c_int32(B),
                           C.c_int32(W), _p(rb), _p(bb))
    return rb, bb


def qsgd_allreduce(layers, lbits, g_ranks, e_ranks, B=128, seed=0, step=0):
    """g_ranks, e_ranks: lists (len W) of flat float32 arrays.  Returns
    (out, [e'_w], [pay1_w], pay2)."""
    W = len(g_ranks)
    N = len(g_ranks[0])
    S, _, _ = layout(layers, lbits, B)
    g = np.ascontiguousarray(np.stack([_f32(x) for x in g_ranks]))
    e = None if e_ranks is None else np.ascontiguousarray(np.stack([_f32(x) for x in e_ranks]))
    p1 = np.zeros(max(W * S, 1), np.uint8)
    p2 = np.zeros(max(S, 1), np.uint8)
    out = np.zeros(N, np.float32)
    st = lib().ref_qsgd_allreduce(_layers(layers), C.c_int32(len(layers)), _p(_i32(lbits)), C.c_int32(B),
                                  C.c_uint64(seed), C.c_uint64(step), C.c_int32(W), C.c_int64(N), _p(g), _p(e),
                                  _p(p1), _p(p2), _p(out))
    _check(st, "qsgd_allreduce")
    es = None if e is None else [e[w] for w in range(W)]
    return out, es, [p1[w * S:(w + 1) * S] for w in range(W)], p2[:S]


def qsgd_reduce_shard(layers, lbits, B, seed, step, W, recv, r0, r1, byte0, shard_bytes, pay2):
    recv = np.ascontiguousarray(recv, dtype=np.uint8)
    st = lib().ref_qsgd_reduce_shard(_layers(layers), C.c_int32(len(layers)), _p(_i32(lbits)), C.c_int32(B),
                                     C.c_uint64(seed), C.c_uint64(step), C.c_int32(W), _p(recv), C.c_int64(r0),
                                     C.c_int64(r1), C.c_int64(byte0), C.c_int64(shard_bytes), _p(pay2))
    _check(st, "qsgd_reduce_shard")


# ---------------------------------------------------------------------- TopK
def topk_k(n, ppm):
    return int(lib().ref_topk_k(C.c_int64(n), C.c_int32(ppm)))


def topk_select(x, k):
    x = _f32(x)
    idx = np.zeros(max(k, 1), np.uint32)
    st = lib().ref_topk_select(_p(x), C.c_int64(x.size), C.c_int64(k), _p(idx))
    _check(st, "topk_select")
    return idx[:k]


def topk_profile(layers, g, e, ppm):
    L, K = len(layers), len(ppm)
    err = np.zeros((L, K), np.float64)
    bits = np.zeros((L, K), np.int64)
    st = lib().ref_topk_profile(_layers(layers), C.c_int32(L), _p(_f32(g)), _p(_f32(e)), _p(_i32(ppm)),
                                C.c_int32(K), _p(err), _p(bits))
    _check(st, "topk_profile")
    return err, bits


def topk_layout(layers, lppm):
    bo = np.zeros(len(layers) + 1, np.int64)
    S = lib().ref_topk_layout(_layers(layers), C.c_int32(len(layers)), _p(_i32(lppm)), _p(bo))
    return int(S), bo


def topk_pack(layers, lppm, g, e):
    S, _ = topk_layout(layers, lppm)
    pay = np.zeros(max(S, 1), np.uint8)
    e2 = None if e is None else _f32(e).copy()
    st = lib().ref_topk_pack(_layers(layers), C.c_int32(len(layers)), _p(_i32(lppm)), _p(_f32(g)), _p(e2),
                             _p(pay))
    _check(st, "topk_pack")
    return pay[:S], e2


def topk_allreduce(layers, lppm, g_ranks, e_ranks):
    W = len(g_ranks)
    N = len(g_ranks[0])
    S, _ = topk_layout(layers, lppm)
    g = np.ascontiguousarray(np.stack([_f32(x) for x in g_ranks]))
    e = None if e_ranks is None else np.ascontiguousarray(np.stack([_f32(x) for x in e_ranks]))
    pays = np.zeros(max(W * S, 1), np.uint8)
    out = np.zeros(N, np.float32)
    st = lib().ref_topk_allreduce(_layers(layers), C.c_int32(len(layers)), _p(_i32(lppm)), C.c_int32(W),
                                  C.c_int64(N), _p(g), _p(e), _p(pays), _p(out))
    _check(st, "topk_allreduce")
    es = None if e is None else [e[w] for w in range(W)]
    return out, es, [pays[w * S:(w + 1) * S] for w in range(W)]


# ------------------------------------------------------------------ PowerSGD
def psgd_init_q(seed, layer, step, k, r):
    Q = np.zeros(k * r, np.float64)
    lib().ref_psgd_init_q(C.c_uint64(seed), C.c_uint32(layer), C.c_uint64(step), C.c_int32(k), C.c_int32(r), _p(Q))
    return Q.reshape(r, k).T.copy()  # (k, r)


def mgs(P):
    """P: (m, r) float64 -> orthonormalised columns (MGS, zero column stays 0)."""
    m, r = P.shape
    cm = np.ascontiguousarray(P.T).copy()
    lib().ref_mgs(_p(cm), C.c_int64(m), C.c_int32(r))
    return cm.T.copy()


def psgd_power(M, Q0, steps):
    """M: (m, k); Q0: (k, r).  Returns (P (m,r), Q (k,r)) after `steps` steps."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, k = M.shape
    r = Q0.shape[1]
    Qc = np.ascontiguousarray(Q0.T).copy()
    Pc = np.zeros((r, m), np.float64)
    lib().ref_psgd_power(_p(M), C.c_int64(m), C.c_int64(k), C.c_int32(r), C.c_int32(steps), _p(Pc), _p(Qc))
    return Pc.T.copy(), Qc.T.copy()


def psgd_err(M, P, Q):
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, k = M.shape
    r = P.shape[1]
    Pc = np.ascontiguousarray(P.T)
    Qc = np.ascontiguousarray(Q.T)
    return float(lib().ref_psgd_err(_p(M), C.c_int64(m), C.c_int64(k), C.c_int32(r), _p(Pc), _p(Qc)))


def psgd_profile(layers, g, e, ranks, steps=5, seed=0, step=0):
    L, K = len(layers), len(ranks)
    err = np.zeros((L, K), np.float64)
    bits = np.zeros((L, K), np.int64)
    st = lib().ref_psgd_profile(_layers(layers), C.c_int32(L), _p(_f32(g)), _p(_f32(e)), _p(_i32(ranks)),
                                C.c_int32(K), C.c_int32(steps), C.c_uint64(seed), C.c_uint64(step), _p(err),
                                _p(bits))
    _check(st, "psgd_profile")
    return err, bits


def psgd_svd_profile(layers, g, e, ranks):
    """NEXT-2: e_r = sqrt(sum_{i > r} sigma_i^2) of the m x k view of
    x = fl32(fl32(g + e) + 0) (R2, R11), singular values by LAPACK (numpy, fp64); lossless
    candidates r (m + k) >= m k and vector / uncompressed layers: err 0, bits 32 n."""
    g = np.asarray(g, np.float32)
    x = g if e is None else (g + np.asarray(e, np.float32)).astype(np.float32)
    x = (x + np.float32(0)).astype(np.float32)
    L, K = len(layers), len(ranks)
    err = np.zeros((L, K), np.float64)
    bits = np.zeros((L, K), np.int64)
    for l, ly in enumerate(layers):
        bits[l, :] = 32 * ly.numel
        if not ly.compress or ly.rows <= 0:
            continue
        m, k = int(ly.rows), int(ly.cols)
        lossy = [not psgd_lossless(m, k, r) for r in ranks]
        if not any(lossy):
            continue
        M = x[ly.offset:ly.offset + ly.numel].astype(np.float64).reshape(m, k)
        sv = np.linalg.svd(M, compute_uv=False)  # descending
        for j, r in enumerate(ranks):
            if lossy[j]:
                err[l, j] = float(np.sqrt(np.sum(sv[r:] ** 2)))
                bits[l, j] = 32 * r * (m + k)
    return err, bits


def psgd_lossless(m, k, r):
    return r * (m + k) >= m * k


def psgd_allreduce(layers, lrank, g_ranks, e_ranks, Qstate):
    """Qstate: dict layer -> (k, r) float64 warm-start Q (updated in place).
    Returns (out, [e'_w], {layer: Pbar_hat (m, r)})."""
    W = len(g_ranks)
    N = len(g_ranks[0])
    L = len(layers)
    qoff = np.zeros(L + 1, np.int64)
    poff = np.zeros(L + 1, np.int64)
    for l, ly in enumerate(layers):
        r = lrank[l]
        active = r > 0 and ly.compress and ly.rows > 0 and not psgd_lossless(ly.rows, ly.cols, r)
        qoff[l + 1] = qoff[l] + (ly.cols * r if active else 0)
        poff[l + 1] = poff[l] + (ly.rows * r if active else 0)
    Qbuf = np.zeros(max(1, qoff[-1]), np.float64)
    for l, ly in enumerate(layers):
        if qoff[l + 1] > qoff[l]:
            Qbuf[qoff[l]:qoff[l + 1]] = np.ascontiguousarray(Qstate[l].T).reshape(-1)
    Pbuf = np.zeros(max(1, poff[-1]), np.float64)
    g = np.ascontiguousarray(np.stack([_f32(x) for x in g_ranks]))
    e = None if e_ranks is None else np.ascontiguousarray(np.stack([_f32(x) for x in e_ranks]))
    out = np.zeros(N, np.float32)
    st = lib().ref_psgd_allreduce(_layers(layers), C.c_int32(L), _p(_i32(lrank)), C.c_int32(W), C.c_int64(N),
                                  _p(g), _p(e), _p(Qbuf), _p(qoff), _p(out), _p(Pbuf), _p(poff))
    _check(st, "psgd_allreduce")
    Ps = {}
    for l, ly in enumerate(layers):
        if qoff[l + 1] > qoff[l]:
            r = lrank[l]
            Qstate[l] = Qbuf[qoff[l]:qoff[l + 1]].reshape(r, ly.cols).T.copy()
            Ps[l] = Pbuf[poff[l]:poff[l + 1]].reshape(r, ly.rows).T.copy()
    es = None if e is None else [e[w] for w in range(W)]
    return out, es, Ps


# ------------------------------------------------------------------------ DP
def solve(err, bits, default_idx, compress=None, D=10000, flags=0):
    err = np.ascontiguousarray(err, dtype=np.float64)
    bits = np.ascontiguousarray(bits, dtype=np.int64)
    L, K = err.shape
    choice = np.zeros(L, np.int32)
    info = SolveInfo()
    st = lib().ref_solve(_p(err), _p(bits), C.c_int32(L), C.c_int32(K), _p(_i32(default_idx)),
                         None if compress is None else _p(_i32(compress)), C.c_int32(D), C.c_uint32(flags),
                         _p(choice), C.byref(info))
    return st, choice, info
