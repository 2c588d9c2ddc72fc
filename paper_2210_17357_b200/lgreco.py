"""Thin ctypes binding of include/lgreco.h (argument marshalling only).

Every step of the hot path runs in liblgreco.so's CUDA kernels; PyTorch only
supplies device memory (tensors), the current stream and process groups.  There
is no CPU fallback: if the library is missing this module raises on import of
any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LGRECO_LIB") or os.path.join(_HERE, "liblgreco.so")  # override: diagnostics only

OK, EINVAL, ENONFINITE, EINFEASIBLE, ECUDA, ENCCL, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7
QSGD, TOPK, POWERSGD = 0, 1, 2
PSGD_POWER, PSGD_SVD, PSGD_AUTO = 0, 1, 2  # PowerSGD profile method (NEXT-2 selector)
SOLVE_NARROW = 8  # lgreco_solve flag: 8-CTA clusters (a solve running beside other work)
PC_CONCURRENT = 1  # lgreco_profile_compress: may run beside the preceding kernel (include/lgreco.h)
CHOICE_SKIP = -2  # (NEXT-4) a compressed layer another family's ctx owns: left untouched
METRIC_SQ, DISC_FLOOR = 1, 2


class LGrecoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"lgreco status {status}: {msg}")
        self.status = status


class Layer(C.Structure):
    _fields_ = [("offset", C.c_int64), ("numel", C.c_int64), ("rows", C.c_int32),
                ("cols", C.c_int32), ("compress", C.c_int32)]


class Candidates(C.Structure):
    _fields_ = [("family", C.c_int32), ("K", C.c_int32), ("params", C.POINTER(C.c_int32)),
                ("qbucket", C.c_int32), ("power_steps", C.c_int32), ("seed", C.c_uint64)]


class SolveInfo(C.Structure):
    _fields_ = [("emax", C.c_double), ("total_err", C.c_double), ("total_bits", C.c_int64),
                ("default_bits", C.c_int64), ("used_default", C.c_int32), ("n_active", C.c_int32),
                ("status", C.c_int32), ("pad", C.c_int32)]


_lib = None
_VP, _I32, _I64, _U32, _U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64

_SIGS = {
    "lgreco_last_error": (C.c_char_p, []),
    "lgreco_version": (_I32, []),
    "lgreco_nccl_unique_id": (C.c_int, [_VP]),
    "lgreco_ctx_create": (C.c_int, [C.POINTER(_VP), _VP, _I32, _VP, _I32, _I32, _VP, _VP]),
    "lgreco_ctx_destroy": (None, [_VP]),
    "lgreco_ctx_check": (C.c_int, [_VP, _VP]),
    "lgreco_ctx_launches": (_I64, [_VP]),
    "lgreco_ctx_timing": (_I32, [_VP, _I32]),
    "lgreco_ctx_kernel_ms": (_I32, [_VP, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "lgreco_accumulate": (C.c_int, [_VP, _VP, _I64, _VP]),
    "lgreco_profile": (C.c_int, [_VP, _VP, _VP, _U64, _VP, _VP, _VP]),
    "lgreco_solve_workspace_bytes": (C.c_size_t, [_I32, _I32, _I32]),
    "lgreco_solve": (C.c_int, [_VP, _VP, _I32, _I32, _VP, _VP, _I32, _U32, _VP, _VP, _VP, C.c_size_t, _VP]),
    "lgreco_weight_costs": (C.c_int, [_VP, _VP, _I32, _I32, _VP, _VP]),
    "lgreco_psgd_profile_svd": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "lgreco_psgd_set_method": (C.c_int, [_VP, C.c_int32]),
    "lgreco_hybrid_table": (C.c_int, [_VP, _VP, _VP, _I32, _I32, _VP, _VP, _VP]),
    "lgreco_hybrid_split": (C.c_int, [_VP, _VP, _I32, _I32, _VP, _VP]),
    "lgreco_psgd_method": (C.c_int, [_VP]),
    "lgreco_layer_norms": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "lgreco_p2p_local": (C.c_int, [_VP, _VP]),
    "lgreco_p2p_export": (C.c_int, [_VP, _VP]),
    "lgreco_p2p_open": (C.c_int, [_VP, _VP]),
    "lgreco_p2p_set_peers": (C.c_int, [_VP, _VP, _VP, _VP]),
    "lgreco_p2p_stage": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _I32, _VP]),
    "lgreco_plan_broadcast": (C.c_int, [_VP, _VP, _VP]),
    "lgreco_compress_allreduce": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP]),
    "lgreco_compress_allreduce_dev": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP]),
    "lgreco_profile_compress": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP, _VP, C.c_uint32, _VP]),
    "lgreco_payload_bytes": (_I64, [_VP, _VP]),
    "lgreco_shard_bounds": (C.c_int, [_VP, _VP, _I32, _VP, _VP]),
    "lgreco_qsgd_pack": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _U32, _U64, _VP]),
    "lgreco_qsgd_reduce": (C.c_int, [_VP, _VP, _I32, _I64, _I64, _VP, _VP, _U64, _VP]),
    "lgreco_qsgd_unpack": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "lgreco_topk_pack": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "lgreco_topk_combine": (C.c_int, [_VP, _VP, _I32, _VP, _VP, _VP]),
    "lgreco_plan_layout": (C.c_int, [_VP, _I32, _VP, _VP, _I32, _VP, _VP, _VP]),
    "lgreco_psgd_sizes": (C.c_int, [_VP, _VP, _VP]),
    "lgreco_psgd_factors": (C.c_int, [_VP, _VP, _VP, _VP]),
    "lgreco_psgd_p": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP]),
    "lgreco_psgd_q": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _I32, _VP, _VP]),
    "lgreco_psgd_out": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _I32, _VP, _VP]),
    "lgreco_psgd_raw_pack": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "lgreco_psgd_raw_combine": (C.c_int, [_VP, _VP, _I32, _VP, _VP, _VP]),
    "lgreco_debug_tc_mq": (C.c_int, [_VP, _VP, _I64, _I32, _VP, _I32, _VP, _VP]),
    "lgreco_debug_tc_mtp": (C.c_int, [_VP, _VP, _I64, _I32, _VP, _I32, _VP, _VP]),
    "lgreco_debug_philox": (C.c_int, [_VP, _U32, _U32, _I64, _VP, _VP]),
}
EXPORTED = tuple(_SIGS)


def lib():
    """Load liblgreco.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make` (or __graft_entry__.build()); "
                              "there is no CPU fallback")
        _lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _check(st, what=""):
    if st != OK:
        raise LGrecoError(st, f"{what}: {lib().lgreco_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    assert t.is_contiguous(), "tensors passed to lgreco must be contiguous"
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _i32(vals):
    arr = (C.c_int32 * max(1, len(vals)))(*[int(v) for v in vals])
    return arr


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().lgreco_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


class Context:
    """Owns an lgreco_ctx (workspaces, NCCL communicator, PowerSGD state)."""

    def __init__(self, layers, family, params, *, qbucket=128, power_steps=5, seed=0, rank=0, world=1,
                 nccl_id: bytes | None = None, stream=None):
        self.layers = list(layers)
        self.L = len(self.layers)
        self.family = family
        self.params = [int(p) for p in params]
        self.K = len(self.params)
        self.rank, self.world = rank, world
        self.N = max(l.offset + l.numel for l in self.layers)
        arr = (Layer * self.L)(*[Layer(l.offset, l.numel, l.rows, l.cols, l.compress) for l in self.layers])
        self._params_arr = _i32(self.params)
        cand = Candidates(family, self.K, C.cast(self._params_arr, C.POINTER(C.c_int32)), qbucket, power_steps,
                          seed)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib().lgreco_ctx_create(C.byref(h), C.cast(arr, C.c_void_p), self.L, C.cast(C.pointer(cand), C.c_void_p),
                                       rank, world, C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                                       _stream(stream)), "ctx_create")
        self.h = h

    def close(self):
        if self.h:
            lib().lgreco_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path ------------------------------------------------------------
    def profile(self, g, ef, step, err, bits, stream=None):
        _check(lib().lgreco_profile(self.h, _ptr(g), _ptr(ef), step, _ptr(err), _ptr(bits), _stream(stream)),
               "profile")

    def set_psgd_method(self, method):
        """PSGD_POWER / PSGD_SVD / PSGD_AUTO (NEXT-2 selector)."""
        _check(lib().lgreco_psgd_set_method(self.h, int(method)), "psgd_set_method")

    def psgd_method(self) -> int:
        v = int(lib().lgreco_psgd_method(self.h))
        if v < 0:
            _check(v, "psgd_method")
        return v

    def profile_svd(self, g, ef, err, bits, stream=None):
        """PowerSGD errors of every candidate rank from the singular values (NEXT-2)."""
        _check(lib().lgreco_psgd_profile_svd(self.h, _ptr(g), _ptr(ef), _ptr(err), _ptr(bits), _stream(stream)),
               "psgd_profile_svd")

    def layer_norms(self, g, ef, norm, stream=None):
        """Per-layer L2 norms of x = g (+ ef) into the L fp64 device tensor `norm`."""
        _check(lib().lgreco_layer_norms(self.h, _ptr(g), _ptr(ef), _ptr(norm), _stream(stream)), "layer_norms")

    # ---- peer-memory exchange (QSGD, world > 1 without NCCL) -------------------------
    def p2p_local(self):
        arr = (C.c_void_p * 3)()
        _check(lib().lgreco_p2p_local(self.h, C.cast(arr, C.c_void_p)), "p2p_local")
        return [int(v or 0) for v in arr]

    def p2p_set_peers(self, recv, stage2, flags):
        W = len(recv)
        mk = lambda v: (C.c_void_p * W)(*[C.c_void_p(x) for x in v])  # noqa: E731
        a, b, c = mk(recv), mk(stage2), mk(flags)
        _check(lib().lgreco_p2p_set_peers(self.h, C.cast(a, C.c_void_p), C.cast(b, C.c_void_p), C.cast(c, C.c_void_p)),
               "p2p_set_peers")

    def p2p_export(self) -> bytes:
        buf = C.create_string_buffer(192)
        _check(lib().lgreco_p2p_export(self.h, C.cast(buf, C.c_void_p)), "p2p_export")
        return buf.raw

    def p2p_open(self, blobs):
        raw = b"".join(blobs)
        buf = C.create_string_buffer(raw, len(raw))
        _check(lib().lgreco_p2p_open(self.h, C.cast(buf, C.c_void_p)), "p2p_open")

    def p2p_stage(self, choice, g, ef, out, step, stage, stream=None):
        _check(lib().lgreco_p2p_stage(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(out), step, stage,
                                      _stream(stream)), "p2p_stage")

    def compress_allreduce(self, choice, g, ef, out, step, stream=None):
        _check(lib().lgreco_compress_allreduce(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(out), step,
                                               _stream(stream)), "compress_allreduce")

    def compress_allreduce_dev(self, d_choice, g, ef, out, step, stream=None):
        _check(lib().lgreco_compress_allreduce_dev(self.h, _ptr(d_choice), _ptr(g), _ptr(ef), _ptr(out), step,
                                                   _stream(stream)), "compress_allreduce_dev")

    def profile_compress(self, d_choice, g, ef, out, step, err, bits, concurrent=False, stream=None):
        """profile(g, ef, step, err, bits) then compress_allreduce_dev(d_choice, ...), one pass
        over g and ef (QSGD, W = 1): the paper's per-step schedule (the plan in force
        compresses the step, the profile feeds the next solve)."""
        _check(lib().lgreco_profile_compress(self.h, _ptr(d_choice), _ptr(g), _ptr(ef), _ptr(out), step, _ptr(err),
                                             _ptr(bits), PC_CONCURRENT if concurrent else 0, _stream(stream)),
               "profile_compress")

    def plan_broadcast(self, d_choice, stream=None):
        _check(lib().lgreco_plan_broadcast(self.h, _ptr(d_choice), _stream(stream)), "plan_broadcast")

    def check(self, stream=None):
        _check(lib().lgreco_ctx_check(self.h, _stream(stream)), "ctx_check")

    def launches(self) -> int:
        return int(lib().lgreco_ctx_launches(self.h))

    def timing(self, enable=True):
        """Record CUDA events around the dominant profile kernel (QSGD K1) per call."""
        _check(lib().lgreco_ctx_timing(self.h, 1 if enable else 0), "timing")

    def kernel_ms(self):
        """(total ms, launches) of the recorded dominant-kernel launches; clears them."""
        t, n = C.c_double(0.0), C.c_int64(0)
        _check(lib().lgreco_ctx_kernel_ms(self.h, C.byref(t), C.byref(n)), "kernel_ms")
        return t.value, n.value

    # ---- stages ----------------------------------------------------------------
    def payload_bytes(self, choice) -> int:
        v = int(lib().lgreco_payload_bytes(self.h, _i32(choice)))
        if v < 0:
            _check(v, "payload_bytes")
        return v

    def shard_bounds(self, choice, W):
        rb = (C.c_int64 * (W + 1))()
        bb = (C.c_int64 * (W + 1))()
        _check(lib().lgreco_shard_bounds(self.h, _i32(choice), W, rb, bb), "shard_bounds")
        return list(rb), list(bb)

    def qsgd_pack(self, choice, g, ef, payload, dec, rank, step, stream=None):
        _check(lib().lgreco_qsgd_pack(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(payload), _ptr(dec), rank, step,
                                      _stream(stream)), "qsgd_pack")

    def qsgd_reduce(self, choice, W, r0, r1, recv, stage2, step, stream=None):
        _check(lib().lgreco_qsgd_reduce(self.h, _i32(choice), W, r0, r1, _ptr(recv), _ptr(stage2), step,
                                        _stream(stream)), "qsgd_reduce")

    def qsgd_unpack(self, choice, payload, out, stream=None):
        _check(lib().lgreco_qsgd_unpack(self.h, _i32(choice), _ptr(payload), _ptr(out), _stream(stream)),
               "qsgd_unpack")


    def topk_pack(self, choice, g, ef, payload, out, stream=None):
        _check(lib().lgreco_topk_pack(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(payload), _ptr(out),
                                      _stream(stream)), "topk_pack")

    def topk_combine(self, choice, W, gathered, out, stream=None):
        _check(lib().lgreco_topk_combine(self.h, _i32(choice), W, _ptr(gathered), _ptr(out), _stream(stream)),
               "topk_combine")


    def psgd_sizes(self):
        p, q = C.c_int64(), C.c_int64()
        _check(lib().lgreco_psgd_sizes(self.h, C.byref(p), C.byref(q)), "psgd_sizes")
        return p.value, q.value

    def psgd_factors(self, Phat, Q, stream=None):
        """Copy the current Phat / warm-start Q slot areas into the float32 cuda tensors."""
        _check(lib().lgreco_psgd_factors(self.h, _ptr(Phat), _ptr(Q), _stream(stream)), "psgd_factors")

    def psgd_p(self, choice, g, ef, P, step, stream=None):
        _check(lib().lgreco_psgd_p(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(P), step, _stream(stream)), "psgd_p")

    def psgd_q(self, choice, g, ef, Psum, W, Q, stream=None):
        _check(lib().lgreco_psgd_q(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(Psum), W, _ptr(Q), _stream(stream)),
               "psgd_q")

    def psgd_out(self, choice, g, ef, Qsum, W, out, stream=None):
        _check(lib().lgreco_psgd_out(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(Qsum), W, _ptr(out),
                                     _stream(stream)), "psgd_out")

    def psgd_raw_pack(self, choice, g, ef, payload, out, stream=None):
        _check(lib().lgreco_psgd_raw_pack(self.h, _i32(choice), _ptr(g), _ptr(ef), _ptr(payload), _ptr(out),
                                          _stream(stream)), "psgd_raw_pack")

    def psgd_raw_combine(self, choice, W, gathered, out, stream=None):
        _check(lib().lgreco_psgd_raw_combine(self.h, _i32(choice), W, _ptr(gathered), _ptr(out), _stream(stream)),
               "psgd_raw_combine")


def plan_layout(layers, family, params, choice, W, qbucket=128):
    """Host-only payload layout / shard bounds (no GPU needed)."""
    L = len(layers)
    arr = (Layer * L)(*[Layer(l.offset, l.numel, l.rows, l.cols, l.compress) for l in layers])
    pa = _i32(params)
    cand = Candidates(family, len(params), C.cast(pa, C.POINTER(C.c_int32)), qbucket, 5, 0)
    S = C.c_int64()
    rb = (C.c_int64 * (W + 1))()
    bb = (C.c_int64 * (W + 1))()
    _check(lib().lgreco_plan_layout(C.cast(arr, C.c_void_p), L, C.cast(C.pointer(cand), C.c_void_p), _i32(choice), W,
                                    C.byref(S), rb, bb), "plan_layout")
    return S.value, list(rb), list(bb)


def solve_workspace_bytes(L, K, D) -> int:
    return int(lib().lgreco_solve_workspace_bytes(L, K, D))


def solve(err, bits, default_idx, compress=None, D=10000, flags=0, choice=None, info=None, workspace=None,
          stream=None):
    """Device-side Algorithm 1.  err (L,K) f64, bits (L,K) i64, default_idx (L,) i32,
    compress (L,) i32 or None, all cuda tensors.  Returns (choice i32 (L,), info u8 tensor)."""
    L, K = err.shape
    dev = err.device
    if choice is None:
        choice = torch.empty(L, dtype=torch.int32, device=dev)
    if info is None:
        info = torch.empty(C.sizeof(SolveInfo), dtype=torch.uint8, device=dev)
    if workspace is None:
        workspace = torch.empty(solve_workspace_bytes(L, K, D), dtype=torch.uint8, device=dev)
    _check(lib().lgreco_solve(_ptr(err), _ptr(bits), L, K, _ptr(default_idx), _ptr(compress), D, flags,
                              _ptr(choice), _ptr(info), _ptr(workspace), workspace.numel(), _stream(stream)),
           "solve")
    return choice, info


def solve_host(err, bits, default_idx, compress=None, D=10000, flags=0, stream=None):
    """lgreco_solve's host mode: numpy tables in, (choice int32 (L,), SolveInfo) out; the DP
    runs in the library's kernels (staged through device scratch), stream-synchronous."""
    import numpy as np
    e = np.ascontiguousarray(err, dtype=np.float64)
    b = np.ascontiguousarray(bits, dtype=np.int64)
    L, K = e.shape
    d = np.ascontiguousarray(default_idx, dtype=np.int32)
    c = None if compress is None else np.ascontiguousarray(compress, dtype=np.int32)
    ch = np.empty(L, dtype=np.int32)
    info = SolveInfo()
    _check(lib().lgreco_solve(e.ctypes.data, b.ctypes.data, L, K, d.ctypes.data, None if c is None else c.ctypes.data,
                              D, flags, ch.ctypes.data, C.addressof(info), None, 0, _stream(stream)), "solve_host")
    return ch, info


def accumulate(G, g, stream=None):
    """K0 (row a1): G += g in fp32 on the device (cuda float32 tensors of equal size)."""
    assert G.dtype == torch.float32 and g.dtype == torch.float32 and G.numel() == g.numel()
    _check(lib().lgreco_accumulate(_ptr(G), _ptr(g), G.numel(), _stream(stream)), "accumulate")
    return G


def weight_costs(bits, weight, out=None, stream=None):
    """Device: out[l, c] = bits[l, c] * weight[l] (int64 cuda tensors; -1 on overflow)."""
    L, K = bits.shape
    if out is None:
        out = torch.empty_like(bits)
    _check(lib().lgreco_weight_costs(_ptr(bits), _ptr(weight), L, K, _ptr(out), _stream(stream)), "weight_costs")
    return out


def hybrid_table(errs, bits, err_out=None, bits_out=None, stream=None):
    """NEXT-4: the families' (L, K_f) device tables side by side -> (L, sum K_f) on the device."""
    F, L = len(errs), errs[0].shape[0]
    Ks = [int(e.shape[1]) for e in errs]
    dev = errs[0].device
    if err_out is None:
        err_out = torch.empty(L, sum(Ks), dtype=torch.float64, device=dev)
    if bits_out is None:
        bits_out = torch.empty(L, sum(Ks), dtype=torch.int64, device=dev)
    pe = (C.c_void_p * F)(*[e.data_ptr() for e in errs])
    pb = (C.c_void_p * F)(*[b.data_ptr() for b in bits])
    _check(lib().lgreco_hybrid_table(C.cast(pe, C.c_void_p), C.cast(pb, C.c_void_p), _i32(Ks), F, L, _ptr(err_out),
                                     _ptr(bits_out), _stream(stream)), "hybrid_table")
    return err_out, bits_out


def hybrid_split(choice, Ks, outs=None, stream=None):
    """NEXT-4: a hybrid plan (device (L,) column indices) -> one device choice vector per
    family (its own index, CHOICE_SKIP where another family owns the layer)."""
    L, F = choice.numel(), len(Ks)
    if outs is None:
        outs = [torch.empty(L, dtype=torch.int32, device=choice.device) for _ in range(F)]
    po = (C.c_void_p * F)(*[o.data_ptr() for o in outs])
    _check(lib().lgreco_hybrid_split(_ptr(choice), _i32(Ks), F, L, C.cast(po, C.c_void_p), _stream(stream)),
           "hybrid_split")
    return outs


def read_info(info_tensor) -> SolveInfo:
    raw = bytes(info_tensor.cpu().numpy().tobytes())
    return SolveInfo.from_buffer_copy(raw)


def debug_philox(ctr, key0, key1, stream=None):
    n = ctr.numel() // 4
    out = torch.empty_like(ctr)
    _check(lib().lgreco_debug_philox(_ptr(ctr), key0, key1, n, _ptr(out), _stream(stream)), "debug_philox")
    return out


def debug_tc_mq(g, e, m, k, Q, r, P, stream=None):
    _check(lib().lgreco_debug_tc_mq(_ptr(g), _ptr(e), m, k, _ptr(Q), r, _ptr(P), _stream(stream)), "debug_tc_mq")


def debug_tc_mtp(g, e, m, k, P, r, Q, stream=None):
    _check(lib().lgreco_debug_tc_mtp(_ptr(g), _ptr(e), m, k, _ptr(P), r, _ptr(Q), _stream(stream)), "debug_tc_mtp")
