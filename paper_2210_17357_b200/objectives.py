"""Per-layer weights for the time-weighted objective and the bucket priorities
(SURVEY.md 8(f) NEXT-1), Accordion-style per-layer defaults and hybrid-family candidate
tables (NEXT-4).  Host-side planning helpers: they produce the integer weight
vector that `lgreco.weight_costs` multiplies into the size table on the device before
`lgreco.solve` (the DP itself is unchanged; only its cost table is).

  PAPER.md:350-356  minimize sum_l size(l, c^l) * T(l)  s.t.  sum_l error(l, c^l) <= Emax,
                    T(b) the per-bucket coefficients of a linear regression of measured
                    synchronisation time on the transmitted bucket sizes.
  PAPER.md:680-682  bucket prioritisation: "multiplying the size of each layer by the
                    index of the bucket the layer is communicated in".
"""
import numpy as np


def ddp_buckets(layers, bucket_bytes=25 * 2 ** 20, first_bucket_bytes=2 ** 20, elem_bytes=4):
    """Bucket index (0 = transmitted first) of every layer, as PyTorch DDP assigns them
    (compute_bucket_assignment_by_size): gradients become ready in reverse layer order,
    so tensors are taken from the last layer backwards; each is appended to the open
    bucket, and the bucket closes once its size reaches the current cap (the first cap
    `first_bucket_bytes`, every later one `bucket_bytes`)."""
    out = [0] * len(layers)
    b, fill, cap = 0, 0, first_bucket_bytes
    for i in reversed(range(len(layers))):
        out[i] = b
        fill += layers[i].numel * elem_bytes
        if fill >= cap:
            b, fill, cap = b + 1, 0, bucket_bytes
    return out


def bucket_priority_weights(layers, **kw):
    """weight of a layer = 1-based index of the bucket it is sent in."""
    return np.array([b + 1 for b in ddp_buckets(layers, **kw)], dtype=np.int64)


def fit_bucket_time(sizes, times, intercept=True):
    """least-squares linear model time ~ sum_b sizes[:, b] * T(b) (+ c)
    over measured samples.  sizes: (S, nb) transmitted bytes (or bits) per bucket,
    times: (S,) synchronisation times.  Returns (T (nb,), c)."""
    A = np.asarray(sizes, dtype=np.float64)
    y = np.asarray(times, dtype=np.float64)
    if intercept:
        A = np.hstack([A, np.ones((A.shape[0], 1))])
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    return (coef[:-1], float(coef[-1])) if intercept else (coef, 0.0)


def time_weights(layers, T, buckets=None, scale=2 ** 16):
    """Integer weights w_l = max(1, round(scale * T(bucket(l)) / max_b T(b))) -- the DP needs
    exact integer costs; `scale` sets the resolution of the quantised coefficients."""
    T = np.asarray(T, dtype=np.float64)
    if buckets is None:
        buckets = ddp_buckets(layers)
    tmax = float(T.max()) if T.size and T.max() > 0 else 1.0
    return np.array([max(1, int(round(scale * max(T[b], 0.0) / tmax))) for b in buckets], dtype=np.int64)


def accordion_defaults(prev_norm, cur_norm, low_idx, high_idx, eta=0.5):
    """NEXT-4: per-layer defaults from an Accordion-style schedule --
    a layer is in a critical regime when its gradient norm changed by at least `eta`
    relative to the previous period (|n_t - n_{t-1}| / n_{t-1} >= eta); critical layers
    get the low-compression candidate `low_idx`, the others `high_idx`.  The result is
    the `default_idx` of lgreco_solve (the defaults set Emax, Alg.1 line 2)."""
    p = np.asarray(prev_norm, dtype=np.float64)
    c = np.asarray(cur_norm, dtype=np.float64)
    crit = np.abs(c - p) >= eta * np.abs(p)
    return np.where(crit, low_idx, high_idx).astype(np.int32)


def hybrid_table(errs, bits, defaults_family=0):
    """NEXT-4 hybrid strategies ("combining different compression techniques
    inside the same model"): candidates of several families side by side in one table,
    so Algorithm 1 picks a (family, parameter) per layer.  errs / bits: lists of (L, K_f)
    arrays (numpy or torch, one per family, rows aligned by layer).  Returns the
    concatenated (err, bits) and the list of (family, index) per column."""
    cols = [(f, j) for f, e in enumerate(errs) for j in range(e.shape[1])]
    try:
        import torch
        if isinstance(errs[0], torch.Tensor):
            return torch.cat(list(errs), 1).contiguous(), torch.cat(list(bits), 1).contiguous(), cols
    except ImportError:  # pragma: no cover
        pass
    return np.concatenate(errs, 1), np.concatenate(bits, 1), cols
