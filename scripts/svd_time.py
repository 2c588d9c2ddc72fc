"""Time the SVD profile (fp64 Grams + the library's eigensolver) against the power profile
on C2 and C5 (device-drawn recipe inputs); prints ms per call."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_17357_b200 import lgreco as lg
from paper_2210_17357_b200 import workloads as W

dev = torch.device("cuda", 0)
for cfg, ranks in (("C2", W.PSGD_RANKS_C2), ("C5", W.PSGD_RANKS_C5)):
    layers = W.config_layers(cfg)
    g, e = W.recipe_device(layers, "low_rank", dev, seed=5)
    L, K = len(layers), len(ranks)
    ctx = lg.Context(layers, lg.POWERSGD, ranks, seed=3)
    err = torch.empty(L, K, dtype=torch.float64, device=dev)
    bits = torch.empty(L, K, dtype=torch.int64, device=dev)
    res = {}
    for name, fn in (("svd", lambda: ctx.profile_svd(g, e, err, bits)), ("power", lambda: ctx.profile(g, e, 0, err, bits))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(2):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / 2
    print(cfg, {k: round(v, 3) for k, v in res.items()}, flush=True)
    ctx.close()
    del g, e
    torch.cuda.empty_cache()
