"""Diagnostic: run the C2 PowerSGD profile (and one compress) a few times on
device-generated inputs, for an ncu launch list.  Not part of the product."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_17357_b200 import lgreco, workloads as W  # noqa: E402

dev = torch.device("cuda:0")
layers = W.config_layers("C2")
N = W.total_numel(layers)
params = W.PSGD_RANKS_C2
L, K = len(layers), len(params)
gen = torch.Generator(device=dev)
gen.manual_seed(3)
g = torch.randn(N, generator=gen, device=dev) * 1e-3
ef = torch.randn(N, generator=gen, device=dev) * 1e-4
err = torch.empty(L, K, dtype=torch.float64, device=dev)
bits = torch.empty(L, K, dtype=torch.int64, device=dev)
ctx = lgreco.Context(layers, lgreco.POWERSGD, params, seed=1)
out = torch.empty_like(g)
choice = [2 if l.compress else -1 for l in layers]
for s in range(3):
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    ctx.profile(g, ef, s, err, bits)
    b.record()
    ctx.compress_allreduce(choice, g, ef, out, s)
    c.record()
    torch.cuda.synchronize()
    print(f"step {s}: profile {a.elapsed_time(b):.3f} ms compress {b.elapsed_time(c):.3f} ms", flush=True)
ctx.close()
