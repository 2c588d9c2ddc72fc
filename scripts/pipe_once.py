"""Diagnostic for ncu captures: a few steps of the pipelined C4 schedule (fused profile +
compress pass, K1b, the narrow solve), nothing else."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_17357_b200 import lgreco as lg
from paper_2210_17357_b200 import workloads as W

dev = torch.device("cuda", 0)
layers = W.config_layers("C4")
L, K = len(layers), len(W.QSGD_BITS)
g_np, e_np = W.gaussian_outliers(layers, seed=W.rank_seed(0x5EED, 0))
g, ef = torch.from_numpy(g_np).to(dev), torch.from_numpy(e_np).to(dev)
out = torch.empty_like(g)
ctx = lg.Context(layers, lg.QSGD, W.QSGD_BITS, seed=0x5EED)
dflt = torch.full((L,), W.QSGD_BITS.index(4), dtype=torch.int32, device=dev)
comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=dev)
plans = [dflt.clone() for _ in range(3)]
tabs = [(torch.empty(L, K, dtype=torch.float64, device=dev), torch.empty(L, K, dtype=torch.int64, device=dev))
        for _ in range(2)]
ws = torch.empty(lg.solve_workspace_bytes(L, K, 10000), dtype=torch.uint8, device=dev)
info = torch.empty(64, dtype=torch.uint8, device=dev)
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    e_t, b_t = tabs[s % 2]
    ctx.profile_compress(plans[s % 3], g, ef, out, s, e_t, b_t, concurrent=s > 0)
    lg.solve(e_t, b_t, dflt, comp, flags=lg.SOLVE_NARROW, choice=plans[(s + 2) % 3], info=info, workspace=ws)
torch.cuda.synchronize()
ctx.check()
print("ok")
