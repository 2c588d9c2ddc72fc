"""Diagnostic: phase cycle counts of k_solve_fast (build/liblgreco_timing.so, built by
`make timing`) and CUDA-event times of the product solve, on the error tables the
product profile kernels produce for C4 (QSGD), C5 (QSGD), C3 (TopK) and C2 (PowerSGD)
from device-generated seeded inputs.  Not part of the product or the tests."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_17357_b200 import lgreco, workloads as W  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "timing":
    lgreco.LIB_PATH = os.path.join(ROOT, "build", "liblgreco_timing.so")

dev = torch.device("cuda:0")
D = 10000
if os.environ.get("DP_ONLY_C4"):
    pass
specs = [("C4", lgreco.QSGD, W.QSGD_BITS, 2), ("C5", lgreco.QSGD, W.QSGD_BITS, 2),
         ("C3", lgreco.TOPK, W.TOPK_PPM_C3, 9), ("C2", lgreco.POWERSGD, W.PSGD_RANKS_C2, 2)]
if os.environ.get("DP_ONLY_C4"):
    specs = specs[:1]
for name, fam, params, di in specs:
    layers = W.config_layers(name)
    N = W.total_numel(layers)
    L, K = len(layers), len(params)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    g = torch.randn(N, generator=gen, device=dev) * 1e-3
    ef = torch.randn(N, generator=gen, device=dev) * 1e-4
    err = torch.empty(L, K, dtype=torch.float64, device=dev)
    bits = torch.empty(L, K, dtype=torch.int64, device=dev)
    ctx = lgreco.Context(layers, fam, params, qbucket=128, seed=1)
    ctx.profile(g, ef, 0, err, bits)
    dflt = torch.full((L,), di, dtype=torch.int32, device=dev)
    comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=dev)
    ch = torch.empty(L, dtype=torch.int32, device=dev)
    info = torch.empty(48, dtype=torch.uint8, device=dev)
    ws = torch.empty(lgreco.solve_workspace_bytes(L, K, D), dtype=torch.uint8, device=dev)
    for fl in ((0, 4) if not os.environ.get('DP_NOPUSH') else (1 << 30,)):  # 4 = LGRECO_SOLVE_SINGLE_CTA
        ts = []
        for it in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lgreco.solve(err, bits, dflt, comp, D=D, flags=fl, choice=ch, info=info, workspace=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        inf = lgreco.read_info(info)
        print(f"{name}: flags={fl} L={L} La={inf.n_active} K={K} solve ms {min(ts[1:]):.4f} "
              f"(all {[round(t, 4) for t in ts]}) used_default={inf.used_default} "
              f"bits {inf.total_bits}/{inf.default_bits} choice {ch[:8].tolist()}", flush=True)
    ctx.close()
    del g, ef
    torch.cuda.empty_cache()
