"""Diagnostic: run one family's profile -> solve -> compress on the SURVEY 8(d) recipe
inputs of a config a few times (device-timed per stage), for ncu launch lists and
captures.  Not part of the product.
  python scripts/family_prof.py C2|C3|C5q|C5t|C5p [steps]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_17357_b200 import lgreco, workloads as W  # noqa: E402

SPECS = {  # config, family, params, default index, generator
    "C2": ("C2", lgreco.POWERSGD, W.PSGD_RANKS_C2, 2, "low_rank"),
    "C3": ("C3", lgreco.TOPK, W.TOPK_PPM_C3, 9, "student_t"),
    "C5q": ("C5", lgreco.QSGD, W.QSGD_BITS, 2, "gaussian"),
    "C5t": ("C5", lgreco.TOPK, W.TOPK_PPM_C5, 9, "student_t"),
    "C5p": ("C5", lgreco.POWERSGD, W.PSGD_RANKS_C5, 16, "low_rank"),
}


def main():
    name = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg, fam, params, di, gen = SPECS[name]
    layers = W.config_layers(cfg)
    t0 = time.time()
    dev = torch.device("cuda:0")
    g, e = W.recipe_device(layers, gen, dev, seed=0x5EED)  # the 8(d) recipe, drawn on the device
    torch.cuda.synchronize()
    print(f"# inputs {time.time() - t0:.1f} s", flush=True)
    L, K = len(layers), len(params)
    err = torch.empty(L, K, dtype=torch.float64, device=dev)
    bits = torch.empty(L, K, dtype=torch.int64, device=dev)
    dflt = torch.full((L,), di, dtype=torch.int32, device=dev)
    comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=dev)
    ch = torch.empty(L, dtype=torch.int32, device=dev)
    info = torch.empty(48, dtype=torch.uint8, device=dev)
    ws = torch.empty(lgreco.solve_workspace_bytes(L, K, 10000), dtype=torch.uint8, device=dev)
    out = torch.empty_like(g)
    ctx = lgreco.Context(layers, fam, params, seed=0x5EED)
    for s in range(steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        ctx.profile(g, e, s, err, bits)
        ev[1].record()
        lgreco.solve(err, bits, dflt, comp, D=10000, choice=ch, info=info, workspace=ws)
        ev[2].record()
        ctx.compress_allreduce_dev(ch, g, e, out, s)
        ev[3].record()
        torch.cuda.synchronize()
        print(f"step {s}: profile {ev[0].elapsed_time(ev[1]):.3f} solve {ev[1].elapsed_time(ev[2]):.3f} "
              f"compress {ev[2].elapsed_time(ev[3]):.3f} ms", flush=True)
    ctx.check()
    ctx.close()


if __name__ == "__main__":
    main()
