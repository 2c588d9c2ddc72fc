"""Seeded synthetic workloads: layer tables shaped like the paper's models and
gradient generators.  This module holds NO arithmetic of the method (no
quantisation, selection, factorisation or DP): it only describes shapes and
draws random numbers, so both the CUDA path and the CPU oracle may use it
(task rule: "only the seeded input generators serve both").

Shapes:
  C1  12 flat layers n_l = round(1024 * 256**(l/11))             (N = 660,492)
  C2  ResNet-18 / CIFAR-10   62 tensors, 11,173,962 params (Table 1)
  C3  Transformer-XL base    180 tensors, 191,948,759 params
  C4  ResNet-50 / ImageNet   161 tensors, 25,557,032 params (Table 1)
  C5  GPT-2-medium-like LM   292 tensors, 354,823,168 params (BASELINE.json C5)
  TLM fairseq transformer_lm 6x512, V=267,744 (ratio pin only)

Layer record: (offset, numel, rows, cols, compress).  Matrix view of a >=2-D
tensor is (shape[0], numel/shape[0]); 1-D tensors are vectors,
sent lossless (compress=0) in the real-model sets.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


# ----------------------------------------------------------------------------
# shape lists (name, shape) in parameter-registration order
# ----------------------------------------------------------------------------

def _bn(name, c):
    return [(name + ".weight", (c,)), (name + ".bias", (c,))]


def resnet18_cifar(num_classes: int = 10):
    s = [("conv1.weight", (64, 3, 3, 3))] + _bn("bn1", 64)
    inp = 64
    for li, (planes, stride) in enumerate([(64, 1), (128, 2), (256, 2), (512, 2)]):
        for bi in range(2):
            st = stride if bi == 0 else 1
            p = f"layer{li + 1}.{bi}"
            s += [(p + ".conv1.weight", (planes, inp, 3, 3))] + _bn(p + ".bn1", planes)
            s += [(p + ".conv2.weight", (planes, planes, 3, 3))] + _bn(p + ".bn2", planes)
            if st != 1 or inp != planes:
                s += [(p + ".shortcut.0.weight", (planes, inp, 1, 1))] + _bn(p + ".shortcut.1", planes)
            inp = planes
    s += [("linear.weight", (num_classes, 512)), ("linear.bias", (num_classes,))]
    return s


def resnet50():
    s = [("conv1.weight", (64, 3, 7, 7))] + _bn("bn1", 64)
    inp = 64
    for li, (planes, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]):
        for bi in range(blocks):
            p = f"layer{li + 1}.{bi}"
            s += [(p + ".conv1.weight", (planes, inp, 1, 1))] + _bn(p + ".bn1", planes)
            s += [(p + ".conv2.weight", (planes, planes, 3, 3))] + _bn(p + ".bn2", planes)
            s += [(p + ".conv3.weight", (planes * 4, planes, 1, 1))] + _bn(p + ".bn3", planes * 4)
            if bi == 0:
                s += [(p + ".downsample.0.weight", (planes * 4, inp, 1, 1))] + _bn(p + ".downsample.1", planes * 4)
            inp = planes * 4
    s += [("fc.weight", (1000, 2048)), ("fc.bias", (1000,))]
    return s


def transformer_xl_base(n_token=267735, d=512, n_layer=16, n_head=8, d_head=64, d_inner=2048):
    s = [("word_emb.emb_layers.0.weight", (n_token, d))]
    for i in range(n_layer):
        p = f"layers.{i}"
        s += [(p + ".dec_attn.qkv_net.weight", (3 * n_head * d_head, d)),
              (p + ".dec_attn.o_net.weight", (d, n_head * d_head)),
              (p + ".dec_attn.layer_norm.weight", (d,)), (p + ".dec_attn.layer_norm.bias", (d,)),
              (p + ".dec_attn.r_net.weight", (n_head * d_head, d)),
              (p + ".pos_ff.CoreNet.0.weight", (d_inner, d)), (p + ".pos_ff.CoreNet.0.bias", (d_inner,)),
              (p + ".pos_ff.CoreNet.3.weight", (d, d_inner)), (p + ".pos_ff.CoreNet.3.bias", (d,)),
              (p + ".pos_ff.layer_norm.weight", (d,)), (p + ".pos_ff.layer_norm.bias", (d,))]
    s += [("crit.out_layers.0.bias", (n_token,)),
          ("r_w_bias", (n_head, d_head)), ("r_r_bias", (n_head, d_head))]
    return s


def gpt2_medium_like(vocab=50257, n_pos=1024, d=1024, n_layer=24, d_ff=4096):
    s = [("wte.weight", (vocab, d)), ("wpe.weight", (n_pos, d))]
    for i in range(n_layer):
        p = f"h.{i}"
        s += [(p + ".ln_1.weight", (d,)), (p + ".ln_1.bias", (d,)),
              (p + ".attn.c_attn.weight", (d, 3 * d)), (p + ".attn.c_attn.bias", (3 * d,)),
              (p + ".attn.c_proj.weight", (d, d)), (p + ".attn.c_proj.bias", (d,)),
              (p + ".ln_2.weight", (d,)), (p + ".ln_2.bias", (d,)),
              (p + ".mlp.c_fc.weight", (d, d_ff)), (p + ".mlp.c_fc.bias", (d_ff,)),
              (p + ".mlp.c_proj.weight", (d_ff, d)), (p + ".mlp.c_proj.bias", (d,))]
    s += [("ln_f.weight", (d,)), ("ln_f.bias", (d,))]
    return s


def fairseq_transformer_lm(vocab=267744, d=512, n_layer=6, d_ff=2048):
    s = [("embed_tokens.weight", (vocab, d))]
    for i in range(n_layer):
        p = f"layers.{i}"
        for proj in ("k_proj", "v_proj", "q_proj", "out_proj"):
            s += [(p + f".self_attn.{proj}.weight", (d, d)), (p + f".self_attn.{proj}.bias", (d,))]
        s += [(p + ".self_attn_layer_norm.weight", (d,)), (p + ".self_attn_layer_norm.bias", (d,)),
              (p + ".fc1.weight", (d_ff, d)), (p + ".fc1.bias", (d_ff,)),
              (p + ".fc2.weight", (d, d_ff)), (p + ".fc2.bias", (d,)),
              (p + ".final_layer_norm.weight", (d,)), (p + ".final_layer_norm.bias", (d,))]
    return s


def synthetic12():
    return [(f"layer{l}", (round(1024 * 256 ** (l / 11)),)) for l in range(12)]


# ----------------------------------------------------------------------------
# layer tables
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Layer:
    offset: int
    numel: int
    rows: int      # 0 -> vector
    cols: int
    compress: int  # 1 -> in the DP / compressed, 0 -> lossless


def layer_table(shapes, compress_vectors: bool = False):
    out, off = [], 0
    for _, shp in shapes:
        n = int(np.prod(shp))
        if len(shp) >= 2:
            out.append(Layer(off, n, int(shp[0]), n // int(shp[0]), 1))
        else:
            out.append(Layer(off, n, 0, 0, 1 if compress_vectors else 0))
        off += n
    return out


def total_numel(layers) -> int:
    return max((l.offset + l.numel for l in layers), default=0)


CONFIGS = {
    # name: (shape fn, compress 1-D tensors?)
    "C1": (synthetic12, True),
    "C2": (resnet18_cifar, False),
    "C3": (transformer_xl_base, False),
    "C4": (resnet50, False),
    "C5": (gpt2_medium_like, False),
    "TLM": (fairseq_transformer_lm, False),
}


def config_layers(name: str):
    fn, cv = CONFIGS[name]
    return layer_table(fn(), compress_vectors=cv)


# Candidate sets (PAPER.md:437-442 range policy)
QSGD_BITS = [2, 3, 4, 5, 6, 7, 8]               # default 4
TOPK_PPM_C3 = [1000 * i for i in range(1, 101)]  # 0.1%..10% step 0.1% (ppm), default 1%
TOPK_PPM_C5 = [10000 * i for i in range(1, 101)]  # 1%..100% step 1%, default 10%
PSGD_RANKS_C2 = [1, 2, 4, 8, 16]                 # default 4
PSGD_RANKS_C5 = list(range(16, 65))              # 16..64, default 32


# ----------------------------------------------------------------------------
# seeded generators (numpy float32 arrays; identical bytes go to GPU and oracle)
# ----------------------------------------------------------------------------

def _gen(seed: int, layer: int) -> torch.Generator:
    g = torch.Generator()
    g.manual_seed((seed * 0x9E3779B1 + layer * 0x85EBCA6B + 0x5EED) % (2 ** 63))
    return g


def _sigma(g: torch.Generator) -> float:
    # log-uniform in [1e-4, 1e-1]
    return float(10.0 ** (-4.0 + 3.0 * torch.rand(1, generator=g, dtype=torch.float64).item()))


def gaussian_outliers(layers, seed: int = 0, with_ef: bool = True):
    """C1/C4 recipe: per-layer sigma log-uniform [1e-4,1e-1]; N(0, sigma^2) with
    1% outliers x10; e ~ N(0, (0.1 sigma)^2).  Returns (g, e) float32 flat."""
    n = total_numel(layers)
    gbuf = torch.zeros(n, dtype=torch.float32)
    ebuf = torch.zeros(n, dtype=torch.float32) if with_ef else None
    for li, L in enumerate(layers):
        g = _gen(seed, li)
        sig = _sigma(g)
        x = torch.randn(L.numel, generator=g, dtype=torch.float32) * sig
        nout = max(0, L.numel // 100)
        if nout:
            idx = torch.randint(0, L.numel, (nout,), generator=g)
            x[idx] *= 10.0
        gbuf[L.offset:L.offset + L.numel] = x
        if with_ef:
            ebuf[L.offset:L.offset + L.numel] = torch.randn(L.numel, generator=g, dtype=torch.float32) * (0.1 * sig)
    return gbuf.numpy(), (ebuf.numpy() if with_ef else None)


def heavy_tailed(layers, seed: int = 0, with_ef: bool = True, sparse_rows_layer: int | None = 0,
                 zero_row_frac: float = 0.9):
    """C3 recipe: Student-t(nu=3) x sigma_l; the embedding gradient (layer
    `sparse_rows_layer`) is row-sparse with `zero_row_frac` of rows zero."""
    n = total_numel(layers)
    gbuf = torch.zeros(n, dtype=torch.float32)
    ebuf = torch.zeros(n, dtype=torch.float32) if with_ef else None
    for li, L in enumerate(layers):
        g = _gen(seed, li)
        sig = _sigma(g)
        z = torch.randn(L.numel, generator=g, dtype=torch.float32)
        chi = torch.randn(3, L.numel, generator=g, dtype=torch.float32).pow_(2).sum(0)
        x = z / torch.sqrt(chi / 3.0) * sig
        if sparse_rows_layer is not None and li == sparse_rows_layer and L.rows > 0:
            keep = torch.rand(L.rows, generator=g) >= zero_row_frac
            x = (x.view(L.rows, L.cols) * keep[:, None].float()).reshape(-1)
        gbuf[L.offset:L.offset + L.numel] = x
        if with_ef:
            ebuf[L.offset:L.offset + L.numel] = torch.randn(L.numel, generator=g, dtype=torch.float32) * (0.1 * sig)
    return gbuf.numpy(), (ebuf.numpy() if with_ef else None)


def low_rank_plus_noise(layers, seed: int = 0, rank: int = 64, noise: float = 0.1, with_ef: bool = False):
    """C2 recipe: per matrix M = U diag(sigma_l / i) V^T (rank 64) + noise with
    ||noise||_F = noise * ||signal||_F; vectors are N(0, sigma^2)."""
    n = total_numel(layers)
    gbuf = torch.zeros(n, dtype=torch.float32)
    ebuf = torch.zeros(n, dtype=torch.float32) if with_ef else None
    for li, L in enumerate(layers):
        g = _gen(seed, li)
        sig = _sigma(g)
        if L.rows > 0:
            r = min(rank, L.rows, L.cols)
            U = torch.randn(L.rows, r, generator=g, dtype=torch.float64) / math.sqrt(L.rows)
            V = torch.randn(L.cols, r, generator=g, dtype=torch.float64) / math.sqrt(L.cols)
            s = sig / torch.arange(1, r + 1, dtype=torch.float64)
            S = (U * s) @ V.T
            N = torch.randn(L.rows, L.cols, generator=g, dtype=torch.float64)
            N *= noise * S.norm() / N.norm()
            x = (S + N).reshape(-1).float()
        else:
            x = torch.randn(L.numel, generator=g, dtype=torch.float32) * sig
        gbuf[L.offset:L.offset + L.numel] = x
        if with_ef:
            ebuf[L.offset:L.offset + L.numel] = torch.randn(L.numel, generator=g, dtype=torch.float32) * (0.1 * sig)
    return gbuf.numpy(), (ebuf.numpy() if with_ef else None)


def rank_seed(base: int, rank: int) -> int:
    """Per-rank seeds: seed = 0x5EED + rank."""
    return base + rank


# ----------------------------------------------------------------------------
# the same recipes drawn on the device (bench.py's large configs: the CPU generators
# above would take minutes at 192M / 355M elements).  Same distributions, different
# bytes -- timing inputs only, never compared with the oracle.
# ----------------------------------------------------------------------------

def recipe_device(layers, recipe: str, dev, seed: int = 0, with_ef: bool = True, sparse_rows_layer: int | None = 0,
                  zero_row_frac: float = 0.9, rank: int = 64, noise: float = 0.1):
    """recipe: "gaussian" (C1/C4: N(0, s^2) + 1% outliers x10), "student_t" (C3:
    Student-t(3) x s, layer `sparse_rows_layer` row-sparse), "low_rank" (C2: rank-64
    signal with 1/i spectrum + 10% noise; vectors Gaussian).  Per-layer s log-uniform
    [1e-4, 1e-1]; e ~ N(0, (0.1 s)^2).  Returns (g, e) flat float32 tensors on dev."""
    n = total_numel(layers)
    gen = torch.Generator(device=dev)
    gen.manual_seed((seed * 0x9E3779B1 + 0x5EED) % (2 ** 63))
    g = torch.zeros(n, dtype=torch.float32, device=dev)
    e = torch.zeros(n, dtype=torch.float32, device=dev) if with_ef else None
    for li, L in enumerate(layers):
        sig = float(10.0 ** (-4.0 + 3.0 * torch.rand(1, generator=gen, device=dev, dtype=torch.float64).item()))
        view = g[L.offset:L.offset + L.numel]
        if recipe == "gaussian" or (recipe == "low_rank" and L.rows == 0):
            torch.randn(L.numel, generator=gen, device=dev, out=view)
            view.mul_(sig)
            if recipe == "gaussian" and L.numel >= 100:
                idx = torch.randint(0, L.numel, (L.numel // 100,), generator=gen, device=dev)
                view[idx] *= 10.0
        elif recipe == "student_t":
            torch.randn(L.numel, generator=gen, device=dev, out=view)
            chi = torch.zeros(L.numel, device=dev)
            for _ in range(3):
                chi.add_(torch.randn(L.numel, generator=gen, device=dev).pow_(2))
            view.div_(chi.div_(3.0).sqrt_()).mul_(sig)
            del chi
            if sparse_rows_layer is not None and li == sparse_rows_layer and L.rows > 0:
                keep = (torch.rand(L.rows, generator=gen, device=dev) >= zero_row_frac).float()
                view.view(L.rows, L.cols).mul_(keep[:, None])
        elif recipe == "low_rank":
            r = min(rank, L.rows, L.cols)
            U = torch.randn(L.rows, r, generator=gen, device=dev) / math.sqrt(L.rows)
            V = torch.randn(L.cols, r, generator=gen, device=dev) / math.sqrt(L.cols)
            s = sig / torch.arange(1, r + 1, device=dev, dtype=torch.float32)
            S = (U * s) @ V.T
            Nz = torch.randn(L.rows, L.cols, generator=gen, device=dev)
            Nz.mul_(noise * S.norm() / Nz.norm())
            view.copy_((S + Nz).reshape(-1))
            del U, V, S, Nz
        else:
            raise ValueError(recipe)
        if with_ef:
            ev = e[L.offset:L.offset + L.numel]
            torch.randn(L.numel, generator=gen, device=dev, out=ev)
            ev.mul_(0.1 * sig)
    return g, e
