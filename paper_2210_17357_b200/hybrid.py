"""NEXT-4: mixed-family L-GreCo ("combining different compression
techniques inside the same model").  One library context per family on
the same layer table; every step of the path runs in the library:

  profile   each family profiles every layer (lgreco_profile)
  table     lgreco_hybrid_table puts the families' (err, bits) tables side by side
  solve     Algorithm 1 on the joint table picks a (family, parameter) per layer
  split     lgreco_hybrid_split -> one choice vector per family (CHOICE_SKIP elsewhere)
  compress  each family's lgreco_compress_allreduce_dev compresses its own layers and
            leaves the others' EF / output untouched, at any W: a CHOICE_SKIP layer has no
            QSGD records and no TopK pairs in its ctx's exchange (R24); PowerSGD
            through its host plan

This module is orchestration only (which call when); the defaults of the joint table
are the column of one family's default (`default_family`, `default_idx`).
"""
import torch

from . import lgreco


class Hybrid:
    def __init__(self, layers, families, *, seed=0, rank=0, world=1, qbucket=128, default_family=0, default_idx=0,
                 D=10000, nccl_ids=None):
        """families: list of (lgreco.QSGD | TOPK | POWERSGD, params)."""
        self.layers, self.D = layers, int(D)
        self.ctxs = [lgreco.Context(layers, fam, params, qbucket=qbucket, seed=seed, rank=rank, world=world,
                                    nccl_id=None if nccl_ids is None else nccl_ids[i])
                     for i, (fam, params) in enumerate(families)]
        self.Ks = [len(p) for _, p in families]
        self.col0 = [sum(self.Ks[:f]) for f in range(len(self.Ks))]
        self.default_col = self.col0[default_family] + int(default_idx)
        self.L = len(layers)

    def profile(self, g, ef, step, stream=None):
        """Per-family tables, then the joint (L, sum K) table on the device."""
        dev = g.device
        errs, bits = [], []
        for ctx, K in zip(self.ctxs, self.Ks):
            e = torch.empty(self.L, K, dtype=torch.float64, device=dev)
            b = torch.empty(self.L, K, dtype=torch.int64, device=dev)
            ctx.profile(g, ef, step, e, b, stream)
            errs.append(e)
            bits.append(b)
        return lgreco.hybrid_table(errs, bits, stream=stream)

    def solve(self, err, bits, compress=None, stream=None):
        dflt = torch.full((self.L,), self.default_col, dtype=torch.int32, device=err.device)
        return lgreco.solve(err, bits, dflt, compress, D=self.D, stream=stream)

    def compress_allreduce(self, choice, g, ef, out, step, stream=None):
        """choice: the joint plan (device, (L,) column indices)."""
        per = lgreco.hybrid_split(choice, self.Ks, stream=stream)
        for ctx, ch in zip(self.ctxs, per):
            ctx.compress_allreduce_dev(ch, g, ef, out, step, stream)
        return per

    def check(self):
        for ctx in self.ctxs:
            ctx.check()

    def close(self):
        for ctx in self.ctxs:
            ctx.close()
