"""The exact path bench.py times, end to end against the oracle (VERDICT r01 "parity
holes"): C4 at full size, QSGD 2..8 bits, default 4, D = 10000, W = 1, in the bench's
launch configuration -- lgreco_profile -> device lgreco_solve (its plan never leaves the
device) -> lgreco_compress_allreduce_dev (fused W = 1 K5) -- over consecutive steps with
the error feedback chained, against the oracle's profile -> Algorithm 1 -> pack/decode
on the same seeded inputs.  Plans bitwise, outputs and EF bitwise, error tables 1e-5."""
import numpy as np
import pytest
import torch

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu

SEED = 0x5EED
D = 10000


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg", ["C4", "C1"])
def test_timed_path_matches_oracle(ref, cfg):
    from paper_2210_17357_b200 import lgreco
    layers = W.config_layers(cfg)
    bits_c = W.QSGD_BITS
    L, K = len(layers), len(bits_c)
    g, e = W.gaussian_outliers(layers, seed=W.rank_seed(SEED, 0))
    dflt_i = bits_c.index(4)
    comp_l = [l.compress for l in layers]
    ctx = lgreco.Context(layers, lgreco.QSGD, bits_c, qbucket=128, seed=SEED)
    gd, ed = _dev(g), _dev(e)
    out = torch.empty_like(gd)
    err = torch.empty(L, K, dtype=torch.float64, device="cuda")
    bits = torch.empty(L, K, dtype=torch.int64, device="cuda")
    dflt = torch.full((L,), dflt_i, dtype=torch.int32, device="cuda")
    comp = torch.tensor(comp_l, dtype=torch.int32, device="cuda")
    ch = torch.empty(L, dtype=torch.int32, device="cuda")
    info = torch.empty(48, dtype=torch.uint8, device="cuda")
    ws = torch.empty(lgreco.solve_workspace_bytes(L, K, D), dtype=torch.uint8, device="cuda")
    e_ref = e.copy()
    mixed = False
    for step in range(3):
        # GPU: the bench's step() with nothing in between (no host synchronisation)
        ctx.profile(gd, ed, step, err, bits)
        lgreco.solve(err, bits, dflt, comp, D=D, choice=ch, info=info, workspace=ws)
        ctx.compress_allreduce_dev(ch, gd, ed, out, step)
        torch.cuda.synchronize()
        # oracle: the same step on the same bytes
        r_err, r_bits = ref.qsgd_profile(layers, g, e_ref, bits_c, seed=SEED, step=step)
        st, r_choice, r_info = ref.solve(r_err, r_bits, [dflt_i] * L, comp_l, D=D)
        assert st == 0
        lbits = [bits_c[c] if c >= 0 else 0 for c in r_choice]
        r_out, r_es, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e_ref], seed=SEED, step=step)
        e_ref = r_es[0]
        assert np.array_equal(bits.cpu().numpy(), r_bits)
        ge = err.cpu().numpy()
        assert (np.abs(ge - r_err) / np.maximum(r_err, 1e-300)).max() <= 1e-5
        assert np.array_equal(ch.cpu().numpy(), r_choice), step
        mixed |= len({int(c) for c, cp in zip(r_choice, comp_l) if cp}) > 1
        assert np.array_equal(out.cpu().numpy().view(np.uint32), r_out.view(np.uint32)), step
        assert np.array_equal(ed.cpu().numpy().view(np.uint32), e_ref.view(np.uint32)), step
        gi = lgreco.read_info(info)
        assert gi.used_default == r_info.used_default and gi.total_bits == r_info.total_bits
    assert mixed, "the solver's plan should mix bit-widths on this workload"
    ctx.check()
    ctx.close()
