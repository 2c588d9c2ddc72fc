"""tcgen05 kind::tf32 (3xTF32) contraction P = M Q used by PowerSGD, against an fp64
reference of the same product (normwise; 3xTF32 is fp32-grade)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,r", [(128, 32, 16), (300, 1000, 16), (1000, 257, 32), (4608, 512, 64), (77, 4608, 4),
                                   (512, 4608, 16)])
def test_tc_mq(m, k, r):
    from paper_2210_17357_b200 import lgreco
    rng = np.random.default_rng(m + k + r)
    g = rng.standard_normal((m, k)).astype(np.float32)
    e = (rng.standard_normal((m, k)) * 0.1).astype(np.float32)
    Q = rng.uniform(-1, 1, (r, k)).astype(np.float32)  # column-major k x r == row-major r x k
    P = torch.zeros(r * m, dtype=torch.float32, device="cuda")
    lgreco.debug_tc_mq(torch.from_numpy(g.ravel()).cuda(), torch.from_numpy(e.ravel()).cuda(), m, k,
                       torch.from_numpy(Q.ravel()).cuda(), r, P)
    x = ((g + e) + np.float32(0)).astype(np.float64)
    ref = x @ Q.astype(np.float64).T  # m x r
    got = P.cpu().numpy().reshape(r, m).T
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 2e-6, rel


@pytest.mark.parametrize("m,k,r", [(32, 128, 16), (300, 1000, 16), (1000, 257, 32), (512, 4608, 64), (2048, 77, 4)])
def test_tc_mtp(m, k, r):
    from paper_2210_17357_b200 import lgreco
    rng = np.random.default_rng(m * 3 + k + r)
    g = rng.standard_normal((m, k)).astype(np.float32)
    e = (rng.standard_normal((m, k)) * 0.1).astype(np.float32)
    P = rng.uniform(-1, 1, (r, m)).astype(np.float32)  # column-major m x r
    Q = torch.zeros(r * k, dtype=torch.float32, device="cuda")
    lgreco.debug_tc_mtp(torch.from_numpy(g.ravel()).cuda(), torch.from_numpy(e.ravel()).cuda(), m, k,
                        torch.from_numpy(P.ravel()).cuda(), r, Q)
    x = ((g + e) + np.float32(0)).astype(np.float64)
    ref = x.T @ P.astype(np.float64).T  # k x r
    got = Q.cpu().numpy().reshape(r, k).T
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 2e-6, rel
