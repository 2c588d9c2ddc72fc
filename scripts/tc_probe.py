import torch, sys, time
sys.path.insert(0, '/root/repo')
from paper_2210_17357_b200 import lgreco
dev = torch.device('cuda')
m, k, r = 4096, 4608, 16
g = torch.randn(m * k, device=dev) * 1e-3
e = torch.randn(m * k, device=dev) * 1e-4
Q = torch.randn(k * r, device=dev)
P = torch.empty(m * r, device=dev)
for name, ee in (("g+e", e), ("g only", None)):
    for _ in range(3): lgreco.debug_tc_mq(g, ee, m, k, Q, r, P)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): lgreco.debug_tc_mq(g, ee, m, k, Q, r, P)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 20
    nb = m * k * (8 if ee is not None else 4)
    print(f"{name}: {t*1e3:.1f} us  {nb/t/1e6:.0f} GB/s")
