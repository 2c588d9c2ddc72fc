"""NEXT-3 measurement (not part of the tests): synthetic ResNet-50 training step on one
GPU under DDP (NCCL group of size 1), plain all-reduce vs the L-GreCo QSGD hook
(paper_2210_17357_b200/ddp.py) after its warm-up, replanning every `replan` steps.
Prints one JSON line with the per-step device times."""
import json
import os
import socket
import sys

import torch
import torch.distributed as dist
import torchvision

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_17357_b200 import lgreco, workloads as W  # noqa: E402
from paper_2210_17357_b200.ddp import LGrecoHook  # noqa: E402


def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def run(use_hook, steps=30, warm=10, batch=64, replan=10):
    torch.manual_seed(0)
    net = torchvision.models.resnet50().cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(net, device_ids=[0])
    state = None
    if use_hook:
        state = LGrecoHook(lgreco.QSGD, W.QSGD_BITS, default_idx=2, warmup_steps=3, replan_every=replan)
        ddp.register_comm_hook(state, LGrecoHook.hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)
    X = torch.randn(batch, 3, 224, 224, device="cuda")
    Y = torch.randint(0, 1000, (batch,), device="cuda")
    ev = []
    for i in range(warm + steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        opt.zero_grad(set_to_none=True)
        torch.nn.functional.cross_entropy(ddp(X), Y).backward()
        opt.step()
        b.record()
        if i >= warm:
            ev.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    if state:
        state.close()
    return ms[len(ms) // 2], sum(ms) / len(ms)


if __name__ == "__main__":
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    base = run(False)
    hook = run(True)
    print(json.dumps({"workload": "ResNet-50 synthetic step, batch 64, fp32, 1 GPU DDP",
                      "allreduce_ms_median": round(base[0], 3), "allreduce_ms_mean": round(base[1], 3),
                      "lgreco_qsgd_ms_median": round(hook[0], 3), "lgreco_qsgd_ms_mean": round(hook[1], 3),
                      "replan_every": 10}))
    dist.destroy_process_group()
