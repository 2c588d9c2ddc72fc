"""NEXT-3: the DDP communication hook on one GPU (NCCL process group
of size 1): warm-up steps are plain all-reduces (bitwise the local gradients), then every
bucket is compressed with the plan solved from the accumulated gradient, bitwise equal
to calling the library directly on the recorded inputs, and training still converges."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2210_17357_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ddp_hook_one_gpu(ref):
    from paper_2210_17357_b200 import lgreco
    from paper_2210_17357_b200.ddp import LGrecoHook
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        torch.manual_seed(0)
        net = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 512),
                                  torch.nn.ReLU(), torch.nn.Linear(512, 10)).cuda()
        ref_net = torch.nn.Sequential(*[type(m)(*([m.in_features, m.out_features] if isinstance(m, torch.nn.Linear)
                                                   else [])) for m in net]).cuda()
        ref_net.load_state_dict(net.state_dict())
        ddp = torch.nn.parallel.DistributedDataParallel(net, device_ids=[0], bucket_cap_mb=0.5)
        from paper_2210_17357_b200.bucket_timer import BucketSyncTimer
        timer = BucketSyncTimer()
        state = LGrecoHook(lgreco.QSGD, W.QSGD_BITS, default_idx=2, warmup_steps=2, replan_every=4, record=True,
                           timer=timer)
        ddp.register_comm_hook(state, LGrecoHook.hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
        g = torch.Generator(device="cuda").manual_seed(1)
        X = torch.randn(512, 256, device="cuda", generator=g)
        Y = torch.randint(0, 10, (512,), device="cuda", generator=g)
        losses = []
        for step in range(12):
            opt.zero_grad(set_to_none=True)
            loss = torch.nn.functional.cross_entropy(ddp(X), Y)
            loss.backward()
            if step < 2:  # warm-up: uncompressed all-reduce of one rank = the local gradient
                ref_net.load_state_dict(net.state_dict())
                torch.nn.functional.cross_entropy(ref_net(X), Y).backward()
                for p, q in zip(net.parameters(), ref_net.parameters()):
                    assert torch.equal(p.grad, q.grad)
                    q.grad = None
            losses.append(float(loss.detach()))
            opt.step()
        torch.cuda.synchronize()
        # NEXT-1: the hook's bucket timer saw every compressed step of every bucket, with
        # the plan's transmitted bytes (lgreco_payload_bytes) and device-timed intervals
        timer.end_step()
        sizes, sync, per = timer.samples()
        assert sizes.shape[0] >= 8 and sizes.shape[1] == len(state.buckets), sizes.shape
        assert np.all(sizes > 0) and np.all(per > 0) and np.all(sync >= per.max(axis=1) - 1e-6)
        for idx, stb in state.buckets.items():
            assert sizes[-1, idx] == stb.ctx.payload_bytes(stb.choice.cpu().tolist())
        assert state.last, "no compressed step was recorded"
        for idx, (gin, ef0, choice, st, out, layers) in state.last.items():
            # the hook's compressed step vs the ORACLE on the recorded inputs (R13, W = 1)
            ch = choice.cpu().numpy()
            lbits = [W.QSGD_BITS[c] if c >= 0 else 0 for c in ch]
            r_out, _, _, _ = ref.qsgd_allreduce(layers, lbits, [gin.cpu().numpy()], [ef0.cpu().numpy()],
                                                seed=state.seed, step=st)
            assert np.array_equal(out.cpu().numpy().view(np.uint32), r_out.view(np.uint32))
            assert int((choice >= 0).sum()) == sum(l.compress for l in layers)
        # accumulation (row a1, K0): G after the last replan = the oracle's G += g over the
        # bucket gradients the hook added since (bitwise)
        n_acc = 0
        for stt in state.buckets.values():
            Gr = np.zeros(stt.G.numel(), np.float32)
            for gi in stt.added:
                Gr = ref.accumulate(Gr, gi.cpu().numpy())
            assert np.array_equal(stt.G.cpu().numpy().view(np.uint32), Gr.view(np.uint32))
            n_acc += len(stt.added)
        assert n_acc > 0
        assert np.mean(losses[-3:]) < losses[0]
        state.close()
    finally:
        dist.destroy_process_group()
