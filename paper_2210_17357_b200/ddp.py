"""NEXT-3: L-GreCo as a PyTorch DDP communication hook (PAPER.md:312-314
"accumulate the gradients ... the designated worker computes the errors ... runs the
dynamic programming ... and broadcasts the mapping", PAPER.md:343 buckets).

Per DDP bucket (its parameters form the layer table, >= 2-D tensors compressed, R8):
  * warm-up steps: plain all-reduce of the bucket (the paper's uncompressed warm-up),
    the local gradient accumulated into G;
  * at every replan boundary (end of the warm-up, then every `replan_every` steps):
    lgreco_profile on the accumulated G (paper mode: no EF, R2), lgreco_solve, the plan
    broadcast from rank 0 (R21), G reset;
  * other steps: lgreco_compress_allreduce_dev with the current plan and the bucket's
    error-feedback buffer -- the compressed exchange and decode -- and G += g.
Every compute step runs in the library's kernels on the current stream; this module is
orchestration only (bucket bookkeeping, which call when).

Usage:
    state = LGrecoHook(lgreco.QSGD, workloads.QSGD_BITS, default_idx=2)
    ddp_model.register_comm_hook(state, LGrecoHook.hook)
"""
import torch
import torch.distributed as dist

from . import lgreco
from . import workloads as W


class _Bucket:
    def __init__(self, owner, layers, shapes, device):
        self.layers = layers
        self.shapes = shapes
        L, K = len(layers), owner.K
        n = W.total_numel(layers)
        kw = dict(qbucket=owner.qbucket, seed=owner.seed, rank=owner.rank, world=owner.world)
        if owner.world > 1 and owner.family == lgreco.QSGD and owner.exchange == "p2p":
            # peer-memory exchange: every rank exports its windows once, all-gathers the
            # IPC handles over the process group and opens its peers' (no NCCL on the data path)
            self.ctx = lgreco.Context(layers, owner.family, owner.params, **kw)
            blobs = [None] * owner.world
            dist.all_gather_object(blobs, self.ctx.p2p_export(), group=owner.pg)
            self.ctx.p2p_open(blobs)
        else:
            nid = None
            if owner.world > 1:
                obj = [lgreco.nccl_unique_id() if owner.rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=owner.pg)
                nid = obj[0]
            self.ctx = lgreco.Context(layers, owner.family, owner.params, nccl_id=nid, **kw)
        self.ef = torch.zeros(n, dtype=torch.float32, device=device)
        self.G = torch.zeros(n, dtype=torch.float32, device=device)
        self.out = torch.empty(n, dtype=torch.float32, device=device)
        self.err = torch.empty(L, K, dtype=torch.float64, device=device)
        self.bits = torch.empty(L, K, dtype=torch.int64, device=device)
        self.dflt = torch.full((L,), owner.default_idx, dtype=torch.int32, device=device)
        self.comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=device)
        self.choice = torch.full((L,), owner.default_idx, dtype=torch.int32, device=device)
        self.info = torch.empty(48, dtype=torch.uint8, device=device)
        self.ws = torch.empty(lgreco.solve_workspace_bytes(L, K, owner.D), dtype=torch.uint8, device=device)
        self.calls = 0
        self.planned = False
        self.added = []  # record=True: the gradients accumulated into G since its last reset


class LGrecoHook:
    def __init__(self, family, params, default_idx, *, warmup_steps=10, replan_every=100, D=10000, seed=0x5EED,
                 qbucket=128, flags=0, process_group=None, record=False, exchange="p2p", timer=None):
        self.family, self.params = family, [int(p) for p in params]
        self.K = len(self.params)
        self.default_idx = int(default_idx)
        self.warmup, self.replan_every = int(warmup_steps), int(replan_every)
        self.D, self.seed, self.qbucket, self.flags = int(D), int(seed), int(qbucket), int(flags)
        self.pg = process_group
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        self.exchange = exchange
        self.buckets: dict[int, _Bucket] = {}
        self.record = record
        self.last = {}  # bucket index -> (g, ef_before, choice, step) when record=True
        # NEXT-1: a bucket_timer.BucketSyncTimer brackets every
        # compressed bucket's synchronisation with device events, recording the bytes the
        # plan transmits (objectives.fit_bucket_time -> time_weights)
        self.timer = timer
        self._timer_open = False

    def _state(self, bucket):
        shapes = tuple(tuple(p.shape) for p in bucket.parameters())
        idx = bucket.index()
        st = self.buckets.get(idx)
        if st is not None and st.shapes != shapes:  # DDP rebuilt its buckets: new layout
            st.ctx.close()
            st = None
        if st is None:
            layers = W.layer_table([(None, s) for s in shapes])
            st = _Bucket(self, layers, shapes, bucket.buffer().device)
            self.buckets[idx] = st
        return st

    def _replan(self, st):
        """Profile the accumulated gradient (paper mode), solve, agree on rank 0's plan."""
        st.ctx.profile(st.G, None, st.calls, st.err, st.bits)
        lgreco.solve(st.err, st.bits, st.dflt, st.comp, D=self.D, flags=self.flags, choice=st.choice, info=st.info,
                     workspace=st.ws)
        st.ctx.plan_broadcast(st.choice)
        st.G.zero_()
        st.added = []
        st.planned = True
        if self.timer is not None:  # the plan's transmitted bytes (one host round trip per replan)
            ch = st.choice.cpu().tolist()
            if self.family != lgreco.POWERSGD:
                st.sent = st.ctx.payload_bytes(ch)
            else:  # R11: 32 r (m + k) bits, raw when r (m + k) >= m k
                st.sent = sum(4 * min(self.params[c] * (l.rows + l.cols), l.numel) if l.compress and c >= 0
                              else 4 * l.numel for l, c in zip(st.layers, ch))

    @staticmethod
    def hook(state: "LGrecoHook", bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
        st = state._state(bucket)
        g = bucket.buffer()
        st.calls += 1
        step = st.calls
        if state.record:
            st.added.append(g.clone())
        if step <= state.warmup or not st.planned:
            lgreco.accumulate(st.G, g)
            if step >= state.warmup:
                state._replan(st)
            fut = dist.all_reduce(g, group=state.pg, async_op=True).get_future()
            world = state.world
            return fut.then(lambda f: f.value()[0].div_(world))
        rec = (g.clone(), st.ef.clone(), st.choice.clone(), step) if state.record else None
        lgreco.accumulate(st.G, g)
        tm = state.timer
        if tm is not None:
            if bucket.index() == 0:  # DDP hands the buckets over in index order every step
                if state._timer_open:
                    tm.end_step()
                tm.begin_step()
                state._timer_open = True
            tm.start(bucket.index())
        st.ctx.compress_allreduce_dev(st.choice, g, st.ef, st.out, step)
        if tm is not None:
            tm.stop(bucket.index(), st.sent)
        g.copy_(st.out)
        if rec is not None:
            state.last[bucket.index()] = rec + (st.out.clone(), st.layers)
        if (step - state.warmup) % state.replan_every == 0:
            state._replan(st)
        fut = torch.futures.Future()
        fut.set_result(g)
        return fut

    def close(self):
        for st in self.buckets.values():
            st.ctx.close()
        self.buckets.clear()
