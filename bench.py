#!/usr/bin/env python
"""bench.py -- L-GreCo data-parallel hot path on B200 (one process per GPU).

One STEP = one pass of the whole hot path over one synthetic gradient batch
(SURVEY.md §8(a)): profile every layer x every candidate (a2) -> Algorithm 1 DP
(a5-a6) -> plan agreement (a7) -> compress + EF + compressed all-reduce (a8-a10).

Default workload: C4 = ResNet-50 / ImageNet gradient shapes (25,557,032 fp32,
161 tensors, 54 compressed), QSGD bits {2..8}, default 4, bucket 128, D = 10000
(BASELINE.json configs[3], the north_star target).  Metric: gradient GB/s =
4 * N bytes per rank per step, aggregated over ranks (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2210_17357_b200 import workloads as W  # noqa: E402

METRIC = "gradient GB/s profile+solve+compress+allreduce"
WORKLOAD = "C4 ResNet-50/ImageNet gradient (25,557,032 fp32), QSGD bits 2..8 default 4, bucket 128, D=10000"
D_BINS = 10000
# K1 algorithmic lane-ops per compressed element, counted on the
# cheapest exact form of the pinned sequence R6: per candidate 7 (v = t*inv, w = RU(v - u),
# ceil, min s, fma dec, x - dec, fma d^2) x 7 candidates = 49; per element 21 (g + e,
# x - mn, 2 min/max, Philox4x32-10 15 per element, u word shift + convert 2)
K1_OPS_PER_ELEM = 70
FUSED_EXTRA_OPS = 5  # the planned candidate's compress in the fused pass: t*inv - u, ceil, min s, dec, x - dec
PIPE_NOTE = ("pipelined (PAPER.md:312-314, re-solved every step): step t = the fused profile + compress pass "
             "(lgreco_profile_compress) with the plan solved from the profile of step t-2, beside the solve of "
             "step t-1 (LGRECO_PC_CONCURRENT; the solve on 2 x 8-SM clusters, LGRECO_SOLVE_NARROW); "
             "value = gradient bytes / (K steps' time / K)")
SEED = 0x5EED


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def _cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return os.cpu_count(), len(os.sched_getaffinity(0)), model


# ------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling (every 2 ms) of SM clock and clock-event reasons in a thread,
    started right before and stopped right after the timed region."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, gpu_index):
        import threading
        self.idx = gpu_index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thr = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.idx)
        self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = {k: getattr(N, v, 0) for k, v in self.REASONS.items()}
        get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            N.nvmlDeviceGetCurrentClocksThrottleReasons

        def sample():
            self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            r = get_reasons(h)
            for k, bit in bits.items():
                if bit and (r & bit):
                    self.reasons.add(k)
        return sample

    def _run(self):
        try:
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(0.001)
        except Exception as ex:
            self.err = f"nvml: {ex}"

    def _smi(self):
        import subprocess
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip().split(",")
        self.sm.append(float(out[0]))
        self.max_mhz = float(out[1])
        for n, v in zip(names, out[2:]):
            if v.strip().lower() == "active":
                self.reasons.add(n)

    def start(self):
        """Called right before the timed region: NVML is initialised here (outside the
        region) so the sampling thread is already polling when the first step launches."""
        import threading
        try:
            self._sample = self._nvml()
            self.source = "nvml ~1 ms"
        except Exception as ex:
            self.err = f"nvml: {ex}"
            self._sample = self._smi
            self.source = "nvidia-smi"
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def stop(self):
        """Called right after the timed region's closing synchronize (one final sample)."""
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=5)
        try:
            self._sample()
        except Exception as ex:
            self.err = getattr(self, "err", "") + f"; final sample: {ex}"
        if not self.sm:
            return {"error": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.source,
                "min_mhz": min(self.sm)}


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2210_17357_b200 import lgreco

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    # (diagnostics: LG_BENCH_ONE_DEVICE=1 puts every rank on device 0 with a gloo group,
    # to exercise the N > 1 code path -- the peer-memory exchange over CUDA IPC -- on a
    # one-GPU box; the driver's runs never set it)
    one_dev = os.environ.get("LG_BENCH_ONE_DEVICE") == "1"
    local = 0 if one_dev else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    layers = W.config_layers("C4")
    N = W.total_numel(layers)
    L, K = len(layers), len(W.QSGD_BITS)
    g_np, e_np = W.gaussian_outliers(layers, seed=W.rank_seed(SEED, rank))
    g = torch.from_numpy(g_np).to(dev)
    e0 = torch.from_numpy(e_np).to(dev)
    ef = e0.clone()
    out = torch.empty_like(g)
    err = torch.empty(L, K, dtype=torch.float64, device=dev)
    bits = torch.empty(L, K, dtype=torch.int64, device=dev)
    dflt = torch.full((L,), W.QSGD_BITS.index(4), dtype=torch.int32, device=dev)
    comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=dev)
    choice_d = torch.empty(L, dtype=torch.int32, device=dev)
    info_d = torch.empty(48, dtype=torch.uint8, device=dev)
    ws = torch.empty(lgreco.solve_workspace_bytes(L, K, D_BINS), dtype=torch.uint8, device=dev)
    choice_h = torch.empty(L, dtype=torch.int32).pin_memory()
    l2_flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    exchange = "local"
    ctx = None
    if world > 1 and os.environ.get("LGRECO_EXCHANGE", "p2p") == "p2p":
        # the product exchange: K5 stores records straight into the owners' windows over
        # NVLink (CUDA IPC handles exchanged here), epoch flags instead of collectives
        try:
            ctx = lgreco.Context(layers, lgreco.QSGD, W.QSGD_BITS, qbucket=128, seed=SEED, rank=rank, world=world)
            blobs = [None] * world
            dist.all_gather_object(blobs, ctx.p2p_export())
            ctx.p2p_open(blobs)
            dist.barrier()
            exchange = "p2p (NVLink peer stores + epoch flags)"
        except Exception as ex:  # fall back to NCCL (reported in the JSON line)
            print(f"# p2p exchange unavailable ({ex}); using NCCL", file=sys.stderr)
            ctx = None
    if ctx is None:
        nccl_id = None
        if world > 1:
            obj = [lgreco.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
            exchange = "nccl (grouped send/recv all-to-all + all-gather)"
        ctx = lgreco.Context(layers, lgreco.QSGD, W.QSGD_BITS, qbucket=128, seed=SEED, rank=rank, world=world,
                             nccl_id=nccl_id)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(s, marks=None, gin=None, gout=None):
        """One step; marks = [begin, end] (headline pass: nothing recorded between the
        kernels, so the library's PDL chaining is undisturbed) or [begin, after profile,
        after solve, end] (stage pass)."""
        gin = g if gin is None else gin
        gout = out if gout is None else gout
        staged = marks is not None and len(marks) == 4
        if marks: marks[0].record(stream)
        ctx.profile(gin, ef, s, err, bits)
        if staged: marks[1].record(stream)
        lgreco.solve(err, bits, dflt, comp, D=D_BINS, choice=choice_d, info=info_d, workspace=ws)
        ctx.plan_broadcast(choice_d)
        if staged: marks[2].record(stream)
        # plan consumed on the device at W = 1 (no host round trip); copied to the host
        # inside the library when the exchange needs the shard sizes (W > 1)
        ctx.compress_allreduce_dev(choice_d, gin, ef, gout, s)
        if marks: marks[-1].record(stream)

    # ---- the pipelined schedule (the plan in force compresses the step,
    # the step's profile feeds the next solve), re-solved EVERY step: step t runs the fused
    # profile + compress pass (lgreco_profile_compress: one read of g and e) with the plan
    # solved from the profile of step t - 2, and the solve of step t - 1 runs beside it on
    # the SMs the fused kernel leaves free (LGRECO_PC_CONCURRENT).  Three plan buffers:
    # step t reads plans[t % 3], the solve of step t writes plans[(t + 2) % 3].
    plans = [dflt.clone() for _ in range(3)]
    # two (err, bits) table pairs: the fused pass of step t writes pair t % 2 while the solve
    # of step t - 1 beside it still reads pair (t - 1) % 2
    tabs = [(err, bits), (torch.empty_like(err), torch.empty_like(bits))]

    def step_pipe(s, gin=None, gout=None, conc=True, marks=None, pre_solve=None):
        gin = g if gin is None else gin
        gout = out if gout is None else gout
        staged = marks is not None and len(marks) == 3
        e_t, b_t = tabs[s % 2]
        if marks: marks[0].record(stream)
        ctx.profile_compress(plans[s % 3], gin, ef, gout, s, e_t, b_t, concurrent=conc)
        if staged: marks[1].record(stream)
        if pre_solve: pre_solve()
        lgreco.solve(e_t, b_t, dflt, comp, D=D_BINS, flags=lgreco.SOLVE_NARROW, choice=plans[(s + 2) % 3],
                     info=info_d, workspace=ws)
        ctx.plan_broadcast(plans[(s + 2) % 3])
        if marks: marks[-1].record(stream)

    pipelined = args.schedule == "pipelined"
    conc = world == 1  # (W > 1: profile + compress are two calls inside the library; no overlap)
    for s in range(args.warmup):
        step(s)
    if pipelined:
        for s in range(args.warmup):
            step_pipe(s, conc=conc and s > 0)
    torch.cuda.synchronize()
    ctx.check()
    pipe = None
    # SM clocks and throttle reasons sampled from here through both timed passes
    clocks = ClockSampler(local)
    clocks.start()
    if pipelined:
        # headline of the pipelined schedule: K consecutive steps between two events (no
        # L2 flush between them: it would serialise the overlap; each step streams 204 MB
        # in and 204 MB out, > the 126 MB L2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        p0, p1 = ev(), ev()
        base = args.warmup
        launches_p0 = ctx.launches()
        p0.record(stream)
        for s in range(args.steps):
            step_pipe(base + s, conc=conc)
        p1.record(stream)
        torch.cuda.synchronize()
        pipe_ms = p0.elapsed_time(p1) / args.steps
        pipe_launches = ctx.launches() - launches_p0 + args.steps
        # the same steps without the overlap (the fused pass waits for the solve before it):
        # what LGRECO_PC_CONCURRENT buys
        q0, q1 = ev(), ev()
        q0.record(stream)
        for s in range(args.steps):
            step_pipe(base + args.steps + s, conc=False)
        q1.record(stream)
        torch.cuda.synchronize()
        serial_ms = q0.elapsed_time(q1) / args.steps
        base += args.steps
        # stage pass of the pipelined step (serial, events between): fused pass, solve
        pt = {"profile_compress": [], "solve": []}
        ctx.timing(True)
        ctx.kernel_ms()
        allm = []
        for s in range(args.steps):
            l2_flush.zero_()
            m = [ev() for _ in range(3)]
            step_pipe(base + args.steps + s, conc=False, marks=m)
            allm.append(m)
        torch.cuda.synchronize()
        for m in allm:
            pt["profile_compress"].append(m[0].elapsed_time(m[1]))
            pt["solve"].append(m[1].elapsed_time(m[2]))
        fk_total, fk_n = ctx.kernel_ms()
        ctx.timing(False)
        if world > 1:
            t = torch.tensor([pipe_ms, sum(pt["profile_compress"]) / args.steps, sum(pt["solve"]) / args.steps],
                             device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pipe_ms = float(t[0])
            pt = {"profile_compress": [float(t[1])], "solve": [float(t[2])]}
        pipe = {"ms": pipe_ms, "launches": pipe_launches, "serial_ms": serial_ms,
                "stage": {k: sum(v) / len(v) for k, v in pt.items()},
                "fused_ms": fk_total / max(1, fk_n), "fused_n": fk_n}
        ctx.check()
        ef.copy_(e0)
        for pl in plans:
            pl.copy_(dflt)
        torch.cuda.synchronize()

    times = {"step": [], "profile": [], "solve": [], "compress_allreduce": []}
    # ---- headline pass: K steps, events only at each step's begin and end
    launches0 = ctx.launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    all_marks = []
    for s in range(args.steps):
        l2_flush.zero_()  # flush L2 between timed steps (outside the timed events)
        marks = [ev() for _ in range(2)]
        step(args.warmup + s, marks)  # enqueued without host synchronisation (W = 1)
        all_marks.append(marks)
    torch.cuda.synchronize()
    for marks in all_marks:
        times["step"].append(marks[0].elapsed_time(marks[1]))
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - t_wall0
    launches = ctx.launches() - launches0 + args.steps  # + one solve kernel per step
    # ---- stage pass (same K steps, not the headline): events between the stages and
    # around K1 (the dominant kernel, `ctx.timing`) for the breakdown and the roofline
    ctx.timing(True)
    ctx.kernel_ms()
    torch.cuda.synchronize()
    all_marks = []
    for s in range(args.steps):
        l2_flush.zero_()
        marks = [ev() for _ in range(4)]
        step(args.warmup + args.steps + s, marks)
        all_marks.append(marks)
    torch.cuda.synchronize()
    for marks in all_marks:
        times["profile"].append(marks[0].elapsed_time(marks[1]))
        times["solve"].append(marks[1].elapsed_time(marks[2]))
        times["compress_allreduce"].append(marks[2].elapsed_time(marks[3]))
    clk = clocks.stop()
    k1_total_ms, k1_n = ctx.kernel_ms()
    ctx.timing(False)
    k1_ms = k1_total_ms / max(1, k1_n)
    ctx.check()

    ms = sum(times["step"]) / args.steps
    stage = {k: sum(v) / len(v) for k, v in times.items()}
    if world > 1:
        t = torch.tensor([ms] + [stage[k] for k in ("profile", "solve", "compress_allreduce")], device=dev,
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        stage.update(profile=float(t[1]), solve=float(t[2]), compress_allreduce=float(t[3]))

    # ---- W > 1: NVLink bus bytes of the exchange (2 (W-1)/W S_packed per
    # rank) over the compress + exchange stage, beside the busbw of a plain NCCL
    # all-gather of the same byte count measured here
    xch = None
    if world > 1:
        ch_list = choice_d.cpu().tolist()
        S = ctx.payload_bytes(ch_list)
        bus = 2.0 * (world - 1) / world * S
        nb = (S + world - 1) // world
        src_t = torch.empty(nb, dtype=torch.uint8, device=dev)
        dst_t = torch.empty(nb * world, dtype=torch.uint8, device=dev)
        ag = None
        if not one_dev:
            for _ in range(3):
                dist.all_gather_into_tensor(dst_t, src_t)
            torch.cuda.synchronize()
            a0, a1 = ev(), ev()
            a0.record(stream)
            for _ in range(20):
                dist.all_gather_into_tensor(dst_t, src_t)
            a1.record(stream)
            torch.cuda.synchronize()
            ag = a0.elapsed_time(a1) / 20
            t = torch.tensor([ag], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ag = float(t[0])
        xch = {"payload_bytes": S, "bus_bytes_per_rank": bus,
               "exchange_busbw_gbs": round(bus / (stage["compress_allreduce"] * 1e-3) / 1e9, 1),
               "busbw_note": "bus bytes / the whole compress + exchange + decode stage (compute included)",
               "nccl_allgather_busbw_gbs": (round((world - 1) / world * nb * world / (ag * 1e-3) / 1e9, 1)
                                            if ag else None),
               "nccl_allgather_ms": round(ag, 4) if ag else None}
        del src_t, dst_t

    # ---- e2e: public API with host buffers.  Every step copies its gradient from pinned
    # host memory (H2D) and reads its mean gradient back (D2H); the copies run on their
    # own streams, double-buffered, so step s+1's H2D and step s-1's D2H overlap step s's
    # kernels (the EF chain stays on the compute stream).  The step's working set (g, e,
    # out: 307 MB) exceeds L2, so no flush here.  Per step = (last D2H end - first H2D
    # start) / steps.
    g_host = torch.from_numpy(g_np).pin_memory()
    out_host = [torch.empty(N, dtype=torch.float32).pin_memory() for _ in range(2)]
    g_dev = [torch.empty_like(g) for _ in range(2)]
    o_dev = [torch.empty_like(out) for _ in range(2)]
    s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ef.copy_(e0)
    torch.cuda.synchronize()
    n_e2e = max(2, args.steps)
    ev_h2d = [torch.cuda.Event() for _ in range(n_e2e)]
    ev_comp = [torch.cuda.Event() for _ in range(n_e2e)]
    ev_d2h = [torch.cuda.Event() for _ in range(n_e2e)]
    t_first, t_last = ev(), ev()
    t_first.record(s_h2d)

    def h2d(s):
        with torch.cuda.stream(s_h2d):
            if s >= 2:
                s_h2d.wait_event(ev_comp[s - 2])  # g_dev[s & 1] consumed by step s-2
            g_dev[s & 1].copy_(g_host, non_blocking=True)
            ev_h2d[s].record(s_h2d)

    def d2h(s):
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_comp[s])
            out_host[s & 1].copy_(o_dev[s & 1], non_blocking=True)
            ev_d2h[s].record(s_d2h)

    if pipelined:
        for pl in plans:
            pl.copy_(dflt)
        h2d(0)
        stream.wait_event(ev_h2d[0])
        for s in range(n_e2e):
            b = s & 1
            if s + 1 < n_e2e:
                h2d(s + 1)

            def waits(s=s):  # step s+1's inputs, enqueued before the solve of step s so the
                # fused pass of step s+1 follows that solve directly (the overlap)
                if s + 1 < n_e2e:
                    stream.wait_event(ev_h2d[s + 1])
                    if s >= 1:
                        stream.wait_event(ev_d2h[s - 1])  # o_dev[(s+1) & 1] drained

            step_pipe(s, gin=g_dev[b], gout=o_dev[b], conc=conc and s > 0,
                      pre_solve=lambda s=s: (ev_comp[s].record(stream), waits()))
            d2h(s)
    else:
        for s in range(n_e2e):
            b = s & 1
            h2d(s)
            stream.wait_event(ev_h2d[s])
            if s >= 2:
                stream.wait_event(ev_d2h[s - 2])  # o_dev[b] drained by step s-2's D2H
            step(s, gin=g_dev[b], gout=o_dev[b])
            ev_comp[s].record(stream)
            d2h(s)
    t_last.record(s_d2h)
    torch.cuda.synchronize()
    e2e = t_first.elapsed_time(t_last) / n_e2e
    if world > 1:
        t = torch.tensor([e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t[0])

    if rank == 0:
        peaks, src = _peaks()
        same_gbs = world * 4.0 * N / (ms * 1e-3) / 1e9
        gbs = world * 4.0 * N / (pipe["ms"] * 1e-3) / 1e9 if pipe else same_gbs
        # dominant kernel: K1 qprofile (ncu launch-list share ~0.4 of the library's device
        # time).  It is bound by instruction issue, not HBM:
        # algorithmic lane-ops = K1_OPS_PER_ELEM per compressed element; peak = one
        # warp-instruction per SMSP per clock = SMs x 128 lanes x SM clock.
        ncomp = sum(l.numel for l in layers if l.compress)
        prof_bytes = 8.0 * ncomp  # g + e read once
        k1_ops = K1_OPS_PER_ELEM * ncomp
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_mhz = float(clk.get("sm_max_mhz") or 1965)
        alu_peak = nsm * 128 * sm_mhz * 1e6 / 1e12  # T lane-ops/s
        k1_tops = k1_ops / (k1_ms * 1e-3) / 1e12
        traffic = _ncu_traffic()
        roof_k1 = {"bound": "alu", "kernel": "k_qprofile_q (K1)", "achieved": round(k1_tops, 3),
                   "peak": round(alu_peak, 3), "unit": "T lane-op/s", "frac": round(k1_tops / alu_peak, 4),
                   "traffic": traffic, "peak_source": f"derived: {nsm} SMs x 4 SMSP x 32 lanes x {sm_mhz:.0f} MHz",
                   "kernel_ms": round(k1_ms, 4), "launches_timed": k1_n,
                   "algorithmic_ops_per_launch": k1_ops, "ops_per_element": K1_OPS_PER_ELEM,
                   "algorithmic_bytes_per_launch": prof_bytes,
                   "hbm_achieved_gbs": round(prof_bytes / (k1_ms * 1e-3) / 1e9, 1),
                   "hbm_frac": round(prof_bytes / (k1_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                   "hbm_peak_gbs": peaks["hbm_gbs"], "hbm_peak_source": src}
        roof = roof_k1
        if pipe:
            # dominant kernel of the pipelined step: the fused pass (K1 + K5's compress).
            # Algorithmic bytes: read g, e and write e', out = 16 B per element (every layer);
            # algorithmic lane-ops: K1's 70 + the planned candidate's 5 (t*inv - u, ceil,
            # min s, dec, x - dec) per compressed element.  Both fractions are reported;
            # `bound` names the higher one.
            fms = pipe["fused_ms"]
            fbytes = 16.0 * N
            fops = (K1_OPS_PER_ELEM + FUSED_EXTRA_OPS) * ncomp
            hbm_gbs = fbytes / (fms * 1e-3) / 1e9
            alu_t = fops / (fms * 1e-3) / 1e12
            fr_h, fr_a = hbm_gbs / peaks["hbm_gbs"], alu_t / alu_peak
            ftraffic = _ncu_traffic("fused_dram_bytes.json")
            common = {"kernel": "k_qprofile_q<7, fused> (K1 + K5 compress)", "kernel_ms": round(fms, 4),
                      "launches_timed": pipe["fused_n"], "traffic": ftraffic,
                      "algorithmic_bytes_per_launch": fbytes, "algorithmic_ops_per_launch": fops,
                      "ops_per_element": K1_OPS_PER_ELEM + FUSED_EXTRA_OPS}
            if fr_h >= fr_a:
                roof = {"bound": "hbm", "achieved": round(hbm_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": round(fr_h, 4), "peak_source": src, **common,
                        "alu_achieved": round(alu_t, 3), "alu_peak": round(alu_peak, 3), "alu_frac": round(fr_a, 4)}
            else:
                roof = {"bound": "alu", "achieved": round(alu_t, 3), "peak": round(alu_peak, 3),
                        "unit": "T lane-op/s", "frac": round(fr_a, 4),
                        "peak_source": f"derived: {nsm} SMs x 4 SMSP x 32 lanes x {sm_mhz:.0f} MHz", **common,
                        "hbm_achieved_gbs": round(hbm_gbs, 1), "hbm_peak_gbs": peaks["hbm_gbs"],
                        "hbm_frac": round(fr_h, 4)}
        line = {
            "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(pipe["ms"] if pipe else ms, 4), "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Gaussian + 1% outliers, EF ~ N(0,(0.1s)^2))",
            "config": {"workload": WORKLOAD, "global_batch": None, "parallelism": f"dp{world}",
                       "schedule": (PIPE_NOTE if pipe else "same-step: profile -> solve -> compress with this step's plan"),
                       "l2": ("not flushed between the K consecutive steps: each streams 204 MB in and 204 MB out "
                              "(> 126 MB L2)" if pipe else "flushed (512 MiB memset) before every timed step"),
                       "family": "qsgd", "exchange": exchange},
            "dp_solve_ms": round(pipe["stage"]["solve"] if pipe else stage["solve"], 4),
            # the same figure for the per-step path alone (compress + exchange
            # with the plan fixed), which is what runs between replans
            "plan_fixed_gbs": round(world * 4.0 * N / (stage["compress_allreduce"] * 1e-3) / 1e9, 2),
            "stage_ms": {k: round(v, 4) for k, v in stage.items()},
            "stage_note": "step: headline pass (events at step begin/end only); profile/solve/compress: a second "
                          "pass of K steps with events between the stages and around K1",
            "roofline": roof,
            "same_step": {"value": round(same_gbs, 3), "unit": "GB/s", "ms_per_step": round(ms, 4),
                          "stage_ms": {k: round(v, 4) for k, v in stage.items()}, "roofline_k1": roof_k1,
                          "l2": "flushed (512 MiB memset) before every timed step",
                          "note": "profile -> solve -> compress with the plan of the same step (round-1 headline)"},
            "pipelined_stage_ms": ({k: round(v, 4) for k, v in pipe["stage"].items()} if pipe else None),
            "pipelined_no_overlap_ms": (round(pipe["serial_ms"], 4) if pipe else None),
            "e2e": {"value": round(world * 4.0 * N / (e2e * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": 4 * N, "d2h_bytes_per_step": 4 * N, "ms_per_step": round(e2e, 4),
                    "steps": n_e2e, "overlap": "H2D(s+1) and D2H(s-1) on copy streams beside step s's kernels",
                    "l2": "not flushed: per-step working set 307 MB > 126 MB L2"},
            "gpu_launches": int(pipe["launches"] if pipe else launches),
            "exchange": xch,
            "clocks": clk,
            "wall_s": round(wall, 3),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_full()
    ctx.close()
    if not args.no_extras:
        ex = run_extras(dev, rank, world, stream, l2_flush, nccl_dist=(world > 1))
        if rank == 0:
            line["extras"] = ex
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_extras(dev, rank, world, stream, l2_flush, nccl_dist):
    """Secondary rows measured the same way (device-timed, L2 flushed before every
    timed step) on the SURVEY.md 8(d) recipes, drawn on the device (same distributions
    as workloads.py's CPU generators): C2 PowerSGD (low rank + noise), C3 TopK
    (Student-t, 90%-zero-row embedding), C5 QSGD (Gaussian + outliers), C5 TopK and C5
    PowerSGD (BASELINE.json configs[4]: the three families with a DP re-solve every
    step), and C4 with the stage-1 payload packed and decoded at W = 1 (K5-with-pack + K9,
    the per-rank work of the W > 1 exchange)."""
    import torch
    import torch.distributed as dist
    from paper_2210_17357_b200 import lgreco
    specs = [("C2", "C2", lgreco.POWERSGD, W.PSGD_RANKS_C2, 2, "low_rank", "ResNet-18 CIFAR-10 PowerSGD r{1,2,4,8,16}"),
             ("C3", "C3", lgreco.TOPK, W.TOPK_PPM_C3, 9, "student_t", "Transformer-XL TopK 0.1%..10%"),
             ("C5", "C5", lgreco.QSGD, W.QSGD_BITS, 2, "gaussian", "GPT-2-medium-like QSGD 2..8 bits"),
             ("C5_topk", "C5", lgreco.TOPK, W.TOPK_PPM_C5, 9, "student_t", "GPT-2-medium-like TopK 1%..100% (K=100)"),
             ("C5_psgd", "C5", lgreco.POWERSGD, W.PSGD_RANKS_C5, 16, "low_rank",
              "GPT-2-medium-like PowerSGD r16..64 (K=49)")]
    only = os.environ.get("LG_EXTRAS")  # diagnostics: comma list of row names to run
    if only:
        specs = [sp for sp in specs if sp[0] in only.split(",")]
    res = {}
    cache = {}
    for name, cfg, fam, params, dflt_i, recipe, desc in specs:
        layers = W.config_layers(cfg)
        N = W.total_numel(layers)
        L, K = len(layers), len(params)
        key = (cfg, recipe)
        if key not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[key] = W.recipe_device(layers, recipe, dev, seed=SEED + rank)
        g, ef0 = cache[key]
        ef = ef0.clone()
        out = torch.empty_like(g)
        err = torch.empty(L, K, dtype=torch.float64, device=dev)
        bits = torch.empty(L, K, dtype=torch.int64, device=dev)
        dflt = torch.full((L,), dflt_i, dtype=torch.int32, device=dev)
        comp = torch.tensor([l.compress for l in layers], dtype=torch.int32, device=dev)
        ch_d = torch.empty(L, dtype=torch.int32, device=dev)
        info = torch.empty(48, dtype=torch.uint8, device=dev)
        ws = torch.empty(lgreco.solve_workspace_bytes(L, K, D_BINS), dtype=torch.uint8, device=dev)
        nid = None
        if world > 1:
            obj = [lgreco.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        ctx = lgreco.Context(layers, fam, params, qbucket=128, seed=SEED, rank=rank, world=world, nccl_id=nid)
        t = {"profile": [], "solve": [], "compress_allreduce": [], "step": []}
        allm = []
        for s in range(7):
            if s >= 2:
                l2_flush.zero_()
            m = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            m[0].record(stream)
            ctx.profile(g, ef, s, err, bits)
            m[1].record(stream)
            lgreco.solve(err, bits, dflt, comp, D=D_BINS, choice=ch_d, info=info, workspace=ws)
            ctx.plan_broadcast(ch_d)
            m[2].record(stream)
            ctx.compress_allreduce_dev(ch_d, g, ef, out, s)
            m[3].record(stream)
            if s >= 2:
                allm.append(m)
        torch.cuda.synchronize()
        for m in allm:
            t["profile"].append(m[0].elapsed_time(m[1]))
            t["solve"].append(m[1].elapsed_time(m[2]))
            t["compress_allreduce"].append(m[2].elapsed_time(m[3]))
            t["step"].append(m[0].elapsed_time(m[3]))
        ctx.check()
        inf = lgreco.read_info(info)
        pipe_ms = None
        if fam == lgreco.QSGD and world == 1:
            # the pipelined schedule of the headline (fused pass + the previous step's narrow
            # solve beside it), K = 5 consecutive steps between two events
            plans = [dflt.clone() for _ in range(3)]
            tabs = [(err, bits), (torch.empty_like(err), torch.empty_like(bits))]

            def pstep(s2):
                e_t, b_t = tabs[s2 % 2]
                ctx.profile_compress(plans[s2 % 3], g, ef, out, s2, e_t, b_t, concurrent=s2 > 0)
                lgreco.solve(e_t, b_t, dflt, comp, D=D_BINS, flags=lgreco.SOLVE_NARROW, choice=plans[(s2 + 2) % 3],
                             info=info, workspace=ws)
            for s2 in range(3):
                pstep(s2)
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for s2 in range(3, 8):
                pstep(s2)
            m1.record(stream)
            torch.cuda.synchronize()
            ctx.check()
            pipe_ms = m0.elapsed_time(m1) / 5
        elif world == 1:
            # the same schedule for TopK / PowerSGD: the profile and the compress (with the
            # plan solved two steps earlier; TopK's compress reuses the profile's thresholds
            # of the same x) on the main stream, the solve of the step on a side stream
            # beside the next step's kernels
            side = torch.cuda.Stream(device=dev)
            plans = [dflt.clone() for _ in range(3)]
            tabs = [(err, bits), (torch.empty_like(err), torch.empty_like(bits))]
            ev_solve = {}

            def pstep(s2):
                e_t, b_t = tabs[s2 % 2]
                if s2 - 2 in ev_solve:  # plans[s2 % 3] and the table pair: solve of step s2-2 done
                    stream.wait_event(ev_solve[s2 - 2])
                ctx.profile(g, ef, s2, e_t, b_t)
                ev_p = torch.cuda.Event()
                ev_p.record(stream)
                ctx.compress_allreduce_dev(plans[s2 % 3], g, ef, out, s2)
                side.wait_event(ev_p)
                with torch.cuda.stream(side):
                    lgreco.solve(e_t, b_t, dflt, comp, D=D_BINS, flags=lgreco.SOLVE_NARROW,
                                 choice=plans[(s2 + 2) % 3], info=info, workspace=ws, stream=side)
                ev_solve[s2] = torch.cuda.Event()
                ev_solve[s2].record(side)
            for s2 in range(3):
                pstep(s2)
            torch.cuda.synchronize()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            for s2 in range(3, 8):
                pstep(s2)
            stream.wait_event(ev_solve[7])
            m1.record(stream)
            torch.cuda.synchronize()
            ctx.check()
            pipe_ms = m0.elapsed_time(m1) / 5
        ctx.close()
        st = {k: sum(v) / len(v) for k, v in t.items()}
        if world > 1:
            tt = torch.tensor([st[k] for k in ("step", "profile", "solve", "compress_allreduce")], device=dev,
                              dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            st = dict(zip(("step", "profile", "solve", "compress_allreduce"), tt.tolist()))
        res[name] = {"workload": desc, "inputs": recipe, "n": N, "K": K,
                     "gbs": round(world * 4.0 * N / (st["step"] * 1e-3) / 1e9, 2),
                     "stage_ms": {k: round(v, 4) for k, v in st.items()}, "steps": 5,
                     "plan_bits_vs_default": round(inf.total_bits / max(1, inf.default_bits), 4)}
        if pipe_ms is not None:
            res[name]["pipelined"] = {"ms_per_step": round(pipe_ms, 4),
                                      "gbs": round(world * 4.0 * N / (pipe_ms * 1e-3) / 1e9, 2),
                                      "note": ("headline schedule: fused pass + the previous step's solve beside it"
                                               if fam == lgreco.QSGD else
                                               "profile + compress with the plan of step t-2, the solve on a side "
                                               "stream beside the next step")}
        del ef, out
    cache.clear()
    torch.cuda.empty_cache()
    if not only or "C4_pack" in only.split(","):
        res["C4_pack"] = _extra_pack_decode(dev, rank, stream, l2_flush)
    return res


def _extra_pack_decode(dev, rank, stream, l2_flush):
    """C4, plan fixed (the default 4-bit everywhere), W = 1: K5 writing the packed
    stage-1 payload + EF, then K9 decoding it (what every rank runs around the
    exchange at W > 1).  Algorithmic bytes per element: K5 12 + (16b+8)/128, K9
    (16b+8)/128 + 4."""
    import torch
    from paper_2210_17357_b200 import lgreco
    layers = W.config_layers("C4")
    N = W.total_numel(layers)
    g, ef = W.recipe_device(layers, "gaussian", dev, seed=SEED + rank)
    ctx = lgreco.Context(layers, lgreco.QSGD, W.QSGD_BITS, qbucket=128, seed=SEED)
    choice = [W.QSGD_BITS.index(4) if l.compress else -1 for l in layers]
    pay = torch.empty(ctx.payload_bytes(choice), dtype=torch.uint8, device=dev)
    out = torch.empty_like(g)
    tp, tu = [], []
    for s in range(7):
        if s >= 2:
            l2_flush.zero_()
        m = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        m[0].record(stream)
        ctx.qsgd_pack(choice, g, ef, pay, None, 0, s)
        m[1].record(stream)
        ctx.qsgd_unpack(choice, pay, out)
        m[2].record(stream)
        if s >= 2:
            tp.append(m)
    torch.cuda.synchronize()
    ctx.check()
    ctx.close()
    pk = sum(m[0].elapsed_time(m[1]) for m in tp) / len(tp)
    up = sum(m[1].elapsed_time(m[2]) for m in tp) / len(tp)
    S = int(pay.numel())
    peaks, _ = _peaks()
    bpk = 12.0 * N + S   # read g, e; write e'; write payload (lossless layers as raw records)
    bup = S + 4.0 * N    # read payload; write out
    return {"workload": "C4, 4-bit plan fixed, W = 1: pack (K5 with payload) + decode (K9)", "n": N,
            "payload_bytes": S, "pack_ms": round(pk, 4), "decode_ms": round(up, 4),
            "pack_hbm_gbs": round(bpk / (pk * 1e-3) / 1e9, 1), "decode_hbm_gbs": round(bup / (up * 1e-3) / 1e9, 1),
            "pack_hbm_frac": round(bpk / (pk * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
            "decode_hbm_frac": round(bup / (up * 1e-3) / 1e9 / peaks["hbm_gbs"], 4), "steps": 5}


def _ncu_traffic(name="k1_dram_bytes.json"):
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if present."""
    p = os.path.join(ROOT, "profiles", name)
    try:
        return json.load(open(p))["dram_bytes_per_launch"]
    except Exception:
        return None


# ------------------------------------------------------------------- oracle arm
def _oracle_step(ref, layers, g, e, step, times=None):
    K = len(W.QSGD_BITS)
    t0 = time.perf_counter()
    err, bits = ref.qsgd_profile(layers, g, e, W.QSGD_BITS, seed=SEED, step=step)
    t1 = time.perf_counter()
    st, choice, info = ref.solve(err, bits, [W.QSGD_BITS.index(4)] * len(layers), [l.compress for l in layers],
                                 D=D_BINS)
    t2 = time.perf_counter()
    lbits = [W.QSGD_BITS[c] if c >= 0 else 0 for c in choice]
    out, es, _, _ = ref.qsgd_allreduce(layers, lbits, [g], [e], seed=SEED, step=step)
    t3 = time.perf_counter()
    if times is not None:
        times.append((t1 - t0, t2 - t1, t3 - t2))
    return es[0]


def _omp_threads():
    try:
        return int(os.environ.get("OMP_NUM_THREADS") or len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline_full():
    """The oracle as it stands on one full C4 step (profile + solve + compress, W=1):
    its OpenMP build (layers on all host cores: the reported value) and the
    single-thread build beside it, each stage timed (the DP is single-threaded in both)."""
    from oracle import ref
    layers = W.config_layers("C4")
    N = W.total_numel(layers)
    g, e = W.gaussian_outliers(layers, seed=SEED)
    res = {}
    for omp in (True, False):
        ref.use_openmp(omp)
        tt = []
        t0 = time.perf_counter()
        _oracle_step(ref, layers, g, e.copy(), 0, tt)
        res[omp] = (time.perf_counter() - t0, tt[0])
    ref.use_openmp(False)
    cores, aff, model = _cpu_info()
    dt, (tp, ts, tc) = res[True]
    dt1, (tp1, ts1, tc1) = res[False]
    thr = _omp_threads()
    return {"value": round(4.0 * N / dt / 1e9, 6), "unit": "GB/s", "cores": thr, "kind": "oracle",
            "sample": f"one full C4 step (N={N}), OpenMP build on {thr} threads, {dt:.2f} s; host {model}, "
                      f"{cores} cpus ({aff} in affinity)",
            "stage_s": {"profile": round(tp, 3), "solve": round(ts, 4), "compress": round(tc, 3)},
            "dp_solve_ms": round(ts * 1e3, 2),
            "single_thread": {"value": round(4.0 * N / dt1 / 1e9, 6), "unit": "GB/s", "cores": 1,
                              "seconds": round(dt1, 2),
                              "stage_s": {"profile": round(tp1, 3), "solve": round(ts1, 4), "compress": round(tc1, 3)}}}


def run_reference(args):
    """--impl reference: the oracle (OpenMP build, all host cores) on the full C4
    workload, one full step (profile + DP + compress, W = 1) per timed step -- the same
    config, metric and unit as our arm."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    ref.use_openmp(True)
    layers = W.config_layers("C4")
    n = W.total_numel(layers)
    g, e = W.gaussian_outliers(layers, seed=SEED)
    for s in range(args.warmup):
        e = _oracle_step(ref, layers, g, e, s)
    t0 = time.perf_counter()
    for s in range(args.steps):
        e = _oracle_step(ref, layers, g, e, args.warmup + s)
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    cores, aff, model = _cpu_info()
    thr = _omp_threads()
    v = 4.0 * n / dt / 1e9
    sample = f"full C4 step ({n} fp32) per timed step, oracle OpenMP build on {thr} threads; host {model}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "parallelism": f"oracle (CPU, OpenMP {thr} threads)", "same_config": True},
        "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": thr, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--schedule", choices=["pipelined", "same_step"], default="pipelined",
                    help="headline step: the paper's pipelined schedule (default) or same-step profile->solve->compress")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2/C3/C5 secondary measurements")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
