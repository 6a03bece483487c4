#!/usr/bin/env python
"""Benchmark of the EP dispatch/combine hot path (BASELINE.json metric:
"LL dispatch+combine us @128 tok; HT dispatch/combine GB/s/GPU").

Default (N=1): configs[1] — LL decode step with DeepSeek-V3 shapes (E=256,
top-8, H=7168), 128 tokens per rank, bf16 tokens quantised to FP8 + block
scales inside the dispatch kernel, bf16 combine; the rank is its own peer
(loopback).  With torchrun (N>1) every rank owns 128 tokens (weak scaling)
and experts are block-placed over the ranks; traffic crosses NVLink through
CUDA-IPC windows.

One step = create_handle (routing layout) + dispatch (send + recv) +
combine (send + recv), captured once as a CUDA graph and replayed; the L2
is flushed (256 MB memset) before every step outside the timed events.
value = mean device time per step in microseconds (max over ranks).

Extra keys: `ht` (configs[2]: 4096 tokens/rank HT dispatch/combine, GB/s),
`e2e` (the same LL step through the public API with host buffers),
`roofline` (dominant kernel vs measured HBM copy bandwidth), `cpu_baseline`
(the CPU oracle port on a bounded sample), `clocks` (NVML during the run).

`--impl reference` times the reference algorithm's CPU restatement
(oracle/, the only executable form of the Python reference on the GPU box)
on the same config and prints the same line with "impl": "reference",
using every usable host core (concurrent oracle rounds in forked processes).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

E, K, H = 256, 8, 7168          # DeepSeek-V3 (BASELINE.json configs[1], [2])
METRIC = "LL dispatch+combine µs @128 tok; HT dispatch/combine GB/s/GPU at 8×B200"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--tokens", type=int, default=128)
    p.add_argument("--ht-tokens", type=int, default=4096)
    p.add_argument("--ht-steps", type=int, default=5)
    p.add_argument("--no-ht", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the C4/C5 configs (extra_configs key)")
    p.add_argument("--cpu-sample-steps", type=int, default=3)
    p.add_argument("--no-sweep", action="store_true", help="skip the LL token sweep 1..128 (ll_sweep_us key)")
    p.add_argument("--ll-zero-copy", action="store_true",
                   help="LL expert outputs in the registered window: the combine pulls them (default: pushed)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def init_dist():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank


def allreduce_max(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allgather_f(v: float, world: int) -> list:
    if world == 1:
        return [v]
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def make_group(world, rank, cfg, strict=False):
    import paper_2603_13606_b200 as ep
    topo = ep.NodeTopology(world, world)
    fab = ep.ProcessFabric(topo) if world > 1 else ep.Fabric(topo)
    return ep.create_group(fab, rank, cfg, strict=strict)


# ---------------------------------------------------------------------------
# clocks (NVML sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self._period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._nv is not None:
            self._stop.set()
            self._t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# LL decode step (configs[1])
# ---------------------------------------------------------------------------

class LLStep:
    def __init__(self, world, rank, b, seed=0, shape=None, zipf=False, zero_copy=False):
        import torch

        import paper_2603_13606_b200 as ep
        from oracle import workload as owl
        self.ep, self.torch = ep, torch
        self.world, self.rank, self.b = world, rank, b
        E, K, H = shape or (globals()["E"], globals()["K"], globals()["H"])
        self.E, self.K, self.H = E, K, H
        # zero_copy: the expert outputs live in the group's registered window
        # (EpHandle.expert_out_buffer); the combine pulls them over NVLink
        self.cfg = ep.EpConfig(ep.Algorithm.LL, world, world, E, K, H, b, ep.Dtype.FP8, True,
                               combine_dtype=ep.Dtype.BF16, expert_out_window=zero_copy)
        self.zero_copy = zero_copy
        self.g = make_group(world, rank, self.cfg, strict=False)
        wl = (owl.make_zipf_workload if zipf else owl.make_workload)(E, world, b, K, H, seed)
        dev = torch.device("cuda", torch.cuda.current_device())
        L = self.cfg.experts_per_rank
        self.x = torch.from_numpy(wl.tokens[rank]).to(dev).to(torch.bfloat16)
        self.topk = torch.from_numpy(wl.routing[rank]).to(dev)
        self.w = torch.from_numpy(wl.weights[rank]).to(dev)
        self.routing_h = wl.routing[rank]
        self.recv = torch.zeros((L, world * b, H), dtype=torch.uint8, device=dev)
        self.recv_sc = torch.zeros((L, world * b, H // 128), dtype=torch.float32, device=dev)
        self.cnt = torch.zeros((L, world), dtype=torch.float32, device=dev)
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)
        self.y = torch.randn((L, world * b, H), dtype=torch.float32, device=dev, generator=gen).to(torch.bfloat16)
        if zero_copy:
            yw = self.g.expert_out_view(L * world * b).view(L, world * b, H)
            yw.copy_(self.y)
            self.y = yw
        self.out = torch.zeros((b, H), dtype=torch.bfloat16, device=dev)
        T = ep.TensorTag
        self.X = ep.tensor_from_torch(self.x, T.TOKENS)
        self.RECV = ep.tensor_from_torch(self.recv, T.TOKENS)
        self.RECV_SC = ep.tensor_from_torch(self.recv_sc, T.SCALES)
        self.CNT = ep.tensor_from_torch(self.cnt, T.RECV_EXPERT_COUNTER_DEVICE)
        self.Y = ep.tensor_from_torch(self.y, T.TOKENS)
        self.W = ep.tensor_from_torch(self.w, T.TOPK_WEIGHTS)
        self.OUT = ep.tensor_from_torch(self.out, T.TOKENS)

    def step(self, upto="combine"):
        """One LL step; `upto` truncates it ("dispatch", "handle") for the
        marginal per-kernel timing in run_ll."""
        h = self.g.create_handle(self.topk)
        if upto == "staged":  # send / complete split (api.py:445-451, :521-540)
            h.dispatch([self.X], [self.RECV, self.RECV_SC, self.CNT], send_only=True)
            h.complete()
            h.combine([self.Y, self.W], [self.OUT], send_only=True)
            h.complete()
            h.destroy()
            return
        if upto != "handle":  # (every dispatch is combined: the arrival protocol counts rounds)
            h.dispatch([self.X], [self.RECV, self.RECV_SC, self.CNT])
            h.combine([self.Y, self.W], [self.OUT])
        h.destroy()

    # algorithmic bytes per kernel launch (this rank), headers not credited
    def algo_bytes(self):
        E, K, H = self.E, self.K, self.H
        L = self.cfg.experts_per_rank
        owner = self.routing_h // L
        dst_per_tok = np.array([len(set(r)) for r in owner]) if self.b else np.zeros(0)
        row8 = H + 4 * (H // 128)
        sent = int(dst_per_tok.sum())
        recv_rows = int(self.b * K)  # balanced estimate; exact value below for N=1
        if self.world == 1:
            recv_rows = int(self.b * K)
            arrive = sent
        else:
            arrive = sent  # symmetric workload: what a rank receives ~ what it sends
        # compulsory HBM bytes per launch: dispatch = read the
        # bf16 tokens + routing, write the FP8 expert-major rows + scales;
        # combine = read the bf16 expert rows + weights, write the bf16 output.
        # Slot traffic in the window is an intermediate (L2-resident at N=1).
        del sent, arrive
        return {
            "epb_routing_layout": self.b * K * 8 + self.b * (K + self.world) * 4 + (E + self.world) * 4,
            "epb_ll_dispatch": self.b * H * 2 + self.b * K * 8 + recv_rows * row8,
            "epb_ll_combine": recv_rows * H * 2 + self.b * K * 4 + self.b * H * 2,
        }, {"dispatch_remote": int(sum(len(set(r) - {self.rank}) for r in owner)) * row8,
            "combine_remote": int((owner != self.rank).sum()) * H * 2}


def capture(step_obj, group, phases: bool, warmup_eager=3):
    """One CUDA graph of a whole step between two timing events; with
    `phases`, every kernel launch inside is also preceded by an event."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warmup_eager):
            step_obj.step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    marks = []
    graph = torch.cuda.CUDAGraph()
    group.trace_phases(marks)
    with torch.cuda.graph(graph):
        group.mark("step:start")
        if not phases:
            group.trace_phases(None)
        step_obj.step()
        group.trace_phases(marks)
        group.mark("step:end")
    group.trace_phases(None)
    torch.cuda.synchronize()
    return graph, marks


def replay_timed(graph, marks, steps, flush, sync_each=False, align=None):
    """Replay `steps` times back to back, the L2 flushed before each step
    outside the timed events.  Without `sync_each` the host never waits
    between steps (per-step events are recorded around each replay on the
    stream), so ranks stay aligned by the exchange itself instead of by host
    jitter.  With `sync_each` the in-graph phase events are read after every
    replay.  Returns (total ms, {phase: ms})."""
    import torch
    names = [m[0] for m in marks]
    phase = {n: 0.0 for n in names[:-1]}
    if not sync_each:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            flush.zero_()
            if align is not None:
                align()  # device barrier of all ranks, outside the timed events
            a.record()
            graph.replay()
            b.record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs), phase
    total = 0.0
    for _ in range(steps):
        flush.zero_()
        if align is not None:
            align()
        graph.replay()
        torch.cuda.synchronize()
        evs = [m[1] for m in marks]
        total += evs[0].elapsed_time(evs[-1])
        for i in range(len(evs) - 1):
            phase[names[i]] += evs[i].elapsed_time(evs[i + 1])
    return total, phase


def capture_steps(step_obj, group, nsteps, flush, phases, upto="combine"):
    """One CUDA graph holding `nsteps` whole steps, each preceded by an L2
    flush and a device barrier of all ranks (untimed) and bracketed by
    external event nodes — per-step device time without the per-launch cost
    of a graph (a decode step's EP ops are nodes inside a bigger graph).
    With `phases`, every kernel launch is also preceded by an event."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step_obj.step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    per_step = []
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(nsteps):
            flush.zero_()
            group.device_barrier()
            marks = []
            group.trace_phases(marks)
            group.mark("step:start")
            if not phases:
                group.trace_phases(None)
            step_obj.step(upto)
            group.trace_phases(marks)
            group.mark("step:end")
            group.trace_phases(None)
            per_step.append(marks)
    torch.cuda.synchronize()
    return graph, per_step


def replay_steps(graph, per_step, replays, samples=None):
    """Replay; returns (sum of step times ms, {phase: summed ms}, steps);
    `samples` (a list) collects every step's time."""
    import torch
    total, phase, n = 0.0, {}, 0
    for _ in range(replays):
        graph.replay()
        torch.cuda.synchronize()
        for marks in per_step:
            evs = [m[1] for m in marks]
            dt = evs[0].elapsed_time(evs[-1])
            total += dt
            if samples is not None:
                samples.append(dt)
            for i in range(len(marks) - 1):
                phase[marks[i][0]] = phase.get(marks[i][0], 0.0) + evs[i].elapsed_time(evs[i + 1])
            n += 1
    return total, phase, n


def steps_per_graph(steps):
    return max(d for d in range(1, min(steps, 10) + 1) if steps % d == 0)


def run_ll(args, world, rank, shape=None, zipf=False, light=False):
    """`light`: only the timed step graph (returns step ms; the sweep)."""
    import torch
    st = LLStep(world, rank, args.tokens, shape=shape, zipf=zipf, zero_copy=getattr(args, "ll_zero_copy", False))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    S = steps_per_graph(args.steps)
    graph, per_step = capture_steps(st, st.g, S, flush, phases=False)
    if not light:
        graph_b, per_step_b = capture_steps(st, st.g, S, flush, phases=True)
    for _ in range(max(1, -(-args.warmup // S))):
        graph.replay()
    torch.cuda.synchronize()
    barrier(world)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier(world)
        samples = []
        total, _, n = replay_steps(graph, per_step, args.steps // S, samples)
        barrier(world)
    assert n == args.steps
    srt = sorted(samples)
    pct = {"median_us": allreduce_max(srt[len(srt) // 2], world) * 1000.0,
           "p99_us": allreduce_max(srt[min(len(srt) - 1, int(0.99 * len(srt)))], world) * 1000.0}
    if light:
        st.pct = pct
        return st, allreduce_max(total, world) / args.steps
    # per-kernel breakdown from the instrumented graph (events between launches)
    barrier(world)
    nb = max(10, min(args.steps, 100))
    _, phase, nph = replay_steps(graph_b, per_step_b, -(-nb // S))
    # per-kernel device time: the instrumented graph's event node before each
    # launch (the nodes themselves add a little to each interval)
    # staged (send_only + complete) steps: step time and the per-launch split
    gs, pss = capture_steps(st, st.g, S, flush, phases=True, upto="staged")
    gs.replay()
    barrier(world)
    ts, phs, ns = replay_steps(gs, pss, -(-nb // S))
    st.staged = {"step_us_with_event_nodes": round(allreduce_max(ts / ns, world) * 1000.0, 2),
                 "launch_us": {k: round(v / ns * 1000.0, 2) for k, v in phs.items()},
                 "note": "dispatch(send_only) -> complete() -> combine(send_only) -> complete(); an event node "
                         "before every launch (send phase, then receive phase of each op)"}
    del gs
    # the same step as its own graph launch per step (graph launch included)
    graph1, marks1 = capture(st, st.g, phases=False)
    for _ in range(3):
        flush.zero_()
        st.g.device_barrier()
        graph1.replay()
    barrier(world)
    t1, _ = replay_timed(graph1, marks1, args.steps, flush, align=st.g.device_barrier)
    st.g.check()
    total_max = allreduce_max(total, world)
    t1_max = allreduce_max(t1, world)
    per_phase = {k: v / nph * 1000.0 for k, v in phase.items()}  # us
    launches = sum(1 for n_, _ in per_step_b[0] if n_.startswith("epb_"))
    kernel_us = {"epb_ll_dispatch": per_phase.get("epb_ll_dispatch", 0.0),
                 "epb_ll_combine": per_phase.get("epb_ll_combine", 0.0)}
    st.pct = pct
    return (st, total_max / args.steps, per_phase, launches * args.steps, clk.report(),
            t1_max / args.steps * 1000.0, kernel_us)


def run_e2e(args, world, rank, st):
    """The LL step through the public API with HOST buffers: pinned host
    tokens / routing / weights in, host combine output back, every step.
    Headline form: the API calls captured once in a CUDA graph (as a decode
    loop captures them; strict=False, no host syncs inside) whose nodes
    include the host->device input copies and the device->host output copy;
    each step = one replay + a host synchronisation, host wall clock.  The
    eager form (API called from Python each step, strict checks on) is
    reported beside it."""
    import torch
    ep = st.ep
    g = st.g
    T = ep.TensorTag
    x_h = st.x.cpu().pin_memory()
    w_h = st.w.cpu().pin_memory()
    topk_h = st.topk.cpu().pin_memory()
    out_h = torch.zeros((st.b, H), dtype=torch.bfloat16).pin_memory()
    X = ep.tensor_from_torch(x_h, T.TOKENS)
    W = ep.tensor_from_torch(w_h, T.TOPK_WEIGHTS)
    OUT = ep.tensor_from_torch(out_h, T.TOKENS)

    def step():
        h = g.create_handle(topk_h)
        h.dispatch([X], [st.RECV, st.RECV_SC, st.CNT])
        h.combine([st.Y, W], [OUT])
        h.destroy()

    n = max(50, args.steps)
    # eager, strict
    g.strict = True
    for _ in range(3):
        step()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    torch.cuda.synchronize()
    dt_eager = allreduce_max((time.perf_counter() - t0) / n, world)
    # graph-captured API calls
    g.strict = False
    from paper_2603_13606_b200 import api as _api
    mapped0, mapped_in0 = _api._HOST_MAPPED, _api._HOST_MAPPED_IN

    def capture(mapped, mapped_in=False):
        _api._HOST_MAPPED, _api._HOST_MAPPED_IN = mapped, mapped_in
        try:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for _ in range(3):
                    step()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
        finally:
            _api._HOST_MAPPED, _api._HOST_MAPPED_IN = mapped0, mapped_in0
        torch.cuda.synchronize()
        for _ in range(3):
            graph.replay()
            torch.cuda.synchronize()
        return graph

    # the three variants' replays are interleaved so box-to-box and drift
    # noise hits them alike
    graphs = [capture(True), capture(False), capture(True, True)]
    barrier(world)
    times = [[] for _ in graphs]
    for _ in range(n):
        for gr, ts in zip(graphs, times):
            t0 = time.perf_counter()
            gr.replay()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
    dt, dt_copies, dt_in_mapped = (allreduce_max(statistics.median(ts), world) for ts in times)
    st.g.check()
    bi = x_h.numel() * 2 + topk_h.numel() * 8 + w_h.numel() * 4
    bo = out_h.numel() * 2
    return {"value": round(dt * 1e6, 2), "unit": "µs", "h2d_bytes_per_step": int(bi),
            "d2h_bytes_per_step": int(bo), "api": "EpGroup.create_handle/EpHandle.dispatch/combine",
            "timing": "host wall clock per step (median): one replay of the graph-captured API calls + host "
                      "sync; pinned host inputs copied H2D as graph nodes, the host combine output written by "
                      "the combine kernel in place over PCIe (default API behaviour)",
            "value_staged_copies": round(dt_copies * 1e6, 2),
            "staged_copies_timing": "same, with a D2H staging copy of the output as well (EPB_HOST_MAPPED=0)",
            "value_mapped_inputs": round(dt_in_mapped * 1e6, 2),
            "mapped_inputs_timing": "same, tokens also read by the dispatch kernel in place over PCIe "
                                    "(EPB_HOST_MAPPED_IN=1)",
            "eager_value": round(dt_eager * 1e6, 2),
            "eager_timing": "host wall clock, API called from Python every step, strict error checks on"}


# ---------------------------------------------------------------------------
# HT prefill (configs[2]) — eager, phase events
# ---------------------------------------------------------------------------

HT_A2A_PULL_GBPS = 650.0  # measured all-to-all NVLink pull, remote bytes per GPU


def run_ht(args, world, rank, shape=None, zipf=False, seed=7):
    import torch

    import paper_2603_13606_b200 as ep
    from oracle import workload as owl
    b = args.ht_tokens
    E, K, H = shape or (globals()["E"], globals()["K"], globals()["H"])
    # expert outputs are written into the group's registered window region
    # (EpHandle.expert_out_buffer), so the combine is pulled, not pushed
    cfg = ep.EpConfig(ep.Algorithm.HT, world, world, E, K, H, b, ep.Dtype.BF16, expert_out_window=True)
    g = make_group(world, rank, cfg, strict=False)
    wl = (owl.make_zipf_workload if zipf else owl.make_workload)(E, world, b, K, H, seed)
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(wl.tokens[rank]).to(dev).to(torch.bfloat16)
    topk = torch.from_numpy(wl.routing[rank]).to(dev)
    w = torch.from_numpy(wl.weights[rank]).to(dev)
    L = cfg.experts_per_rank
    T = ep.TensorTag
    X, Wt = ep.tensor_from_torch(x, T.TOKENS), ep.tensor_from_torch(w, T.TOPK_WEIGHTS)
    out = torch.zeros((b, H), dtype=torch.bfloat16, device=dev)
    OUT = ep.tensor_from_torch(out, T.TOKENS)
    cnt = torch.zeros((L, world), dtype=torch.float32, device=dev)
    CNT = ep.tensor_from_torch(cnt, T.TOKENS_PER_EXPERTS)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    bufs = {}

    t_handle = []

    def step(marks, zero_copy=True):
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        h = g.create_handle(topk)  # routing layout + metadata all-gather (ht.py open_round); host-synchronous
        t_handle.append(time.perf_counter() - t0)
        tot = h.get_num_recv_tokens()
        if tot not in bufs:
            bufs[tot] = (torch.zeros((tot, H), dtype=torch.bfloat16, device=dev),
                         torch.randn((tot, H), device=dev).to(torch.bfloat16))
        rt, yt = bufs[tot]
        yw = h.expert_out_buffer()
        yw.copy_(yt)  # stand-in for the expert GEMM writing its output (untimed)
        flush.zero_()
        g.device_barrier()
        g.trace_phases(marks)
        h.dispatch([X, Wt], [ep.tensor_from_torch(rt, T.TOKENS), CNT])
        g.mark("dispatch:end")
        h.combine([ep.tensor_from_torch(yw if zero_copy else yt, T.TOKENS), Wt], [OUT])
        g.mark("combine:end")
        g.trace_phases(None)
        h.destroy()
        return tot

    for _ in range(2):
        step([])
    barrier(world)
    td, tc, tphase = [], [], {}
    for _ in range(args.ht_steps):
        marks = []
        tot = step(marks)
        torch.cuda.synchronize()
        ev = {}
        for n_, e_ in marks:
            ev.setdefault(n_, e_)
        names = [m[0] for m in marks]
        for i in range(len(marks) - 1):
            tphase[names[i]] = tphase.get(names[i], 0.0) + marks[i][1].elapsed_time(marks[i + 1][1])
        td.append(ev["epb_ht_dispatch"].elapsed_time(ev["dispatch:end"]))
        tc.append(ev["epb_ht_combine"].elapsed_time(ev["combine:end"]))
    # the same combine with the expert rows in an ordinary tensor (pushed
    # into the homes' slots, then reduced there)
    tpush = []
    for _ in range(2):
        marks = []
        step(marks, zero_copy=False)
        torch.cuda.synchronize()
        ev = {}
        for n_, e_ in marks:
            ev.setdefault(n_, e_)
        tpush.append(ev["epb_ht_combine"].elapsed_time(ev["combine:end"]))
    t_push = allreduce_max(min(tpush), world) / 1e3
    g.check()
    barrier(world)
    t_h = allreduce_max(statistics.median(t_handle[-args.ht_steps:]), world)
    per_d = allgather_f(statistics.median(td), world)
    per_c = allgather_f(statistics.median(tc), world)
    ph_send = allgather_f(tphase.get("epb_ht_dispatch", 0.0) / args.ht_steps, world)
    ph_recv = allgather_f(tphase.get("epb_ht_dispatch:recv", 0.0) / args.ht_steps, world)
    t_d = max(per_d) / 1e3
    t_c = max(per_c) / 1e3
    owner = wl.routing[rank] // L
    dsts = [set(r) for r in owner]
    d_all = sum(len(s) for s in dsts) * H * 2
    d_remote = sum(len(s - {rank}) for s in dsts) * H * 2
    c_all = b * K * H * 2
    c_remote = int((owner != rank).sum()) * H * 2
    g.destroy()
    return {
        "tokens_per_rank": b, "dtype": "bf16", "recv_rows": tot,
        "dispatch_us": round(t_d * 1e6, 1), "combine_us": round(t_c * 1e6, 1),
        "create_handle_us": round(t_h * 1e6, 1),
        "combine_push_us": round(t_push * 1e6, 1),
        "combine_push_note": "combine input in an ordinary tensor: rows pushed to the homes' slots, then reduced",
        "create_handle_timing": "host wall clock of EpGroup.create_handle (routing layout + metadata "
                                "all-gather, receive count on the host on return; ht.py open_round)",
        "dispatch_payload_GBps": round(d_all / t_d / 1e9, 1),
        "combine_payload_GBps": round(c_all / t_c / 1e9, 1),
        "dispatch_nvlink_GBps": round(d_remote / t_d / 1e9, 1) if world > 1 else None,
        "combine_nvlink_GBps": round(c_remote / t_c / 1e9, 1) if world > 1 else None,
        # every GPU pulling from every peer at once (tools/a2a_micro.cu, N=2/4)
        "nvlink_a2a_pull_bound_GBps": HT_A2A_PULL_GBPS if world > 1 else None,
        "dispatch_frac_of_a2a": round(d_remote / t_d / 1e9 / HT_A2A_PULL_GBPS, 3) if world > 1 else None,
        "combine_frac_of_a2a": round(c_remote / t_c / 1e9 / HT_A2A_PULL_GBPS, 3) if world > 1 else None,
        "phase_us": {k: round(v / args.ht_steps * 1e3, 1) for k, v in tphase.items()},
        "per_rank_us": {"dispatch": [round(v * 1e3, 1) for v in per_d], "combine": [round(v * 1e3, 1) for v in per_c],
                        "dispatch_send": [round(v * 1e3, 1) for v in ph_send],
                        "dispatch_recv": [round(v * 1e3, 1) for v in ph_recv]},
        "transport": "dispatch: pull (rows staged in the sender's window, read once per (token, rank) over "
                     "NVLink); combine: pull (expert outputs in the registered window, read by the token's home)",
        "note": "payload = bf16 rows per (token, destination rank) for dispatch and per (token, k) "
                "for combine, all destinations incl. self; nvlink = remote part only",
    }


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------

def cpu_oracle_ll(b, n_ranks, steps, seed=0):
    """Time LL dispatch + combine of the CPU restatement (oracle/ll.py) for
    one rank group of the bench config; returns us per step and the sample."""
    from oracle import ll as oll
    from oracle import workload as owl
    wl = owl.make_workload(E, n_ranks, b, K, H, seed)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        d = oll.dispatch(wl.tokens, wl.routing, E, n_ranks, b, H, "fp8", True)
        outs = [d[r]["recv"] for r in range(n_ranks)]
        oll.combine(outs, wl.routing, wl.weights, E, n_ranks, b, H, "bf16")
        times.append(time.perf_counter() - t0)
        del d, outs
    per = statistics.median(times) / n_ranks  # one rank's share of the simulated group
    return per * 1e6, f"{steps} oracle LL rounds (dispatch FP8+scales, bf16 combine), " \
                      f"{n_ranks} simulated rank(s) x {b} tokens, DeepSeek-V3 shapes, median, per rank"


# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return main_reference(args)
    import torch
    world, rank = init_dist()
    st, step_ms, phases, launches, clocks, own_graph_us, kernel_us = run_ll(args, world, rank)
    value_us = step_ms * 1000.0
    # roofline of the dominant kernel
    algo, remote = st.algo_bytes()
    kernels = kernel_us
    dom = max(kernels, key=kernels.get)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = algo[dom] / (kernels[dom] * 1e-6) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = prof.get(dom)
    except Exception:  # noqa: BLE001
        pass
    result = {
        "metric": METRIC,
        "value": round(value_us, 2),
        "unit": "µs",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 5),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp8 dispatch (e4m3 + f32 block-128 scales) / bf16 combine, f32 accumulate",
        "data": "synthetic (oracle.make_workload: U(-3,3) tokens, uniform distinct top-8 routing, U(0.1,1) weights)",
        "config": {"workload": "configs[1] LL decode, DeepSeek-V3 shapes", "experts": E, "top_k": K,
                   "hidden": H, "tokens_per_rank": args.tokens, "ranks": world,
                   "parallelism": f"ep{world}", "l2": "flushed (256 MB memset) before every step",
                   "align": "device barrier of all ranks before each step (untimed)",
                   "graph": (f"{steps_per_graph(args.steps)} steps per CUDA graph (create_handle+dispatch+combine "
                             "each, bracketed by in-graph events; flush + barrier between, untimed)")},
        "step_us_own_graph_launch": round(own_graph_us, 2),
        "ll_staged": st.staged,
        "step_us_median": round(st.pct["median_us"], 2), "step_us_p99": round(st.pct["p99_us"], 2),
        "kernel_us": {k: round(v, 2) for k, v in kernel_us.items()},
        "phase_us_event_nodes": {k: round(v, 2) for k, v in phases.items()},
        "gpu_launches": launches,
        "roofline": {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "algorithmic_bytes": int(algo[dom]), "traffic": traffic,
                     "duration": "kernel_us: in-graph event nodes before each launch (CUDA events on the "
                                 "launching stream)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"},
        "nvlink_bytes_per_step": remote if world > 1 else None,
        "clocks": clocks,
    }
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, world, rank, st)
    if not args.no_ht:
        result["ht"] = run_ht(args, world, rank)
    if not args.no_ht and not args.no_extra:
        # the other BASELINE configs at this N (parity for them: tests/test_gpu_parity.py)
        extra = {}
        a2 = argparse.Namespace(**vars(args))
        a2.ht_steps = 3
        extra["C4 HT Mixtral E=8 K=2 H=4096, 4096 tok"] = run_ht(a2, world, rank, shape=(8, 2, 4096))
        extra["C5 HT Qwen3 E=128 K=8 H=4096, 4096 tok, Zipf routing"] = run_ht(
            a2, world, rank, shape=(128, 8, 4096), zipf=True)
        a3 = argparse.Namespace(**vars(args))
        a3.steps, a3.warmup = 50, 10
        s3, ms3, _, _, _, _, k3 = run_ll(a3, world, rank, shape=(128, 8, 4096), zipf=True)
        extra["C5 LL Qwen3 E=128 K=8 H=4096, 128 tok, Zipf routing, fp8 dispatch / bf16 combine"] = {
            "step_us": round(ms3 * 1000, 2), "kernel_us": {k: round(v, 2) for k, v in k3.items()}}
        s3.g.destroy()
        result["extra_configs"] = extra
    if not args.no_sweep:
        # configs[1]'s 1-128 tokens/rank sweep (step time only)
        sweep = {}
        for bb in (1, 2, 4, 8, 16, 32, 64, 128):
            a2 = argparse.Namespace(**vars(args))
            a2.tokens, a2.steps, a2.warmup = bb, 20, 10
            s2, ms2 = run_ll(a2, world, rank, light=True)
            sweep[bb] = round(ms2 * 1000, 2)
            s2.g.destroy()
        result["ll_sweep_us"] = sweep
    if rank == 0 and world == 1 and not args.no_cpu:
        us, sample = cpu_oracle_ll(args.tokens, 1, args.cpu_sample_steps)
        result["cpu_baseline"] = {"value": round(us, 1), "unit": "µs", "cores": 1, "kind": "port",
                                  "sample": sample}
    st.g.destroy()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


def _cpu_oracle_worker(b, n_ranks, steps, seed, barrier_, q):
    from oracle import ll as oll
    from oracle import workload as owl
    wl = owl.make_workload(E, n_ranks, b, K, H, seed)

    def one():
        d = oll.dispatch(wl.tokens, wl.routing, E, n_ranks, b, H, "fp8", True)
        oll.combine([d[r]["recv"] for r in range(n_ranks)], wl.routing, wl.weights, E, n_ranks, b, H, "bf16")

    one()  # warm-up
    barrier_.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    q.put((t0, time.perf_counter()))


def cpu_oracle_ll_parallel(b, n_ranks, steps):
    """The oracle LL round on every usable host core: P independent rounds
    run concurrently in P processes (the oracle is single-threaded numpy), so
    the per-step figure is the amortised wall time (max end - min start) /
    (P * steps).  P is capped by the free host memory (a round peaks at
    ~0.7 GB per simulated rank at DeepSeek-V3 shapes; 1 GB per rank + 1 GB is
    budgeted) and at 32."""
    import multiprocessing as mp
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # pragma: no cover
        avail = 16 << 30
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    p = max(1, min(ncpu, int(avail // ((1 + n_ranks) << 30)), 32))
    if p == 1:
        us, sample = cpu_oracle_ll(b, n_ranks, steps)
        return us, 1, sample
    ctx = mp.get_context("fork")
    barrier_ = ctx.Barrier(p)
    q = ctx.Queue()
    procs = [ctx.Process(target=_cpu_oracle_worker, args=(b, n_ranks, steps, i, barrier_, q)) for i in range(p)]
    for pr in procs:
        pr.start()
    spans = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    wall = max(e for _, e in spans) - min(s_ for s_, _ in spans)
    us = wall / (p * steps) / n_ranks * 1e6
    return us, p, (f"{p} processes x {steps} oracle LL rounds each, run concurrently (dispatch FP8+scales, "
                   f"bf16 combine), {n_ranks} simulated rank(s) x {b} tokens, DeepSeek-V3 shapes; amortised "
                   f"wall time per round, per rank")


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    steps = max(1, min(args.steps, args.cpu_sample_steps))
    us, cores, sample = cpu_oracle_ll_parallel(args.tokens, world, steps)
    result = {
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": "µs",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(us / 1000, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp8 dispatch / bf16 combine (numpy f32 arithmetic)",
        "data": "synthetic (oracle.make_workload)",
        "config": {"workload": "configs[1] LL decode, DeepSeek-V3 shapes", "experts": E, "top_k": K,
                   "hidden": H, "tokens_per_rank": args.tokens, "ranks": world,
                   "parallelism": f"ep{world} (simulated on host)"},
        "cpu_baseline": {"value": round(us, 1), "unit": "µs", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(us, 1), "unit": "µs", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (epsim) is pure Python and absent on the GPU box; this is its "
                "CPU restatement in oracle/ (pinned bit-exact to the reference by tests/golden)",
    }
    print(json.dumps(result))


if __name__ == "__main__":
    main()
