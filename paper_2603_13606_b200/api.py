"""Group / handle lifecycle of the reference API (epsim api.py), driving the
sm_100a kernels of libepb200.

Same names, argument meaning and error behaviour as epsim.api:
create_group / EpGroup / EpHandle / HandleState / AllocationHooks and the
module-level dispatch / combine / complete / get_num_recv_tokens /
create_handle / destroy_handle / destroy_group.  Tagged-tensor validation
runs on the host before any kernel is launched (api.py:116-170, 386-426);
routing validation (ids in range, distinct per row) runs in the routing
layout kernel and is raised from create_handle.

Extensions (all opt-in through tensor dtypes, the reference forms keep
working unchanged):
* dispatch TOKENS input may be f32/bf16/f16 under an FP8 config: the send
  kernel quantises (block 128, reference tie rule) — no SCALES input then;
* dispatch TOKENS output may be the wire dtype instead of f32 (plus a SCALES
  output [L, N*B, H/128] for FP8 with scales) — no f32 widening pass;
* combine TOKENS input may be bf16 and the combine output f32 or bf16.
"""

from __future__ import annotations

import ctypes
import warnings
import weakref
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional, Sequence

import os

import numpy as np
import torch

from . import _lib
from . import stats as _stats
from .core import (FP8_BLOCK, Algorithm, Dtype, EpConfig, EpError, ErrorCode, NDTensor,
                   TensorTag, raise_status)

ALLOC_ALIGNMENT = 256
LAYOUTS = ("optimized", "legacy")
# LL: a pinned host combine output is written by the combine kernel in place
# over PCIe (posted writes overlap the reduction) instead of through a D2H
# staging copy; EPB_HOST_MAPPED=0 restores the copy.  Pinned host token
# inputs are read in place only with EPB_HOST_MAPPED_IN=1: GPU-initiated
# PCIe reads measured slower than the copy engine (e2e 152 vs 116-132 us).
_HOST_MAPPED = os.environ.get("EPB_HOST_MAPPED", "1") != "0"
_HOST_MAPPED_IN = os.environ.get("EPB_HOST_MAPPED_IN", "0") == "1"
# HT create_handle in one launch (epb_ht_open) where every rank's kernel can
# run concurrently; EPB_HT_OPEN_FUSED=0 keeps the separate layout / metadata
# launches
_HT_OPEN_FUSED = os.environ.get("EPB_HT_OPEN_FUSED", "1") != "0"


# entry points that never read or write a window (local routing layout)
_WINDOW_FREE = frozenset({"epb_routing_layout"})


@dataclass
class AllocationHooks:
    """Caller-supplied provider of the group window (api.py:43-55).

    allocate(nbytes, alignment) must return a CUDA uint8 tensor of at least
    nbytes (or an integer device pointer), or None to refuse; release(buffer)
    is called once at group destruction or failed setup."""

    allocate: Callable[[int, int], object]
    release: Callable[[object], None]


class HandleState(Enum):
    CREATED = "Created"
    DISPATCH_STAGED = "DispatchStaged"
    DISPATCHED = "Dispatched"
    COMBINE_STAGED = "CombineStaged"
    COMBINED = "Combined"
    DESTROYED = "Destroyed"


def _ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def _by_tag(tensors: Sequence[NDTensor], wanted: set, where: str) -> dict:
    found: dict = {}
    for t in tensors:
        if not isinstance(t, NDTensor):
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"{where}: expected NDTensor, got {type(t).__name__}")
        if t.tag in found:
            raise EpError(ErrorCode.TAG_MISMATCH, f"{where}: duplicate tensor for tag {t.tag.value}")
        found[t.tag] = t
    missing = wanted - found.keys()
    if missing:
        raise EpError(ErrorCode.TAG_MISMATCH, f"{where}: missing {sorted(t.value for t in missing)}")
    extra = found.keys() - wanted
    if extra:
        raise EpError(ErrorCode.TAG_MISMATCH, f"{where}: unexpected {sorted(t.value for t in extra)}")
    return found


def _expect_dtype(t: NDTensor, dtypes, what: str) -> None:
    dtypes = dtypes if isinstance(dtypes, tuple) else (dtypes,)
    if t.dtype not in dtypes:
        raise EpError(ErrorCode.TAG_MISMATCH,
                      f"{what}: dtype {t.dtype.value}, want {'|'.join(d.value for d in dtypes)}")


def _expect_shape(t: NDTensor, shape, what: str) -> None:
    if tuple(t.shape) != tuple(shape):
        raise EpError(ErrorCode.SHAPE_MISMATCH, f"{what}: shape {tuple(t.shape)}, want {tuple(shape)}")


def _peek_tag(tensors, tag):
    for t in tensors:
        if isinstance(t, NDTensor) and t.tag is tag:
            return t
    return None


@dataclass
class LLDispatchResult:
    recv: torch.Tensor          # [L, N*B, H] (valid rows per counts)
    counts: torch.Tensor        # [L, N] int32 (device)
    src_info: torch.Tensor      # [L, N*B] int32: t*K + k of each valid row
    scales: Optional[torch.Tensor] = None
    _total: Optional[int] = None
    _stats_fn: Optional[Callable] = None
    _stats: object = None

    @property
    def recv_total(self) -> int:
        if self._total is None:
            self._total = int(self.counts.sum().item())
        return self._total

    @property
    def stats(self):
        """LLStats of this dispatch (ll.py:39-55), computed on demand."""
        if self._stats is None and self._stats_fn is not None:
            self._stats = self._stats_fn()
        return self._stats


@dataclass
class HTDispatchResult:
    rows: torch.Tensor          # [recv_total, H] sorted by (expert, src, token)
    origin: torch.Tensor        # [recv_total, 4] int32 (e, src, t, k)
    origin_w: torch.Tensor      # [recv_total] f32 weights
    meta_m: np.ndarray          # [N, E] tokens_per_expert
    meta_q: np.ndarray          # [N, N] records_per_pair
    recv_total: int
    _stats_fn: Optional[Callable] = None
    _stats: object = None

    @property
    def stats(self):
        """HTStats of this dispatch (ht.py:57-74), computed on demand."""
        if self._stats is None and self._stats_fn is not None:
            self._stats = self._stats_fn()
        return self._stats


class _Scratch:
    """A handle's small device state in one int32 allocation (pooled per
    group, reused by later handles of the same batch size): the routing
    layout (m, q, tok_rank, tok_slot), the LL round word and the LL round
    state (counts, src_info, self_row, owner_row).  Pointers are handed to
    the kernels; torch views exist only for what the API exposes."""

    def __init__(self, group: "EpGroup", b: int):
        cfg = group.config
        n, e, k = cfg.num_ranks, cfg.num_experts, cfg.top_k
        ell = cfg.experts_per_rank
        bb = max(b, 1)
        ll_rows = ell * n * cfg.max_tokens_per_rank if cfg.algorithm is Algorithm.LL else 1
        sizes = [("m", e), ("q", n), ("tok_rank", bb * k), ("tok_slot", bb * n), ("hseq", 1),
                 ("counts", ell * n), ("src_info", ll_rows), ("self_row", bb * k), ("owner_row", bb * k)]
        off, self.off = 0, {}
        for name, size in sizes:
            self.off[name] = (off, size)
            off += (size + 3) // 4 * 4  # 16-B aligned pieces
        self.b = b
        self.buf = torch.empty(off, dtype=torch.int32, device=group.device)
        base = self.buf.data_ptr()
        self.ptr = {name: base + o * 4 for name, (o, _) in self.off.items()}
        self._views = {}

    def view(self, name: str, shape) -> torch.Tensor:
        v = self._views.get(name)
        if v is None:
            o, size = self.off[name]
            v = self._views[name] = self.buf[o:o + size].view(shape)
        return v


class EpGroup:
    """One rank's context: config, window, peers, handles (api.py:178-253)."""

    def __init__(self, fabric, rank: int, config: EpConfig, layout: str, cgroup: ctypes.c_void_p,
                 logical_bytes: int, physical_bytes: int, hooks, hook_buffer, strict: bool):
        self.fabric = fabric
        self.rank = rank
        self.config = config
        self.layout = layout
        self._g = cgroup
        self._logical = logical_bytes
        self._physical = physical_bytes
        self._hooks = hooks
        self._buffer = hook_buffer
        self._handles: list = []
        self._next_seq = 0
        self._ht_round = 0
        # HT: the handle whose round is open (opened by create_handle or a
        # reused handle's dispatch, closed by its combine or by destroying it
        # before dispatch) — one open round per group (ht.py:355-357, :619)
        self._ht_active: Optional["EpHandle"] = None
        # enqueued library entry points: all of them, and those that touch any
        # window (the analogue of the reference fabric's put/signal/lsa
        # counters that its tests assert unchanged on rejected calls)
        self.launches = 0
        self.traffic = 0
        self._alive = True
        self.strict = strict
        self._marks = None
        self._scratch_pool: dict = {}
        # pinned host mirror of the device error word (read after a sync)
        word = ctypes.c_void_p()
        _lib.call("epb_group_error_word", cgroup, ctypes.byref(word))
        self._err_word = ctypes.c_int32.from_address(word.value)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        # op trace (fabric `trace`): a device ring the kernels append to,
        # drained into the fabric's sink after every call
        self._op_ring = None
        sink = getattr(fabric, "trace", None)
        if sink is not None and sink.active:
            self._op_ring = torch.zeros(4 + 4 * sink.capacity, dtype=torch.int64, device=self.device)
            _lib.call("epb_group_set_op_trace", cgroup, ctypes.c_void_p(self._op_ring.data_ptr()), sink.capacity)
        # the group's kernels go to whatever stream is current at the call
        self._follows_current = bool(getattr(fabric, "process_mode", False)) or config.num_ranks == 1
        self._call_sp = 0  # raw stream of the call in progress (set by _on_stream)

    # -- properties -----------------------------------------------------------
    @property
    def alive(self) -> bool:
        return self._alive

    @property
    def buffer_bytes(self) -> int:
        """The reference's window size for this config (ll.py:107-121,
        ht.py:167-174) — footprint parity with the paper."""
        return self._logical

    @property
    def physical_bytes(self) -> int:
        """Bytes actually registered on the device (16-B padded slots)."""
        return self._physical

    @property
    def stream(self) -> torch.cuda.Stream:
        return self.fabric.stream(self.rank)

    def _check_alive(self) -> None:
        if not self._alive:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "group has been destroyed")

    def _alloc_seq(self) -> int:
        seq = self._next_seq
        self._next_seq += 1
        return seq

    def expert_out_view(self, rows: int) -> torch.Tensor:
        """[rows, H] bf16 view of the window's registered expert-output
        region (config.expert_out_window)."""
        off, cap = getattr(self, "_expert_out", (0, 0))
        if not cap or not isinstance(self._buffer, torch.Tensor):
            raise EpError(ErrorCode.INVALID_ARGUMENT, "group has no expert-output region (EpConfig.expert_out_window)")
        if rows > cap:
            raise EpError(ErrorCode.CAPACITY_EXCEEDED, f"{rows} expert rows exceed the region ({cap})")
        h = self.config.hidden
        return self._buffer[off:off + rows * h * 2].view(torch.bfloat16).view(rows, h)

    def token_in_view(self, rows: int) -> torch.Tensor:
        """HT: [rows, H] view (the wire dtype) of this rank's token stage in
        the registered window.  Tokens written here and passed unchanged as
        the dispatch TOKENS input skip the stage copy: peers read them in
        place (zero-copy input).  Needs a torch-backed window
        (EpConfig.expert_out_window or allocation hooks returning a tensor).
        The rows must stay unchanged until the round's combine."""
        off, cap = getattr(self, "_token_in", (0, 0))
        if not cap or not isinstance(self._buffer, torch.Tensor):
            raise EpError(ErrorCode.INVALID_ARGUMENT, "group has no torch-backed HT token stage")
        if rows > cap:
            raise EpError(ErrorCode.CAPACITY_EXCEEDED, f"{rows} rows exceed the stage ({cap})")
        dt = self.config.token_dtype.torch_dtype
        h = self.config.hidden
        rb = h * self.config.token_dtype.byte_width
        if rb % 16:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "stage rows are padded to 16 B; hidden * width must be a multiple")
        nb = rows * rb
        return self._buffer[off:off + nb].view(dt).view(rows, h)

    def _in_expert_out(self, t: torch.Tensor) -> bool:
        off, cap = getattr(self, "_expert_out", (0, 0))
        return bool(cap) and isinstance(self._buffer, torch.Tensor) and t.dtype == torch.bfloat16 and \
            t.data_ptr() == self._buffer.data_ptr() + off

    def _take_scratch(self, b: int) -> _Scratch:
        free = self._scratch_pool.get(b)
        return free.pop() if free else _Scratch(self, b)

    def _give_scratch(self, sc: _Scratch) -> None:
        # later work reusing it is enqueued on this group's stream, after
        # everything that used it (stream order)
        self._scratch_pool.setdefault(sc.b, []).append(sc)

    def _pinned_i32(self, n: int) -> torch.Tensor:
        buf = getattr(self, "_pinned_buf", None)
        if buf is None or buf.numel() < n:
            buf = self._pinned_buf = torch.empty(max(n, 1024), dtype=torch.int32).pin_memory()
        return buf[:n]

    def _on_stream(self):
        """Context for a call's device work: the group's stream, ordered after
        the caller's current stream (inputs the caller just produced) and
        followed by it (outputs the caller consumes next).  When the group
        follows the caller's stream (ProcessFabric, one emulated rank) the
        scope only looks up the raw current stream once per call."""
        if self._follows_current:
            self._call_sp = _raw_current_stream(self._dev_index)
            scope = _NULL_SCOPE
        else:
            scope = _StreamScope(self)
        return scope if self._op_ring is None else _TraceScope(self, scope)

    def _drain_ops(self) -> None:
        """Hand the op records of the call just made to the fabric's trace
        sink (waits for the call's kernels)."""
        ring = self._op_ring
        torch.cuda.current_stream(self.device).synchronize()
        n = int(ring[0].item())
        if n == 0:
            return
        sink = self.fabric.trace
        m = min(n, sink.capacity)
        recs = ring[4:4 + 4 * m].view(m, 4).cpu().numpy().view(np.uint64)
        ring[0].zero_()
        sink.emit(recs, dropped=n - m)
        if n > m:
            warnings.warn(f"op trace: {n - m} records beyond the ring capacity {sink.capacity} were dropped")

    def check(self) -> None:
        """Synchronise and raise any error the kernels recorded (timeouts,
        routing validation, weight mismatch).  The whole device is
        synchronised: the group's kernels may have gone to any stream that
        was current at the call (ProcessFabric follows the caller's stream)."""
        torch.cuda.synchronize(self.device)
        if self._err_word.value == 0:  # the kernels mirror any failure to host memory
            return
        code = ctypes.c_int32(0)
        _lib.call("epb_group_poll_error", self._g, 1, ctypes.byref(code))
        if code.value:
            raise_status(code.value, "device-side failure recorded by the EP kernels")

    def set_timeout(self, seconds: float) -> None:
        _lib.call("epb_group_set_timeout", self._g, int(seconds * 1e9))

    def device_barrier(self) -> None:
        """Stream-ordered barrier of all ranks over the peer windows (no host
        sync, capturable in a CUDA graph).  Collective.  Emulated ranks share
        one stream, so a host barrier already orders them (a spinning kernel
        per rank on one GPU would wait on kernels queued behind it)."""
        if not self.fabric.process_mode and self.config.num_ranks > 1:
            self.fabric.phase(self.rank)
            return
        with self._on_stream():
            _lib.call("epb_group_barrier", self._g, ctypes.c_void_p(self._call_sp))

    # -- kernel launches (optionally bracketed by timing marks) -------------
    def trace_phases(self, marks: Optional[list]) -> None:
        """With a list, every kernel launch of this group is preceded by a
        timing event (external, so it survives CUDA-graph capture) appended
        as (kernel name, event); pass None to stop."""
        self._marks = marks

    def mark(self, name: str) -> None:
        if getattr(self, "_marks", None) is not None:
            ev = torch.cuda.Event(enable_timing=True, external=True)
            ev.record(self.stream)
            self._marks.append((name, ev))

    def _launch(self, name: str, *args) -> None:
        """Call a C entry point; `name` may carry a ":label" suffix that
        only names the timing mark."""
        self.mark(name)
        fn = name.split(":")[0]
        self.launches += 1
        if fn not in _WINDOW_FREE:
            self.traffic += 1
        _lib.call(fn, *args)

    def _fused_ok(self) -> bool:
        """Send and receive halves may share one (cooperative) launch unless
        several ranks are emulated on this GPU, where every rank's send must
        be enqueued before any rank's receive."""
        return self.fabric.process_mode or self.config.num_ranks == 1

    # -- handles ----------------------------------------------------------------
    def create_handle(self, topk_idx) -> "EpHandle":
        """Snapshot a routing decision (api.py:218-239).  LL: local; HT:
        collective (metadata exchange), receive count known on return."""
        self._check_alive()
        routing = _validated_routing(topk_idx, self.config, self.device, snapshot=self.strict)
        handle = EpHandle(self, routing)
        with self._on_stream():
            if self.config.algorithm is Algorithm.HT:
                self._open_ht_round(handle)
            elif self.strict:
                # the LL dispatch kernel validates and lays out the routing
                # itself; strict mode also validates here so a bad routing
                # raises from create_handle like the reference (api.py:233)
                handle._run_layout()
                self.check()
        self._handles.append(handle)
        return handle

    def _open_ht_round(self, handle: "EpHandle") -> None:
        """Run the metadata collective for `handle` (HTRank.open_round,
        ht.py:335-368): refused while any round of this group is open, i.e.
        until the previous round's combine (ht.py:355-357, reset at :619)."""
        if self._ht_active is not None:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "previous round still open; combine first")
        rnd = self._ht_round
        self._ht_round += 1
        self._ht_active = handle
        try:
            handle._open_round(rnd)
        except BaseException:
            self._ht_active = None
            raise

    def _close_ht_round(self, handle: "EpHandle") -> None:
        if self._ht_active is handle:
            self._ht_active = None

    def destroy(self) -> None:
        """Release the window; all handles must be destroyed (api.py:241-253)."""
        self._check_alive()
        live = [h for h in self._handles if h.state is not HandleState.DESTROYED]
        if live:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, f"group still owns {len(live)} live handle(s)")
        self._alive = False
        torch.cuda.synchronize(self.device)
        _lib.call("epb_group_destroy", self._g)
        self.fabric.registered[self.rank] = 0
        if self._hooks is not None:
            self._hooks.release(self._buffer)


def _raw_current_stream(device_index: int) -> int:
    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(device_index)
    return torch.cuda.current_stream(device_index).cuda_stream


class _NullScope:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_NULL_SCOPE = _NullScope()


class _TraceScope:
    """A call scope that drains the op trace when the call's work is issued."""

    def __init__(self, group, inner):
        self._g = group
        self._inner = inner

    def __enter__(self):
        self._inner.__enter__()
        return self

    def __exit__(self, *exc):
        self._inner.__exit__(*exc)
        self._g._drain_ops()
        return False


class _StreamScope:
    """A group with its own stream (ranks emulated on one GPU): that stream
    waits for the caller's, runs the call, and the caller's waits for it."""

    def __init__(self, group):
        self._g = group
        self._s = group.stream
        self._cur = None
        self._ctx = None

    def __enter__(self):
        self._cur = torch.cuda.current_stream()
        if self._cur != self._s:
            self._s.wait_stream(self._cur)
        self._ctx = torch.cuda.stream(self._s)
        self._ctx.__enter__()
        self._g._call_sp = self._s.cuda_stream
        return self

    def __exit__(self, *exc):
        self._ctx.__exit__(*exc)
        if self._cur != self._s:
            self._cur.wait_stream(self._s)
        return False


def _validated_routing(topk_idx, cfg: EpConfig, device, snapshot: bool = True) -> torch.Tensor:
    """Host-side shape/dtype/capacity checks (api.py:150-170); range and
    distinctness are checked by the routing-layout kernel."""
    if isinstance(topk_idx, torch.Tensor):
        r = topk_idx
        integral = not (r.is_floating_point() or r.is_complex() or r.dtype == torch.bool)
    else:
        arr = np.asarray(topk_idx)
        integral = np.issubdtype(arr.dtype, np.integer) or arr.size == 0
        r = arr
    if r.ndim != 2 or r.shape[1] != cfg.top_k:
        raise EpError(ErrorCode.INVALID_ARGUMENT,
                      f"topk_idx shape {tuple(r.shape)}, want (tokens, {cfg.top_k})")
    if r.shape[0] and not integral:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"topk_idx dtype {r.dtype} is not integral")
    b = r.shape[0]
    if b > cfg.max_tokens_per_rank:
        raise EpError(ErrorCode.INVALID_ARGUMENT,
                      f"{b} routed tokens exceed max_tokens_per_rank {cfg.max_tokens_per_rank}")
    if isinstance(r, np.ndarray):
        r = torch.from_numpy(np.ascontiguousarray(r.astype(np.int64, copy=False)))
    if not snapshot and r.device == device and r.dtype == torch.int64 and r.is_contiguous():
        return r  # perf mode: the caller keeps topk_idx unchanged until dispatch
    out = r.to(device=device, dtype=torch.int64, non_blocking=True).contiguous()
    return out.clone() if out is r else out


def create_group(fabric, rank: int, config: EpConfig, hooks: Optional[AllocationHooks] = None,
                 layout: str = "optimized", strict: bool = True) -> EpGroup:
    """Collectively create one rank's group (api.py:256-319).

    Every rank must call with an identical config and layout, or all fail
    with ConfigMismatch.  The fingerprints are agreed BEFORE any device
    memory is registered; then each rank allocates its window (library
    cudaMalloc or `hooks`), the window descriptors are all-gathered and
    every peer window is mapped (CUDA IPC across processes)."""
    if not 0 <= rank < config.num_ranks:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"rank {rank} outside 0..{config.num_ranks - 1}")
    if getattr(fabric, "devices", None) is not None:
        torch.cuda.set_device(fabric.device_of(rank))  # ranks of one process on several GPUs
    topo = fabric.topology
    if topo.num_ranks != config.num_ranks or topo.ranks_per_node != config.ranks_per_node:
        raise EpError(ErrorCode.INVALID_ARGUMENT, "fabric topology does not match the config")
    if layout not in LAYOUTS:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"unknown layout {layout!r}")
    fingerprint = config.fingerprint() + layout.encode()
    prints = fabric.exchange(rank, fingerprint)
    if any(p != fingerprint for p in prints):
        raise EpError(ErrorCode.CONFIG_MISMATCH, "ranks disagree on group config/layout")

    ccfg = config.to_c(layout)
    info = _lib.WindowInfo()
    _lib.call("epb_window_geometry", ctypes.byref(ccfg), ctypes.byref(info))
    if config.expert_out_window and hooks is None:
        # the expert-output region is handed out as a torch view of the window
        hooks = AllocationHooks(allocate=lambda n, a: torch.empty(n, dtype=torch.uint8, device=torch.device(
            "cuda", torch.cuda.current_device())), release=lambda b: None)
    buffer, wptr, wbytes = None, 0, 0
    if hooks is not None:
        buffer = hooks.allocate(int(info.physical_bytes), ALLOC_ALIGNMENT)
        if buffer is None:
            raise EpError(ErrorCode.CAPACITY_EXCEEDED, f"allocation hook refused {info.physical_bytes} bytes")
        if isinstance(buffer, torch.Tensor):
            if not buffer.is_cuda:
                hooks.release(buffer)
                raise EpError(ErrorCode.INVALID_ARGUMENT, "allocation hook must return device memory")
            wptr, wbytes = buffer.data_ptr(), buffer.numel() * buffer.element_size()
        else:
            wptr, wbytes = int(buffer), int(info.physical_bytes)
    stream = fabric.stream(rank)
    cg = ctypes.c_void_p()
    try:
        _lib.call("epb_group_create", ctypes.byref(ccfg), rank, ctypes.c_void_p(wptr), wbytes,
                  ctypes.c_void_p(stream.cuda_stream), ctypes.byref(cg))
    except BaseException:
        if hooks is not None:
            hooks.release(buffer)
        raise
    try:
        if fabric.process_mode:
            desc = _lib.IpcDesc()
            _lib.call("epb_group_ipc_desc", cg, ctypes.byref(desc))
            descs = fabric.exchange(rank, bytes(desc))
            arr = (_lib.IpcDesc * config.num_ranks)()
            for r, blob in enumerate(descs):
                ctypes.memmove(ctypes.byref(arr[r]), blob, ctypes.sizeof(_lib.IpcDesc))
            _lib.call("epb_group_open_peers", cg, arr)
            fabric.barrier()
        else:
            win, nb = ctypes.c_void_p(), ctypes.c_uint64()
            _lib.call("epb_group_window", cg, ctypes.byref(win), ctypes.byref(nb))
            ptrs = fabric.exchange(rank, int(win.value))
            arr = (ctypes.c_uint64 * config.num_ranks)(*ptrs)
            _lib.call("epb_group_set_peers", cg, arr)
    except BaseException:
        _lib.call("epb_group_destroy", cg)
        if hooks is not None:
            hooks.release(buffer)
        raise
    fabric.registered[rank] = int(info.physical_bytes)
    grp = EpGroup(fabric, rank, config, layout, cg, int(info.logical_bytes), int(info.physical_bytes),
                  hooks, buffer, strict)
    grp._expert_out = (int(info.expert_out_offset), int(info.expert_out_rows))
    grp._token_in = (int(info.token_in_offset), int(info.token_in_rows))
    return grp


def destroy_group(group: EpGroup) -> None:
    group.destroy()


# ---------------------------------------------------------------------------
# handles
# ---------------------------------------------------------------------------


class EpHandle:
    """A routing snapshot moving through dispatch/combine rounds
    (api.py:331-581); owns the state machine and the per-round device state
    (routing layout, counts, source info / origin)."""

    def __init__(self, group: EpGroup, routing: torch.Tensor):
        self.group = group
        self.routing = routing
        self.state = HandleState.CREATED
        cfg = group.config
        dev = group.device
        self._b = routing.shape[0]
        del dev
        sc = self._sc = group._take_scratch(self._b)
        self._lay = _lib.Layout(sc.ptr["m"], sc.ptr["q"], sc.ptr["tok_rank"], sc.ptr["tok_slot"], self._b)
        self._hseq_p = ctypes.c_void_p(sc.ptr["hseq"])  # LL round sequence (device word)
        self._round: Optional[int] = None
        self._round_open = False
        self._meta = None
        self._staged = None
        self._dispatch_result = None
        self._combine_stats = None
        self._weights = None
        # LL per-round device state
        self._counts_i32 = None
        self._src_info = None

    @property
    def config(self) -> EpConfig:
        return self.group.config

    @property
    def num_tokens(self) -> int:
        return self._b

    def _require(self, states: tuple, verb: str) -> None:
        if self.state not in states:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, f"cannot {verb} in state {self.state.value}")

    def _sp(self) -> ctypes.c_void_p:
        """The stream of the public call in progress (EpGroup._on_stream)."""
        return ctypes.c_void_p(self.group._call_sp)

    def _run_layout(self) -> None:
        self.group._launch("epb_routing_layout", self.group._g, _ptr(self.routing), self._b,
                  ctypes.byref(self._lay), self._sp())

    # -- HT metadata round ------------------------------------------------------
    def _open_round(self, rnd: int) -> None:
        g = self.group
        cfg = g.config
        n, e = cfg.num_ranks, cfg.num_experts
        self._round = rnd
        nm = n * (e + n)
        # one round is open per group at a time (ht.py:355-357), so the round
        # buffers (meta rows | receive total, group offsets) are the group's
        if getattr(g, "_ht_bufs", None) is None:
            mt = torch.empty(nm + 1, dtype=torch.int32, device=g.device)
            g._ht_bufs = (mt, torch.empty((e, n), dtype=torch.int32, device=g.device),
                          ctypes.c_void_p(mt.data_ptr()), ctypes.c_void_p(mt.data_ptr() + nm * 4))
        mt, offsets, meta_p, total_p = g._ht_bufs
        host = g._pinned_i32(nm + 2)
        fused = g._fused_ok() and _HT_OPEN_FUSED
        if fused:
            # layout + metadata all-gather in one launch, the shapes written
            # straight into pinned host memory with the error word after them
            try:
                g._launch("epb_ht_open", g._g, rnd, _ptr(self.routing), self._b, ctypes.byref(self._lay),
                          ctypes.c_void_p(host.data_ptr()), _ptr(offsets), self._sp())
            except EpError as err:
                # more chunks than can be co-resident (refused before any
                # launch): the separate launches speak the same protocol
                if err.code is not ErrorCode.CAPACITY_EXCEEDED:
                    raise
                fused = False
            else:
                g.check()  # one synchronisation: receive shapes are host-known on return (api.py:235-237)
        if not fused:
            # ranks emulated on one GPU: every rank's row is sent before any
            # rank waits for its peers'
            self._run_layout()
            g._launch("epb_ht_meta_send", g._g, rnd, ctypes.byref(self._lay), self._sp())
            g.fabric.phase(g.rank)
            g._launch("epb_ht_meta_recv", g._g, rnd, meta_p, _ptr(offsets), total_p, self._sp())
            host[:nm + 1].copy_(mt, non_blocking=True)
            g.check()  # one synchronisation: receive shapes are host-known on return (api.py:235-237)
        meta_h = host.numpy()[:nm].reshape(n, e + n).astype(np.int64)
        ell = cfg.experts_per_rank
        lo = g.rank * ell
        hi = min(lo + ell, e)
        counts = np.zeros((ell, n), dtype=np.float32)  # TOKENS_PER_EXPERTS (api.py:437-441)
        counts[:hi - lo] = meta_h[:, lo:hi].T
        self._meta = dict(m=meta_h[:, :e], q=meta_h[:, e:], recv_total=int(host[nm]), offsets=offsets,
                          counts_host=counts)
        self._round_open = True

    # -- staging helpers ----------------------------------------------------------
    def _dev_in(self, t: NDTensor, mapped: bool = False) -> torch.Tensor:
        """Device view of an input.  `mapped`: a pinned, contiguous host
        tensor is read by the kernel in place over PCIe (pinned memory is
        device-mapped under UVA), so the host->device transfer overlaps the
        kernel's own work instead of preceding it as a copy."""
        v = t.view()
        if mapped and _HOST_MAPPED and _HOST_MAPPED_IN and v.device.type == "cpu" and v.is_pinned() and v.is_contiguous():
            return v
        if v.device != self.group.device:
            v = v.to(self.group.device, non_blocking=True)
        return v.contiguous()

    def _dev_out(self, t: NDTensor, full: bool = False, mapped: bool = False):
        """(device tensor to write, needs_copy_back).  `full`: the kernel
        overwrites every element, so a host output needs no upload.
        `mapped`: a pinned host tensor is written in place by the kernel
        (pinned memory is device-mapped under UVA) — for small outputs such
        as the expert counters."""
        v = t.view()
        if v.device == self.group.device and v.is_contiguous():
            return v, False
        if mapped and v.device.type == "cpu" and v.is_pinned() and v.is_contiguous():
            return v, False
        if full:
            return torch.empty(t.shape, dtype=t.dtype.torch_dtype, device=self.group.device), True
        # rows the kernels do not write keep the caller's contents
        return v.to(self.group.device, non_blocking=True).contiguous(), True

    # -- dispatch -----------------------------------------------------------------
    def dispatch(self, inputs: Sequence[NDTensor], outputs: Sequence[NDTensor],
                 send_only: bool = False) -> None:
        """Move tokens to their experts (api.py:361-453)."""
        cfg = self.config
        g = self.group
        g._check_alive()
        self._require((HandleState.CREATED, HandleState.COMBINED), "dispatch")
        ht = cfg.algorithm is Algorithm.HT
        if ht and send_only:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "send_only staging is an LL feature")
        b = self._b
        tok_peek = _peek_tag(inputs, TensorTag.TOKENS)
        quant_in_kernel = (cfg.token_dtype is Dtype.FP8 and tok_peek is not None
                           and tok_peek.dtype in (Dtype.F32, Dtype.BF16, Dtype.F16))
        in_want = {TensorTag.TOKENS}
        if cfg.with_scales and not quant_in_kernel:
            in_want.add(TensorTag.SCALES)
        if ht:
            in_want.add(TensorTag.TOPK_WEIGHTS)
        named_in = _by_tag(inputs, in_want, "dispatch input")
        out_peek = _peek_tag(outputs, TensorTag.TOKENS)
        wire_out = out_peek is not None and out_peek.dtype is cfg.token_dtype and \
            cfg.token_dtype is not Dtype.F32
        counter_tag = TensorTag.TOKENS_PER_EXPERTS if ht else (
            TensorTag.RECV_EXPERT_COUNTER_DEVICE
            if _peek_tag(outputs, TensorTag.RECV_EXPERT_COUNTER_DEVICE) is not None
            else TensorTag.RECV_EXPERT_COUNTER_HOST)
        out_want = {TensorTag.TOKENS, counter_tag}
        if wire_out and cfg.with_scales:
            out_want.add(TensorTag.SCALES)
        named_out = _by_tag(outputs, out_want, "dispatch output")

        tokens = named_in[TensorTag.TOKENS]
        if quant_in_kernel:
            _expect_dtype(tokens, (Dtype.F32, Dtype.BF16, Dtype.F16), "dispatch TOKENS input")
        else:
            _expect_dtype(tokens, cfg.token_dtype, "dispatch TOKENS input")
        _expect_shape(tokens, (b, cfg.hidden), "dispatch TOKENS input")
        scales = None
        if TensorTag.SCALES in named_in:
            scales = named_in[TensorTag.SCALES]
            _expect_dtype(scales, Dtype.F32, "SCALES")
            _expect_shape(scales, (b, cfg.hidden // FP8_BLOCK), "SCALES")
        weights = None
        if ht:
            weights = named_in[TensorTag.TOPK_WEIGHTS]
            _expect_dtype(weights, Dtype.F32, "TOPK_WEIGHTS")
            _expect_shape(weights, (b, cfg.top_k), "TOPK_WEIGHTS")
        ell, n = cfg.experts_per_rank, cfg.num_ranks
        out_tokens = named_out[TensorTag.TOKENS]
        out_counts = named_out[counter_tag]
        _expect_dtype(out_tokens, (Dtype.F32, cfg.token_dtype), "dispatch TOKENS output")
        _expect_dtype(out_counts, Dtype.F32, f"{counter_tag.value} output")
        _expect_shape(out_counts, (ell, n), f"{counter_tag.value} output")
        out_scales = named_out.get(TensorTag.SCALES)
        if ht:
            if not self._round_open:
                # handle reuse (e.g. backward): a fresh collective round
                with g._on_stream():
                    g._open_ht_round(self)
            _expect_shape(out_tokens, (self._meta["recv_total"], cfg.hidden), "dispatch TOKENS output")
        else:
            _expect_shape(out_tokens, (ell, n * cfg.max_tokens_per_rank, cfg.hidden),
                          "dispatch TOKENS output")
        if out_scales is not None:
            _expect_dtype(out_scales, Dtype.F32, "SCALES output")
            _expect_shape(out_scales, tuple(out_tokens.shape[:-1]) + (cfg.hidden // FP8_BLOCK,),
                          "SCALES output")

        with g._on_stream():
            if ht:
                self._ht_dispatch(tokens, weights, out_tokens, out_counts)
                return
            x = self._dev_in(tokens, mapped=True)
            xs = self._dev_in(scales) if scales is not None else None
            g._alloc_seq()
            dev = g.device
            out_t, back_t = self._dev_out(out_tokens)
            out_s, back_s = self._dev_out(out_scales) if out_scales is not None else (None, False)
            cnt_f, back_c = self._dev_out(out_counts, full=True, mapped=True)
            sc = self._sc
            self._counts_i32 = sc.view("counts", (ell, n))
            self._src_info = sc.view("src_info", (ell, n * cfg.max_tokens_per_rank))
            a = _lib.LLDispatchArgs(x.data_ptr(), tokens.dtype.code, xs.data_ptr() if xs is not None else None,
                                    self.routing.data_ptr(), b, out_t.data_ptr(), out_tokens.dtype.code,
                                    out_s.data_ptr() if out_s is not None else None, cnt_f.data_ptr(),
                                    sc.ptr["counts"], sc.ptr["src_info"], sc.ptr["self_row"],
                                    sc.ptr["owner_row"] if g._expert_out[1] else None)
            self._ll_args = a
            self._keep_alive = (x, xs)
            self._staged = (out_tokens, out_counts, out_scales, out_t, out_s, cnt_f, back_t, back_s, back_c)
            if send_only:
                g._launch("epb_ll_dispatch", g._g, self._hseq_p, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
                self.state = HandleState.DISPATCH_STAGED
                return
            if g._fused_ok():
                g._launch("epb_ll_dispatch", g._g, self._hseq_p, _lib.PHASE_BOTH, ctypes.byref(a), self._sp())
            else:
                g._launch("epb_ll_dispatch", g._g, self._hseq_p, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
                g.fabric.phase(g.rank)
                g._launch("epb_ll_dispatch:recv", g._g, self._hseq_p, _lib.PHASE_RECV, ctypes.byref(a), self._sp())
            self._ll_recv()

    def _ll_recv(self) -> None:
        """Finish a dispatch whose receive phase has been launched."""
        g = self.group
        out_tokens, out_counts, out_scales, out_t, out_s, cnt_f, back_t, back_s, back_c = self._staged
        self._staged = None
        if g.strict:
            g.check()
        if back_t:
            out_tokens.view().copy_(out_t, non_blocking=not g.strict)
        if back_s:
            out_scales.view().copy_(out_s, non_blocking=not g.strict)
        if back_c:
            out_counts.view().copy_(cnt_f, non_blocking=not g.strict)
        self._dispatch_result = LLDispatchResult(out_t, self._counts_i32, self._src_info, out_s,
                                                 _stats_fn=self._ll_dispatch_stats)
        self._keep_alive = None
        self.state = HandleState.DISPATCHED

    def _ht_dispatch(self, tokens, weights, out_tokens, out_counts) -> None:
        g = self.group
        cfg = g.config
        meta = self._meta
        x = self._dev_in(tokens)
        w = self._dev_in(weights)
        self._weights = w.clone()
        rnd = self._round
        total = meta["recv_total"]
        out_t, back_t = self._dev_out(out_tokens, full=True)
        origin = torch.empty((max(total, 1), 4), dtype=torch.int32, device=g.device)
        origin_w = torch.empty(max(total, 1), dtype=torch.float32, device=g.device)
        a = _lib.HTDispatchArgs(x.data_ptr(), tokens.dtype.code, w.data_ptr(), self.routing.data_ptr(), self._b,
                                self._sc.ptr["q"], self._sc.ptr["tok_rank"], self._sc.ptr["tok_slot"],
                                meta["offsets"].data_ptr(), out_t.data_ptr(), out_tokens.dtype.code,
                                origin.data_ptr(), origin_w.data_ptr())
        if g._fused_ok():
            g._launch("epb_ht_dispatch", g._g, rnd, _lib.PHASE_BOTH, ctypes.byref(a), self._sp())
        else:
            g._launch("epb_ht_dispatch", g._g, rnd, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
            if not g._fused_ok():
                g.fabric.phase(g.rank)
            g._launch("epb_ht_dispatch:recv", g._g, rnd, _lib.PHASE_RECV, ctypes.byref(a), self._sp())
        if g.strict:
            g.check()
        if back_t:
            out_tokens.view().copy_(out_t, non_blocking=not g.strict)
        ell, n = cfg.experts_per_rank, cfg.num_ranks
        lo = g.rank * ell
        hi = min(lo + ell, cfg.num_experts)
        oc = out_counts.view()  # host-known since the meta round
        oc.copy_(torch.from_numpy(meta["counts_host"]).reshape(oc.shape), non_blocking=oc.device.type != "cpu")
        self._round_open = False
        self._dispatch_result = HTDispatchResult(out_t, origin[:total], origin_w[:total], meta["m"],
                                                 meta["q"], total, _stats_fn=self._ht_dispatch_stats)
        self.state = HandleState.DISPATCHED

    # -- combine ------------------------------------------------------------------
    def combine(self, inputs: Sequence[NDTensor], outputs: Sequence[NDTensor],
                send_only: bool = False) -> None:
        """Return weighted expert outputs to this rank's tokens (api.py:463-519)."""
        cfg = self.config
        g = self.group
        g._check_alive()
        self._require((HandleState.DISPATCHED,), "combine")
        ht = cfg.algorithm is Algorithm.HT
        if ht and send_only:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "send_only staging is an LL feature")
        b = self._b
        named_in = _by_tag(inputs, {TensorTag.TOKENS, TensorTag.TOPK_WEIGHTS}, "combine input")
        named_out = _by_tag(outputs, {TensorTag.TOKENS}, "combine output")
        rows_in = named_in[TensorTag.TOKENS]
        _expect_dtype(rows_in, (Dtype.F32, Dtype.BF16), "combine TOKENS input")
        wt = named_in[TensorTag.TOPK_WEIGHTS]
        _expect_dtype(wt, Dtype.F32, "TOPK_WEIGHTS")
        _expect_shape(wt, (b, cfg.top_k), "TOPK_WEIGHTS")
        out = named_out[TensorTag.TOKENS]
        _expect_dtype(out, (Dtype.F32, Dtype.BF16), "combine TOKENS output")
        _expect_shape(out, (b, cfg.hidden), "combine TOKENS output")
        ell, n = cfg.experts_per_rank, cfg.num_ranks
        if ht:
            _expect_shape(rows_in, (self._meta["recv_total"], cfg.hidden), "combine TOKENS input")
        else:
            _expect_shape(rows_in, (ell, n * cfg.max_tokens_per_rank, cfg.hidden), "combine TOKENS input")
        with g._on_stream():
            y = self._dev_in(rows_in)
            w = self._dev_in(wt)
            if ht:
                self._ht_combine(y, rows_in.dtype, w, out)
                return
            o, back = self._dev_out(out, full=True, mapped=_HOST_MAPPED)
            sc = self._sc
            a = _lib.LLCombineArgs(y.data_ptr(), rows_in.dtype.code, sc.ptr["counts"],
                                   sc.ptr["src_info"], w.data_ptr(), b, o.data_ptr(), out.dtype.code,
                                   sc.ptr["self_row"], self.routing.data_ptr() if b else None,
                                   sc.ptr["owner_row"] if g._expert_out[1] else None, int(g._in_expert_out(y)))
            self._ll_cargs = a
            self._staged = (out, o, back, w, y)
            if send_only:
                g._launch("epb_ll_combine", g._g, self._hseq_p, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
                self.state = HandleState.COMBINE_STAGED
                return
            if g._fused_ok():
                g._launch("epb_ll_combine", g._g, self._hseq_p, _lib.PHASE_BOTH, ctypes.byref(a), self._sp())
            else:
                g._launch("epb_ll_combine", g._g, self._hseq_p, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
                g.fabric.phase(g.rank)
                g._launch("epb_ll_combine:recv", g._g, self._hseq_p, _lib.PHASE_RECV, ctypes.byref(a), self._sp())
            self._ll_combine_recv()

    def _ll_combine_recv(self) -> None:
        """Finish a combine whose receive phase has been launched."""
        g = self.group
        out, o, back, _w, _y = self._staged
        self._staged = None
        if g.strict:
            g.check()
        if back:
            out.view().copy_(o, non_blocking=not g.strict)
        self._combine_stats = None
        self.state = HandleState.COMBINED

    def _ht_combine(self, y, y_dtype, w, out) -> None:
        g = self.group
        res = self._dispatch_result
        # combine weights must equal the dispatched ones (ht.py:605-609),
        # checked on the device before any combine traffic
        # (the weights-equal check runs first inside epb_ht_combine; a
        # mismatch aborts the combine kernels before any traffic)
        o, back = self._dev_out(out, full=True)
        a = _lib.HTCombineArgs(y.data_ptr(), y_dtype.code, res.origin.data_ptr(), res.recv_total,
                               self.routing.data_ptr(), w.data_ptr(), self._b, self._sc.ptr["tok_rank"],
                               self._meta["offsets"].data_ptr(), o.data_ptr(), out.dtype.code,
                               self._weights.data_ptr(), self._row_ptr_scratch().data_ptr(),
                               int(g._in_expert_out(y)))
        if g._fused_ok() and g._marks is None:
            g._launch("epb_ht_combine", g._g, self._round, _lib.PHASE_BOTH, ctypes.byref(a), self._sp())
        else:
            g._launch("epb_ht_combine", g._g, self._round, _lib.PHASE_SEND, ctypes.byref(a), self._sp())
            if not g._fused_ok():
                g.fabric.phase(g.rank)
            g._launch("epb_ht_combine:recv", g._g, self._round, _lib.PHASE_RECV, ctypes.byref(a), self._sp())
        if g.strict:
            g.check()
        if back:
            out.view().copy_(o, non_blocking=not g.strict)
        self._combine_stats = None
        g._close_ht_round(self)
        self.state = HandleState.COMBINED

    def expert_out_buffer(self) -> torch.Tensor:
        """EpConfig.expert_out_window: a bf16 tensor in the group's
        registered window for this round's expert outputs — HT [recv_total,
        H], LL [L, N*B, H] (the dispatch output layout).  Passing it
        (unchanged) as the combine input makes the combine zero-copy: each
        home rank pulls its tokens' rows from the owners over NVLink.  One
        region per group: its contents must stay until every rank's combine
        of the round is done (the next round's dispatch orders that), so LL
        rounds pipelined on two handles must not both use it."""
        if self.config.algorithm is Algorithm.LL:
            cfg = self.config
            rows = cfg.experts_per_rank * cfg.num_ranks * cfg.max_tokens_per_rank
            return self.group.expert_out_view(rows).view(cfg.experts_per_rank, -1, cfg.hidden)
        return self.group.expert_out_view(self._meta["recv_total"])

    def _row_ptr_scratch(self) -> torch.Tensor:
        n = max(1, self._b * self.config.top_k)
        if getattr(self, "_row_ptr", None) is None or self._row_ptr.numel() < n:
            self._row_ptr = torch.empty(n, dtype=torch.int64, device=self.group.device)
        return self._row_ptr

    def complete(self) -> None:
        """Finish a staged LL dispatch or combine (api.py:521-540)."""
        g = self.group
        g._check_alive()
        if self.state is HandleState.DISPATCH_STAGED:
            with g._on_stream():
                g.fabric.phase(g.rank)
                g._launch("epb_ll_dispatch:recv", g._g, self._hseq_p, _lib.PHASE_RECV,
                          ctypes.byref(self._ll_args), self._sp())
                self._ll_recv()
            return
        if self.state is HandleState.COMBINE_STAGED:
            with g._on_stream():
                g.fabric.phase(g.rank)
                g._launch("epb_ll_combine:recv", g._g, self._hseq_p, _lib.PHASE_RECV,
                          ctypes.byref(self._ll_cargs), self._sp())
                self._ll_combine_recv()
            return
        raise EpError(ErrorCode.HANDLE_STATE_ERROR, f"nothing staged to complete in state {self.state.value}")

    # -- queries --------------------------------------------------------------------
    def get_num_recv_tokens(self) -> int:
        """HT: known at creation; LL: after dispatch completes (api.py:544-559)."""
        if self.state is HandleState.DESTROYED:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "handle destroyed")
        if self.config.algorithm is Algorithm.HT:
            return self._meta["recv_total"]
        valid = (HandleState.DISPATCHED, HandleState.COMBINE_STAGED, HandleState.COMBINED)
        if self.state not in valid or self._dispatch_result is None:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "LL receive count is known after dispatch completes")
        return self._dispatch_result.recv_total

    @property
    def dispatch_result(self):
        return self._dispatch_result

    @property
    def combine_stats(self):
        """LLStats / HTStats of the last combine (ll.py:427-459,
        ht.py:616-735), computed on demand from the receive plan."""
        if self._combine_stats is None and self.state is HandleState.COMBINED:
            self._combine_stats = self._combine_stats_now()
        return self._combine_stats

    # -- stats (host-side accounting, never on the kernel path) -------------------
    def _routing_np(self) -> np.ndarray:
        return self.routing.detach().cpu().numpy().reshape(-1, self.config.top_k)

    def _ll_dispatch_stats(self):
        g = self.group
        return _stats.ll_dispatch_stats(self.config, g.layout, self._routing_np(), g.buffer_bytes)

    def _ht_dispatch_stats(self):
        g = self.group
        return _stats.ht_dispatch_stats(self.config, g.rank, self._routing_np(), self._dispatch_result.meta_q,
                                        g.buffer_bytes)

    def _combine_stats_now(self):
        g, cfg = self.group, self.config
        res = self._dispatch_result
        if cfg.algorithm is Algorithm.HT:
            return _stats.ht_combine_stats(cfg, g.rank, self._routing_np(), res.recv_total, res.meta_m,
                                           g.buffer_bytes)
        return _stats.ll_combine_stats(cfg, g.layout, g.rank, res.counts.cpu().numpy(), res.src_info.cpu().numpy(),
                                       g.buffer_bytes)

    def destroy(self) -> None:
        """Retire the handle; legal only with no round in flight."""
        self._require((HandleState.CREATED, HandleState.COMBINED), "destroy handle")
        if self._round_open:
            # HT: metadata went out, payload never followed; every rank drops
            # the round with its handle (HTRank.abort_round, ht.py:370-377)
            self._round_open = False
            self.group._close_ht_round(self)
        self.state = HandleState.DESTROYED
        sc, self._sc = self._sc, None
        if sc is not None:
            self.group._give_scratch(sc)
        try:
            self.group._handles.remove(self)
        except ValueError:
            pass


def create_handle(group: EpGroup, topk_idx) -> EpHandle:
    return group.create_handle(topk_idx)


def destroy_handle(handle: EpHandle) -> None:
    handle.destroy()


def dispatch(handle: EpHandle, inputs, outputs, send_only: bool = False) -> None:
    handle.dispatch(inputs, outputs, send_only=send_only)


def combine(handle: EpHandle, inputs, outputs, send_only: bool = False) -> None:
    handle.combine(inputs, outputs, send_only=send_only)


def complete(handle: EpHandle) -> None:
    handle.complete()


def get_num_recv_tokens(handle: EpHandle) -> int:
    return handle.get_num_recv_tokens()
