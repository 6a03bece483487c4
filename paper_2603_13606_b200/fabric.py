"""Rank groups and their bootstrap (replaces epsim fabric.py + the
_Rendezvous of api.py:67-94).

The reference's Fabric is a simulated one-sided transport between threads.
Here the transport is NVLink load/store between GPUs, done inside the CUDA
kernels; what remains on the host is:

* `exchange(rank, obj)`  — collective all-gather used once per group to agree
  on the config fingerprint and to trade window descriptors;
* `phase(rank)`          — the point between a collective's send half and its
  receive half.  One process per GPU needs nothing there (peers run
  concurrently); N ranks emulated on ONE GPU must have every rank's send
  kernel enqueued before any rank's receive kernel, so the local fabric
  barriers its rank threads;
* `stream(rank)`         — where a rank's kernels go.

* `trace`                — optional op log (the reference fabric's trace
  sink, fabric.py:83-111): a callable receiving one CSV line per transport
  op, or a file path.  The kernels record their window transfers on the
  device (epb_group_set_op_trace); the groups drain them after each call.

Two fabrics:
  Fabric(topology)                       N ranks as threads on one GPU
                                         (the reference's test model,
                                          harness.py:20-67)
  ProcessFabric(topology, process_group) one process per GPU, torch.distributed
                                         (NCCL or gloo) for bootstrap only
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import torch

from .core import EpError, ErrorCode

# op codes of the device op-trace records (include/epb200.h)
OP_PUT, OP_SIGNAL, OP_GET = 1, 2, 3
DEFAULT_TRACE_CAPACITY = 1 << 17  # records per group per call


class TraceSink:
    """Where op-trace lines go: a callable or a file path, like the
    reference fabric's `trace` argument (fabric.py:83-111).  Lines follow the
    reference's columns `op,src,dst,window,offset,len,signal_id,value,seq`:
      put,src,dst,window,offset,len,,,seq     row record / count row stored
                                              into dst's window by src
      get,src,dst,window,offset,len,,,seq     row read from dst's window by
                                              src (pulled transports; B200)
      signal,src,dst,,,,signal_id,value,seq   arrival counter add or flag
                                              store into dst's window
    `seq` numbers the lines of the whole fabric in the order they were
    drained (within one kernel the device append order)."""

    def __init__(self, trace, capacity: int = DEFAULT_TRACE_CAPACITY):
        self._file = None
        self.capacity = int(capacity)
        if trace is None:
            self.fn = None
        elif callable(trace):
            self.fn = trace
        else:
            self._file = open(trace, "w")
            self.fn = lambda line: self._file.write(line + "\n")
        self.seq = 0
        self.dropped = 0
        self._lock = threading.Lock()

    @property
    def active(self) -> bool:
        return self.fn is not None

    @staticmethod
    def format(rec, seq: int) -> str:
        w0, off, ln, val = (int(x) for x in rec)
        op, wid = w0 & 0xF, (w0 >> 4) & 0xF
        src, dst, sig = (w0 >> 8) & 0xFFF, (w0 >> 20) & 0xFFF, w0 >> 32
        if op == OP_SIGNAL:
            return f"signal,{src},{dst},,,,{sig},{val},{seq}"
        name = "put" if op == OP_PUT else "get" if op == OP_GET else f"op{op}"
        return f"{name},{src},{dst},{wid},{off},{ln},,,{seq}"

    def emit(self, records, dropped: int = 0) -> None:
        """records: [n, 4] uint64 device records (w0, offset, len, value)."""
        if self.fn is None:
            return
        with self._lock:
            self.dropped += dropped
            for rec in records:
                self.seq += 1
                self.fn(self.format(rec, self.seq))

    def close(self) -> None:
        if self._file is not None:
            self._file.close()
            self._file = None
            self.fn = None


@dataclass(frozen=True)
class NodeTopology:
    """Which ranks share a node (fabric.py:25-50)."""

    num_ranks: int
    ranks_per_node: int

    def __post_init__(self):
        if self.num_ranks < 1 or self.ranks_per_node < 1 or self.num_ranks % self.ranks_per_node:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          f"bad topology ({self.num_ranks} ranks, {self.ranks_per_node} per node)")

    @property
    def num_nodes(self) -> int:
        return self.num_ranks // self.ranks_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.ranks_per_node

    def rail_of(self, rank: int) -> int:
        return rank % self.ranks_per_node

    def same_node(self, a: int, b: int) -> bool:
        return self.node_of(a) == self.node_of(b)


class _Barrier:
    def __init__(self, n: int, timeout: float):
        self._b = threading.Barrier(n)
        self._timeout = timeout

    def wait(self):
        try:
            self._b.wait(self._timeout)
        except threading.BrokenBarrierError:
            raise EpError(ErrorCode.TRANSPORT_CLOSED, "fabric shut down or a rank stopped participating")

    def abort(self):
        self._b.abort()


class Fabric:
    """N emulated ranks on one GPU, one host thread per rank.

    Every rank's window lives on the same device; kernels store into peer
    windows through plain device pointers, exactly as they store into
    CUDA-IPC-mapped windows of other GPUs in ProcessFabric."""

    process_mode = False

    def __init__(self, topology: NodeTopology, seed: int = 0, device=None, timeout: float = 120.0, devices=None,
                 trace=None, trace_capacity: int = DEFAULT_TRACE_CAPACITY):
        """`devices`: one CUDA device per rank — ranks on several GPUs of one
        process (threads; peer windows through peer access, system-scope
        ordering); default: every rank on `device` (the current one).
        `trace`: op-trace sink (callable or path; TraceSink)."""
        self.topology = topology
        self.trace = TraceSink(trace, trace_capacity)
        self.seed = seed
        n = topology.num_ranks
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices] \
            if devices is not None else None
        if self.devices is not None and len(self.devices) != n:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"{len(self.devices)} devices for {n} ranks")
        if self.devices is not None:
            self._streams = [torch.cuda.Stream(device=d) for d in self.devices]
            self._stream = None
        else:
            self._streams = None
            self._stream = torch.cuda.Stream(device=self.device) if n > 1 else None
        self._barrier = _Barrier(n, timeout)
        self._lock = threading.Lock()
        self._calls = {}
        self._slots = {}
        self._closed = False
        self.registered = [0] * n  # bytes of live windows per rank (fabric.registered_bytes)

    # -- collectives ----------------------------------------------------------
    def exchange(self, rank: int, value) -> list:
        if self._closed:
            raise EpError(ErrorCode.TRANSPORT_CLOSED, "fabric shut down")
        with self._lock:
            gen = self._calls.get(rank, 0)
            self._calls[rank] = gen + 1
            self._slots.setdefault(gen, {})[rank] = value
        self._barrier.wait()
        with self._lock:
            slot = self._slots[gen]
            out = [slot[r] for r in range(self.topology.num_ranks)]
        self._barrier.wait()
        return out

    def phase(self, rank: int) -> None:
        if self.topology.num_ranks > 1:
            self._barrier.wait()

    def device_of(self, rank: int) -> torch.device:
        return self.devices[rank] if self.devices is not None else self.device

    def stream(self, rank: int):
        if self._streams is not None:
            return self._streams[rank]
        return self._stream if self._stream is not None else torch.cuda.current_stream(self.device)

    def registered_bytes(self, rank: int) -> int:
        return self.registered[rank]

    def shutdown(self) -> None:
        self._closed = True
        self._barrier.abort()
        self.trace.close()


class ProcessFabric:
    """One process per GPU; `process_group` (torch.distributed) carries only
    the bootstrap all-gather and barriers — never token data."""

    process_mode = True

    def __init__(self, topology: NodeTopology, process_group=None, trace=None,
                 trace_capacity: int = DEFAULT_TRACE_CAPACITY):
        import torch.distributed as dist

        self.topology = topology
        self.trace = TraceSink(trace, trace_capacity)
        self.group = process_group
        self._dist = dist
        world = dist.get_world_size(process_group)
        if world != topology.num_ranks:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          f"process group has {world} ranks, topology {topology.num_ranks}")
        self.rank = dist.get_rank(process_group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
        self.registered = [0] * topology.num_ranks

    def exchange(self, rank: int, value) -> list:
        if rank != self.rank:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"rank {rank} is not this process ({self.rank})")
        out = [None] * self.topology.num_ranks
        self._dist.all_gather_object(out, value, group=self.group)
        return out

    def phase(self, rank: int) -> None:
        return None

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)

    def stream(self, rank: int):
        return torch.cuda.current_stream()

    def registered_bytes(self, rank: int) -> int:
        return self.registered[rank] if rank == self.rank else 0

    def shutdown(self) -> None:
        self.trace.close()
