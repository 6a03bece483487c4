"""Index math, slot geometry, footprints and the header codec
(epsim layout.py).  Pure host functions: they size and describe buffers,
they never touch token data.

The receive windows this library allocates follow these formulas
(`footprint`, `EpGroup.buffer_bytes`) except that each slot is padded to a
16-byte multiple on the device (see csrc/geometry.h); the reference's byte
counts are what `footprint` reports, so the paper's memory-reduction claim
(2E/(N+K)) is preserved exactly.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

from .core import FP8_BLOCK, Dtype, EpError, ErrorCode


@dataclass(frozen=True)
class MoeShape:
    """Routing geometry (layout.py:32-59): expert e lives on rank e // L."""

    num_experts: int
    num_ranks: int
    tokens_per_rank: int
    top_k: int
    hidden: int

    def __post_init__(self):
        if self.num_experts < self.num_ranks:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          f"{self.num_experts} experts on {self.num_ranks} ranks")
        if not (1 <= self.top_k <= self.num_experts):
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"top_k {self.top_k}")

    @property
    def experts_per_rank(self) -> int:
        return math.ceil(self.num_experts / self.num_ranks)

    def owner_rank(self, expert: int) -> int:
        return expert // self.experts_per_rank

    def local_experts(self, rank: int) -> range:
        lo = rank * self.experts_per_rank
        return range(lo, min(lo + self.experts_per_rank, self.num_experts))


def idx_dp_legacy(expert: int, src_rank: int, shape: MoeShape, mod_by_ranks: bool = False) -> int:
    """Legacy dispatch sub-region (layout.py:81-95): (e mod L)*N + r."""
    n = shape.num_ranks
    if mod_by_ranks:
        if shape.experts_per_rank != n:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "strict (e mod N)*N + r indexing requires L == N")
        return (expert % n) * n + src_rank
    return (expert % shape.experts_per_rank) * n + src_rank


def idx_e(expert: int) -> int:
    return expert


def idx_d_opt(src_rank: int) -> int:
    return src_rank


def idx_c_opt(token: int, k: int, top_k: int) -> int:
    """Optimized combine slot t*K + k (layout.py:108-110)."""
    return token * top_k + k


def header_bytes(top_k: int) -> int:
    return 8 + 4 * top_k


@dataclass(frozen=True)
class SlotGeometry:
    header_bytes: int
    token_bytes: int
    scale_bytes: int

    @property
    def dispatch_bytes(self) -> int:
        return self.header_bytes + self.token_bytes + self.scale_bytes

    @property
    def combine_bytes(self) -> int:
        return self.token_bytes

    @staticmethod
    def for_config(hidden: int, dtype: Dtype, top_k: int, with_scales: bool) -> "SlotGeometry":
        return SlotGeometry(header_bytes(top_k), hidden * dtype.byte_width,
                            (hidden // FP8_BLOCK) * 4 if with_scales else 0)


@dataclass(frozen=True)
class FootprintReport:
    dispatch_bytes: int
    combine_bytes: int
    coordination_bytes: int

    @property
    def total(self) -> int:
        return self.dispatch_bytes + self.combine_bytes

    @property
    def total_with_coordination(self) -> int:
        return self.total + self.coordination_bytes


def footprint(shape: MoeShape, geom: SlotGeometry, layout: str) -> FootprintReport:
    """Receive bytes per rank, double buffered (layout.py:164-181)."""
    e, n, b, k = shape.num_experts, shape.num_ranks, shape.tokens_per_rank, shape.top_k
    if layout == "legacy":
        ds, cs = e * b, e * b
    elif layout == "optimized":
        ds, cs = n * b, b * k
    else:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"unknown layout {layout!r}")
    return FootprintReport(2 * ds * geom.dispatch_bytes, 2 * cs * geom.combine_bytes, 2 * (2 * e * 8))


def footprint_ratio(shape: MoeShape, geom: SlotGeometry | None = None) -> float:
    """legacy / optimized; closed form 2E/(N+K) without a geometry."""
    if geom is None:
        return 2.0 * shape.num_experts / (shape.num_ranks + shape.top_k)
    return footprint(shape, geom, "legacy").total / footprint(shape, geom, "optimized").total


def encode_header(src_token_idx: int, routing, top_k: int, num_experts: int | None = None) -> bytes:
    """Little-endian u32 token, u32 k_count, K u32 ids (layout.py:282-295);
    the dispatch slots on the device start with exactly these words."""
    routing = [int(e) for e in routing]
    if len(routing) > top_k:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"{len(routing)} routing entries exceed top_k {top_k}")
    if src_token_idx < 0:
        raise EpError(ErrorCode.INVALID_ARGUMENT, "negative token index")
    if num_experts is not None and any(not 0 <= e < num_experts for e in routing):
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"routing entry outside [0, {num_experts})")
    return struct.pack(f"<II{top_k}I", src_token_idx, len(routing), *(routing + [0] * (top_k - len(routing))))


def decode_header(blob: bytes, top_k: int):
    need = header_bytes(top_k)
    if len(blob) < need:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"header needs {need} bytes, got {len(blob)}")
    fields = struct.unpack_from(f"<II{top_k}I", blob)
    if fields[1] > top_k:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"k_count {fields[1]} > {top_k}")
    return fields[0], list(fields[2:2 + fields[1]])


def row_wire_bytes(hidden: int, dtype: Dtype, with_scales: bool = False) -> int:
    return hidden * dtype.byte_width + ((hidden // FP8_BLOCK) * 4 if with_scales else 0)
