"""Index math, region sizes and the header codec, restated from epsim
(test infrastructure only).

* L = ceil(E/N); expert e on rank e // L; tail rank may own fewer   layout.py:49-59
* header: little-endian u32 token, u32 k_count, K x u32 ids         layout.py:282-308
* slot geometry (hdr + H*w + 4*H/128 scales)                        layout.py:122-143
* footprint (legacy E*B / optimized N*B + B*K slots, double-buffered) layout.py:164-194
* LL window = 2 parities x [L*N + E counters][disp slots][comb slots] ll.py:58-121
* HT window plan                                                    ht.py:78-174
"""

from __future__ import annotations

import math
import struct

WIDTH = {"f32": 4, "bf16": 2, "f16": 2, "fp8": 1}


def experts_per_rank(e: int, n: int) -> int:
    return math.ceil(e / n)


def owner(expert, e: int, n: int):
    return expert // experts_per_rank(e, n)


def local_range(rank: int, e: int, n: int) -> range:
    lo = rank * experts_per_rank(e, n)
    return range(lo, min(lo + experts_per_rank(e, n), e))


def header_bytes(k: int) -> int:
    return 8 + 4 * k


def encode_header(token: int, routing, k: int) -> bytes:
    routing = [int(x) for x in routing]
    if len(routing) > k or token < 0:
        raise ValueError("bad header")
    return struct.pack(f"<II{k}I", token, len(routing), *(routing + [0] * (k - len(routing))))


def decode_header(blob: bytes, k: int):
    f = struct.unpack_from(f"<II{k}I", blob)
    if f[1] > k:
        raise ValueError("k_count")
    return f[0], list(f[2:2 + f[1]])


def slot_geometry(h: int, dtype: str, k: int, with_scales: bool):
    """(header, token, scale) bytes of one LL dispatch slot."""
    return header_bytes(k), h * WIDTH[dtype], (h // 128) * 4 if with_scales else 0


def footprint(e, n, b, k, h, dtype, with_scales, layout):
    """(dispatch, combine, coordination) receive bytes, double buffered."""
    hb, tb, sb = slot_geometry(h, dtype, k, with_scales)
    if layout == "legacy":
        ds, cs = e * b, e * b
    elif layout == "optimized":
        ds, cs = n * b, b * k
    else:
        raise ValueError(layout)
    return 2 * ds * (hb + tb + sb), 2 * cs * tb, 2 * (2 * e * 8)


def ll_window_bytes(e, n, b, k, h, dtype, with_scales, layout):
    hb, tb, sb = slot_geometry(h, dtype, k, with_scales)
    pairs = experts_per_rank(e, n) * n
    if layout == "legacy":
        ds, cs = pairs * b, e * b
    else:
        ds, cs = n * b, b * k
    parity = pairs * 8 + e * 8 + ds * (hb + tb + sb) + cs * tb
    return 2 * parity


def ht_window_bytes(e, n, rpn, b, k, h, dtype, with_scales=False, chunk=4, depth=8):
    nodes = n // rpn
    record = header_bytes(k) + 4 * k + h * WIDTH[dtype] + ((h // 128) * 4 if with_scales else 0)
    meta = 2 * n * (e + n) * 4
    rcount = n * 8
    rrec = n * b * record
    fifo = (nodes - 1) * depth * (8 + chunk * record)
    ccount = rpn * nodes * 8
    crow = nodes * b * k * (4 + 4 * h)
    partial = nodes * b * 4 * h
    return meta + rcount + rrec + fifo + ccount + crow + partial
