"""Issue-side accounting of one collective op, field for field the
reference's LLStats / HTStats (epsim ll.py:39-55, ht.py:57-74).

The reference counts what its message model issues: one `put`/LSA store per
contiguous blob (msgs, bytes_put), one counter write or signal per flag
(signals), one slot per token row placed (slots_used), plus the window size
(buffer_bytes).  Those numbers are deterministic functions of the routing and
the config, so here they are computed on the host from the handle's routing
(dispatch) or from the receive plan the dispatch kernel recorded (combine:
counts + src_info), only when a caller asks for them — the kernels never pay
for observability.  Byte counts use the reference's wire formats (header
8 + 4K B, row H*w, FP8 scales 4*H/128 B, HT record = header + 4K weights +
row, HT contribution = 4 + 4H B), not this library's padded slots.

Multi-node HT (ranks_per_node < num_ranks) is reported for the source side
and this rank's fan-out from the metadata; the forwarder's head-credit
signals and the aggregator runs of remote sources need other ranks' routing
and are left out (`exact` is False then).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import FP8_BLOCK, EpConfig

COUNTER_BYTES = 8        # ll.py / ht.py counter words
VALID_BYTES = 4          # ht.py:49 contribution valid marker
CHUNK_HEADER_BYTES = 8   # ht.py:47


@dataclass
class LLStats:
    op: str
    bytes_put: int = 0
    msgs: int = 0
    signals: int = 0
    slots_used: int = 0
    buffer_bytes: int = 0

    FIELDS = ("op", "bytes_put", "msgs", "signals", "slots_used", "buffer_bytes")

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f in self.FIELDS}


@dataclass
class HTStats:
    op: str
    bytes_put: int = 0
    msgs: int = 0
    signals: int = 0
    slots_used: int = 0
    buffer_bytes: int = 0
    inter_node_msgs: int = 0
    intra_node_msgs: int = 0
    fifo_stalls: int = 0     # scheduling-dependent in the reference; 0 here
    exact: bool = True

    FIELDS = ("op", "bytes_put", "msgs", "signals", "slots_used", "buffer_bytes", "inter_node_msgs",
              "intra_node_msgs", "fifo_stalls")

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f in self.FIELDS}


def _owner(e, ell):
    return np.asarray(e) // ell


def _ll_slot_bytes(cfg: EpConfig) -> int:
    sb = (cfg.hidden // FP8_BLOCK) * 4 if cfg.with_scales else 0
    return 8 + 4 * cfg.top_k + cfg.hidden * cfg.token_dtype.byte_width + sb


def _local_count(cfg: EpConfig, rank: int) -> int:
    ell = cfg.experts_per_rank
    return max(0, min(cfg.num_experts, (rank + 1) * ell) - rank * ell)


def ll_dispatch_stats(cfg: EpConfig, layout: str, routing: np.ndarray, buffer_bytes: int) -> LLStats:
    """ll.py:271-308: optimized = one blob per destination rank holding the
    tokens that touch it, then one counter per (destination's local expert);
    legacy = one blob per expert, one counter per expert."""
    st = LLStats("dispatch", buffer_bytes=buffer_bytes)
    routing = np.asarray(routing, dtype=np.int64).reshape(-1, cfg.top_k)
    slot = _ll_slot_bytes(cfg)
    ell, n, e = cfg.experts_per_rank, cfg.num_ranks, cfg.num_experts
    if layout == "legacy":
        per_e = np.bincount(routing.ravel(), minlength=e) if routing.size else np.zeros(e, np.int64)
        used = int(np.count_nonzero(per_e))
        st.msgs, st.bytes_put, st.slots_used = used, int(per_e.sum()) * slot, int(per_e.sum())
        st.signals = e
        return st
    own = _owner(routing, ell)
    for d in range(n):
        toks = int(np.any(own == d, axis=1).sum()) if routing.size else 0
        if toks:
            st.msgs += 1
            st.bytes_put += toks * slot
            st.slots_used += toks
        st.signals += _local_count(cfg, d)
    return st


def ll_combine_stats(cfg: EpConfig, layout: str, rank: int, counts: np.ndarray, src_info: np.ndarray,
                     buffer_bytes: int) -> LLStats:
    """ll.py:404-462: per source rank, its rows sorted by combine slot
    (optimized t*K + k, legacy e*B + t) and merged into runs of consecutive
    slots, one message per run; one counter per (source, local expert)."""
    st = LLStats("combine", buffer_bytes=buffer_bytes)
    n, b, k = cfg.num_ranks, cfg.max_tokens_per_rank, cfg.top_k
    ell = cfg.experts_per_rank
    row_bytes = cfg.hidden * cfg.combine_wire.byte_width
    counts = np.asarray(counts, dtype=np.int64).reshape(ell, n)
    src_info = np.asarray(src_info, dtype=np.int64).reshape(ell, n * b)
    nloc = _local_count(cfg, rank)
    for r in range(n):
        lin = []
        for l in range(nloc):
            info = src_info[l, r * b:r * b + counts[l, r]]
            if layout == "legacy":
                lin.append((rank * ell + l) * b + info // k)
            else:
                lin.append(info)
        lin = np.sort(np.concatenate(lin)) if lin else np.zeros(0, np.int64)
        if len(lin):
            runs = 1 + int(np.count_nonzero(np.diff(lin) != 1))
            st.msgs += runs
            st.bytes_put += len(lin) * row_bytes
        st.slots_used += len(lin)
        st.signals += nloc
    return st


def _ht_record_bytes(cfg: EpConfig) -> int:
    return 8 + 4 * cfg.top_k + 4 * cfg.top_k + cfg.hidden * cfg.token_dtype.byte_width


def ht_dispatch_stats(cfg: EpConfig, rank: int, routing: np.ndarray, meta_q: np.ndarray,
                      buffer_bytes: int) -> HTStats:
    """ht.py:291-331 (metadata all-gather) + ht.py:381-461 (records to
    same-node ranks, chunked streams to remote nodes) + this rank's
    forwarder fan-out (ht.py:532-551)."""
    st = HTStats("dispatch", buffer_bytes=buffer_bytes)
    n, e, rpn = cfg.num_ranks, cfg.num_experts, cfg.ranks_per_node
    node = rank // rpn
    routing = np.asarray(routing, dtype=np.int64).reshape(-1, cfg.top_k)
    own = _owner(routing, cfg.experts_per_rank)
    # metadata: one (E+N) u32 row store + one signal per destination
    for d in range(n):
        st.msgs += 1
        st.bytes_put += (e + n) * 4
        st.signals += 1
    rec = _ht_record_bytes(cfg)
    for d in range(n):
        if d // rpn != node:
            continue
        toks = int(np.any(own == d, axis=1).sum()) if routing.size else 0
        if not toks:
            continue
        st.msgs += 2                      # records, then the count word
        st.bytes_put += toks * rec + COUNTER_BYTES
        st.intra_node_msgs += toks
        st.slots_used += toks
    nodes = n // rpn
    if nodes > 1:
        st.exact = False
        cap = cfg.ht_chunk_tokens
        own_node = own // rpn
        for nd in range(nodes):
            if nd == node:
                continue
            toks = int(np.any(own_node == nd, axis=1).sum()) if routing.size else 0
            chunks = (toks + cap - 1) // cap
            st.msgs += chunks + 1         # data chunks + end-of-stream chunk
            st.bytes_put += chunks * CHUNK_HEADER_BYTES + toks * rec + CHUNK_HEADER_BYTES
            st.inter_node_msgs += toks
            st.slots_used += toks
            st.signals += chunks + 1      # tail signal per chunk
        # forwarder: records from same-rail ranks of other nodes fanned out
        # to this node's ranks (two stores each)
        q = np.asarray(meta_q, dtype=np.int64).reshape(n, n)
        rail = rank % rpn
        for src in range(n):
            if src // rpn == node or src % rpn != rail:
                continue
            fan = int(q[src, node * rpn:(node + 1) * rpn].sum())
            st.msgs += 2 * fan
            st.bytes_put += fan * (rec + COUNTER_BYTES)
            st.intra_node_msgs += fan
    return st


def ht_combine_stats(cfg: EpConfig, rank: int, routing: np.ndarray, recv_total: int, meta_m: np.ndarray,
                     buffer_bytes: int) -> HTStats:
    """ht.py:626-735 (hierarchical): every received row goes, weighted, to
    the node aggregator of its source (4 + 4H B), one count word per source
    that received contributions; the aggregator ships partial rows back in
    runs of consecutive tokens and signals the source."""
    st = HTStats("combine", buffer_bytes=buffer_bytes)
    n, rpn = cfg.num_ranks, cfg.ranks_per_node
    node = rank // rpn
    ell = cfg.experts_per_rank
    st.msgs += recv_total
    st.bytes_put += recv_total * (VALID_BYTES + 4 * cfg.hidden)
    st.intra_node_msgs += recv_total
    st.slots_used += recv_total
    m = np.asarray(meta_m, dtype=np.int64).reshape(n, cfg.num_experts)
    lo, hi = rank * ell, min(cfg.num_experts, (rank + 1) * ell)
    for src in range(n):
        if int(m[src, lo:hi].sum()):
            st.msgs += 1
            st.bytes_put += COUNTER_BYTES
    # aggregator duty: on one node the aggregator of a source is the source
    # itself, i.e. this rank aggregates its own tokens touching this node
    routing = np.asarray(routing, dtype=np.int64).reshape(-1, cfg.top_k)
    own_node = _owner(routing, ell) // rpn
    toks = np.nonzero(np.any(own_node == node, axis=1))[0] if routing.size else np.zeros(0, np.int64)
    if len(toks):
        runs = 1 + int(np.count_nonzero(np.diff(toks) != 1))
        st.msgs += runs
        st.bytes_put += len(toks) * 4 * cfg.hidden
        st.intra_node_msgs += len(toks)
        st.signals += 1
    if n // rpn > 1:
        st.exact = False  # same-rail sources on other nodes: their routing is not local
    return st
