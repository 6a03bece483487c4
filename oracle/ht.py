"""High-throughput dispatch/combine semantics restated from epsim ht.py
(test infrastructure only).

Metadata (ht.py:291-331): m[src, e] tokens of src routed to e; q[src, d]
tokens of src touching rank d (dedup); recv_total(r) = sum over local e, src.
Dispatch (ht.py:553-583): output rows sorted by (local e asc, src asc, t asc);
origin = (e, src, t, k, w); rows are the wire image (f32/bf16/f16).
Combine (ht.py:587-735): p = f32(w * y) with y the f32 expert row (no wire
rounding, ht.py:622-624).  Per token, for each node holding one of its
experts (ascending node), partial = first present p, then f32(acc + p) in
ascending k over that node's experts (ht.py:680-694); the source then forms
out = f32(f32(0 + partial_0) + partial_1) ... (ht.py:727-734).  On one node
this equals the LL/oracle ascending-k order bit-for-bit.
"""

from __future__ import annotations

import numpy as np

from .codecs import wire_roundtrip
from .layout import experts_per_rank
from .ll import expert_ranks


def meta(routing, e, n):
    ell = experts_per_rank(e, n)
    m = np.zeros((n, e), dtype=np.int64)
    q = np.zeros((n, n), dtype=np.int64)
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        if rt.shape[0] == 0:
            continue
        np.add.at(m[s], rt.reshape(-1), 1)
        touch = np.zeros((rt.shape[0], n), dtype=bool)
        touch[np.repeat(np.arange(rt.shape[0]), rt.shape[1]), (rt // ell).reshape(-1)] = True
        q[s] = touch.sum(axis=0)
    return m, q


def recv_total(m, rank, e, n):
    ell = experts_per_rank(e, n)
    lo, hi = rank * ell, min(rank * ell + ell, e)
    return int(m[:, lo:hi].sum())


def expert_offsets(m, rank, e, n):
    """offsets[l, src] of each (local expert, src) group (ht.py:185-193)."""
    ell = experts_per_rank(e, n)
    lo, hi = rank * ell, min(rank * ell + ell, e)
    grp = m[:, lo:hi].T.reshape(-1)                  # (l asc, src asc)
    off = np.concatenate([[0], np.cumsum(grp)[:-1]]) if grp.size else grp
    return off.reshape(hi - lo, n)


def dispatch_plan(routing, weights, e, n, d):
    """Where every (src, token, k) routed to rank d lands in d's sorted
    output (ht.py:553-583 order, offsets of ht.py:185-193): arrays
    pos, e, src, t, k, w over those entries, plus recv_total and counts."""
    ell = experts_per_rank(e, n)
    m, _ = meta(routing, e, n)
    off = expert_offsets(m, d, e, n)
    cols = [[], [], [], [], [], []]
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        if rt.shape[0] == 0:
            continue
        ranks = expert_ranks(rt, e)
        tt, kk = np.nonzero(rt // ell == d)
        ee = rt[tt, kk]
        cols[0].append(off[ee - d * ell, s] + ranks[tt, kk])
        cols[1].append(ee)
        cols[2].append(np.full(len(tt), s, dtype=np.int64))
        cols[3].append(tt)
        cols[4].append(kk)
        cols[5].append(np.asarray(weights[s], dtype=np.float32)[tt, kk])
    pos, ee, src, tt, kk = (np.concatenate(c) if c else np.zeros(0, np.int64) for c in cols[:5])
    w = np.concatenate(cols[5]) if cols[5] else np.zeros(0, np.float32)
    counts = np.zeros((ell, n), dtype=np.int64)
    lo, hi = d * ell, min(d * ell + ell, e)
    counts[:hi - lo] = m[:, lo:hi].T
    return dict(pos=pos, e=ee, src=src, t=tt, k=kk, w=w, recv_total=recv_total(m, d, e, n), counts=counts)


def dispatch(tokens, routing, weights, e, n, h, dtype):
    """Per destination rank dict(rows [R, H], origin [R, 5] as
    (e, src, t, k) int64 + w f32 column separately, counts [L, N])."""
    m, q = meta(routing, e, n)
    out = []
    for d in range(n):
        pl = dispatch_plan(routing, weights, e, n, d)
        total = pl["recv_total"]
        rows = np.zeros((total, h), dtype=np.float32)
        origin = np.zeros((total, 4), dtype=np.int64)
        wts = np.zeros((total,), dtype=np.float32)
        pos = pl["pos"]
        for s in range(n):
            sel = pl["src"] == s
            if np.any(sel):
                rows[pos[sel]] = wire_roundtrip(tokens[s][pl["t"][sel]], dtype, False)
        origin[pos, 0], origin[pos, 1], origin[pos, 2], origin[pos, 3] = pl["e"], pl["src"], pl["t"], pl["k"]
        wts[pos] = pl["w"]
        out.append(dict(rows=rows, origin=origin, weights=wts, counts=pl["counts"],
                        recv_total=total))
    return out, m, q


def combine(expert_rows, routing, weights, e, n, rpn):
    """expert_rows[d] = [recv_total_d, H] f32 aligned with dispatch rows."""
    ell = experts_per_rank(e, n)
    m, _ = meta(routing, e, n)
    offs = [expert_offsets(m, d, e, n) for d in range(n)]
    res = []
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        w = np.asarray(weights[s], dtype=np.float32)
        b, k = rt.shape
        h = expert_rows[0].shape[1] if expert_rows else 0
        out = np.zeros((b, h), dtype=np.float32)
        if b == 0:
            res.append(out)
            continue
        ranks = expert_ranks(rt, e)
        own = rt // ell
        node = own // rpn
        p = np.zeros((b, k, h), dtype=np.float32)
        for kk in range(k):
            pos = np.array([offs[own[t, kk]][rt[t, kk] - own[t, kk] * ell, s] + ranks[t, kk]
                            for t in range(b)])
            y = np.stack([expert_rows[own[t, kk]][pos[t]] for t in range(b)])
            p[:, kk] = (w[:, kk:kk + 1] * y).astype(np.float32)
        for nd in range(n // rpn):
            present = node == nd                          # [b, k]
            part = np.zeros((b, h), dtype=np.float32)
            started = np.zeros(b, dtype=bool)
            for kk in range(k):
                sel = present[:, kk]
                first = sel & ~started
                more = sel & started
                part[first] = p[first, kk]
                part[more] = (part[more] + p[more, kk]).astype(np.float32)
                started |= sel
            out[started] = (out[started] + part[started]).astype(np.float32)
        res.append(out)
    return res


def apply_experts(rows, origin, expert_fn):
    """Stub expert on sorted 2D rows (harness.py:584-589)."""
    out = np.zeros_like(rows)
    for ex in np.unique(origin[:, 0]) if len(origin) else []:
        sel = origin[:, 0] == ex
        out[sel] = expert_fn(int(ex), rows[sel])
    return out
