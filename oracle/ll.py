"""Low-latency dispatch/combine semantics restated from epsim ll.py
(test infrastructure only).  Vectorised numpy; no transport is modelled —
only what lands where.

Dispatch, per source rank s (ll.py:255-308, 378-400):
  * each token t touching destination d gets one slot, slots ordered by t;
  * on d, the row lands at recv[l, s*B + i] for every k with e_tk local to d
    (l = e_tk - d*L), i = rank of t among s's tokens routed to e_tk;
  * counts[l, s] = m(e, s)  (counter value m + 1, minus 1; ll.py:333-338);
  * plan rows (l, s, i, t, k) in (s asc, slot asc, k asc) order;
  * the row is the wire image of the token in the config dtype.
Combine (ll.py:404-507): the expert output at recv position is re-encoded in
the token dtype (FP8 without scales), and the home rank accumulates
  acc = 0; acc = f32(acc + f32(w[t,k] * y_k)) for k = 0..K-1.
"""

from __future__ import annotations

import numpy as np

from .codecs import wire_roundtrip
from .layout import experts_per_rank


def expert_ranks(routing: np.ndarray, e: int) -> np.ndarray:
    """i[t, k] = #{t' < t : e_tk in routing[t']} (distinct ids per row)."""
    b, k = routing.shape
    flat = routing.reshape(-1)
    order = np.argsort(flat, kind="stable")           # t-major within expert
    sorted_e = flat[order]
    first = np.searchsorted(sorted_e, sorted_e, side="left")
    rank = np.empty(b * k, dtype=np.int64)
    rank[order] = np.arange(b * k) - first
    return rank.reshape(b, k)


def dedup_slots(routing: np.ndarray, e: int, n: int) -> np.ndarray:
    """slot[t, d] = index of t among tokens touching rank d, or -1."""
    b = routing.shape[0]
    touch = np.zeros((b, n), dtype=bool)
    if b:
        touch[np.repeat(np.arange(b), routing.shape[1]),
              (routing // experts_per_rank(e, n)).reshape(-1)] = True
    csum = np.cumsum(touch, axis=0) - 1
    return np.where(touch, csum, -1)


def dispatch(tokens, routing, e, n, bmax, h, dtype, with_scales):
    """Returns per destination rank dict(recv, counts, plan)."""
    ell = experts_per_rank(e, n)
    out = []
    for d in range(n):
        out.append(dict(recv=np.zeros((ell, n * bmax, h), dtype=np.float32),
                        counts=np.zeros((ell, n), dtype=np.int64),
                        plan=[]))
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        b = rt.shape[0]
        if b == 0:
            continue
        wire = wire_roundtrip(tokens[s], dtype, with_scales)
        ranks = expert_ranks(rt, e)
        own = rt // ell
        for d in range(n):
            lo = d * ell
            tt, kk = np.nonzero(own == d)            # (t asc, k asc)
            if tt.size == 0:
                continue
            ll_ = rt[tt, kk] - lo
            ii = ranks[tt, kk]
            out[d]["recv"][ll_, s * bmax + ii] = wire[tt]
            np.add.at(out[d]["counts"], (ll_, np.full_like(ll_, s)), 1)
            out[d]["plan"].extend(zip(ll_.tolist(), [s] * tt.size, ii.tolist(),
                                      tt.tolist(), kk.tolist()))
    for d in range(n):
        out[d]["plan"] = np.array(out[d]["plan"], dtype=np.int64).reshape(-1, 5)
    return out


def combine(expert_out, routing, weights, e, n, bmax, h, dtype):
    """expert_out[d] = [L, N*B, H] f32 expert outputs on rank d.
    Returns per home rank the [b, H] f32 reduction."""
    ell = experts_per_rank(e, n)
    res = []
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        b, k = rt.shape
        w = np.asarray(weights[s], dtype=np.float32)
        acc = np.zeros((b, h), dtype=np.float32)
        if b:
            ranks = expert_ranks(rt, e)
            for kk in range(k):
                ek = rt[:, kk]
                d = ek // ell
                y = np.stack([expert_out[d[t]][ek[t] - d[t] * ell, s * bmax + ranks[t, kk]]
                              for t in range(b)])
                y = wire_roundtrip(y, dtype, False)
                acc = (acc + (w[:, kk:kk + 1] * y).astype(np.float32)).astype(np.float32)
        res.append(acc)
    return res


def apply_experts(recv, counts, rank, e, n, bmax, expert_fn):
    """Stub expert on the valid rows of one rank's [L, N*B, H] grid
    (harness.py:518-530): unused rows stay zero."""
    ell = experts_per_rank(e, n)
    out = np.zeros_like(recv)
    for l in range(counts.shape[0]):
        for r in range(counts.shape[1]):
            c = int(counts[l, r])
            if c:
                out[l, r * bmax:r * bmax + c] = expert_fn(rank * ell + l,
                                                          recv[l, r * bmax:r * bmax + c])
    return out


def dispatch_plan(routing, e, n, d):
    """Destination d only (no payload): plan rows (l, s, i, t, k) in the
    order of `dispatch` and counts [L, N] — the checker for large runs,
    where every source's full [L, N*B, H] grid would not fit."""
    ell = experts_per_rank(e, n)
    counts = np.zeros((ell, n), dtype=np.int64)
    plan = []
    for s in range(n):
        rt = np.asarray(routing[s], dtype=np.int64)
        if rt.shape[0] == 0:
            continue
        ranks = expert_ranks(rt, e)
        tt, kk = np.nonzero(rt // ell == d)
        ll_ = rt[tt, kk] - d * ell
        np.add.at(counts, (ll_, np.full_like(ll_, s)), 1)
        plan.append(np.stack([ll_, np.full_like(ll_, s), ranks[tt, kk], tt, kk], axis=1))
    plan = np.concatenate(plan) if plan else np.zeros((0, 5), dtype=np.int64)
    return plan, counts


def combine_scaled_experts(wire, routing, weights, scale_of, dtype):
    """One home rank's combine (ll.py:464-507) when every expert e returns
    its input row times scale_of(e) (exact in the wire dtype): the row of
    (t, k) is wire[t] * scale_of(e_tk), re-encoded in `dtype`, then
    acc = f32(acc + f32(w * y)) for ascending k."""
    rt = np.asarray(routing, dtype=np.int64)
    w = np.asarray(weights, dtype=np.float32)
    b, k = rt.shape
    acc = np.zeros(wire.shape, dtype=np.float32)
    for kk in range(k):
        y = wire_roundtrip((wire * scale_of(rt[:, kk])[:, None]).astype(np.float32), dtype, False)
        acc = (acc + (w[:, kk:kk + 1] * y).astype(np.float32)).astype(np.float32)
    return acc
