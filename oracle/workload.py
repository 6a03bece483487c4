"""Seeded synthetic inputs (test infrastructure only).

`make_workload` replays the reference generator's exact RNG call sequence
(epsim oracle.py:32-45): per rank, tokens ~ U(-3, 3) [B, H] f32, then one
`permutation(E)[:K]` per token, then weights ~ U(0.1, 1.0) [B, K] f32, all
from one `np.random.default_rng(seed)`.  Identical seeds therefore give the
reference and this repo bit-identical inputs.

`make_zipf_workload` is the C5 skewed-routing generator the reference lacks
(SURVEY.md §8c divergence 3): K distinct experts per token drawn without
replacement with p ~ 1/(rank+1)^s over a seeded permutation of expert ids.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    tokens: list    # per rank f32 [B, H]
    routing: list   # per rank int64 [B, K]
    weights: list   # per rank f32 [B, K]


def make_workload(e: int, n: int, b: int, k: int, h: int, seed: int) -> Workload:
    rng = np.random.default_rng(seed)
    tokens, routing, weights = [], [], []
    for _ in range(n):
        tokens.append(rng.uniform(-3.0, 3.0, (b, h)).astype(np.float32))
        if b:
            rows = np.stack([rng.permutation(e)[:k] for _ in range(b)])
        else:
            rows = np.zeros((0, k), dtype=np.int64)
        routing.append(rows.astype(np.int64))
        weights.append(rng.uniform(0.1, 1.0, (b, k)).astype(np.float32))
    return Workload(tokens, routing, weights)


def make_zipf_workload(e: int, n: int, b: int, k: int, h: int, seed: int,
                       s: float = 1.0) -> Workload:
    rng = np.random.default_rng(seed)
    order = rng.permutation(e)                 # expert popularity ranking
    p = 1.0 / np.arange(1, e + 1, dtype=np.float64) ** s
    p /= p.sum()
    tokens, routing, weights = [], [], []
    for _ in range(n):
        tokens.append(rng.uniform(-3.0, 3.0, (b, h)).astype(np.float32))
        # Gumbel-top-k == sampling K without replacement proportional to p
        g = rng.gumbel(size=(b, e)) + np.log(p)[None, :]
        top = np.argsort(-g, axis=1, kind="stable")[:, :k]
        routing.append(order[top].astype(np.int64))
        weights.append(rng.uniform(0.1, 1.0, (b, k)).astype(np.float32))
    return Workload(tokens, routing, weights)


def expert_identity(e, rows):
    return rows


def expert_scale(e, rows):
    return (rows * np.float32(e + 1)).astype(np.float32)


def _affine(e):
    rng = np.random.default_rng(e)
    return np.float32(rng.uniform(0.5, 1.5)), np.float32(rng.uniform(-0.5, 0.5))


def expert_affine(e, rows):
    a, c = _affine(e)
    return (rows * a + c).astype(np.float32)


EXPERT_STUBS = {"identity": expert_identity, "scale": expert_scale,
                "affine": expert_affine}
