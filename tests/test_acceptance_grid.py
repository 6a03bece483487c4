"""The reference's acceptance grid (epsim tests/test_acceptance.py:34-105,
driver.verify_grid: driver.py:386-448) on the CUDA path: every
configuration point N in {1, 2, 4, 8} x nodes in {1, 2} x E in {8, 16, 32}
x B in {1, 16, 32} x K in {1, 2, 8}, for LL in both layouts (staged and
unstaged alternating) and HT, ranks emulated on one B200, checked
bit-for-bit against the CPU oracle (counts, every received row at its
oracle position, HT origins, and the combine output) — stricter than the
reference's 1e-6 / 1e-5 tolerances.  A second pass is the reference's
round-trip identity (integer tokens, weights 1/K, identity experts): every
token must come back exactly."""

import numpy as np
import pytest
import torch

from oracle import ht as oht
from oracle import ll as oll
from oracle import workload as owl
from tests.gpu_util import make_cfg, run_ht, run_ll

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda_required():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def grid_shapes():
    for n in (1, 2, 4, 8):
        for nodes in (1, 2):
            if nodes > n or n % nodes:
                continue
            for e in (8, 16, 32):
                if e < n:
                    continue
                for b in (1, 16, 32):
                    for k in (1, 2, 8):
                        if k > e:
                            continue
                        yield n, n // nodes, e, b, k


H = 8


def _check_ll_case(n, rpn, e, b, k, wl, layout, staged, stub):
    cfg = make_cfg("ll", n, rpn, e, b, k, H)
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, stub, staged=staged, layout=layout)
    d = oll.dispatch(wl.tokens, wl.routing, e, n, b, H, "f32", False)
    ys = [oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, n, b, stub) for r in range(n)]
    comb = oll.combine(ys, wl.routing, wl.weights, e, n, b, H, "f32")
    label = f"LL N={n} rpn={rpn} E={e} B={b} K={k} {layout} staged={staged}"
    for r in range(n):
        np.testing.assert_array_equal(res[r]["counts"], d[r]["counts"], err_msg=label)
        plan = d[r]["plan"]
        if len(plan):
            idx = (plan[:, 0], plan[:, 1] * b + plan[:, 2])
            np.testing.assert_array_equal(res[r]["recv"][idx], d[r]["recv"][idx], err_msg=label)
        np.testing.assert_array_equal(res[r]["out"], comb[r], err_msg=label)
    return res


def _check_ht_case(n, rpn, e, b, k, wl, stub):
    cfg = make_cfg("ht", n, rpn, e, b, k, H)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, stub)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, n, H, "f32")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], stub) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, e, n, rpn)
    label = f"HT N={n} rpn={rpn} E={e} B={b} K={k}"
    for r in range(n):
        np.testing.assert_array_equal(res[r]["m"], m, err_msg=label)
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"], err_msg=label)
        np.testing.assert_array_equal(res[r]["origin"], dd[r]["origin"], err_msg=label)
        np.testing.assert_array_equal(res[r]["out"], comb[r], err_msg=label)
    return res


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_oracle_equivalence_grid(n):
    cases = 0
    for nn, rpn, e, b, k in grid_shapes():
        if nn != n:
            continue
        wl = owl.make_workload(e, n, b, k, H, seed=e * 1000 + b * 10 + k)
        _check_ll_case(n, rpn, e, b, k, wl, "optimized", cases % 2 == 1, owl.expert_affine)
        _check_ll_case(n, rpn, e, b, k, wl, "legacy", cases % 2 == 0, owl.expert_affine)
        _check_ht_case(n, rpn, e, b, k, wl, owl.expert_affine)
        cases += 3
    assert cases > 0


@pytest.mark.parametrize("n", [2, 8])
def test_round_trip_identity_exact(n):
    """test_acceptance.py:77-105: integer tokens and 1/K weights keep every
    partial sum exact, so the combine must return the tokens bit-for-bit."""
    for nn, rpn, e, b, k in grid_shapes():
        if nn != n:
            continue
        rng = np.random.default_rng(e * 1000 + b * 10 + k)
        tokens = [rng.integers(-512, 512, (b, H)).astype(np.float32) for _ in range(n)]
        routing = [np.stack([rng.permutation(e)[:k] for _ in range(b)]).astype(np.int64) for _ in range(n)]
        weights = [np.full((b, k), 1.0 / k, dtype=np.float32) for _ in range(n)]
        wl = owl.Workload(tokens, routing, weights)
        for layout in ("optimized", "legacy"):
            res = run_ll(make_cfg("ll", n, rpn, e, b, k, H), tokens, routing, weights, owl.expert_identity,
                         layout=layout)
            for r in range(n):
                np.testing.assert_array_equal(res[r]["out"], tokens[r], err_msg=f"LL {layout} E={e} B={b} K={k}")
        res = run_ht(make_cfg("ht", n, rpn, e, b, k, H), wl.tokens, wl.routing, wl.weights, owl.expert_identity)
        for r in range(n):
            np.testing.assert_array_equal(res[r]["out"], tokens[r], err_msg=f"HT E={e} B={b} K={k}")
