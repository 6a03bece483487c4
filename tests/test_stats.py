"""Stats parity: LLStats / HTStats (ll.py:39-55,
ht.py:57-74) from the host-side accounting in paper_2603_13606_b200.stats
against the values the reference engine reported for the golden rounds
(tests/golden/make_golden.py stores them).  CPU only: the receive plan comes
from the oracle here; the GPU tests check the same numbers through the API.
"""

import numpy as np
import pytest

import paper_2603_13606_b200 as ep
from oracle import layout as olay
from oracle import ll as oll
from paper_2603_13606_b200 import stats as st
from tests._golden import HT_NAMES, LL_NAMES, ht_case, ll_case

LL_F = ("bytes_put", "msgs", "signals", "slots_used", "buffer_bytes")
HT_F = LL_F + ("inter_node_msgs", "intra_node_msgs")
DT = {"f32": ep.Dtype.F32, "bf16": ep.Dtype.BF16, "f16": ep.Dtype.F16, "fp8": ep.Dtype.FP8}


def _vec(s, fields):
    return np.array([getattr(s, f) for f in fields], dtype=np.int64)


def _cfg(algo, c, b):
    return ep.EpConfig(algorithm=algo, num_ranks=c["n"], ranks_per_node=c["rpn"], num_experts=c["e"],
                       top_k=c["k"], hidden=c["h"], max_tokens_per_rank=b, token_dtype=DT[c["dtype"]],
                       with_scales=c.get("scales", False))


def ll_plan_arrays(c, rank):
    """counts [L, N] and src_info [L, N*B] (t*K + k per valid row) of one
    rank, from the oracle's receive plan."""
    n, e, bmax, k = c["n"], c["e"], c["bmax"], c["k"]
    d = oll.dispatch(c["tokens"], c["routing"], e, n, bmax, c["h"], c["dtype"], c["scales"])[rank]
    ell = -(-e // n)
    src_info = np.full((ell, n * bmax), -1, np.int64)
    for l, s, i, t, kk in d["plan"]:
        src_info[l, s * bmax + i] = t * k + kk
    return d["counts"], src_info


@pytest.mark.parametrize("layout", ["optimized", "legacy"])
@pytest.mark.parametrize("name", LL_NAMES)
def test_ll_stats_match_reference(name, layout):
    c = ll_case(name)
    cfg = _cfg(ep.Algorithm.LL, c, c["bmax"])
    buf = olay.ll_window_bytes(c["e"], c["n"], c["bmax"], c["k"], c["h"], c["dtype"], c["scales"], layout)
    sfx = "" if layout == "optimized" else "_leg"
    for r in range(c["n"]):
        ds = st.ll_dispatch_stats(cfg, layout, c["routing"][r], buf)
        np.testing.assert_array_equal(_vec(ds, LL_F), c["g"][f"dstats{sfx}{r}"])
        counts, src_info = ll_plan_arrays(c, r)
        cs = st.ll_combine_stats(cfg, layout, r, counts, src_info, buf)
        np.testing.assert_array_equal(_vec(cs, LL_F), c["g"][f"cstats{sfx}{r}"])


@pytest.mark.parametrize("name", HT_NAMES)
def test_ht_stats_match_reference(name):
    c = ht_case(name)
    cfg = _cfg(ep.Algorithm.HT, c, c["b"])
    g = c["g"]
    buf = olay.ht_window_bytes(c["e"], c["n"], c["rpn"], c["b"], c["k"], c["h"], c["dtype"])
    for r in range(c["n"]):
        ds = st.ht_dispatch_stats(cfg, r, c["routing"][r], g["q"], buf)
        cs = st.ht_combine_stats(cfg, r, c["routing"][r], int(g[f"recv_total{r}"]), g["m"], buf)
        if c["rpn"] == c["n"]:
            assert ds.exact and cs.exact
            np.testing.assert_array_equal(_vec(ds, HT_F), g[f"dstats{r}"])
            np.testing.assert_array_equal(_vec(cs, HT_F), g[f"cstats{r}"])
        else:
            # multi-node: the forwarder's credits and remote aggregator runs
            # need other ranks' routing; the source-side fields still agree
            assert not ds.exact and not cs.exact
            for f in ("slots_used", "buffer_bytes", "inter_node_msgs"):
                assert getattr(ds, f) == g[f"dstats{r}"][HT_F.index(f)], f
            assert cs.slots_used == g[f"cstats{r}"][HT_F.index("slots_used")]
