"""Pin the CPU oracle restatement against fixtures produced by the reference
simulator itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import codecs, ht as oht, layout as olay, ll as oll, workload as owl
from tests._golden import HT_NAMES, LL_NAMES, ht_case, ll_case, load


def test_e4m3_table_and_encoder_match_reference():
    g = load("codecs")
    np.testing.assert_array_equal(codecs.E4M3, g["table"])
    np.testing.assert_array_equal(codecs.encode_e4m3(g["e_x"]), g["e_codes"])


def test_block_quantisation_matches_reference():
    g = load("codecs")
    c, s = codecs.quantize_block(g["q_rows"])
    np.testing.assert_array_equal(c, g["q_codes"])
    np.testing.assert_array_equal(s.view(np.uint32), g["q_scales"].view(np.uint32))
    np.testing.assert_array_equal(codecs.dequantize_block(c, s), g["q_deq"])


def test_bf16_codec_matches_reference():
    g = load("codecs")
    np.testing.assert_array_equal(codecs.f32_to_bf16(g["bf_in"]), g["bf_out"])


def test_header_golden_bytes():
    g = load("codecs")
    assert olay.encode_header(3, [5, 9], 4) == g["hdr"].tobytes()
    assert olay.encode_header(0, list(range(8)), 8) == g["hdr8"].tobytes()
    assert olay.decode_header(g["hdr"].tobytes(), 4) == (3, [5, 9])


def test_window_geometry_matches_reference():
    g = load("codecs")
    names = ["f32", "bf16", "f16", "fp8"]
    for e, n, rpn, b, k, h, dt, sc, w_opt, w_leg, w_ht in g["geo"]:
        dt = names[dt]
        assert olay.ll_window_bytes(e, n, b, k, h, dt, bool(sc), "optimized") == w_opt
        assert olay.ll_window_bytes(e, n, b, k, h, dt, bool(sc), "legacy") == w_leg
        if w_ht >= 0:
            assert olay.ht_window_bytes(e, n, rpn, b, k, h, dt) == w_ht


def test_workload_replays_reference_rng():
    c = ll_case("ll_f32_n4")
    wl = owl.make_workload(c["e"], c["n"], c["b"], c["k"], c["h"], c["seed"])
    for r in range(c["n"]):
        np.testing.assert_array_equal(wl.tokens[r], c["tokens"][r])
        np.testing.assert_array_equal(wl.routing[r], c["routing"][r])
        np.testing.assert_array_equal(wl.weights[r], c["weights"][r])


@pytest.mark.parametrize("name", LL_NAMES)
def test_ll_oracle_matches_reference_engine(name):
    c = ll_case(name)
    n, e, bmax, h, k = c["n"], c["e"], c["bmax"], c["h"], c["k"]
    res = oll.dispatch(c["tokens"], c["routing"], e, n, bmax, h, c["dtype"], c["scales"])
    stub = owl.EXPERT_STUBS[c["stub"]]
    outs = []
    for r in range(n):
        g = c["g"]
        np.testing.assert_array_equal(res[r]["counts"], g[f"counts{r}"])
        pos = g[f"recvpos{r}"]
        got = res[r]["recv"][pos[:, 0], pos[:, 1] * bmax + pos[:, 2]] if len(pos) else \
            np.zeros((0, h), np.float32)
        np.testing.assert_array_equal(got, g[f"recvrows{r}"])
        assert int(res[r]["counts"].sum()) == int(g[f"recv_total{r}"])
        outs.append(oll.apply_experts(res[r]["recv"], res[r]["counts"], r, e, n, bmax, stub))
    comb = oll.combine(outs, c["routing"], c["weights"], e, n, bmax, h, c["dtype"])
    for r in range(n):
        np.testing.assert_array_equal(comb[r], c["g"][f"out{r}"])


@pytest.mark.parametrize("name", HT_NAMES)
def test_ht_oracle_matches_reference_engine(name):
    c = ht_case(name)
    n, e, h = c["n"], c["e"], c["h"]
    res, m, q = oht.dispatch(c["tokens"], c["routing"], c["weights"], e, n, h, c["dtype"])
    g = c["g"]
    np.testing.assert_array_equal(m, g["m"])
    np.testing.assert_array_equal(q, g["q"])
    stub = owl.EXPERT_STUBS[c["stub"]]
    rows = []
    for r in range(n):
        np.testing.assert_array_equal(res[r]["rows"], g[f"rows{r}"])
        np.testing.assert_array_equal(res[r]["origin"], g[f"origin{r}"])
        np.testing.assert_array_equal(res[r]["weights"], g[f"originw{r}"])
        rows.append(oht.apply_experts(res[r]["rows"], res[r]["origin"], stub))
    comb = oht.combine(rows, c["routing"], c["weights"], e, n, c["rpn"])
    for r in range(n):
        np.testing.assert_array_equal(comb[r], g[f"out{r}"])
