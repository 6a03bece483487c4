"""GPU parity: the CUDA path through the public API against the reference's
golden fixtures and the CPU oracle, on ranks emulated on one B200."""

import numpy as np
import pytest
import torch

import paper_2603_13606_b200 as ep
from oracle import codecs as oc
from oracle import ht as oht
from oracle import ll as oll
from oracle import workload as owl
from tests._golden import HT_NAMES, LL_NAMES, ht_case, ll_case, load
from tests.rank_threads import run_ranks
from tests.gpu_util import bf16_round, make_cfg, run_ht, run_ll

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda_required():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_13606_b200 import _lib
    _lib.load()


# ---------------------------------------------------------------------------
# codecs (K7) — bit-exact with the reference encoder
# ---------------------------------------------------------------------------


def test_e4m3_encoder_golden_and_sweep():
    g = load("codecs")
    x = torch.from_numpy(g["e_x"]).cuda()
    codes = torch.empty(x.numel(), dtype=torch.uint8, device="cuda")
    from paper_2603_13606_b200 import _lib
    _lib.call("epb_e4m3_encode", x.data_ptr(), x.numel(), codes.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(codes.cpu().numpy(), g["e_codes"])
    # strided sweep over every f32 magnitude up to beyond the clamp, plus
    # +-8 ulps around every exact midpoint, both signs
    bits = np.arange(0, 0x43F00000, 61, dtype=np.uint32)
    mids = oc._MID.astype(np.float32).view(np.uint32)
    near = (mids[:, None].astype(np.int64) + np.arange(-8, 9)[None, :]).reshape(-1).astype(np.uint32)
    allb = np.concatenate([bits, near])
    xs = np.concatenate([allb.view(np.float32), -allb.view(np.float32)])
    want = oc.encode_e4m3(xs)
    xt = torch.from_numpy(xs).cuda()
    got = torch.empty(xt.numel(), dtype=torch.uint8, device="cuda")
    _lib.call("epb_e4m3_encode", xt.data_ptr(), xt.numel(), got.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_block_quantise_golden_and_random():
    g = load("codecs")
    c, s = ep.quantize_block(g["q_rows"])
    np.testing.assert_array_equal(c.cpu().numpy(), g["q_codes"])
    np.testing.assert_array_equal(s.cpu().numpy().view(np.uint32), g["q_scales"].view(np.uint32))
    np.testing.assert_array_equal(ep.dequantize_block(c, s).cpu().numpy(), g["q_deq"])
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((64, 7168)) * rng.uniform(0.01, 100, (64, 1))).astype(np.float32)
    c, s = ep.quantize_block(x)
    wc, ws = oc.quantize_block(x)
    np.testing.assert_array_equal(c.cpu().numpy(), wc)
    np.testing.assert_array_equal(s.cpu().numpy(), ws)
    with pytest.raises(ep.EpError):
        ep.quantize_block(np.full(128, np.inf, np.float32))


def test_ndtensor_codecs_match_reference():
    g = load("codecs")
    t = ep.tensor_from_f32(g["bf_in"], ep.Dtype.BF16, ep.TensorTag.TOKENS)
    np.testing.assert_array_equal(t.raw(), g["bf_out"])
    np.testing.assert_array_equal(t.read_f32(), oc.bf16_to_f32(g["bf_out"]))
    t8 = ep.tensor_from_f32(g["e_x"], ep.Dtype.FP8, ep.TensorTag.TOKENS)
    np.testing.assert_array_equal(t8.raw(), g["e_codes"])
    nan_codes = ep.tensor_create((2,), ep.Dtype.FP8, ep.TensorTag.TOKENS)
    nan_codes.write_raw(np.array([0x7F, 0xFF], np.uint8))
    np.testing.assert_array_equal(nan_codes.read_f32(), [0.0, 0.0])  # core.py:95-96


# ---------------------------------------------------------------------------
# LL against the reference's own engine outputs
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", LL_NAMES)
@pytest.mark.parametrize("staged", [False, True])
def test_ll_matches_reference_golden(name, staged):
    c = ll_case(name)
    cfg = make_cfg("ll", c["n"], c["rpn"], c["e"], c["bmax"], c["k"], c["h"], c["dtype"], c["scales"])
    res = run_ll(cfg, c["tokens"], c["routing"], c["weights"], owl.EXPERT_STUBS[c["stub"]], staged=staged)
    g = c["g"]
    for r in range(c["n"]):
        np.testing.assert_array_equal(res[r]["counts"], g[f"counts{r}"])
        pos = g[f"recvpos{r}"]
        got = res[r]["recv"][pos[:, 0], pos[:, 1] * c["bmax"] + pos[:, 2]] if len(pos) else \
            np.zeros((0, c["h"]), np.float32)
        np.testing.assert_array_equal(got, g[f"recvrows{r}"])
        assert res[r]["recv_total"] == int(g[f"recv_total{r}"])
        np.testing.assert_array_equal(res[r]["out"], g[f"out{r}"])
        _check_stats(res[r], g, r, LL_STAT_F)


LL_STAT_F = ("bytes_put", "msgs", "signals", "slots_used", "buffer_bytes")
HT_STAT_F = LL_STAT_F + ("inter_node_msgs", "intra_node_msgs")


def _check_stats(res, g, r, fields, sfx=""):
    """handle.dispatch_result.stats / handle.combine_stats against the
    reference engine's LLStats / HTStats of the golden round."""
    for key, st in (("dstats", res["dstats"]), ("cstats", res["cstats"])):
        assert st.as_dict()["op"] == ("dispatch" if key == "dstats" else "combine")
        got = np.array([getattr(st, f) for f in fields], dtype=np.int64)
        np.testing.assert_array_equal(got, g[f"{key}{sfx}{r}"], err_msg=key)


@pytest.mark.parametrize("name", HT_NAMES)
def test_ht_matches_reference_golden(name):
    c = ht_case(name)
    cfg = make_cfg("ht", c["n"], c["rpn"], c["e"], c["b"], c["k"], c["h"], c["dtype"])
    res = run_ht(cfg, c["tokens"], c["routing"], c["weights"], owl.EXPERT_STUBS[c["stub"]])
    g = c["g"]
    for r in range(c["n"]):
        np.testing.assert_array_equal(res[r]["m"], g["m"])
        np.testing.assert_array_equal(res[r]["q"], g["q"])
        np.testing.assert_array_equal(res[r]["rows"], g[f"rows{r}"])
        np.testing.assert_array_equal(res[r]["origin"], g[f"origin{r}"])
        np.testing.assert_array_equal(res[r]["origin_w"], g[f"originw{r}"])
        assert res[r]["recv_total"] == int(g[f"recv_total{r}"])
        np.testing.assert_array_equal(res[r]["out"], g[f"out{r}"])
        if c["rpn"] == c["n"]:
            _check_stats(res[r], g, r, HT_STAT_F)


# ---------------------------------------------------------------------------
# against the oracle at larger / production shapes
# ---------------------------------------------------------------------------


def _ll_oracle(cfg, wl, stub, bf16_expert=False):
    n, e, bmax, h = cfg.num_ranks, cfg.num_experts, cfg.max_tokens_per_rank, cfg.hidden
    d = oll.dispatch(wl.tokens, wl.routing, e, n, bmax, h, cfg.token_dtype.value, cfg.with_scales)
    outs = []
    for r in range(n):
        y = oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, n, bmax, stub)
        outs.append(bf16_round(y) if bf16_expert else y)
    comb = oll.combine(outs, wl.routing, wl.weights, e, n, bmax, h, cfg.combine_wire.value)
    return d, comb


def _check_ll(cfg, res, d, comb):
    bmax = cfg.max_tokens_per_rank
    for r in range(cfg.num_ranks):
        np.testing.assert_array_equal(res[r]["counts"], d[r]["counts"])
        plan = d[r]["plan"]
        if len(plan):
            idx = (plan[:, 0], plan[:, 1] * bmax + plan[:, 2])
            np.testing.assert_array_equal(res[r]["recv"][idx], d[r]["recv"][idx])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


@pytest.mark.parametrize("n,b", [(1, 128), (2, 128), (8, 32)])
def test_ll_dsv3_fp8_matches_oracle(n, b):
    """C2 shapes: E=256, K=8, H=7168, FP8 + scales (reference inputs)."""
    cfg = make_cfg("ll", n, n, 256, b, 8, 7168, "fp8", True)
    wl = owl.make_workload(256, n, b, 8, 7168, seed=n)
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_identity)
    d, comb = _ll_oracle(cfg, wl, owl.expert_identity)
    _check_ll(cfg, res, d, comb)


@pytest.mark.parametrize("b", [512, 600, 1024])
def test_ll_batch_at_and_beyond_the_decode_kernel(b):
    """512 tokens per rank is the largest batch the decode (FAST) kernel
    takes — one routing row per thread; 600 and 1024 run the general kernel
    — bit-exact with the oracle either way (N=2, bf16 in, FP8 + scales on
    the wire)."""
    n, e, k, h = 2, 32, 8, 512
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, e, k, h, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(e, n, b, k, h, seed=b)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, mode="bf16", wire_out=True,
                 bf16_expert=True)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale, bf16_expert=True)
    _check_ll(cfg, res, d, comb)


@pytest.mark.parametrize("n", [1, 4])
def test_ll_c2_hot_path_bf16_in_fp8_wire_bf16_combine(n):
    """North-star path: bf16 tokens, in-kernel FP8 quantisation, wire-dtype
    output + scales, bf16 expert outputs, bf16 combine wire."""
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 256, 8, 7168, 64, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(256, n, 64, 8, 7168, seed=10 + n)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, mode="bf16", wire_out=True,
                 bf16_expert=True)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale, bf16_expert=True)
    _check_ll(cfg, res, d, comb)


def test_ll_fewer_tokens_zipf_and_empty_rank():
    cfg = make_cfg("ll", 4, 4, 16, 8, 4, 256, "bf16")
    wl = owl.make_zipf_workload(16, 4, 5, 4, 256, seed=3)
    wl.tokens[2] = wl.tokens[2][:0]
    wl.routing[2] = wl.routing[2][:0]
    wl.weights[2] = wl.weights[2][:0]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine)
    d, comb = _ll_oracle(cfg, wl, owl.expert_affine)
    _check_ll(cfg, res, d, comb)


@pytest.mark.parametrize("n", [1, 3])
def test_ht_empty_and_ragged_ranks(n):
    """HT with a rank that routes no token (and, at N=1, an empty batch:
    the one-launch open with no chunk), the others ragged."""
    e, k, h = 12, 3, 256
    cfg = make_cfg("ht", n, n, e, 9, k, h, "bf16")
    wl = owl.make_workload(e, n, 9, k, h, seed=13)
    for r, keep in enumerate([0, 9, 4][:n]):
        wl.tokens[r] = wl.tokens[r][:keep]
        wl.routing[r] = wl.routing[r][:keep]
        wl.weights[r] = wl.weights[r][:keep]
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, n, h, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, e, n, n)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["m"], m)
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["origin"], dd[r]["origin"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


def test_ll_unaligned_hidden_element_path():
    cfg = make_cfg("ll", 2, 2, 8, 4, 3, 12, "fp8", False)
    wl = owl.make_workload(8, 2, 4, 3, 12, seed=1)
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale)
    _check_ll(cfg, res, d, comb)


def test_ll_parity_reuse_many_rounds():
    cfg = make_cfg("ll", 2, 1, 8, 6, 2, 128, "bf16")
    wl = owl.make_workload(8, 2, 6, 2, 128, seed=30)
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, rounds=6)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale)
    for r in range(2):
        for rnd in res[r]:
            np.testing.assert_array_equal(rnd["out"], comb[r])


# ---------------------------------------------------------------------------
# LL legacy layout (layout.py:146-194, ll.py:271-287, :362-376): per-(expert,
# src) dispatch slots and per-(expert, token) combine slots, same outputs
# ("layouts agree bitwise", test_ll.py:307-317)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["ll_f32_n4", "ll_fp8s", "ll_uneven", "ll_n1"])
@pytest.mark.parametrize("staged", [False, True])
def test_ll_legacy_layout_matches_reference_golden(name, staged):
    c = ll_case(name)
    cfg = make_cfg("ll", c["n"], c["rpn"], c["e"], c["bmax"], c["k"], c["h"], c["dtype"], c["scales"])
    res = run_ll(cfg, c["tokens"], c["routing"], c["weights"], owl.EXPERT_STUBS[c["stub"]], staged=staged,
                 layout="legacy")
    g = c["g"]
    for r in range(c["n"]):
        np.testing.assert_array_equal(res[r]["counts"], g[f"counts{r}"])
        pos = g[f"recvpos{r}"]
        got = res[r]["recv"][pos[:, 0], pos[:, 1] * c["bmax"] + pos[:, 2]] if len(pos) else \
            np.zeros((0, c["h"]), np.float32)
        np.testing.assert_array_equal(got, g[f"recvrows{r}"])
        np.testing.assert_array_equal(res[r]["out"], g[f"out{r}"])
        _check_stats(res[r], g, r, LL_STAT_F, sfx="_leg")


@pytest.mark.parametrize("n", [1, 4])
def test_ll_legacy_layout_c2_hot_path(n):
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 256, 8, 7168, 32, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(256, n, 32, 8, 7168, seed=40 + n)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, mode="bf16", wire_out=True,
                 bf16_expert=True, layout="legacy", rounds=3)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale, bf16_expert=True)
    for rnd in range(3):
        _check_ll(cfg, [res[r][rnd] for r in range(n)], d, comb)


@pytest.mark.parametrize("n,layout", [(1, "optimized"), (4, "optimized"), (4, "legacy")])
def test_ll_zero_copy_combine_pulls_from_window(n, layout):
    """EpConfig.expert_out_window (LL): expert outputs written into the
    registered [L, N*B, H] bf16 region; each home pulls its tokens' rows."""
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 64, 8, 2048, 32, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16,
                      expert_out_window=True)
    wl = owl.make_workload(64, n, 32, 8, 2048, seed=60 + n)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, mode="bf16", wire_out=True,
                 bf16_expert=True, layout=layout, zero_copy=True, rounds=3)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale, bf16_expert=True)
    for rnd in range(3):
        _check_ll(cfg, [res[r][rnd] for r in range(n)], d, comb)


def test_ll_legacy_window_is_the_reference_footprint():
    from oracle import layout as olay
    cfg = ep.EpConfig(ep.Algorithm.LL, 2, 2, 64, 8, 1024, 16, ep.Dtype.FP8, True)
    fabric = ep.Fabric(ep.NodeTopology(2, 2))

    def body(rank):
        out = {}
        for lay in ("optimized", "legacy"):
            g = ep.create_group(fabric, rank, cfg, layout=lay)
            out[lay] = g.buffer_bytes
            g.destroy()
        return out

    try:
        res = run_ranks(2, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()
    for lay in ("optimized", "legacy"):
        assert res[0][lay] == olay.ll_window_bytes(64, 2, 16, 8, 1024, "fp8", True, lay)
    assert res[0]["legacy"] > res[0]["optimized"]


@pytest.mark.parametrize("n,rpn", [(2, 2), (8, 8), (8, 2)])
def test_ht_dsv3_like_matches_oracle(n, rpn):
    cfg = make_cfg("ht", n, rpn, 64, 256, 8, 2048, "bf16")
    wl = owl.make_workload(64, n, 256, 8, 2048, seed=7)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 64, n, 2048, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, 64, n, rpn)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["m"], m)
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["origin"], dd[r]["origin"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


@pytest.mark.parametrize("n,rpn", [(1, 1), (2, 2), (8, 8), (8, 2)])
def test_ht_zero_copy_combine_pulls_from_window(n, rpn):
    """EpConfig.expert_out_window: expert rows written into the registered
    window region; the home ranks pull them (no push pass), bit-exact."""
    cfg = ep.EpConfig(ep.Algorithm.HT, n, rpn, 64, 8, 2048, 256, ep.Dtype.BF16, expert_out_window=True)
    wl = owl.make_workload(64, n, 256, 8, 2048, seed=17)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine, zero_copy=True)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 64, n, 2048, "bf16")
    ys = [bf16_round(oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine)) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, 64, n, rpn)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


@pytest.mark.parametrize("n,k", [(2, 4), (1, 4), (1, 10)])
@pytest.mark.parametrize("b", [1500, 4096])
def test_ht_multi_cta_routing_layout(b, n, k):
    """Batches over several 128-token chunks: emulated ranks (N=2) take the
    three-kernel layout (per-chunk histograms, column prefix, rebase); one
    rank (N=1) the fused open — one grid barrier for top-k <= 8, the
    two-barrier form above — same receive order and rows either way."""
    cfg = make_cfg("ht", n, n, 32, b, k, 256, "bf16")
    wl = owl.make_workload(32, n, b, k, 256, seed=21)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 32, n, 256, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_scale) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, 32, n, n)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["m"], m)
        np.testing.assert_array_equal(res[r]["q"], q)
        np.testing.assert_array_equal(res[r]["origin"], dd[r]["origin"])
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


def test_ht_open_beyond_coresident_chunks_uses_separate_launches():
    """More 128-token chunks than fit on the GPU at once (E=2048: one
    layout CTA per SM): the one-launch open is refused before any work and
    create_handle takes the separate layout / metadata launches."""
    n, e, b, k, h = 1, 2048, 20000, 2, 16
    cfg = make_cfg("ht", n, n, e, b, k, h, "bf16")
    wl = owl.make_workload(e, n, b, k, h, seed=41)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, n, h, "bf16")
    ys = [oht.apply_experts(dd[0]["rows"], dd[0]["origin"], owl.expert_scale)]
    comb = oht.combine(ys, wl.routing, wl.weights, e, n, n)
    np.testing.assert_array_equal(res[0]["m"], m)
    np.testing.assert_array_equal(res[0]["origin"], dd[0]["origin"])
    np.testing.assert_array_equal(res[0]["rows"], dd[0]["rows"])
    np.testing.assert_array_equal(res[0]["out"], comb[0])


# BASELINE configs[3] / [4] shapes: Mixtral (E=8, K=2, H=4096, one expert per
# rank at N=8) and Qwen3-MoE (E=128, K=8, H=4096, Zipf routing)
@pytest.mark.parametrize("n", [2, 8])
def test_ht_mixtral_shape(n):
    cfg = make_cfg("ht", n, n, 8, 256, 2, 4096, "bf16")
    wl = owl.make_workload(8, n, 256, 2, 4096, seed=31)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 8, n, 4096, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, 8, n, n)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


def test_ht_qwen3_shape_zipf():
    n = 2
    cfg = make_cfg("ht", n, n, 128, 256, 8, 4096, "bf16")
    wl = owl.make_zipf_workload(128, n, 256, 8, 4096, seed=32)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 128, n, 4096, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_scale) for r in range(n)]
    comb = oht.combine(ys, wl.routing, wl.weights, 128, n, n)
    for r in range(n):
        np.testing.assert_array_equal(res[r]["m"], m)
        np.testing.assert_array_equal(res[r]["rows"], dd[r]["rows"])
        np.testing.assert_array_equal(res[r]["out"], comb[r])


def test_ll_qwen3_shape_zipf_fp8_bf16():
    n = 2
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 128, 8, 4096, 64, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_zipf_workload(128, n, 64, 8, 4096, seed=33)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, mode="bf16", wire_out=True,
                 bf16_expert=True)
    d, comb = _ll_oracle(cfg, wl, owl.expert_scale, bf16_expert=True)
    _check_ll(cfg, res, d, comb)


def test_ht_bf16_expert_rows_are_exact():
    cfg = make_cfg("ht", 4, 4, 32, 64, 4, 512, "bf16")
    wl = owl.make_workload(32, 4, 64, 4, 512, seed=9)
    res = run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, bf16_expert=True)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, 32, 4, 512, "bf16")
    ys = [bf16_round(oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_scale)) for r in range(4)]
    comb = oht.combine(ys, wl.routing, wl.weights, 32, 4, 4)
    for r in range(4):
        np.testing.assert_array_equal(res[r]["out"], comb[r])


# ---------------------------------------------------------------------------
# API behaviour on the device
# ---------------------------------------------------------------------------


def _solo(algo="ll", **kw):
    cfg = make_cfg(algo, 1, 1, kw.get("e", 4), kw.get("b", 3), kw.get("k", 2), kw.get("h", 16))
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    return cfg, fab, ep.create_group(fab, 0, cfg)


@pytest.mark.parametrize("routing", [[[2, 2]], [[0, 7]], [[-1, 0]]])
def test_bad_routing_rejected_at_create_handle(routing):
    cfg, fab, g = _solo()
    with pytest.raises(ep.EpError) as ei:
        g.create_handle(np.array(routing))
    assert ei.value.code == ep.ErrorCode.INVALID_ARGUMENT
    g.destroy()


@pytest.mark.parametrize("bad", [-1, 99, "dup"])
def test_bad_routing_rejected_by_multi_cta_layout(bad):
    """HT create_handle with > 512 tokens (multi-CTA layout): an invalid
    row anywhere raises InvalidArgument, no fault."""
    cfg = make_cfg("ht", 1, 1, 16, 1000, 2, 16)
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    g = ep.create_group(fab, 0, cfg)
    r = np.tile(np.array([[0, 1]], np.int64), (1000, 1))
    if bad == "dup":
        r[777] = [5, 5]
    else:
        r[901, 1] = bad
    with pytest.raises(ep.EpError) as ei:
        g.create_handle(r)
    assert ei.value.code == ep.ErrorCode.INVALID_ARGUMENT
    g.destroy()


def test_too_many_tokens_and_shape_errors():
    cfg, fab, g = _solo()
    with pytest.raises(ep.EpError) as ei:
        g.create_handle(np.tile([0, 1], (4, 1)))
    assert ei.value.code == ep.ErrorCode.INVALID_ARGUMENT
    h = g.create_handle(np.array([[0, 1]]))
    with pytest.raises(ep.EpError) as ei:
        h.combine([], [])
    assert ei.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    bad = ep.tensor_create((2, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    out = ep.tensor_create((2, 3, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    cnt = ep.tensor_create((2, 1), ep.Dtype.F32, ep.TensorTag.RECV_EXPERT_COUNTER_HOST)
    with pytest.raises(ep.EpError) as ei:
        h.dispatch([bad], [out, cnt])
    assert ei.value.code == ep.ErrorCode.SHAPE_MISMATCH
    with pytest.raises(ep.EpError) as ei:
        h.dispatch([ep.tensor_create((1, 16), ep.Dtype.BF16, ep.TensorTag.TOKENS)], [out, cnt])
    assert ei.value.code == ep.ErrorCode.TAG_MISMATCH
    h.destroy()
    g.destroy()


def test_ht_combine_weights_must_match_dispatch():
    cfg = make_cfg("ht", 1, 1, 4, 3, 2, 16)
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    g = ep.create_group(fab, 0, cfg)
    h = g.create_handle(np.array([[0, 1], [2, 3]]))
    w = np.full((2, 2), 0.5, np.float32)
    tok = ep.tensor_from_f32(np.ones((2, 16), np.float32), ep.Dtype.F32, ep.TensorTag.TOKENS)
    total = h.get_num_recv_tokens()
    assert total == 4
    out = ep.tensor_create((total, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    cnt = ep.tensor_create((4, 1), ep.Dtype.F32, ep.TensorTag.TOKENS_PER_EXPERTS)
    h.dispatch([tok, ep.tensor_from_f32(w, ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)], [out, cnt])
    comb_out = ep.tensor_create((2, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    with pytest.raises(ep.EpError) as ei:
        h.combine([out, ep.tensor_from_f32(w * 2, ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)], [comb_out])
    assert ei.value.code == ep.ErrorCode.INVALID_ARGUMENT
    h.combine([out, ep.tensor_from_f32(w, ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)], [comb_out])
    np.testing.assert_array_equal(comb_out.read_f32(), np.ones((2, 16), np.float32))
    h.destroy()
    g.destroy()


def test_group_buffer_report_matches_footprint():
    from paper_2603_13606_b200.layout import MoeShape, SlotGeometry, footprint
    cfg = make_cfg("ll", 1, 1, 64, 128, 8, 7168)
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    g = ep.create_group(fab, 0, cfg)
    geom = SlotGeometry.for_config(7168, ep.Dtype.F32, 8, False)
    want = 2 * (64 * 8 + 64 * 8) + 2 * (1 * 128 * geom.dispatch_bytes) + 2 * 128 * 8 * geom.combine_bytes
    assert g.buffer_bytes == want
    assert g.physical_bytes >= g.buffer_bytes
    g.destroy()


def test_allocation_hooks_back_the_window():
    cfg = make_cfg("ll", 1, 1, 4, 3, 2, 16)
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    allocs, released = [], []

    def alloc(nbytes, align):
        t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        allocs.append((nbytes, align, t))
        return t

    g = ep.create_group(fab, 0, cfg, hooks=ep.AllocationHooks(alloc, released.append))
    assert allocs[0][1] == 256 and allocs[0][0] == g.physical_bytes
    h = g.create_handle(np.array([[0, 1], [2, 3]]))
    tok = ep.tensor_from_f32(np.ones((2, 16), np.float32), ep.Dtype.F32, ep.TensorTag.TOKENS)
    out = ep.tensor_create((4, 3, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    cnt = ep.tensor_create((4, 1), ep.Dtype.F32, ep.TensorTag.RECV_EXPERT_COUNTER_HOST)
    h.dispatch([tok], [out, cnt])
    import ctypes
    from paper_2603_13606_b200 import _lib
    win, nb = ctypes.c_void_p(), ctypes.c_uint64()
    _lib.call("epb_group_window", g._g, ctypes.byref(win), ctypes.byref(nb))
    assert win.value == allocs[0][2].data_ptr() and nb.value == allocs[0][0]  # the hook storage is the window
    comb = ep.tensor_create((2, 16), ep.Dtype.F32, ep.TensorTag.TOKENS)
    h.combine([out, ep.tensor_from_f32(np.ones((2, 2), np.float32), ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)], [comb])
    np.testing.assert_array_equal(comb.read_f32(), np.full((2, 16), 2.0, np.float32))
    h.destroy()
    g.destroy()
    assert released == [allocs[0][2]]


def test_host_buffers_round_trip():
    """Reference-style usage: inputs/outputs backed by host numpy arrays."""
    cfg = make_cfg("ll", 1, 1, 8, 4, 2, 32, "bf16")
    fab = ep.Fabric(ep.NodeTopology(1, 1))
    g = ep.create_group(fab, 0, cfg)
    wl = owl.make_workload(8, 1, 4, 2, 32, seed=2)
    h = g.create_handle(wl.routing[0])
    tok_host = ep.tensor_create((4, 32), ep.Dtype.BF16, ep.TensorTag.TOKENS, buffer=np.zeros(4 * 32, np.uint16))
    tok_host.write_f32(wl.tokens[0])
    out = ep.tensor_create((8, 4, 32), ep.Dtype.F32, ep.TensorTag.TOKENS, buffer=np.zeros(8 * 4 * 32, np.float32))
    cnt = ep.tensor_create((8, 1), ep.Dtype.F32, ep.TensorTag.RECV_EXPERT_COUNTER_HOST, buffer=np.zeros(8, np.float32))
    h.dispatch([tok_host], [out, cnt])
    assert out.data.device.type == "cpu"
    d, comb = _ll_oracle(cfg, wl, owl.expert_identity)
    np.testing.assert_array_equal(cnt.read_f32(), d[0]["counts"])
    np.testing.assert_array_equal(out.read_f32(), d[0]["recv"])
    w_host = ep.tensor_create((4, 2), ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS, buffer=wl.weights[0].copy())
    comb = ep.tensor_create((4, 32), ep.Dtype.F32, ep.TensorTag.TOKENS, buffer=np.zeros(4 * 32, np.float32))
    h.combine([out, w_host], [comb])
    np.testing.assert_array_equal(comb.read_f32(), comb_ref := comb.read_f32())
    np.testing.assert_array_equal(comb_ref, comb.data.numpy().reshape(4, 32))
    np.testing.assert_array_equal(comb_ref, _ll_oracle(cfg, wl, owl.expert_identity)[1][0])
    h.destroy()
    g.destroy()


@pytest.mark.parametrize("strict,mapped_in", [(True, False), (False, False), (True, True), (False, True)])
def test_ll_pinned_host_tokens_and_output_are_mapped(strict, mapped_in, monkeypatch):
    """C2 path with pinned host tokens and a pinned host combine output: the
    combine kernel writes the output in place over PCIe (api._HOST_MAPPED);
    with `mapped_in` the dispatch kernel also reads the tokens in place.
    Outputs are bit-identical to the all-device call."""
    from paper_2603_13606_b200 import api as _api
    monkeypatch.setattr(_api, "_HOST_MAPPED", True)
    monkeypatch.setattr(_api, "_HOST_MAPPED_IN", mapped_in)
    E, K, H, b = 256, 8, 7168, 128
    cfg = ep.EpConfig(ep.Algorithm.LL, 1, 1, E, K, H, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    g = ep.create_group(ep.Fabric(ep.NodeTopology(1, 1)), 0, cfg, strict=strict)
    wl = owl.make_workload(E, 1, b, K, H, seed=31)
    dev = torch.device("cuda", 0)
    T = ep.TensorTag
    x_d = torch.from_numpy(wl.tokens[0]).to(dev).to(torch.bfloat16)
    w_d = torch.from_numpy(wl.weights[0]).to(dev)
    topk = torch.from_numpy(wl.routing[0]).to(dev)
    y = torch.randn((E, b, H), device=dev).to(torch.bfloat16)
    outs = {}
    for where in ("device", "host"):
        x = x_d if where == "device" else x_d.cpu().pin_memory()
        out = torch.zeros((b, H), dtype=torch.bfloat16, device=dev)
        if where == "host":
            out = out.cpu().pin_memory()
        recv = torch.zeros((E, b, H), dtype=torch.uint8, device=dev)
        sc = torch.zeros((E, b, H // 128), dtype=torch.float32, device=dev)
        cnt = torch.zeros((E, 1), dtype=torch.float32, device=dev)
        h = g.create_handle(topk)
        h.dispatch([ep.tensor_from_torch(x, T.TOKENS)],
                   [ep.tensor_from_torch(recv, T.TOKENS), ep.tensor_from_torch(sc, T.SCALES),
                    ep.tensor_from_torch(cnt, T.RECV_EXPERT_COUNTER_DEVICE)])
        h.combine([ep.tensor_from_torch(y, T.TOKENS), ep.tensor_from_torch(w_d, T.TOPK_WEIGHTS)],
                  [ep.tensor_from_torch(out, T.TOKENS)])
        torch.cuda.synchronize()
        g.check()
        h.destroy()
        valid = cnt.cpu().numpy().astype(np.int64)[:, 0]
        rows = [recv[e, :valid[e]].cpu() for e in range(E)]
        scs = [sc[e, :valid[e]].cpu() for e in range(E)]
        outs[where] = (rows, scs, out.cpu())
    g.destroy()
    for a, c in zip(outs["device"][0] + outs["device"][1], outs["host"][0] + outs["host"][1]):
        assert torch.equal(a, c)
    assert torch.equal(outs["device"][2], outs["host"][2])
    assert outs["host"][2].abs().sum() > 0
