"""Parity at exactly the shapes and data paths bench.py times (BASELINE
configs[1]-[4]): ranks emulated on one B200, device tensors in the bench's
dtypes, checked against the CPU oracle.

* HT (configs[2], [3], [4]): 4096 tokens per rank, bf16 tokens in, bf16
  wire output (the bulk-copy receive), expert outputs written into the
  group's registered window (the pulled combine) or an ordinary tensor
  (pushed combine), f32 combine output.  Every received row is checked
  bit-for-bit at the position the oracle's index math (oracle/ht.py
  dispatch_plan: ht.py:185-193, :553-583) gives it, with its origin
  (e, src, t, k) and weight; the combine of every token is checked against
  the reference formula (single node: acc = p_0, acc += p_k ascending k,
  out = 0 + acc; ht.py:680-734) evaluated with IEEE f32 torch ops, and that
  evaluation is itself pinned to the numpy oracle (oracle.ht.combine) on a
  sub-workload of each rank's first tokens.
* LL (configs[1]): DeepSeek-V3 shapes at 8 ranks, 128 tokens, bf16 tokens
  quantised to FP8 + block scales inside the dispatch kernel, wire-dtype
  outputs, bf16 expert rows, bf16 combine wire — against oracle/ll.py.

The expert is x * 2^((e % 3) - 1): exact in bf16, so the expert outputs the
kernels combine are known exactly to the checker."""

import numpy as np
import pytest
import torch

import paper_2603_13606_b200 as ep
from oracle import ht as oht
from oracle import workload as owl
from tests.gpu_util import bf16_round, run_ll
from tests.rank_threads import run_ranks
from tests.test_gpu_parity import _check_ll, _ll_oracle

pytestmark = pytest.mark.gpu
T = ep.TensorTag


@pytest.fixture(scope="module", autouse=True)
def cuda_required():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def pow2_scale(e):
    return 2.0 ** ((np.asarray(e) % 3) - 1)


def expert_pow2(e, rows):
    return (rows * np.float32(pow2_scale(e))).astype(np.float32)


def run_ht_device(cfg, wl, zero_copy, zc_in=False):
    n, h = cfg.num_ranks, cfg.hidden
    ell = cfg.experts_per_rank
    fabric = ep.Fabric(ep.NodeTopology(n, cfg.ranks_per_node))
    dev = torch.device("cuda", torch.cuda.current_device())

    def body(rank):
        g = ep.create_group(fabric, rank, cfg)
        try:
            x = torch.from_numpy(wl.tokens[rank]).to(dev).to(torch.bfloat16)
            if zc_in:  # tokens written into the registered stage: peers read them in place
                xs = g.token_in_view(x.shape[0])
                xs.copy_(x)
                x = xs
            topk = torch.from_numpy(wl.routing[rank]).to(dev)
            w = torch.from_numpy(wl.weights[rank]).to(dev)
            hd = g.create_handle(topk)
            tot = hd.get_num_recv_tokens()
            recv = torch.empty((tot, h), dtype=torch.bfloat16, device=dev)
            cnt = torch.empty((ell, n), dtype=torch.float32, device=dev)
            W = ep.tensor_from_torch(w, T.TOPK_WEIGHTS)
            hd.dispatch([ep.tensor_from_torch(x, T.TOKENS), W],
                        [ep.tensor_from_torch(recv, T.TOKENS), ep.tensor_from_torch(cnt, T.TOKENS_PER_EXPERTS)])
            res = hd.dispatch_result
            sc = torch.exp2(((res.origin[:, 0].long() % 3) - 1).float())
            y = (recv.float() * sc[:, None]).to(torch.bfloat16)  # exact: power-of-two scale
            if zero_copy:
                yb = hd.expert_out_buffer()
                yb.copy_(y)
                yin = ep.tensor_from_torch(yb, T.TOKENS)
            else:
                yin = ep.tensor_from_torch(y, T.TOKENS)
            out = torch.empty((x.shape[0], h), dtype=torch.float32, device=dev)
            hd.combine([yin, W], [ep.tensor_from_torch(out, T.TOKENS)])
            torch.cuda.synchronize()
            r = dict(x=x.clone(), recv=recv, origin=res.origin.clone(), origin_w=res.origin_w.clone(), counts=cnt,
                     out=out, total=tot)
            hd.destroy()
            return r
        finally:
            for hh in list(g._handles):
                hh.state = ep.HandleState.DESTROYED
            if g.alive:
                g.destroy()

    try:
        return run_ranks(n, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()


def check_ht(cfg, wl, res, pin_tokens=48):
    n, e, k = cfg.num_ranks, cfg.num_experts, cfg.top_k
    dev = res[0]["x"].device
    xs = [r["x"] for r in res]
    for d in range(n):
        pl = oht.dispatch_plan(wl.routing, wl.weights, e, n, d)
        got = res[d]
        assert got["total"] == pl["recv_total"]
        np.testing.assert_array_equal(got["counts"].cpu().numpy(), pl["counts"])
        pos = torch.from_numpy(pl["pos"]).to(dev)
        origin = got["origin"].long()[pos].cpu().numpy()
        np.testing.assert_array_equal(origin[:, 0], pl["e"])
        np.testing.assert_array_equal(origin[:, 1], pl["src"])
        np.testing.assert_array_equal(origin[:, 2], pl["t"])
        np.testing.assert_array_equal(origin[:, 3], pl["k"])
        np.testing.assert_array_equal(got["origin_w"][pos].cpu().numpy(), pl["w"])
        for s in range(n):  # payload bits, row by row at the oracle positions
            sel = torch.from_numpy(np.nonzero(pl["src"] == s)[0]).to(dev)
            want = xs[s][torch.from_numpy(pl["t"]).to(dev)[sel]]
            assert torch.equal(got["recv"][pos[sel]].view(torch.int16), want.view(torch.int16)), (d, s)
    # combine: every token with the reference order in IEEE f32 torch ops
    assert cfg.ranks_per_node == n
    for s in range(n):
        rt = torch.from_numpy(wl.routing[s]).to(dev)
        w = torch.from_numpy(wl.weights[s]).to(dev)
        xf = xs[s].float()
        acc = None
        for kk in range(k):
            y = (xf * torch.exp2(((rt[:, kk] % 3) - 1).float())[:, None]).to(torch.bfloat16).float()
            p = w[:, kk:kk + 1] * y
            acc = p if acc is None else acc + p
        want = torch.zeros_like(acc) + acc
        assert torch.equal(res[s]["out"].view(torch.int32), want.view(torch.int32)), s
    # the formula above against the numpy oracle on a sub-workload (each
    # token's combine depends only on its own rows)
    b = min(pin_tokens, wl.routing[0].shape[0])
    sub = owl.Workload([res[s]["x"][:b].float().cpu().numpy() for s in range(n)],
                       [wl.routing[s][:b] for s in range(n)], [wl.weights[s][:b] for s in range(n)])
    dd, _, _ = oht.dispatch(sub.tokens, sub.routing, sub.weights, e, n, cfg.hidden, "bf16")
    ys = [bf16_round(oht.apply_experts(dd[r]["rows"], dd[r]["origin"], expert_pow2)) for r in range(n)]
    comb = oht.combine(ys, sub.routing, sub.weights, e, n, cfg.ranks_per_node)
    for s in range(n):
        np.testing.assert_array_equal(res[s]["out"][:b].cpu().numpy(), comb[s])


HT_CASES = {
    # name: (E, K, H, N, zipf)
    "C3_dsv3_n2": (256, 8, 7168, 2, False),
    "C3_dsv3_n8": (256, 8, 7168, 8, False),
    "C4_mixtral_n8": (8, 2, 4096, 8, False),
    "C5_qwen3_zipf_n8": (128, 8, 4096, 8, True),
}


@pytest.mark.parametrize("zero_copy", [True, False], ids=["pulled_combine", "pushed_combine"])
@pytest.mark.parametrize("case", list(HT_CASES))
def test_ht_bench_shape_4096_tokens(case, zero_copy):
    e, k, h, n, zipf = HT_CASES[case]
    b = 4096
    cfg = ep.EpConfig(ep.Algorithm.HT, n, n, e, k, h, b, ep.Dtype.BF16, expert_out_window=zero_copy)
    wl = (owl.make_zipf_workload if zipf else owl.make_workload)(e, n, b, k, h, seed=101 + n)
    res = run_ht_device(cfg, wl, zero_copy)
    check_ht(cfg, wl, res)


@pytest.mark.parametrize("n", [2, 8])
def test_ll_bench_path_dsv3_128_tokens(n):
    """configs[1]: bf16 tokens -> in-kernel FP8 + scales, wire outputs, bf16
    expert rows and combine wire, 128 tokens per rank."""
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 256, 8, 7168, 128, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(256, n, 128, 8, 7168, seed=200 + n)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, expert_pow2, mode="bf16", wire_out=True, bf16_expert=True)
    d, comb = _ll_oracle(cfg, wl, expert_pow2, bf16_expert=True)
    _check_ll(cfg, res, d, comb)


def test_ll_qwen3_zipf_n8():
    cfg = ep.EpConfig(ep.Algorithm.LL, 8, 8, 128, 8, 4096, 128, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_zipf_workload(128, 8, 128, 8, 4096, seed=207)
    wl.tokens = [bf16_round(t) for t in wl.tokens]
    res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, expert_pow2, mode="bf16", wire_out=True, bf16_expert=True)
    d, comb = _ll_oracle(cfg, wl, expert_pow2, bf16_expert=True)
    _check_ll(cfg, res, d, comb)


def test_ll_fp8_quantiser_at_midpoints():
    """In-kernel FP8 quantisation when x / scale lands exactly on, and within a
    few ulp of, every E4M3 rounding midpoint (the reference rounds ties to
    the smaller magnitude), plus tiny and signed-zero elements."""
    from oracle import codecs as oc
    h, b = 1024, 96
    rng = np.random.default_rng(5)
    mids = np.unique(np.abs(oc._MID.astype(np.float32)))
    mids = mids[(mids > 0) & (mids < 448)]
    rows = []
    for t in range(b):
        amax = np.float32(2.0 ** rng.integers(-20, 20)) * np.float32(rng.uniform(1, 2))
        scale = np.float32(amax / np.float32(448.0))
        q = rng.choice(mids, h)
        ulp = rng.integers(-3, 4, h).astype(np.int64)
        qv = (q.view(np.int32).astype(np.int64) + ulp).astype(np.int32).view(np.float32)
        x = (qv * scale).astype(np.float32) * rng.choice([-1, 1], h).astype(np.float32)
        x[rng.integers(0, h, 4)] = np.float32(-0.0)
        x[rng.integers(0, h, 4)] = np.float32(1e-35)
        x[::128] = amax  # every block's absmax, so each block's scale is `scale`
        rows.append(x)
    x = np.stack(rows).astype(np.float32)
    cfg = ep.EpConfig(ep.Algorithm.LL, 1, 1, 8, 2, h, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    routing = np.stack([np.array([t % 8, (t + 3) % 8]) for t in range(b)]).astype(np.int64)
    wts = np.ones((b, 2), np.float32)
    res = run_ll(cfg, [x], [routing], [wts], owl.expert_identity, mode="f32", wire_out=True, bf16_expert=True)
    d, comb = _ll_oracle(cfg, owl.Workload([x], [routing], [wts]), owl.expert_identity, bf16_expert=True)
    _check_ll(cfg, res, d, comb)
    # codes and scales bit for bit (signed zeros included)
    codes, scales = oc.quantize_block(x)
    plan = d[0]["plan"]  # (l, src, i, t, k)
    rows = (plan[:, 0], plan[:, 1] * b + plan[:, 2])
    np.testing.assert_array_equal(res[0]["recv_raw"][rows], codes[plan[:, 3]])
    np.testing.assert_array_equal(res[0]["scales_raw"][rows].view(np.uint32), scales[plan[:, 3]].view(np.uint32))
    assert (codes == 0x80).any() and (codes[:, 1:] != 0).any()


@pytest.mark.parametrize("n", [2, 8])
def test_ht_zero_copy_input_and_combine(n):
    """Tokens in the registered token stage (no stage copy) and expert
    outputs in the registered window: both directions zero-copy."""
    e, k, h, b = 256, 8, 7168, 4096
    cfg = ep.EpConfig(ep.Algorithm.HT, n, n, e, k, h, b, ep.Dtype.BF16, expert_out_window=True)
    wl = owl.make_workload(e, n, b, k, h, seed=121 + n)
    res = run_ht_device(cfg, wl, True, zc_in=True)
    check_ht(cfg, wl, res)
