"""Buffer-style wrapper (PAPER.md Table "Buffer operations")
against the oracle: wire-dtype outputs from the caching allocator, counts in
pinned mapped host memory, cached dispatch, comm stream and events."""

import numpy as np
import pytest
import torch

import paper_2603_13606_b200 as ep
from oracle import codecs as oc
from oracle import ht as oht
from oracle import ll as oll
from oracle import workload as owl
from tests.rank_threads import run_ranks

pytestmark = pytest.mark.gpu


def bf16r(x):
    return oc.bf16_to_f32(oc.f32_to_bf16(x))


def _run(n, body):
    fabric = ep.Fabric(ep.NodeTopology(n, n))
    try:
        return run_ranks(n, lambda r: body(fabric, r), on_error=fabric.shutdown)
    finally:
        fabric.shutdown()


@pytest.mark.parametrize("n", [1, 4])
def test_buffer_ll_c2_path_and_cached_dispatch(n):
    e, k, h, b = 256, 8, 7168, 32
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, e, k, h, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(e, n, b, k, h, seed=50 + n)
    wl.tokens = [bf16r(t) for t in wl.tokens]
    d = oll.dispatch(wl.tokens, wl.routing, e, n, b, h, "fp8", True)
    ys = [bf16r(oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, n, b, owl.expert_scale)) for r in range(n)]
    want = oll.combine(ys, wl.routing, wl.weights, e, n, b, h, "bf16")

    def body(fabric, r):
        dev = torch.device("cuda", 0)
        buf = ep.Buffer(fabric, r, cfg)
        x = torch.from_numpy(wl.tokens[r]).to(dev).to(torch.bfloat16)
        topk = torch.from_numpy(wl.routing[r]).to(dev)
        w = torch.from_numpy(wl.weights[r]).to(dev)
        y = torch.from_numpy(ys[r]).to(dev).to(torch.bfloat16)
        outs = []
        hd = None
        for _ in range(2):  # second round: cached dispatch on the same handle
            (rx, rs), ri, rw, hd, ev = buf.dispatch(x, topk, w, handle=hd)
            assert isinstance(ev, torch.cuda.Event) and rw is None
            assert rx.dtype == torch.uint8 and rs.dtype == torch.float32
            tpe = buf.get_tokens_per_expert_list()
            assert tpe == d[r]["counts"].sum(axis=1).tolist()
            np.testing.assert_array_equal(ri.cpu().numpy(), d[r]["counts"])
            plan = d[r]["plan"]
            if len(plan):
                idx = (plan[:, 0], plan[:, 1] * b + plan[:, 2])
                got = oc.dequantize_block(rx.cpu().numpy()[idx], rs.cpu().numpy()[idx])
                np.testing.assert_array_equal(got, d[r]["recv"][idx])
            out, ow, ev2 = buf.combine(y, hd, w)
            assert out.dtype == torch.bfloat16 and ow is w
            outs.append(out.float().cpu().numpy())
        buf.destroy_handle(hd)
        assert buf._counts_host.is_pinned()
        assert buf.get_comm_stream() is not None and isinstance(buf.capture(), torch.cuda.Event)
        buf.destroy()
        return outs

    res = _run(n, body)
    for r in range(n):
        for out in res[r]:
            np.testing.assert_array_equal(out, bf16r(want[r]))


@pytest.mark.parametrize("n", [2])
def test_buffer_ht_and_cached_dispatch(n):
    e, k, h, b = 32, 4, 512, 64
    cfg = ep.EpConfig(ep.Algorithm.HT, n, n, e, k, h, b, ep.Dtype.BF16)
    wl = owl.make_workload(e, n, b, k, h, seed=60)
    wl.tokens = [bf16r(t) for t in wl.tokens]
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, n, h, "bf16")
    ys = [bf16r(oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine)) for r in range(n)]
    want = oht.combine(ys, wl.routing, wl.weights, e, n, n)

    def body(fabric, r):
        dev = torch.device("cuda", 0)
        buf = ep.Buffer(fabric, r, cfg)
        x = torch.from_numpy(wl.tokens[r]).to(dev).to(torch.bfloat16)
        topk = torch.from_numpy(wl.routing[r]).to(dev)
        w = torch.from_numpy(wl.weights[r]).to(dev)
        outs = []
        hd = None
        for _ in range(2):
            rx, ri, rw, hd, ev = buf.dispatch(x, topk, w, handle=hd)
            assert rx.dtype == torch.bfloat16
            np.testing.assert_array_equal(rx.float().cpu().numpy(), dd[r]["rows"])
            np.testing.assert_array_equal(ri.cpu().numpy(), dd[r]["origin"][:, 0])
            np.testing.assert_array_equal(rw.cpu().numpy(), dd[r]["weights"])
            ell = cfg.experts_per_rank
            assert buf.get_tokens_per_expert_list() == m[:, r * ell:(r + 1) * ell].sum(axis=0).tolist()
            y = buf.get_expert_out_buffer(hd)  # zero-copy: expert rows written in the window
            y.copy_(torch.from_numpy(ys[r]).to(dev).to(torch.bfloat16))
            out, _, _ = buf.combine(y, hd, w, out_dtype=torch.float32)
            outs.append(out.cpu().numpy())
        buf.destroy_handle(hd)
        buf.destroy()
        return outs

    res = _run(n, body)
    for r in range(n):
        for out in res[r]:
            np.testing.assert_array_equal(out, want[r])
