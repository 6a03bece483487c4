"""The reference's API conformance suite (epsim tests/test_api.py and the HT
round rule of tests/test_ht.py:316-345) ported onto this API, on ranks
emulated on one B200: handle creation is local (LL) or collective (HT),
validation completes before any window traffic, staging / complete /
destroy rules, the one-open-round HT rule, handle reuse, and random walks
over the handle state machine (test_api.py:688-761).

"No traffic" is checked two ways: the group's count of enqueued entry
points that touch a window is unchanged, and the window bytes themselves
are unchanged (the window comes from allocation hooks, so the test holds it
as a tensor)."""

import numpy as np
import pytest
import torch

import paper_2603_13606_b200 as ep
from oracle import ht as oht
from oracle import ll as oll
from oracle import workload as owl
from tests.gpu_util import dispatch_inputs
from tests.rank_threads import run_ranks

pytestmark = pytest.mark.gpu

T = ep.TensorTag
S = ep.HandleState
LL, HT = ep.Algorithm.LL, ep.Algorithm.HT


@pytest.fixture(scope="module", autouse=True)
def cuda_required():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def make_cfg(algo=LL, n=2, rpn=1, e=8, b=4, k=2, h=16, dtype=ep.Dtype.F32, scales=False):
    return ep.EpConfig(algorithm=algo, num_ranks=n, ranks_per_node=rpn, num_experts=e, top_k=k, hidden=h,
                       max_tokens_per_rank=b, token_dtype=dtype, with_scales=scales)


class _Hooks:
    """Window from a torch tensor the test can inspect."""

    def __init__(self):
        self.buf = None

    def hooks(self):
        def alloc(nbytes, align):
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
            return self.buf
        return ep.AllocationHooks(allocate=alloc, release=lambda b: None)


def solo_group(algo=LL, **kw):
    cfg = make_cfg(algo=algo, n=1, rpn=1, **kw)
    fabric = ep.Fabric(ep.NodeTopology(1, 1))
    h = _Hooks()
    g = ep.create_group(fabric, 0, cfg, hooks=h.hooks())
    g._test_window = h
    return cfg, fabric, g


def teardown(g):
    for hd in list(g._handles):
        hd.state = S.DESTROYED
    g._handles.clear()
    g._ht_active = None
    if g.alive:
        g.destroy()


def on_ranks(cfg, fn):
    fabric = ep.Fabric(ep.NodeTopology(cfg.num_ranks, cfg.ranks_per_node))

    def body(rank):
        g = ep.create_group(fabric, rank, cfg)
        try:
            return fn(rank, g)
        finally:
            teardown(g)

    try:
        return run_ranks(cfg.num_ranks, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()


def dispatch_outputs(cfg, recv_total=None):
    """(TOKENS, counter) outputs of the reference forms (driver.py:91-103)."""
    ell, n = cfg.experts_per_rank, cfg.num_ranks
    if cfg.algorithm is HT:
        return (ep.tensor_create((recv_total, cfg.hidden), ep.Dtype.F32, T.TOKENS),
                ep.tensor_create((ell, n), ep.Dtype.F32, T.TOKENS_PER_EXPERTS))
    return (ep.tensor_create((ell, n * cfg.max_tokens_per_rank, cfg.hidden), ep.Dtype.F32, T.TOKENS),
            ep.tensor_create((ell, n), ep.Dtype.F32, T.RECV_EXPERT_COUNTER_HOST))


def window_snapshot(g):
    torch.cuda.synchronize()
    return g._test_window.buf.clone()


# ---------------------------------------------------------------------------
# handle creation (test_api.py:302-345)
# ---------------------------------------------------------------------------


def test_ll_handle_creation_is_local():
    cfg, fabric, g = solo_group()
    w0, t0 = window_snapshot(g), g.traffic
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    assert g.traffic == t0
    assert torch.equal(window_snapshot(g), w0)
    assert hd.state is S.CREATED
    hd.destroy()
    g.destroy()


def test_ht_handle_knows_recv_count_at_creation():
    cfg = make_cfg(algo=HT, n=2, rpn=1, e=4, b=3, k=2)
    wl = owl.make_workload(4, 2, 3, 2, cfg.hidden, seed=9)
    m = oht.meta(wl.routing, 4, 2)[0]

    def body(rank, g):
        hd = g.create_handle(wl.routing[rank])
        n = hd.get_num_recv_tokens()
        hd.destroy()  # round aborted collectively, never dispatched
        assert g._ht_active is None
        return n

    outs = on_ranks(cfg, body)
    assert outs == [oht.recv_total(m, r, 4, 2) for r in range(2)]


@pytest.mark.parametrize("bad", [np.array([[0, 0], [1, 2]]), np.array([[0, 9], [1, 2]]), np.array([[0, 1]] * 5),
                                 np.array([0, 1]), np.array([[0.5, 1.5]])],
                         ids=["repeated", "out_of_range", "over_capacity", "not_2d", "not_integral"])
@pytest.mark.parametrize("algo", [LL, HT])
def test_bad_routing_rejected_at_handle_creation(bad, algo):
    cfg, fabric, g = solo_group(algo=algo, e=4, b=3, k=2)
    with pytest.raises(ep.EpError) as err:
        g.create_handle(bad)
    assert err.value.code == ep.ErrorCode.INVALID_ARGUMENT
    assert g._ht_active is None
    g.check()  # the device error word was consumed by the rejection
    teardown(g)


# ---------------------------------------------------------------------------
# tag and shape validation, all before any traffic (test_api.py:350-426)
# ---------------------------------------------------------------------------


class TestTagValidation:
    def _staged(self, algo=LL):
        cfg, fabric, g = solo_group(algo=algo, e=4, b=3, k=2)
        hd = g.create_handle(np.array([[0, 1], [2, 3]]))
        tokens = np.random.default_rng(0).standard_normal((2, cfg.hidden)).astype(np.float32)
        weights = np.ones((2, 2), np.float32)
        inputs = dispatch_inputs(cfg, tokens, weights)
        outputs = list(dispatch_outputs(cfg, hd.get_num_recv_tokens() if algo is HT else None))
        return cfg, g, hd, inputs, outputs

    def _expect(self, hd, inputs, outputs, code):
        g = hd.group
        w0, t0, st = window_snapshot(g), g.traffic, hd.state
        with pytest.raises(ep.EpError) as err:
            hd.dispatch(inputs, outputs)
        assert err.value.code == code
        assert g.traffic == t0, "rejected dispatch enqueued window traffic"
        assert torch.equal(window_snapshot(g), w0), "rejected dispatch changed the window"
        assert hd.state is st
        teardown(g)

    @pytest.mark.parametrize("algo", [LL, HT])
    def test_missing_tag(self, algo):
        cfg, g, hd, inputs, outputs = self._staged(algo)
        self._expect(hd, [], outputs, ep.ErrorCode.TAG_MISMATCH)

    @pytest.mark.parametrize("algo", [LL, HT])
    def test_duplicate_tag(self, algo):
        cfg, g, hd, inputs, outputs = self._staged(algo)
        self._expect(hd, inputs + inputs, outputs, ep.ErrorCode.TAG_MISMATCH)

    def test_unexpected_tag(self):
        cfg, g, hd, inputs, outputs = self._staged()
        stray = ep.tensor_from_f32(np.zeros((2, 2), np.float32), ep.Dtype.F32, T.TOPK_WEIGHTS)
        self._expect(hd, inputs + [stray], outputs, ep.ErrorCode.TAG_MISMATCH)

    def test_wrong_dtype_is_tag_mismatch(self):
        cfg, g, hd, inputs, outputs = self._staged()
        wrong = ep.tensor_from_f32(np.zeros((2, cfg.hidden), np.float32), ep.Dtype.F16, T.TOKENS)
        self._expect(hd, [wrong], outputs, ep.ErrorCode.TAG_MISMATCH)

    def test_wrong_output_leading_dim_is_shape_mismatch(self):
        cfg, g, hd, inputs, outputs = self._staged()
        bad = ep.tensor_create((cfg.experts_per_rank + 1, cfg.num_ranks * cfg.max_tokens_per_rank, cfg.hidden),
                               ep.Dtype.F32, T.TOKENS)
        self._expect(hd, inputs, [bad, outputs[1]], ep.ErrorCode.SHAPE_MISMATCH)

    @pytest.mark.parametrize("algo", [LL, HT])
    def test_wrong_token_count_is_shape_mismatch(self, algo):
        cfg, g, hd, inputs, outputs = self._staged(algo)
        wrong = ep.tensor_from_f32(np.zeros((3, cfg.hidden), np.float32), ep.Dtype.F32, T.TOKENS)
        self._expect(hd, [wrong] + inputs[1:], outputs, ep.ErrorCode.SHAPE_MISMATCH)

    def test_ht_wrong_recv_shape_is_shape_mismatch(self):
        cfg, g, hd, inputs, outputs = self._staged(HT)
        bad = ep.tensor_create((hd.get_num_recv_tokens() + 1, cfg.hidden), ep.Dtype.F32, T.TOKENS)
        self._expect(hd, inputs, [bad, outputs[1]], ep.ErrorCode.SHAPE_MISMATCH)

    def test_combine_rejections_before_traffic(self):
        cfg, g, hd, inputs, outputs = self._staged()
        hd.dispatch(inputs, outputs)
        w0, t0 = window_snapshot(g), g.traffic
        rows = ep.tensor_from_f32(np.zeros(outputs[0].shape, np.float32), ep.Dtype.F32, T.TOKENS)
        wts = ep.tensor_from_f32(np.ones((2, 2), np.float32), ep.Dtype.F32, T.TOPK_WEIGHTS)
        out = ep.tensor_create((2, cfg.hidden), ep.Dtype.F32, T.TOKENS)
        for ins, outs, code in (
                ([rows], [out], ep.ErrorCode.TAG_MISMATCH),
                ([rows, wts, wts], [out], ep.ErrorCode.TAG_MISMATCH),
                ([rows, ep.tensor_from_f32(np.ones((3, 2), np.float32), ep.Dtype.F32, T.TOPK_WEIGHTS)], [out],
                 ep.ErrorCode.SHAPE_MISMATCH),
                ([rows, wts], [ep.tensor_create((2, cfg.hidden + 1), ep.Dtype.F32, T.TOKENS)],
                 ep.ErrorCode.SHAPE_MISMATCH)):
            with pytest.raises(ep.EpError) as err:
                hd.combine(ins, outs)
            assert err.value.code == code
        assert g.traffic == t0 and torch.equal(window_snapshot(g), w0)
        assert hd.state is S.DISPATCHED
        teardown(g)


def test_fp8_dispatch_without_scales_is_tag_mismatch():
    cfg, fabric, g = solo_group(e=4, b=2, k=2, h=256, dtype=ep.Dtype.FP8, scales=True)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    tokens = ep.tensor_create((2, cfg.hidden), ep.Dtype.FP8, T.TOKENS)
    t0 = g.traffic
    with pytest.raises(ep.EpError) as err:
        hd.dispatch([tokens], list(dispatch_outputs(cfg)))
    assert err.value.code == ep.ErrorCode.TAG_MISMATCH
    assert "SCALES" in err.value.detail.upper()
    assert g.traffic == t0
    teardown(g)


# ---------------------------------------------------------------------------
# staging (test_api.py:434-520)
# ---------------------------------------------------------------------------


def test_ht_rejects_staging_and_complete():
    cfg, fabric, g = solo_group(algo=HT, e=4, b=2, k=2)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    inputs = dispatch_inputs(cfg, np.ones((2, cfg.hidden), np.float32), np.ones((2, 2), np.float32))
    outputs = list(dispatch_outputs(cfg, hd.get_num_recv_tokens()))
    with pytest.raises(ep.EpError) as err:
        hd.dispatch(inputs, outputs, send_only=True)
    assert err.value.code == ep.ErrorCode.INVALID_ARGUMENT
    with pytest.raises(ep.EpError) as err:
        hd.complete()
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    teardown(g)


def test_complete_with_nothing_staged_is_state_error():
    cfg, fabric, g = solo_group()
    hd = g.create_handle(np.array([[0, 1]]))
    with pytest.raises(ep.EpError) as err:
        hd.complete()
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    teardown(g)


def _round_through(cfg, rank, hd, wl, expert_fn, send_only=False):
    """One dispatch -> expert -> combine over the tagged-tensor surface
    (epsim driver.run_handle_round, driver.py:143-179)."""
    recv = hd.get_num_recv_tokens() if cfg.algorithm is HT else None
    out_tok, out_cnt = dispatch_outputs(cfg, recv)
    hd.dispatch(dispatch_inputs(cfg, wl.tokens[rank], wl.weights[rank]), [out_tok, out_cnt], send_only=send_only)
    if send_only:
        hd.complete()
    if cfg.algorithm is HT:
        res = hd.dispatch_result
        rows = oht.apply_experts(out_tok.read_f32(), res.origin.cpu().numpy().astype(np.int64), expert_fn)
    else:
        rows = oll.apply_experts(out_tok.read_f32(), out_cnt.read_f32().astype(np.int64), rank, cfg.num_experts,
                                 cfg.num_ranks, cfg.max_tokens_per_rank, expert_fn)
    comb_in = [ep.tensor_from_f32(rows, ep.Dtype.F32, T.TOKENS),
               ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)]
    comb_out = ep.tensor_create((wl.routing[rank].shape[0], cfg.hidden), ep.Dtype.F32, T.TOKENS)
    hd.combine(comb_in, [comb_out], send_only=send_only)
    if send_only:
        hd.complete()
    return comb_out.read_f32()


def _ref_combine(cfg, wl, expert_fn):
    n, e = cfg.num_ranks, cfg.num_experts
    if cfg.algorithm is HT:
        d, _, _ = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, n, cfg.hidden, "f32")
        ys = [oht.apply_experts(d[r]["rows"], d[r]["origin"], expert_fn) for r in range(n)]
        return oht.combine(ys, wl.routing, wl.weights, e, n, cfg.ranks_per_node)
    b = cfg.max_tokens_per_rank
    d = oll.dispatch(wl.tokens, wl.routing, e, n, b, cfg.hidden, "f32", False)
    ys = [oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, n, b, expert_fn) for r in range(n)]
    return oll.combine(ys, wl.routing, wl.weights, e, n, b, cfg.hidden, "f32")


def test_two_handles_pipeline_like_sequential():
    """test_api.py:441-494: two LL handles staged back to back give the
    same bytes as two sequential rounds."""
    cfg = make_cfg(n=2, rpn=1, e=8, b=3, k=2)
    wls = [owl.make_workload(8, 2, 3, 2, cfg.hidden, seed=s) for s in (31, 32)]
    fn = owl.expert_scale

    def sequential(rank, g):
        outs = []
        for wl in wls:
            hd = g.create_handle(wl.routing[rank])
            outs.append(_round_through(cfg, rank, hd, wl, fn))
            hd.destroy()
        return outs

    def pipelined(rank, g):
        hs, staged = [], []
        for wl in wls:
            hd = g.create_handle(wl.routing[rank])
            out_tok, out_cnt = dispatch_outputs(cfg)
            hd.dispatch(dispatch_inputs(cfg, wl.tokens[rank], wl.weights[rank]), [out_tok, out_cnt],
                        send_only=True)
            hs.append(hd)
            staged.append((wl, out_tok, out_cnt))
        for hd in hs:
            hd.complete()
        outs = []
        for hd, (wl, out_tok, out_cnt) in zip(hs, staged):
            rows = oll.apply_experts(out_tok.read_f32(), out_cnt.read_f32().astype(np.int64), rank, 8, 2, 3, fn)
            comb_out = ep.tensor_create((3, cfg.hidden), ep.Dtype.F32, T.TOKENS)
            hd.combine([ep.tensor_from_f32(rows, ep.Dtype.F32, T.TOKENS),
                        ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)], [comb_out],
                       send_only=True)
            outs.append(comb_out)
        for hd in hs:
            hd.complete()
            hd.destroy()
        return [o.read_f32() for o in outs]

    seq = on_ranks(cfg, sequential)
    pipe = on_ranks(cfg, pipelined)
    for r in range(2):
        for i in range(2):
            np.testing.assert_array_equal(seq[r][i], pipe[r][i])
            np.testing.assert_array_equal(seq[r][i], _ref_combine(cfg, wls[i], fn)[r])


# ---------------------------------------------------------------------------
# handle reuse and teardown (test_api.py:527-660)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("algo", [LL, HT])
def test_training_step_reuses_handle_for_backward(algo):
    cfg = make_cfg(algo=algo, n=2, rpn=1, e=8, b=3, k=2)
    wl = owl.make_workload(8, 2, 3, 2, cfg.hidden, seed=41)
    ref = _ref_combine(cfg, wl, owl.expert_scale)

    def body(rank, g):
        hd = g.create_handle(wl.routing[rank])
        outs = [_round_through(cfg, rank, hd, wl, owl.expert_scale) for _ in range(2)]  # forward, backward
        hd.destroy()
        return outs

    outs = on_ranks(cfg, body)
    for r in range(2):
        np.testing.assert_allclose(outs[r][0], ref[r], rtol=1e-5)
        np.testing.assert_array_equal(outs[r][0], outs[r][1])


def test_destroy_rules_guard_rounds_in_flight():
    cfg, fabric, g = solo_group(e=4, b=2, k=2)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    tokens = np.random.default_rng(0).standard_normal((2, cfg.hidden)).astype(np.float32)
    inputs, outputs = dispatch_inputs(cfg, tokens, None), list(dispatch_outputs(cfg))
    hd.dispatch(inputs, outputs)
    for victim in (hd.destroy, g.destroy):  # mid-round; group with a live handle
        with pytest.raises(ep.EpError) as err:
            victim()
        assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    rows = ep.tensor_from_f32(np.zeros(outputs[0].shape, np.float32), ep.Dtype.F32, T.TOKENS)
    comb_in = [rows, ep.tensor_from_f32(np.ones((2, 2), np.float32), ep.Dtype.F32, T.TOPK_WEIGHTS)]
    comb_out = ep.tensor_create((2, cfg.hidden), ep.Dtype.F32, T.TOKENS)
    hd.combine(comb_in, [comb_out], send_only=True)
    with pytest.raises(ep.EpError) as err:
        hd.destroy()  # staged
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    hd.complete()
    hd.destroy()
    for again in (hd.destroy, lambda: hd.dispatch(inputs, outputs)):  # twice; use after destroy
        with pytest.raises(ep.EpError) as err:
            again()
        assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    g.destroy()
    assert fabric.registered_bytes(0) == 0
    for dead in (lambda: g.create_handle(np.array([[0, 1]])), g.destroy):
        with pytest.raises(ep.EpError) as err:
            dead()
        assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR


def test_ht_destroying_fresh_handles_frees_the_round():
    cfg = make_cfg(algo=HT, n=2, rpn=1, e=4, b=2, k=2)
    wl = owl.make_workload(4, 2, 2, 2, cfg.hidden, seed=13)
    ref = _ref_combine(cfg, wl, owl.expert_identity)

    def body(rank, g):
        first = g.create_handle(wl.routing[rank])
        first.destroy()  # round opened by creation is dropped collectively
        hd = g.create_handle(wl.routing[rank])
        out = _round_through(cfg, rank, hd, wl, owl.expert_identity)
        hd.destroy()
        return out

    outs = on_ranks(cfg, body)
    for r in range(2):
        np.testing.assert_allclose(outs[r], ref[r], rtol=1e-5)


def test_second_ht_handle_while_round_open_is_state_error():
    """test_api.py:631-643 and test_ht.py:316-329: one open round per group,
    from creation until the round's combine — including a round that has
    dispatched but not yet combined (its metadata rows are still in use)."""
    cfg, fabric, g = solo_group(algo=HT, e=4, b=2, k=2)
    first = g.create_handle(np.array([[0, 1]]))
    with pytest.raises(ep.EpError) as err:
        g.create_handle(np.array([[2, 3]]))
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    first.destroy()
    second = g.create_handle(np.array([[2, 3]]))  # now legal
    wl = owl.Workload([np.ones((1, cfg.hidden), np.float32)], [np.array([[2, 3]])], [np.ones((1, 2), np.float32)])
    out_tok, out_cnt = dispatch_outputs(cfg, second.get_num_recv_tokens())
    second.dispatch(dispatch_inputs(cfg, wl.tokens[0], wl.weights[0]), [out_tok, out_cnt])
    t0 = g.traffic
    with pytest.raises(ep.EpError) as err:  # dispatched, not combined: still open
        g.create_handle(np.array([[0, 1]]))
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    assert g.traffic == t0
    second.combine([out_tok, ep.tensor_from_f32(wl.weights[0], ep.Dtype.F32, T.TOPK_WEIGHTS)],
                   [ep.tensor_create((1, cfg.hidden), ep.Dtype.F32, T.TOKENS)])
    third = g.create_handle(np.array([[0, 1]]))  # combined: the next round may open
    with pytest.raises(ep.EpError) as err:  # and the reused handle cannot reopen while `third` is open
        second.dispatch(dispatch_inputs(cfg, wl.tokens[0], wl.weights[0]), [out_tok, out_cnt])
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    assert second.state is S.COMBINED
    third.destroy()
    second.destroy()
    ep.destroy_group(g)


def test_ll_recv_count_needs_completed_dispatch():
    cfg, fabric, g = solo_group(e=4, b=2, k=2)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    with pytest.raises(ep.EpError) as err:
        hd.get_num_recv_tokens()
    assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
    tokens = np.ones((2, cfg.hidden), np.float32)
    hd.dispatch(dispatch_inputs(cfg, tokens, None), list(dispatch_outputs(cfg)), send_only=True)
    with pytest.raises(ep.EpError):
        hd.get_num_recv_tokens()  # still staged
    hd.complete()
    assert hd.get_num_recv_tokens() == 4  # 2 tokens x k=2, all local
    teardown(g)


# ---------------------------------------------------------------------------
# state machine random walks (test_api.py:688-761)
# ---------------------------------------------------------------------------


def _walk_op(cfg, hd, op):
    b = hd.num_tokens
    if op in ("dispatch", "dispatch_staged"):
        inputs = dispatch_inputs(cfg, np.ones((b, cfg.hidden), np.float32), np.ones((b, cfg.top_k), np.float32))
        recv = hd.get_num_recv_tokens() if cfg.algorithm is HT else None
        hd.dispatch(inputs, list(dispatch_outputs(cfg, recv)), send_only=op.endswith("staged"))
    elif op in ("combine", "combine_staged"):
        shape = (hd.get_num_recv_tokens(), cfg.hidden) if cfg.algorithm is HT else \
            (cfg.experts_per_rank, cfg.num_ranks * cfg.max_tokens_per_rank, cfg.hidden)
        comb_in = [ep.tensor_from_f32(np.zeros(shape, np.float32), ep.Dtype.F32, T.TOKENS),
                   ep.tensor_from_f32(np.ones((b, cfg.top_k), np.float32), ep.Dtype.F32, T.TOPK_WEIGHTS)]
        hd.combine(comb_in, [ep.tensor_create((b, cfg.hidden), ep.Dtype.F32, T.TOKENS)],
                   send_only=op.endswith("staged"))
    elif op == "complete":
        hd.complete()
    elif op == "destroy":
        hd.destroy()


_LL_MODEL = {
    S.CREATED: {"dispatch": S.DISPATCHED, "dispatch_staged": S.DISPATCH_STAGED, "destroy": S.DESTROYED},
    S.DISPATCH_STAGED: {"complete": S.DISPATCHED},
    S.DISPATCHED: {"combine": S.COMBINED, "combine_staged": S.COMBINE_STAGED},
    S.COMBINE_STAGED: {"complete": S.COMBINED},
    S.COMBINED: {"dispatch": S.DISPATCHED, "dispatch_staged": S.DISPATCH_STAGED, "destroy": S.DESTROYED},
    S.DESTROYED: {},
}
_HT_MODEL = {
    S.CREATED: {"dispatch": S.DISPATCHED, "destroy": S.DESTROYED},
    S.DISPATCHED: {"combine": S.COMBINED},
    S.COMBINED: {"dispatch": S.DISPATCHED, "destroy": S.DESTROYED},
    S.DESTROYED: {},
}


@pytest.mark.parametrize("seed", range(4))
def test_ll_state_machine_random_walk(seed):
    cfg, fabric, g = solo_group(e=4, b=2, k=2)
    ops = ("dispatch", "dispatch_staged", "combine", "combine_staged", "complete", "destroy")
    rng = np.random.default_rng(seed)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    for _ in range(120):
        op = ops[rng.integers(len(ops))]
        legal = _LL_MODEL[hd.state]
        if op in legal:
            _walk_op(cfg, hd, op)
            assert hd.state is legal[op]
        else:
            before = hd.state
            with pytest.raises(ep.EpError) as err:
                _walk_op(cfg, hd, op)
            assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
            assert hd.state is before
        if hd.state is S.DESTROYED:
            hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    g.check()
    teardown(g)


@pytest.mark.parametrize("seed", range(2))
def test_ht_state_machine_random_walk(seed):
    cfg, fabric, g = solo_group(algo=HT, e=4, b=2, k=2)
    ops = ("dispatch", "combine", "complete", "destroy", "dispatch_staged")
    rng = np.random.default_rng(seed)
    hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    for _ in range(80):
        op = ops[rng.integers(len(ops))]
        legal = _HT_MODEL[hd.state]
        if op in legal:
            _walk_op(cfg, hd, op)
            assert hd.state is legal[op]
        else:
            with pytest.raises(ep.EpError) as err:
                _walk_op(cfg, hd, op)
            if op == "dispatch_staged" and hd.state in (S.CREATED, S.COMBINED):
                assert err.value.code == ep.ErrorCode.INVALID_ARGUMENT
            else:
                assert err.value.code == ep.ErrorCode.HANDLE_STATE_ERROR
        # the open round belongs to the handle until its combine / abort
        assert (g._ht_active is hd) == (hd.state in (S.CREATED, S.DISPATCHED) and hd.state is not S.DESTROYED)
        if hd.state is S.DESTROYED:
            hd = g.create_handle(np.array([[0, 1], [2, 3]]))
    g.check()
    teardown(g)
