"""Multi-GPU parity worker: one process per GPU (torchrun), ProcessFabric
over NCCL for the bootstrap, CUDA-IPC peer windows for all token traffic.
Every rank runs LL and HT rounds through the public API and checks its own
outputs bit-for-bit against the CPU oracle (which computes every rank's
expected values from the same seeded workload).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tests/mp_worker.py
"""

import contextlib
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_13606_b200 as ep  # noqa: E402
from paper_2603_13606_b200 import api as _api  # noqa: E402
from oracle import codecs as oc  # noqa: E402
from oracle import ht as oht  # noqa: E402
from oracle import ll as oll  # noqa: E402
from oracle import workload as owl  # noqa: E402

T = ep.TensorTag


@contextlib.contextmanager
def host_mapped_input(on: bool):
    """Pinned host token inputs read in place by the dispatch kernel for the
    duration of the block (api._HOST_MAPPED_IN), restored on any exit."""
    prev = _api._HOST_MAPPED_IN
    _api._HOST_MAPPED_IN = bool(on)
    try:
        yield
    finally:
        _api._HOST_MAPPED_IN = prev


def bf16r(x):
    return oc.bf16_to_f32(oc.f32_to_bf16(x))


def ll_case(world, rank, e, k, h, bmax, dtype, scales, combine_dtype, seed, staged, mode, rounds=1,
            layout="optimized", zero_copy=False, host_io=False, ragged=False):
    cfg = ep.EpConfig(ep.Algorithm.LL, world, world, e, k, h, bmax, dtype, scales, combine_dtype=combine_dtype,
                      expert_out_window=zero_copy)
    fab = ep.ProcessFabric(ep.NodeTopology(world, world))
    g = ep.create_group(fab, rank, cfg, layout=layout)
    ell = cfg.experts_per_rank
    for rnd in range(rounds):
        wl = owl.make_workload(e, world, bmax, k, h, seed + rnd)
        if ragged:  # rank 0 routes no token, rank 1 a full batch, the rest part of one
            for r in range(world):
                keep = 0 if r == 0 else (bmax if r == 1 else (bmax * r) // (world + 1))
                wl.tokens[r], wl.routing[r], wl.weights[r] = (wl.tokens[r][:keep], wl.routing[r][:keep],
                                                              wl.weights[r][:keep])
        if mode == "bf16":
            wl.tokens = [bf16r(t) for t in wl.tokens]
        d = oll.dispatch(wl.tokens, wl.routing, e, world, bmax, h, dtype.value, scales)
        ys = [bf16r(oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, world, bmax, owl.expert_scale))
              for r in range(world)]
        want = oll.combine(ys, wl.routing, wl.weights, e, world, bmax, h, cfg.combine_wire.value)[rank]
        hd = g.create_handle(wl.routing[rank])
        if mode == "bf16" and host_io:  # pinned host tokens: staged H2D (even rounds), read in place (odd)
            xh = torch.from_numpy(wl.tokens[rank]).to(torch.bfloat16).pin_memory()
            inputs = [ep.tensor_from_torch(xh, T.TOKENS)]
        elif mode == "bf16":
            inputs = [ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.BF16, T.TOKENS)]
        elif scales:
            c, s = oc.quantize_block(wl.tokens[rank])
            tok = ep.tensor_create(c.shape, ep.Dtype.FP8, T.TOKENS)
            tok.write_raw(c)
            sc = ep.tensor_create(s.shape, ep.Dtype.F32, T.SCALES)
            sc.write_raw(s)
            inputs = [tok, sc]
        else:
            inputs = [ep.tensor_from_f32(wl.tokens[rank], dtype, T.TOKENS)]
        out = ep.tensor_create((ell, world * bmax, h), ep.Dtype.F32, T.TOKENS)
        cnt = ep.tensor_create((ell, world), ep.Dtype.F32, T.RECV_EXPERT_COUNTER_HOST)
        with host_mapped_input(host_io and rnd % 2 == 1):
            hd.dispatch(inputs, [out, cnt], send_only=staged)
            if staged:
                hd.complete()
        counts = cnt.read_f32()
        np.testing.assert_array_equal(counts, d[rank]["counts"])
        recv = out.read_f32()
        plan = d[rank]["plan"]
        if len(plan):
            idx = (plan[:, 0], plan[:, 1] * bmax + plan[:, 2])
            np.testing.assert_array_equal(recv[idx], d[rank]["recv"][idx])
        y = ys[rank]
        if zero_copy:
            yb = hd.expert_out_buffer()
            yb.copy_(torch.from_numpy(y).cuda().to(torch.bfloat16))
            yin = ep.tensor_from_torch(yb, T.TOKENS)
        else:
            yin = ep.tensor_from_f32(y, ep.Dtype.BF16, T.TOKENS)
        comb_in = [yin, ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)]
        b_me = wl.routing[rank].shape[0]
        if host_io:  # pinned host output: written by the combine kernel in place over PCIe
            comb_out = ep.tensor_from_torch(torch.zeros((b_me, h), dtype=torch.float32).pin_memory(), T.TOKENS)
        else:
            comb_out = ep.tensor_create((b_me, h), ep.Dtype.F32, T.TOKENS)
        hd.combine(comb_in, [comb_out], send_only=staged)
        if staged:
            hd.complete()
        np.testing.assert_array_equal(comb_out.read_f32(), want)
        hd.destroy()
    g.destroy()


def ll_pipelined(world, rank):
    """Two handles in flight (parities 0 and 1), ll.py:171-218."""
    e, k, h, b = 32, 4, 512, 16
    cfg = ep.EpConfig(ep.Algorithm.LL, world, world, e, k, h, b, ep.Dtype.BF16)
    fab = ep.ProcessFabric(ep.NodeTopology(world, world))
    g = ep.create_group(fab, rank, cfg)
    ell = cfg.experts_per_rank
    wls = [owl.make_workload(e, world, b, k, h, s) for s in (20, 21)]
    hds, outs = [], []
    for wl in wls:
        hd = g.create_handle(wl.routing[rank])
        out = ep.tensor_create((ell, world * b, h), ep.Dtype.F32, T.TOKENS)
        cnt = ep.tensor_create((ell, world), ep.Dtype.F32, T.RECV_EXPERT_COUNTER_HOST)
        hd.dispatch([ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.BF16, T.TOKENS)], [out, cnt], send_only=True)
        hds.append(hd)
        outs.append((out, cnt))
    for hd in hds:
        hd.complete()
    combs = []
    for wl, hd, (out, cnt) in zip(wls, hds, outs):
        y = oll.apply_experts(out.read_f32(), cnt.read_f32().astype(np.int64), rank, e, world, b, owl.expert_identity)
        co = ep.tensor_create((b, h), ep.Dtype.F32, T.TOKENS)
        hd.combine([ep.tensor_from_f32(y, ep.Dtype.F32, T.TOKENS),
                    ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)], [co], send_only=True)
        combs.append(co)
    for hd in hds:
        hd.complete()
    for wl, co in zip(wls, combs):
        d = oll.dispatch(wl.tokens, wl.routing, e, world, b, h, "bf16", False)
        ys = [oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, world, b, owl.expert_identity)
              for r in range(world)]
        want = oll.combine(ys, wl.routing, wl.weights, e, world, b, h, "bf16")[rank]
        np.testing.assert_array_equal(co.read_f32(), want)
    for hd in hds:
        hd.destroy()
    g.destroy()


def buffer_ll(world, rank):
    """Buffer wrapper, one process per GPU: own comm stream, pinned mapped
    counters, cached dispatch."""
    e, k, h, b = 256, 8, 7168, 64
    cfg = ep.EpConfig(ep.Algorithm.LL, world, world, e, k, h, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    wl = owl.make_workload(e, world, b, k, h, 70)
    wl.tokens = [bf16r(t) for t in wl.tokens]
    d = oll.dispatch(wl.tokens, wl.routing, e, world, b, h, "fp8", True)
    ys = [bf16r(oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, world, b, owl.expert_scale))
          for r in range(world)]
    want = oll.combine(ys, wl.routing, wl.weights, e, world, b, h, "bf16")[rank]
    buf = ep.Buffer(ep.ProcessFabric(ep.NodeTopology(world, world)), rank, cfg)
    x = torch.from_numpy(wl.tokens[rank]).cuda().to(torch.bfloat16)
    topk = torch.from_numpy(wl.routing[rank]).cuda()
    w = torch.from_numpy(wl.weights[rank]).cuda()
    y = torch.from_numpy(ys[rank]).cuda().to(torch.bfloat16)
    hd = None
    for _ in range(2):
        (rx, rs), ri, _, hd, _ = buf.dispatch(x, topk, w, handle=hd)
        assert buf.get_tokens_per_expert_list() == d[rank]["counts"].sum(axis=1).tolist()
        out, _, ev = buf.combine(y, hd, w)
        ev.synchronize()
        np.testing.assert_array_equal(out.float().cpu().numpy(), bf16r(want))
    buf.destroy_handle(hd)
    buf.destroy()


def ht_case(world, rank, rpn, e, k, h, b, seed, bf16_expert, zero_copy=False):
    cfg = ep.EpConfig(ep.Algorithm.HT, world, rpn, e, k, h, b, ep.Dtype.BF16, expert_out_window=zero_copy)
    fab = ep.ProcessFabric(ep.NodeTopology(world, rpn))
    g = ep.create_group(fab, rank, cfg)
    wl = owl.make_workload(e, world, b, k, h, seed)
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, world, h, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine) for r in range(world)]
    if bf16_expert:
        ys = [bf16r(y) for y in ys]
    want = oht.combine(ys, wl.routing, wl.weights, e, world, rpn)[rank]
    hd = g.create_handle(wl.routing[rank])
    tot = hd.get_num_recv_tokens()
    assert tot == dd[rank]["recv_total"], (tot, dd[rank]["recv_total"])
    out = ep.tensor_create((tot, h), ep.Dtype.F32, T.TOKENS)
    cnt = ep.tensor_create((cfg.experts_per_rank, world), ep.Dtype.F32, T.TOKENS_PER_EXPERTS)
    w = ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)
    hd.dispatch([ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.BF16, T.TOKENS), w], [out, cnt])
    np.testing.assert_array_equal(out.read_f32(), dd[rank]["rows"])
    np.testing.assert_array_equal(hd.dispatch_result.origin.cpu().numpy(), dd[rank]["origin"])
    ydt = ep.Dtype.BF16 if bf16_expert else ep.Dtype.F32
    co = ep.tensor_create((b, h), ep.Dtype.F32, T.TOKENS)
    if zero_copy:
        yb = hd.expert_out_buffer()
        yb.copy_(torch.from_numpy(ys[rank]).cuda().to(torch.bfloat16))
        hd.combine([ep.tensor_from_torch(yb, T.TOKENS), w], [co])
    else:
        hd.combine([ep.tensor_from_f32(ys[rank], ydt, T.TOKENS), w], [co])
    np.testing.assert_array_equal(co.read_f32(), want)
    hd.destroy()
    g.destroy()


def ht_ragged(world, rank):
    """HT in process mode with rank 0 routing no token and the others ragged
    (the one-launch open with one chunk on some ranks, several on others)."""
    e, k, h, bmax = 8 * world, 4, 512, 700
    cfg = ep.EpConfig(ep.Algorithm.HT, world, world, e, k, h, bmax, ep.Dtype.BF16)
    wl = owl.make_workload(e, world, bmax, k, h, 57)
    for r in range(world):
        keep = 0 if r == 0 else (bmax if r == 1 else 300 + 37 * r)
        wl.tokens[r], wl.routing[r], wl.weights[r] = wl.tokens[r][:keep], wl.routing[r][:keep], wl.weights[r][:keep]
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, world, h, "bf16")
    ys = [oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_affine) for r in range(world)]
    want = oht.combine(ys, wl.routing, wl.weights, e, world, world)[rank]
    g = ep.create_group(ep.ProcessFabric(ep.NodeTopology(world, world)), rank, cfg)
    hd = g.create_handle(wl.routing[rank])
    tot = hd.get_num_recv_tokens()
    assert tot == dd[rank]["recv_total"], (tot, dd[rank]["recv_total"])
    out = ep.tensor_create((tot, h), ep.Dtype.F32, T.TOKENS)
    cnt = ep.tensor_create((cfg.experts_per_rank, world), ep.Dtype.F32, T.TOKENS_PER_EXPERTS)
    w = ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)
    hd.dispatch([ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.BF16, T.TOKENS), w], [out, cnt])
    np.testing.assert_array_equal(out.read_f32(), dd[rank]["rows"])
    co = ep.tensor_create((wl.routing[rank].shape[0], h), ep.Dtype.F32, T.TOKENS)
    hd.combine([ep.tensor_from_f32(ys[rank], ep.Dtype.F32, T.TOKENS), w], [co])
    np.testing.assert_array_equal(co.read_f32(), want)
    hd.destroy()
    g.destroy()


def traced_rounds(world, rank):
    """The op trace in process mode (one GPU per rank, CUDA-IPC windows):
    every line this rank's kernels record is one it initiated, with the
    multiplicities the routing implies (tests/test_op_trace.py for the
    emulated form)."""
    e, k, h, b = 4 * world, 3, 512, 16
    wl = owl.make_workload(e, world, b, k, h, seed=77)
    for algo in ("ll", "ht"):
        lines = []
        fab = ep.ProcessFabric(ep.NodeTopology(world, world), trace=lines.append)
        if algo == "ll":
            cfg = ep.EpConfig(ep.Algorithm.LL, world, world, e, k, h, b, ep.Dtype.BF16)
        else:
            cfg = ep.EpConfig(ep.Algorithm.HT, world, world, e, k, h, b, ep.Dtype.BF16)
        g = ep.create_group(fab, rank, cfg)
        ell = cfg.experts_per_rank
        hd = g.create_handle(wl.routing[rank])
        x = ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.BF16, T.TOKENS)
        w = ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, T.TOPK_WEIGHTS)
        if algo == "ll":
            out = ep.tensor_create((ell, world * b, h), ep.Dtype.F32, T.TOKENS)
            cnt = ep.tensor_create((ell, world), ep.Dtype.F32, T.RECV_EXPERT_COUNTER_HOST)
            hd.dispatch([x], [out, cnt])
            y = ep.tensor_from_f32(out.read_f32(), ep.Dtype.BF16, T.TOKENS)
        else:
            tot = hd.get_num_recv_tokens()
            out = ep.tensor_create((tot, h), ep.Dtype.F32, T.TOKENS)
            cnt = ep.tensor_create((ell, world), ep.Dtype.F32, T.TOKENS_PER_EXPERTS)
            hd.dispatch([x, w], [out, cnt])
            y = ep.tensor_from_f32(out.read_f32(), ep.Dtype.BF16, T.TOKENS)
        hd.combine([y, w], [ep.tensor_create((b, h), ep.Dtype.F32, T.TOKENS)])
        hd.destroy()
        g.destroy()
        ops = [ln.split(",") for ln in lines]
        assert ops and all(int(o[1]) == rank for o in ops), "a record names another initiator"
        owners = [set(int(v) // ell for v in row) for row in wl.routing[rank]]
        for d in range(world):
            q = sum(d in os_ for os_ in owners)
            sig = [o for o in ops if o[0] == "signal" and int(o[2]) == d]
            if algo == "ll":
                rec_len = h * 2 + 4 * (2 + 2 * k)
                puts = [o for o in ops if o[0] == "put" and int(o[2]) == d and int(o[5]) == rec_len]
                assert len(puts) == (q if d != rank else 0), (algo, d, len(puts), q)
                if d != rank:
                    assert sum(int(o[7]) for o in sig) == 2 * 148 or os.environ.get("EPB_LL_CTAS"), (d, sig)
            else:
                gets = [o for o in ops if o[0] == "get" and int(o[2]) == d and int(o[5]) == h * 2]
                srcq = sum(rank in set(int(v) // ell for v in row) for row in wl.routing[d])
                assert len(gets) == srcq, (algo, d, len(gets), srcq)  # rows pulled from d's stage
                assert len([o for o in sig if int(o[6]) // world == 0]) == 1  # metadata tag to d


def ll_stress(world, rank, rounds, b=64):
    """`rounds` back-to-back LL rounds (C2 path: bf16 -> FP8 + scales, bf16
    combine) on one handle per round, every round checked bit-for-bit on the
    device against oracle-derived expectations; mismatches accumulate on the
    device and are read once at the end.  Run under EPB_CHAOS_NS the kernels
    sleep a random time before stores and releases (test_acceptance.py:286-292
    analogue: ordering must not depend on timing)."""
    e, k, h = 256, 8, 7168
    cfg = ep.EpConfig(ep.Algorithm.LL, world, world, e, k, h, b, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    fab = ep.ProcessFabric(ep.NodeTopology(world, world))
    g = ep.create_group(fab, rank, cfg, strict=False)
    wl = owl.make_workload(e, world, b, k, h, 90)
    wl.tokens = [bf16r(t) for t in wl.tokens]
    d = oll.dispatch(wl.tokens, wl.routing, e, world, b, h, "fp8", True)
    ys = [bf16r(oll.apply_experts(d[r]["recv"], d[r]["counts"], r, e, world, b, owl.expert_scale))
          for r in range(world)]
    want = torch.from_numpy(oll.combine(ys, wl.routing, wl.weights, e, world, b, h, "bf16")[rank]).cuda()
    ell = cfg.experts_per_rank
    codes, scales = oc.quantize_block(np.concatenate(wl.tokens))
    plan = d[rank]["plan"]
    rows = torch.from_numpy(plan[:, 0] * (world * b) + plan[:, 1] * b + plan[:, 2]).cuda()
    gtok = torch.from_numpy(plan[:, 1] * b + plan[:, 3]).cuda()  # source row in the concatenated batch
    want_codes = torch.from_numpy(codes).cuda()[gtok]
    want_scales = torch.from_numpy(scales).cuda()[gtok]
    want_cnt = torch.from_numpy(d[rank]["counts"].astype(np.float32)).cuda()
    x = torch.from_numpy(wl.tokens[rank]).cuda().to(torch.bfloat16)
    topk = torch.from_numpy(wl.routing[rank]).cuda()
    w = torch.from_numpy(wl.weights[rank]).cuda()
    y = torch.from_numpy(ys[rank]).cuda().to(torch.bfloat16)
    recv = torch.zeros((ell, world * b, h), dtype=torch.uint8, device="cuda")
    rsc = torch.zeros((ell, world * b, h // 128), dtype=torch.float32, device="cuda")
    cnt = torch.zeros((ell, world), dtype=torch.float32, device="cuda")
    out = torch.zeros((b, h), dtype=torch.float32, device="cuda")
    X, W, Y = ep.tensor_from_torch(x, T.TOKENS), ep.tensor_from_torch(w, T.TOPK_WEIGHTS), ep.tensor_from_torch(y, T.TOKENS)
    outs = [ep.tensor_from_torch(recv, T.TOKENS), ep.tensor_from_torch(rsc, T.SCALES),
            ep.tensor_from_torch(cnt, T.RECV_EXPERT_COUNTER_DEVICE)]
    OUT = ep.tensor_from_torch(out, T.TOKENS)
    bad = torch.zeros(4, dtype=torch.int64, device="cuda")
    for rnd in range(rounds):
        hd = g.create_handle(topk)
        hd.dispatch([X], outs, send_only=(rnd % 3 == 1))
        if rnd % 3 == 1:
            hd.complete()
        flat = recv.view(-1, h)
        bad[0] += (flat[rows] != want_codes).any(1).sum()
        bad[1] += (rsc.view(-1, h // 128)[rows] != want_scales).any(1).sum()
        bad[2] += (cnt != want_cnt).sum()
        hd.combine([Y, W], [OUT], send_only=(rnd % 3 == 2))
        if rnd % 3 == 2:
            hd.complete()
        bad[3] += (out.view(torch.int32) != want.view(torch.int32)).any(1).sum()
        hd.destroy()
        recv.zero_()
        out.zero_()
    g.check()
    res = bad.cpu().tolist()
    print(f"rank {rank}: ll stress {rounds} rounds, mismatching (rows, scale rows, counts, tokens) = {res}", flush=True)
    assert res == [0, 0, 0, 0], res
    g.destroy()


def ht_stress(world, rank, rounds):
    """HT rounds (4096 tokens would be slow in Python per round; 512 tokens,
    DeepSeek-like E=64, K=8, H=2048) under EPB_CHAOS_NS, bit-exact every
    round on the device."""
    e, k, h, b = 64, 8, 2048, 512
    cfg = ep.EpConfig(ep.Algorithm.HT, world, world, e, k, h, b, ep.Dtype.BF16, expert_out_window=True)
    fab = ep.ProcessFabric(ep.NodeTopology(world, world))
    g = ep.create_group(fab, rank, cfg, strict=False)
    wl = owl.make_workload(e, world, b, k, h, 91)
    wl.tokens = [bf16r(t) for t in wl.tokens]
    dd, m, q = oht.dispatch(wl.tokens, wl.routing, wl.weights, e, world, h, "bf16")
    ys = [bf16r(oht.apply_experts(dd[r]["rows"], dd[r]["origin"], owl.expert_scale)) for r in range(world)]
    want = torch.from_numpy(oht.combine(ys, wl.routing, wl.weights, e, world, world)[rank]).cuda()
    want_rows = torch.from_numpy(dd[rank]["rows"]).cuda().to(torch.bfloat16)
    x = torch.from_numpy(wl.tokens[rank]).cuda().to(torch.bfloat16)
    topk = torch.from_numpy(wl.routing[rank]).cuda()
    w = torch.from_numpy(wl.weights[rank]).cuda()
    y = torch.from_numpy(ys[rank]).cuda().to(torch.bfloat16)
    tot = dd[rank]["recv_total"]
    recv = torch.zeros((tot, h), dtype=torch.bfloat16, device="cuda")
    cnt = torch.zeros((cfg.experts_per_rank, world), dtype=torch.float32, device="cuda")
    out = torch.zeros((b, h), dtype=torch.float32, device="cuda")
    X, W = ep.tensor_from_torch(x, T.TOKENS), ep.tensor_from_torch(w, T.TOPK_WEIGHTS)
    outs = [ep.tensor_from_torch(recv, T.TOKENS), ep.tensor_from_torch(cnt, T.TOKENS_PER_EXPERTS)]
    OUT = ep.tensor_from_torch(out, T.TOKENS)
    bad = torch.zeros(2, dtype=torch.int64, device="cuda")
    for rnd in range(rounds):
        hd = g.create_handle(topk)
        hd.dispatch([X, W], outs)
        bad[0] += (recv.view(torch.int16) != want_rows.view(torch.int16)).any(1).sum()
        yb = hd.expert_out_buffer()
        yb.copy_(y)
        hd.combine([ep.tensor_from_torch(yb, T.TOKENS), W], [OUT])
        bad[1] += (out.view(torch.int32) != want.view(torch.int32)).any(1).sum()
        hd.destroy()
        recv.zero_()
        out.zero_()
    g.check()
    res = bad.cpu().tolist()
    print(f"rank {rank}: ht stress {rounds} rounds, mismatching (rows, tokens) = {res}", flush=True)
    assert res == [0, 0], res
    g.destroy()


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    os.environ.setdefault("EPB_TIMEOUT_MS", "20000")
    cases = [
        ("ll fp8+scales dsv3 b=64", lambda: ll_case(world, rank, 256, 8, 7168, 64, ep.Dtype.FP8, True, None, 1, False, "ref")),
        ("ll c2 hot path bf16->fp8 / bf16 comb", lambda: ll_case(world, rank, 256, 8, 7168, 128, ep.Dtype.FP8, True,
                                                                  ep.Dtype.BF16, 2, False, "bf16")),
        ("ll staged bf16 uneven", lambda: ll_case(world, rank, 3 * world + 1, 3, 256, 12, ep.Dtype.BF16, False, None,
                                                  3, True, "ref", rounds=3)),
        ("ll pipelined parities", lambda: ll_pipelined(world, rank)),
        ("ll zero-copy combine (pull) c2", lambda: ll_case(world, rank, 256, 8, 7168, 128, ep.Dtype.FP8, True,
                                                            ep.Dtype.BF16, 9, False, "bf16", rounds=3, zero_copy=True)),
        ("ll legacy layout c2 hot path", lambda: ll_case(world, rank, 256, 8, 7168, 64, ep.Dtype.FP8, True,
                                                          ep.Dtype.BF16, 6, False, "bf16", rounds=2, layout="legacy")),
        ("ll legacy layout staged uneven", lambda: ll_case(world, rank, 3 * world + 1, 3, 256, 12, ep.Dtype.BF16, False,
                                                            None, 7, True, "ref", rounds=3, layout="legacy")),
        ("ll c2 pinned host tokens + in-place host output", lambda: ll_case(
            world, rank, 256, 8, 7168, 128, ep.Dtype.FP8, True, ep.Dtype.BF16, 11, False, "bf16", rounds=2,
            host_io=True)),
        ("ll staged, pinned host output", lambda: ll_case(world, rank, 256, 8, 7168, 32, ep.Dtype.FP8, True,
                                                           ep.Dtype.BF16, 12, True, "bf16", rounds=2, host_io=True)),
        ("buffer wrapper ll c2 path", lambda: buffer_ll(world, rank)),
        ("ht bf16 single node", lambda: ht_case(world, rank, world, 64, 8, 2048, 256, 4, False)),
        ("ht zero-copy combine (pull)", lambda: ht_case(world, rank, world, 64, 8, 2048, 256, 8, True, zero_copy=True)),
        ("ht bf16 rpn=2 hierarchical order", lambda: ht_case(world, rank, max(1, world // 2), 32, 4, 512, 64, 5, True)),
        ("ht empty + ragged ranks", lambda: ht_ragged(world, rank)),
        ("ll c2 hot path, empty + ragged ranks", lambda: ll_case(world, rank, 256, 8, 7168, 128, ep.Dtype.FP8, True,
                                                                  ep.Dtype.BF16, 61, False, "bf16", rounds=2,
                                                                  ragged=True)),
        ("op trace ll + ht (process mode)", lambda: traced_rounds(world, rank)),
    ]
    stress = int(os.environ.get("EPB_MP_STRESS", "0"))
    if stress:
        cases = [(f"ll stress {stress} rounds (chaos {os.environ.get('EPB_CHAOS_NS', '0')} ns)",
                  lambda: ll_stress(world, rank, stress)),
                 (f"ll stress {max(1, stress // 2)} rounds, 2 tokens (chaos {os.environ.get('EPB_CHAOS_NS', '0')} ns)",
                  lambda: ll_stress(world, rank, max(1, stress // 2), b=2)),
                 (f"ht stress {max(1, stress // 20)} rounds (chaos {os.environ.get('EPB_CHAOS_NS', '0')} ns)",
                  lambda: ht_stress(world, rank, max(1, stress // 20)))]
    failures = []
    for name, fn in cases:
        try:
            fn()
            ok = 1
        except Exception:  # noqa: BLE001 - reported below
            ok = 0
            failures.append(name + "\n" + traceback.format_exc())
        t = torch.tensor([ok], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"[{'PASS' if t.item() else 'FAIL'}] N={world} {name}", flush=True)
    for f in failures:
        print(f"rank {rank} FAILURE: {f}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
