"""The op trace: the reference fabric's per-op log (fabric.py:83-111,
186-201; line format put/signal/lsa_store,src,dst,window,offset,len,
signal_id,value,seq), here recorded by the transport kernels themselves.

CPU: the line format and the sinks (callable, file).  GPU: one traced round
of LL (pushed and pulled combine) and HT on emulated ranks, decoded like the
reference's own trace tests (test_ll.py:250-300 reads the counter signals
back out of the trace; test_ht.py:170-200 counts the puts of a stream):
every transfer the protocol implies appears exactly once per round with the
oracle's multiplicity, and every arrival adds up to the launch's grid."""

import os
from collections import Counter

import numpy as np
import pytest

import paper_2603_13606_b200 as ep
from oracle import workload as owl
from paper_2603_13606_b200.fabric import OP_GET, OP_PUT, OP_SIGNAL, TraceSink


def rec(op, src, dst, off=0, ln=0, sig=0, val=0, wid=0):
    w0 = op | (wid << 4) | (src << 8) | (dst << 20) | (sig << 32)
    return np.array([w0, off, ln, val], dtype=np.uint64)


def test_line_format_matches_reference_columns():
    assert TraceSink.format(rec(OP_PUT, 1, 3, off=4096, ln=1048), 7) == "put,1,3,0,4096,1048,,,7"
    assert TraceSink.format(rec(OP_GET, 2, 0, off=64, ln=512), 8) == "get,2,0,0,64,512,,,8"
    assert TraceSink.format(rec(OP_SIGNAL, 0, 5, off=8, ln=8, sig=11, val=148), 9) == "signal,0,5,,,,11,148,9"


def test_callable_sink_numbers_lines():
    lines = []
    sink = TraceSink(lines.append)
    sink.emit(np.stack([rec(OP_PUT, 0, 1, 16, 32), rec(OP_SIGNAL, 0, 1, sig=1, val=2)]))
    sink.emit(np.stack([rec(OP_GET, 1, 0, 0, 8)]), dropped=3)
    assert [ln.split(",")[-1] for ln in lines] == ["1", "2", "3"]
    assert lines[1].startswith("signal,0,1,")
    assert sink.dropped == 3


def test_file_sink(tmp_path):
    path = tmp_path / "ops.trace"
    sink = TraceSink(str(path))
    sink.emit(np.stack([rec(OP_PUT, 0, 1, 16, 32)]))
    sink.close()
    assert path.read_text().strip().split("\n") == ["put,0,1,0,16,32,,,1"]
    assert not TraceSink(None).active


# ---------------------------------------------------------------------------
# GPU: traced rounds
# ---------------------------------------------------------------------------

def _parse(lines):
    out = []
    for ln in lines:
        f = ln.split(",")
        out.append(dict(op=f[0], src=int(f[1]), dst=int(f[2]), off=int(f[4]) if f[4] else None,
                        len=int(f[5]) if f[5] else None, sig=int(f[6]) if f[6] else None,
                        val=int(f[7]) if f[7] else None, seq=int(f[8])))
    return out


def _grid():
    v = os.environ.get("EPB_LL_CTAS")
    return int(v) if v else 148


def _owner_sets(routing, ell):
    return [[set(int(e) // ell for e in row) for row in r] for r in routing]


@pytest.mark.gpu
@pytest.mark.parametrize("pulled", [False, True])
def test_ll_round_trace(pulled):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from tests.gpu_util import make_cfg, run_ll
    n, e, b, k, h = 3, 12, 6, 3, 256
    if pulled:  # expert outputs in the registered bf16 window region, pulled by the homes
        cfg = ep.EpConfig(ep.Algorithm.LL, n, n, e, k, h, b, ep.Dtype.F32, False, combine_dtype=ep.Dtype.BF16,
                          expert_out_window=True)
    else:
        cfg = make_cfg("ll", n, n, e, b, k, h)
    wl = owl.make_workload(e, n, b, k, h, seed=5)
    lines = []
    run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine, zero_copy=pulled, bf16_expert=pulled,
           trace=lines.append)
    ops = _parse(lines)
    assert [o["seq"] for o in ops] == list(range(1, len(ops) + 1))
    ell = cfg.experts_per_rank
    owners = _owner_sets(wl.routing, ell)
    rec_len = h * 4 + 4 * (2 + 2 * k)      # f32 row + header (t, K, ids, ranks)
    cnt_len = 4 * (ell + 1)                # count row: m per local expert, then q
    row_len = h * (2 if pulled else 4)     # combine row: bf16 window rows, or the f32 wire
    disp = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "put" and o["len"] == rec_len)
    cnt = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "put" and o["len"] == cnt_len)
    for s in range(n):
        for d in range(n):
            if s == d:
                assert disp[(s, d)] == 0 and cnt[(s, d)] == 0  # own rows never enter the window
                continue
            assert disp[(s, d)] == sum(d in os_ for os_ in owners[s]), (s, d)
            assert cnt[(s, d)] == 1
    # arrivals: dispatch counters (ids parity*N + src) and combine counters
    # (2N + parity*N + src) each add up to the grid once per round and pair
    sig = Counter()
    for o in ops:
        if o["op"] == "signal":
            assert o["sig"] % n == o["src"] and o["src"] != o["dst"]
            sig[("c" if o["sig"] >= 2 * n else "d", o["src"], o["dst"])] += o["val"]
    for s in range(n):
        for d in range(n):
            if s != d:
                assert sig[("d", s, d)] == _grid() and sig[("c", s, d)] == _grid(), (s, d)
    # combine: one transfer per (token, k) whose expert lives off the home
    kind = "get" if pulled else "put"
    comb = Counter((o["src"], o["dst"]) for o in ops if o["op"] == kind and o["len"] == row_len)
    other = "put" if pulled else "get"
    assert not any(o["op"] == other and o["len"] == row_len for o in ops)
    for home in range(n):
        for owner in range(n):
            if owner == home:
                continue
            want = int(sum((wl.routing[home] // ell == owner).sum(axis=1)))
            key = (home, owner) if pulled else (owner, home)
            assert comb[key] == want, (home, owner)


@pytest.mark.gpu
def test_ht_round_trace():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from tests.gpu_util import make_cfg, run_ht
    n, e, b, k, h = 3, 12, 7, 3, 256
    cfg = make_cfg("ht", n, n, e, b, k, h)
    wl = owl.make_workload(e, n, b, k, h, seed=9)
    lines = []
    run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_affine, trace=lines.append)
    ops = _parse(lines)
    ell = cfg.experts_per_rank
    owners = _owner_sets(wl.routing, ell)
    q = [[sum(d in os_ for os_ in owners[s]) for d in range(n)] for s in range(n)]
    meta_len = 4 * (e + n)
    meta = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "put" and o["len"] == meta_len)
    row_len = h * 4
    gets = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "get" and o["len"] == row_len)
    recs = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "put" and o["len"] not in (meta_len, row_len))
    pushes = Counter((o["src"], o["dst"]) for o in ops if o["op"] == "put" and o["len"] == row_len)
    sigs = Counter((o["sig"] // n, o["src"], o["dst"]) for o in ops if o["op"] == "signal")
    for s in range(n):
        for d in range(n):
            assert meta[(s, d)] == 1  # metadata row to every rank, itself included
            assert sigs[(0, s, d)] == 1  # its tag (round 0: parity 0)
            assert recs[(s, d)] == q[s][d]  # one record per (token, rank it touches)
            assert gets[(d, s)] == q[s][d]  # the receiver pulls each row once
            if s != d:
                assert sigs[(2, s, d)] == 1 and sigs[(3, s, d)] == 1  # dispatch / combine flags
                want = int(sum((wl.routing[d] // ell == s).sum(axis=1)))
                assert pushes[(s, d)] == want  # expert rows pushed to their tokens' homes
    flags = [o for o in ops if o["op"] == "signal" and o["sig"] // n == 2]
    for o in flags:
        assert o["val"] & 0xFFFFFFFF == q[o["src"]][o["dst"]]  # flag value carries the record count


@pytest.mark.gpu
@pytest.mark.filterwarnings("ignore:op trace")
def test_trace_ring_overflow_keeps_the_first_records_and_warns():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from tests.gpu_util import make_cfg
    n, e, b, k, h = 2, 8, 6, 2, 64
    cfg = make_cfg("ll", n, n, e, b, k, h)
    wl = owl.make_workload(e, n, b, k, h, seed=3)
    lines = []
    fabric = ep.Fabric(ep.NodeTopology(n, n), trace=lines.append, trace_capacity=3)
    from tests.rank_threads import run_ranks

    def body(rank):
        g = ep.create_group(fabric, rank, cfg)
        hd = g.create_handle(wl.routing[rank])
        out = ep.tensor_create((cfg.experts_per_rank, n * b, h), ep.Dtype.F32, ep.TensorTag.TOKENS)
        cnt = ep.tensor_create((cfg.experts_per_rank, n), ep.Dtype.F32, ep.TensorTag.RECV_EXPERT_COUNTER_HOST)
        hd.dispatch([ep.tensor_from_f32(wl.tokens[rank], ep.Dtype.F32, ep.TensorTag.TOKENS)], [out, cnt])
        y = ep.tensor_from_f32(out.read_f32(), ep.Dtype.F32, ep.TensorTag.TOKENS)
        w = ep.tensor_from_f32(wl.weights[rank], ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)
        hd.combine([y, w], [ep.tensor_create((b, h), ep.Dtype.F32, ep.TensorTag.TOKENS)])
        hd.destroy()
        g.destroy()

    try:
        run_ranks(n, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()
    assert fabric.trace.dropped > 0  # counted (and warned about) when a call overflows its ring
    assert lines and all(len(ln.split(",")) == 9 for ln in lines)
    assert [int(ln.split(",")[-1]) for ln in lines] == list(range(1, len(lines) + 1))
