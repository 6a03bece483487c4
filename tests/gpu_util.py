"""Shared drivers for the GPU parity tests: run one dispatch -> expert stub ->
combine round through the public API on N ranks emulated on one GPU (one
host thread per rank, `Fabric`), mirroring epsim.driver.run_handle_round
(driver.py:143-179).  The expert stub and all expected values come from the
CPU oracle (test infrastructure)."""

from __future__ import annotations

import numpy as np
import torch

import paper_2603_13606_b200 as ep
from oracle import codecs as oc
from oracle import ht as oht
from oracle import ll as oll
from tests.rank_threads import run_ranks

DT = {"f32": ep.Dtype.F32, "bf16": ep.Dtype.BF16, "f16": ep.Dtype.F16, "fp8": ep.Dtype.FP8}


def make_cfg(algo, n, rpn, e, bmax, k, h, dtype="f32", scales=False):
    return ep.EpConfig(algorithm=ep.Algorithm(algo), num_ranks=n, ranks_per_node=rpn, num_experts=e,
                       top_k=k, hidden=h, max_tokens_per_rank=bmax, token_dtype=DT[dtype],
                       with_scales=scales)


def dispatch_inputs(cfg, tokens, weights, mode="reference"):
    """reference: tokens in the config dtype (+ SCALES from quantize_block),
    like epsim driver.dispatch_inputs (driver.py:71-88).  mode="bf16": bf16
    tokens and in-kernel quantisation (the north-star hot path)."""
    t = []
    if mode == "bf16":
        t.append(ep.tensor_from_f32(tokens, ep.Dtype.BF16, ep.TensorTag.TOKENS))
    elif mode == "f32":  # f32 tokens quantised by the dispatch kernel (FP8 configs)
        t.append(ep.tensor_from_f32(tokens, ep.Dtype.F32, ep.TensorTag.TOKENS))
    elif cfg.with_scales:
        codes, scales = oc.quantize_block(tokens)
        tok = ep.tensor_create(codes.shape, ep.Dtype.FP8, ep.TensorTag.TOKENS)
        tok.write_raw(codes)
        sc = ep.tensor_create(scales.shape, ep.Dtype.F32, ep.TensorTag.SCALES)
        sc.write_raw(scales)
        t += [tok, sc]
    else:
        t.append(ep.tensor_from_f32(tokens, cfg.token_dtype, ep.TensorTag.TOKENS))
    if cfg.algorithm is ep.Algorithm.HT:
        t.append(ep.tensor_from_f32(weights, ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS))
    return t


def run_ll(cfg, tokens, routing, weights, expert_fn, staged=False, mode="reference",
           wire_out=False, bf16_expert=False, rounds=1, layout="optimized", zero_copy=False, trace=None):
    """Returns per rank dict(recv, counts, out, recv_total).  `trace`: the
    fabric's op-trace sink."""
    n = cfg.num_ranks
    bmax, h = cfg.max_tokens_per_rank, cfg.hidden
    ell = cfg.experts_per_rank
    fabric = ep.Fabric(ep.NodeTopology(n, cfg.ranks_per_node), trace=trace)

    def body(rank):
        g = ep.create_group(fabric, rank, cfg, layout=layout)
        res = []
        try:
            for _ in range(rounds):
                hd = g.create_handle(routing[rank])
                inputs = dispatch_inputs(cfg, tokens[rank], weights[rank], mode)
                if wire_out:
                    out_tok = ep.tensor_create((ell, n * bmax, h), cfg.token_dtype, ep.TensorTag.TOKENS)
                    outs = [out_tok]
                    if cfg.with_scales:
                        out_sc = ep.tensor_create((ell, n * bmax, h // 128), ep.Dtype.F32, ep.TensorTag.SCALES)
                        outs.append(out_sc)
                else:
                    out_tok = ep.tensor_create((ell, n * bmax, h), ep.Dtype.F32, ep.TensorTag.TOKENS)
                    outs = [out_tok]
                out_cnt = ep.tensor_create((ell, n), ep.Dtype.F32, ep.TensorTag.RECV_EXPERT_COUNTER_HOST)
                outs.append(out_cnt)
                hd.dispatch(inputs, outs, send_only=staged)
                if staged:
                    hd.complete()
                counts = out_cnt.read_f32()
                if wire_out and cfg.with_scales:
                    recv = oc.dequantize_block(out_tok.raw(), outs[1].raw())
                else:
                    recv = out_tok.read_f32()
                rows = oll.apply_experts(recv, counts.astype(np.int64), rank, cfg.num_experts, n, bmax, expert_fn)
                ydt = ep.Dtype.BF16 if bf16_expert else ep.Dtype.F32
                if zero_copy:  # expert outputs written into the registered window region
                    yb = hd.expert_out_buffer()
                    yb.copy_(torch.from_numpy(rows).to(yb.device).to(torch.bfloat16))
                    yin = ep.tensor_from_torch(yb, ep.TensorTag.TOKENS)
                else:
                    yin = ep.tensor_from_f32(rows, ydt, ep.TensorTag.TOKENS)
                comb_in = [yin, ep.tensor_from_f32(weights[rank], ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)]
                comb_out = ep.tensor_create((routing[rank].shape[0], h), ep.Dtype.F32, ep.TensorTag.TOKENS)
                hd.combine(comb_in, [comb_out], send_only=staged)
                if staged:
                    hd.complete()
                raw = dict(recv_raw=out_tok.raw(), scales_raw=outs[1].raw()) if wire_out and cfg.with_scales else {}
                res.append(dict(recv=recv, counts=counts, out=comb_out.read_f32(), **raw,
                                recv_total=hd.get_num_recv_tokens(), rows=rows,
                                dstats=hd.dispatch_result.stats, cstats=hd.combine_stats))
                hd.destroy()
        finally:
            _teardown(g)
        return res if rounds > 1 else res[0]

    try:
        return run_ranks(n, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()


def run_ht(cfg, tokens, routing, weights, expert_fn, bf16_expert=False, zero_copy=False, trace=None):
    n = cfg.num_ranks
    h = cfg.hidden
    fabric = ep.Fabric(ep.NodeTopology(n, cfg.ranks_per_node), trace=trace)

    def body(rank):
        g = ep.create_group(fabric, rank, cfg)
        try:
            hd = g.create_handle(routing[rank])
            total = hd.get_num_recv_tokens()
            out_tok = ep.tensor_create((total, h), ep.Dtype.F32, ep.TensorTag.TOKENS)
            out_cnt = ep.tensor_create((cfg.experts_per_rank, n), ep.Dtype.F32, ep.TensorTag.TOKENS_PER_EXPERTS)
            hd.dispatch(dispatch_inputs(cfg, tokens[rank], weights[rank]), [out_tok, out_cnt])
            rows = out_tok.read_f32()
            res = hd.dispatch_result
            origin = res.origin.cpu().numpy().astype(np.int64)
            origin_w = res.origin_w.cpu().numpy()
            y = oht.apply_experts(rows, origin, expert_fn)
            ydt = ep.Dtype.BF16 if bf16_expert else ep.Dtype.F32
            if zero_copy:  # expert rows written into the registered window region
                yb = hd.expert_out_buffer()
                yb.copy_(torch.from_numpy(y).to(yb.device).to(torch.bfloat16))
                yin = ep.tensor_from_torch(yb, ep.TensorTag.TOKENS)
            else:
                yin = ep.tensor_from_f32(y, ydt, ep.TensorTag.TOKENS)
            comb_in = [yin, ep.tensor_from_f32(weights[rank], ep.Dtype.F32, ep.TensorTag.TOPK_WEIGHTS)]
            comb_out = ep.tensor_create((routing[rank].shape[0], h), ep.Dtype.F32, ep.TensorTag.TOKENS)
            hd.combine(comb_in, [comb_out])
            out = dict(rows=rows, origin=origin, origin_w=origin_w, counts=out_cnt.read_f32(),
                       out=comb_out.read_f32(), recv_total=total, m=res.meta_m, q=res.meta_q, y=y,
                       dstats=res.stats, cstats=hd.combine_stats)
            hd.destroy()
            return out
        finally:
            _teardown(g)

    try:
        return run_ranks(n, body, on_error=fabric.shutdown)
    finally:
        fabric.shutdown()


def _teardown(g):
    """Destroy a group even when a test body failed mid-round (the original
    exception must surface, not the live-handle complaint)."""
    for h in g._handles:
        h.state = ep.HandleState.DESTROYED
    if g.alive:
        g.destroy()


def bf16_round(x):
    return oc.bf16_to_f32(oc.f32_to_bf16(x))
