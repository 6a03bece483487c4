"""Generate golden fixtures by running the REFERENCE simulator (`epsim`).

Run in the build container, where the read-only reference is mounted:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference is imported from /root/reference/pkg/src and driven through its
own engine harness (`epsim.harness.run_ll_round` / `run_ht_round`) and codecs,
so every array stored here is the reference's output, not ours.  The GPU box
never runs this script (the reference is absent there); the tests only read
the committed .npz files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _epsim():
    sys.path.insert(0, REF)
    import epsim  # noqa: F401
    from epsim import core, harness, layout, oracle, ht, ll
    return core, harness, layout, oracle, ht, ll


LL_CASES = {
    # name: (n, rpn, e, bmax, b_used, k, h, dtype, scales, stub, seed)
    "ll_f32_n4": (4, 2, 8, 5, 5, 2, 16, "f32", False, "scale", 11),
    "ll_uneven": (4, 4, 10, 3, 3, 3, 16, "f32", False, "affine", 11),
    "ll_n1": (1, 1, 4, 3, 3, 2, 16, "f32", False, "scale", 2),
    "ll_fewer": (4, 2, 8, 8, 3, 2, 16, "f32", False, "identity", 4),
    "ll_bf16": (4, 2, 8, 4, 4, 2, 256, "bf16", False, "scale", 6),
    "ll_f16": (4, 2, 8, 4, 4, 2, 256, "f16", False, "scale", 6),
    "ll_fp8s": (4, 2, 8, 4, 4, 2, 256, "fp8", True, "scale", 6),
    "ll_fp8": (4, 2, 8, 4, 4, 2, 256, "fp8", False, "scale", 6),
    "ll_dsv3_tiny": (8, 8, 256, 4, 4, 8, 256, "fp8", True, "affine", 3),
    "ll_dsv3_bf16": (8, 8, 256, 6, 6, 8, 128, "bf16", False, "scale", 5),
}

HT_CASES = {
    # name: (n, rpn, e, b, k, h, dtype, stub, seed)
    "ht_f32_2node": (4, 2, 8, 5, 2, 16, "f32", "scale", 11),
    "ht_uneven": (4, 4, 10, 3, 3, 16, "f32", "affine", 11),
    "ht_bf16": (4, 2, 8, 4, 2, 32, "bf16", "scale", 23),
    "ht_node8": (8, 8, 16, 6, 4, 16, "f32", "affine", 3),
    "ht_4node": (8, 2, 16, 3, 4, 16, "f32", "scale", 7),
    "ht_n1": (1, 1, 4, 3, 2, 16, "f32", "scale", 1),
}


# issue-side accounting (ll.py:39-55, ht.py:57-74); fifo_stalls is
# scheduling-dependent and never compared
LL_STAT_FIELDS = ("bytes_put", "msgs", "signals", "slots_used", "buffer_bytes")
HT_STAT_FIELDS = ("bytes_put", "msgs", "signals", "slots_used", "buffer_bytes", "inter_node_msgs",
                  "intra_node_msgs")


def _stat_vec(st, fields):
    return np.array([getattr(st, f) for f in fields], dtype=np.int64)


def make_ll(core, harness, layout_mod, oracle, name, spec):
    n, rpn, e, bmax, b, k, h, dt, scales, stub, seed = spec
    cfg = core.EpConfig(algorithm=core.Algorithm.LL, num_ranks=n, ranks_per_node=rpn,
                        num_experts=e, top_k=k, hidden=h, max_tokens_per_rank=bmax,
                        token_dtype=core.Dtype(dt), with_scales=scales)
    shape = layout_mod.MoeShape(e, n, b, k, h)
    wl = oracle.make_workload(shape, seed)
    res = harness.run_ll_round(cfg, "optimized", wl, oracle.EXPERT_STUBS[stub], delay_seed=seed)
    out = dict(spec=np.array([n, rpn, e, bmax, b, k, h, int(scales), seed]),
               dtype=np.array(dt), stub=np.array(stub))
    for r in range(n):
        d = res.per_rank[r].dispatch
        rnd_plan = []
        # rebuild the plan the engine used: valid rows in (src, i) order per l
        ell = cfg.experts_per_rank
        rows = []
        for l in range(ell):
            for s in range(n):
                for i in range(int(d.counts[l, s])):
                    rows.append(d.recv[l, s * bmax + i])
                    rnd_plan.append((l, s, i))
        out[f"tokens{r}"] = wl.tokens[r]
        out[f"routing{r}"] = wl.routing[r]
        out[f"weights{r}"] = wl.weights[r]
        out[f"counts{r}"] = d.counts
        out[f"recvpos{r}"] = np.array(rnd_plan, dtype=np.int64).reshape(-1, 3)
        out[f"recvrows{r}"] = np.array(rows, dtype=np.float32).reshape(-1, h)
        out[f"out{r}"] = res.per_rank[r].tokens_out
        out[f"recv_total{r}"] = np.array(d.recv_total)
        out[f"dstats{r}"] = _stat_vec(d.stats, LL_STAT_FIELDS)
        out[f"cstats{r}"] = _stat_vec(res.per_rank[r].combine_stats, LL_STAT_FIELDS)
    # the legacy layout: same outputs (test_ll.py:307-317), its own stats
    leg = harness.run_ll_round(cfg, "legacy", wl, oracle.EXPERT_STUBS[stub], delay_seed=seed)
    for r in range(n):
        assert np.array_equal(leg.per_rank[r].tokens_out, res.per_rank[r].tokens_out)
        out[f"dstats_leg{r}"] = _stat_vec(leg.per_rank[r].dispatch.stats, LL_STAT_FIELDS)
        out[f"cstats_leg{r}"] = _stat_vec(leg.per_rank[r].combine_stats, LL_STAT_FIELDS)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def make_ht(core, harness, layout_mod, oracle, name, spec):
    n, rpn, e, b, k, h, dt, stub, seed = spec
    cfg = core.EpConfig(algorithm=core.Algorithm.HT, num_ranks=n, ranks_per_node=rpn,
                        num_experts=e, top_k=k, hidden=h, max_tokens_per_rank=b,
                        token_dtype=core.Dtype(dt))
    shape = layout_mod.MoeShape(e, n, b, k, h)
    wl = oracle.make_workload(shape, seed)
    res = harness.run_ht_round(cfg, wl, oracle.EXPERT_STUBS[stub], delay_seed=seed)
    out = dict(spec=np.array([n, rpn, e, b, k, h, seed]), dtype=np.array(dt),
               stub=np.array(stub))
    for r in range(n):
        d = res.per_rank[r].dispatch
        out[f"tokens{r}"] = wl.tokens[r]
        out[f"routing{r}"] = wl.routing[r]
        out[f"weights{r}"] = wl.weights[r]
        out[f"rows{r}"] = d.rows
        out[f"origin{r}"] = np.array([o[:4] for o in d.origin], dtype=np.int64).reshape(-1, 4)
        out[f"originw{r}"] = np.array([o[4] for o in d.origin], dtype=np.float32)
        out[f"out{r}"] = res.per_rank[r].tokens_out
        if r == 0:
            out["m"] = d.meta.tokens_per_expert
            out["q"] = d.meta.records_per_pair
        out[f"recv_total{r}"] = np.array(d.meta.recv_total)
        out[f"dstats{r}"] = _stat_vec(d.stats, HT_STAT_FIELDS)
        out[f"cstats{r}"] = _stat_vec(res.per_rank[r].combine_stats, HT_STAT_FIELDS)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def make_codecs(core, layout_mod, ll, ht):
    rng = np.random.default_rng(1234)
    rows = np.concatenate([
        rng.uniform(-3, 3, (6, 256)),
        rng.standard_normal((4, 256)) * 100,
        rng.uniform(-1e-3, 1e-3, (2, 256)),
    ]).astype(np.float32)
    rows[0, :128] = 0.0                                   # zero block
    rows[1, 5] = -0.0
    codes, scales = core.quantize_block(rows)
    deq = core.dequantize_block(codes, scales)
    # every exact midpoint between adjacent magnitudes, both signs, plus
    # random values over the whole range and beyond the clamp
    mag = core.E4M3_VALUES[:0x7F].astype(np.float64)
    mids = ((mag[:-1] + mag[1:]) / 2).astype(np.float32)
    xs = np.concatenate([mids, -mids, core.E4M3_VALUES[:0x7F], -core.E4M3_VALUES[:0x7F],
                         rng.uniform(-500, 500, 2000).astype(np.float32),
                         rng.uniform(-2.0 ** -6, 2.0 ** -6, 500).astype(np.float32),
                         np.float32([1e4, -1e4, 448.0, 464.0, 463.99, -0.0, 0.0])]).astype(np.float32)
    enc = core.encode_e4m3(xs)
    bf_in = rng.standard_normal(4096).astype(np.float32) * np.float32(1e3)
    bf_in[:4] = np.float32([1.00390625, 1.01171875, -2.5, 3.0e38])
    bf = core.f32_to_bf16(bf_in)
    hdr = layout_mod.encode_header(3, [5, 9], 4)
    hdr8 = layout_mod.encode_header(0, list(range(8)), 8)
    # frozen sizes: (e, n, rpn, b, k, h, dtype, scales)
    geo = []
    for (e, n, rpn, b, k, h, dt, sc) in [(8, 2, 1, 4, 4, 16, "f32", False),
                                         (64, 8, 8, 128, 8, 7168, "f32", False),
                                         (256, 8, 8, 128, 8, 7168, "fp8", True),
                                         (256, 8, 8, 128, 8, 7168, "bf16", False),
                                         (10, 4, 2, 3, 3, 16, "bf16", False),
                                         (512, 64, 8, 128, 8, 7168, "fp8", True)]:
            cfg = core.EpConfig(algorithm=core.Algorithm.LL, num_ranks=n, ranks_per_node=rpn,
                                num_experts=e, top_k=k, hidden=h, max_tokens_per_rank=b,
                                token_dtype=core.Dtype(dt), with_scales=sc)
            w_opt = ll.ll_regions(cfg, "optimized").window_bytes
            w_leg = ll.ll_regions(cfg, "legacy").window_bytes
            if dt != "fp8":
                hcfg = core.EpConfig(algorithm=core.Algorithm.HT, num_ranks=n, ranks_per_node=rpn,
                                     num_experts=e, top_k=k, hidden=h, max_tokens_per_rank=b,
                                     token_dtype=core.Dtype(dt))
                w_ht = ht.ht_regions(hcfg).window_bytes
            else:
                w_ht = -1
            geo.append([e, n, rpn, b, k, h, {"f32": 0, "bf16": 1, "f16": 2, "fp8": 3}[dt], int(sc),
                        w_opt, w_leg, w_ht])
    np.savez_compressed(os.path.join(HERE, "codecs.npz"), q_rows=rows, q_codes=codes,
                        q_scales=scales, q_deq=deq, e_x=xs, e_codes=enc,
                        table=core.E4M3_VALUES, bf_in=bf_in, bf_out=bf,
                        hdr=np.frombuffer(hdr, np.uint8), hdr8=np.frombuffer(hdr8, np.uint8),
                        geo=np.array(geo, dtype=np.int64))


def main():
    core, harness, layout_mod, oracle, ht, ll = _epsim()
    for name, spec in LL_CASES.items():
        make_ll(core, harness, layout_mod, oracle, name, spec)
    for name, spec in HT_CASES.items():
        make_ht(core, harness, layout_mod, oracle, name, spec)
    make_codecs(core, layout_mod, ll, ht)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
