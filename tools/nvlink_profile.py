"""Diagnostics: NVLink byte counters of the EP kernels.  ncu profiles one
process, so the ranks here are threads of one process on two GPUs
(Fabric(devices=[0, 1]): peer windows through peer access, system-scope
ordering, send and receive phases as separate launches), each running
`--rounds` LL rounds (configs[1]: DeepSeek-V3, 128 tokens, FP8 dispatch /
bf16 combine) and HT rounds (configs[2]: 4096 tokens, bf16, tokens and expert
outputs in the registered window).  Outputs are checked against the oracle
on the first round (run it once without ncu before profiling).

    python tools/nvlink_profile.py
    ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,\\
dram__bytes_read.sum,dram__bytes_write.sum -k regex:"ll_|ht_" python tools/nvlink_profile.py --rounds 2
"""

import argparse
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_13606_b200 as ep  # noqa: E402
from oracle import workload as owl  # noqa: E402

T = ep.TensorTag


def ll_rank(fab, rank, n, rounds, out):
    cfg = ep.EpConfig(ep.Algorithm.LL, n, n, 256, 8, 7168, 128, ep.Dtype.FP8, True, combine_dtype=ep.Dtype.BF16)
    g = ep.create_group(fab, rank, cfg, strict=False)
    wl = owl.make_workload(256, n, 128, 8, 7168, 0)
    dev = torch.device("cuda", torch.cuda.current_device())
    L = cfg.experts_per_rank
    x = torch.from_numpy(wl.tokens[rank]).to(dev).to(torch.bfloat16)
    topk = torch.from_numpy(wl.routing[rank]).to(dev)
    w = torch.from_numpy(wl.weights[rank]).to(dev)
    recv = torch.zeros((L, n * 128, 7168), dtype=torch.uint8, device=dev)
    rsc = torch.zeros((L, n * 128, 56), dtype=torch.float32, device=dev)
    cnt = torch.zeros((L, n), dtype=torch.float32, device=dev)
    o = torch.zeros((128, 7168), dtype=torch.bfloat16, device=dev)
    outs = [ep.tensor_from_torch(recv, T.TOKENS), ep.tensor_from_torch(rsc, T.SCALES),
            ep.tensor_from_torch(cnt, T.RECV_EXPERT_COUNTER_DEVICE)]
    y = torch.zeros((L, n * 128, 7168), dtype=torch.bfloat16, device=dev)
    for rnd in range(rounds):
        h = g.create_handle(topk)
        h.dispatch([ep.tensor_from_torch(x, T.TOKENS)], outs)
        if rnd == 0:
            deq = recv.view(torch.float8_e4m3fn).float().view(L, n * 128, 56, 128) * rsc[..., None]
            eids = torch.arange(L, device=dev) + rank * L
            y.copy_((deq.view(L, n * 128, 7168) * bench.pow2_torch(eids)[:, None, None]).to(torch.bfloat16))
        h.combine([ep.tensor_from_torch(y, T.TOKENS), ep.tensor_from_torch(w, T.TOPK_WEIGHTS)],
                  [ep.tensor_from_torch(o, T.TOKENS)])
        h.destroy()
        if rnd == 0:
            g.check()
            st = type("S", (), {})()
            st.wl, st.E, st.H, st.b, st.world, st.rank = wl, 256, 7168, 128, n, rank
            st.recv, st.recv_sc, st.cnt, st.out = recv, rsc, cnt, o
            out[("ll", rank)] = bench.LLStep.parity(st)
    g.check()
    g.destroy()


def ht_rank(fab, rank, n, rounds, out):
    b = 4096
    cfg = ep.EpConfig(ep.Algorithm.HT, n, n, 256, 8, 7168, b, ep.Dtype.BF16, expert_out_window=True)
    g = ep.create_group(fab, rank, cfg, strict=False)
    wl = owl.make_workload(256, n, b, 8, 7168, 7)
    dev = torch.device("cuda", torch.cuda.current_device())
    xs = g.token_in_view(b)
    xs.copy_(torch.from_numpy(wl.tokens[rank]).to(dev).to(torch.bfloat16))
    topk = torch.from_numpy(wl.routing[rank]).to(dev)
    w = torch.from_numpy(wl.weights[rank]).to(dev)
    W = ep.tensor_from_torch(w, T.TOPK_WEIGHTS)
    cnt = torch.zeros((cfg.experts_per_rank, n), dtype=torch.float32, device=dev)
    o = torch.zeros((b, 7168), dtype=torch.bfloat16, device=dev)
    for rnd in range(rounds):
        h = g.create_handle(topk)
        tot = h.get_num_recv_tokens()
        rt = torch.zeros((tot, 7168), dtype=torch.bfloat16, device=dev)
        h.dispatch([ep.tensor_from_torch(xs, T.TOKENS), W],
                   [ep.tensor_from_torch(rt, T.TOKENS), ep.tensor_from_torch(cnt, T.TOKENS_PER_EXPERTS)])
        res = h.dispatch_result
        yw = h.expert_out_buffer()
        yw.copy_((rt.float() * bench.pow2_torch(res.origin[:, 0])[:, None]).to(torch.bfloat16))
        h.combine([ep.tensor_from_torch(yw, T.TOKENS), W], [ep.tensor_from_torch(o, T.TOKENS)])
        if rnd == 0:
            g.check()
            out[("ht", rank)] = bench.ht_parity(cfg, wl, rank, xs.clone(), rt, res.origin, res.origin_w, cnt, o,
                                                256, 8, 7168)
        h.destroy()
    g.check()
    g.destroy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--only", choices=["ll", "ht"], default=None)
    a = ap.parse_args()
    n = a.n
    out = {}
    for fn in [f for f in (ll_rank, ht_rank) if a.only is None or f.__name__.startswith(a.only)]:
        fab = ep.Fabric(ep.NodeTopology(n, n), devices=list(range(n)))
        errs = []

        def body(r):
            try:
                torch.cuda.set_device(r)
                fn(fab, r, n, a.rounds, out)
            except BaseException as ex:  # noqa: BLE001
                errs.append((r, ex))
                fab.shutdown()

        ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0][1]
    for k in sorted(out):
        print(k, out[k])
    assert all(v["ok"] for v in out.values())
    print("nvlink_profile: ok")


if __name__ == "__main__":
    main()
