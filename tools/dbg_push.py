import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2603_13606_b200 as ep
from oracle import workload as owl
from tests.test_parity_bench_shapes import run_ht_device
for n, b, h, e, k in [(1, 4096, 7168, 256, 8), (2, 64, 7168, 256, 8), (2, 4096, 512, 256, 8), (2, 4096, 7168, 256, 8), (2, 1024, 7168, 256, 8)]:
    cfg = ep.EpConfig(ep.Algorithm.HT, n, n, e, k, h, b, ep.Dtype.BF16, expert_out_window=False)
    wl = owl.make_workload(e, n, b, k, h, seed=103)
    res = run_ht_device(cfg, wl, False)
    dev = res[0]['x'].device
    bad = []
    for s in range(n):
        rt = torch.from_numpy(wl.routing[s]).to(dev); w = torch.from_numpy(wl.weights[s]).to(dev)
        xf = res[s]['x'].float(); acc = None
        for kk in range(k):
            y = (xf * torch.exp2(((rt[:, kk] % 3) - 1).float())[:, None]).to(torch.bfloat16).float()
            p = w[:, kk:kk+1] * y; acc = p if acc is None else acc + p
        want = torch.zeros_like(acc) + acc
        got = res[s]['out']
        ne = (got != want)
        bad.append((int(ne.sum()), int(ne.any(1).sum()), int(ne.any(0).sum())))
    print(n, b, h, 'mismatches (elems, rows, cols) per rank:', bad, flush=True)
