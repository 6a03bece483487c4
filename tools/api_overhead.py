"""Diagnostics: host-side cost of the public API per call, N=1.

    python tools/api_overhead.py

Times an eager LL step (create_handle + dispatch + combine + destroy,
device tensors, perf mode and strict mode) and an HT create_handle, then
prints the top functions of a cProfile of the perf-mode LL step.
"""

import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def timeit(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    torch.cuda.set_device(0)
    st = bench.LLStep(1, 0, 128)
    g = st.g
    for strict in (False, True):
        g.strict = strict
        print(f"LL eager step, strict={strict}: {timeit(st.step):8.1f} us per step")
    g.strict = False
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        st.step()
    t_issue = (time.perf_counter() - t0) / 200 * 1e6
    torch.cuda.synchronize()
    print(f"LL eager step, host issue time only (perf mode): {t_issue:8.1f} us per step")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        st.step()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)

    import paper_2603_13606_b200 as ep
    from oracle import workload as owl
    cfg = ep.EpConfig(ep.Algorithm.HT, 1, 1, 256, 8, 7168, 4096, ep.Dtype.BF16)
    hg = bench.make_group(1, 0, cfg, strict=True)
    wl = owl.make_workload(256, 1, 4096, 8, 7168, 7)
    topk = torch.from_numpy(wl.routing[0]).cuda()

    def handle():
        h = hg.create_handle(topk)
        h.destroy()
    print(f"HT create_handle + destroy (4096 tok): {timeit(handle, 50):8.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        handle()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)


if __name__ == "__main__":
    main()
