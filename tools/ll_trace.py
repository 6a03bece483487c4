"""Diagnostics: per-CTA %globaltimer stamps of the fused LL kernels.

    python tools/ll_trace.py [--tokens 128] [--reps 5]

Prints, for the dispatch and the combine kernel, each checkpoint's
(min, median, max) over CTAs in microseconds after the earliest CTA start.
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_13606_b200 import _lib  # noqa: E402

# stamp indices of ll_dispatch_kernel / ll_combine_kernel (csrc/ll.cu LL_STAMP)
DISP = ["start", "", "emitted", "tokens-done", "arrived", "recv", "first-src-seen", "recv-done", "rows-in",
        "quantised(w1)", "after-barrier"]
COMB = ["start", "prefix", "sent", "arrived", "recv", "fetched", "reduced", "srcs-seen"]


def show(name, buf, labels):
    t = buf.cpu().numpy().astype(np.int64).reshape(-1, 16)
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"-- {name}")
    for i, lab in enumerate(labels):
        col = t[:, i]
        col = col[col > 0]
        if len(col) == 0:
            continue
        d = (col - t0) / 1e3
        print(f"  {i} {lab:10s} n={len(col):4d}  min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flush", default="write", choices=["write", "read", "none"])
    a = ap.parse_args()
    world, rank = bench.init_dist()
    st = bench.LLStep(world, rank, a.tokens)
    g = st.g
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tr_d = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    tr_c = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        st.step()
    for rep in range(a.reps):
        tr_d.zero_()
        tr_c.zero_()
        if a.flush == "write":
            flush.zero_()
        elif a.flush == "read":
            flush.view(torch.int32).sum()
        bench.barrier(world)
        g.device_barrier()  # ranks start the step together (as bench.py does)
        h = g.create_handle(st.topk)
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_d.data_ptr()))
        h.dispatch([st.X], [st.RECV, st.RECV_SC, st.CNT])
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_c.data_ptr()))
        h.combine([st.Y, st.W], [st.OUT])
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(0))
        h.destroy()
        torch.cuda.synchronize()
        t0s = bench.allgather_f(float(tr_d.view(-1, 16)[:, 0][tr_d.view(-1, 16)[:, 0] > 0].min().item()), world)
        if rank == 0:
            print(f"== rep {rep} (rank 0 of {world}, L2 flush: {a.flush}); dispatch start per rank vs rank 0 "
                  f"(globaltimer, comparable only if the GPUs' timers agree): "
                  f"{[round((t - t0s[0]) / 1e3, 2) for t in t0s]} us")
            show("dispatch", tr_d, DISP)
            show("combine", tr_c, COMB)
            td = tr_d.view(-1, 16).cpu().numpy().astype(np.int64)
            tc = tr_c.view(-1, 16).cpu().numpy().astype(np.int64)
            d0 = td[:, 0][td[:, 0] > 0].min()
            c0 = tc[:, 0][tc[:, 0] > 0].min()
            print(f"  dispatch span {(td.max() - d0) / 1e3:.2f} us; combine starts {(c0 - d0) / 1e3:.2f} us after "
                  f"the dispatch start, ends {(tc.max() - d0) / 1e3:.2f} us after it")
        bench.barrier(world)


if __name__ == "__main__":
    main()
