"""Diagnostics: the LL step's device timeline inside a CUDA graph, as bench.py
times it (256 MB L2 flush, device barrier, create_handle + dispatch +
combine), from the kernels' per-CTA %globaltimer stamps.

    python tools/ll_graph_trace.py [--tokens 128] [--reps 5]
    torchrun --nproc-per-node 2 ... tools/ll_graph_trace.py

Prints per rank: dispatch span (first CTA start -> last stamp), the gap to
the combine's first CTA, the combine span, and the step (dispatch start ->
combine end), all on that GPU's clock.
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
from paper_2603_13606_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--push", action="store_true", help="expert outputs in an ordinary tensor (pushed combine)")
    a = ap.parse_args()
    world, rank = bench.init_dist()
    st = bench.LLStep(world, rank, a.tokens, zero_copy=not a.push)
    g = st.g
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tr_d = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    tr_c = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")

    def step():
        h = g.create_handle(st.topk)
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_d.data_ptr()))
        h.dispatch([st.X], [st.RECV, st.RECV_SC, st.CNT])
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_c.data_ptr()))
        h.combine([st.Y, st.W], [st.OUT])
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(0))
        h.destroy()

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        flush.zero_()
        g.device_barrier()
        step()
    torch.cuda.synchronize()
    rows = []
    for rep in range(a.reps + 2):
        tr_d.zero_()
        tr_c.zero_()
        bench.barrier(world)
        graph.replay()
        torch.cuda.synchronize()
        td = tr_d.view(-1, 16).cpu().numpy().astype(np.int64)
        tc = tr_c.view(-1, 16).cpu().numpy().astype(np.int64)
        d0 = td[:, 0][td[:, 0] > 0].min()
        c0 = tc[:, 0][tc[:, 0] > 0].min()
        if rep >= 2:
            rows.append(((td.max() - d0) / 1e3, (c0 - td.max()) / 1e3, (tc.max() - c0) / 1e3, (tc.max() - d0) / 1e3))
    if os.environ.get("LL_GRAPH_TRACE_STAMPS") and rank == 0:
        import ll_trace  # noqa: E402  (tools/)
        ll_trace.show("dispatch (last replay)", tr_d, ll_trace.DISP)
        ll_trace.show("combine (last replay)", tr_c, ll_trace.COMB)
    r = np.array(rows)
    med = np.median(r, axis=0)
    res = bench.allgather_f(float(med[3]), world)
    print(f"rank {rank}/{world} tokens {a.tokens}: dispatch span {med[0]:.2f} us, gap {med[1]:.2f} us, "
          f"combine span {med[2]:.2f} us, dispatch start -> combine end {med[3]:.2f} us "
          f"(all ranks: {[round(x, 2) for x in res]})", flush=True)
    bench.barrier(world)


if __name__ == "__main__":
    main()
