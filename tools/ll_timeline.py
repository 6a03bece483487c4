"""Diagnostics: where the time of one graph-replayed LL step goes.

    python tools/ll_timeline.py [--tokens 128] [--reps 5]

Captures  stamp -> dispatch -> stamp -> combine -> stamp  in one CUDA graph
(the LL kernels with per-CTA %globaltimer stamps on) and replays it after an
L2 flush, like bench.py.  A stamp is a 1-thread kernel writing the global
timer, so the gaps show the launch/drain cost each LL kernel pays outside its
CTAs' own first..last stamps.  Builds its stamp kernel with nvcc at run time.
"""

import argparse
import ctypes
import os
import subprocess
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_13606_b200 import _lib  # noqa: E402

STAMP_SRC = r"""
#include <cstdint>
#include <cuda_runtime.h>
__global__ void stamp_kernel(uint64_t* dst) {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); *dst = t;
}
extern "C" int stamp(uint64_t* dst, cudaStream_t s) { stamp_kernel<<<1, 1, 0, s>>>(dst); return (int)cudaGetLastError(); }
"""


def build_stamp():
    d = tempfile.mkdtemp()
    src, so = os.path.join(d, "stamp.cu"), os.path.join(d, "libstamp.so")
    open(src, "w").write(STAMP_SRC)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, src])
    lib = ctypes.CDLL(so)
    lib.stamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    return lib


def span(buf):
    t = buf.cpu().numpy().astype(np.int64).reshape(-1, 16)
    v = t[t > 0]
    return (int(v.min()), int(v.max())) if len(v) else (0, 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    world, rank = bench.init_dist()
    lib = build_stamp()
    st = bench.LLStep(world, rank, a.tokens)
    g = st.g
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    marks = torch.zeros(8, dtype=torch.int64, device="cuda")
    tr_d = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    tr_c = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    for _ in range(5):
        st.step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        h = g.create_handle(st.topk)
        lib.stamp(ctypes.c_void_p(marks.data_ptr()), cs)
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_d.data_ptr()))
        h.dispatch([st.X], [st.RECV, st.RECV_SC, st.CNT])
        lib.stamp(ctypes.c_void_p(marks.data_ptr() + 8), cs)
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr_c.data_ptr()))
        h.combine([st.Y, st.W], [st.OUT])
        _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(0))
        lib.stamp(ctypes.c_void_p(marks.data_ptr() + 16), cs)
        h.destroy()
    torch.cuda.synchronize()
    rows = []
    for rep in range(a.reps + 1):
        tr_d.zero_()
        tr_c.zero_()
        marks.zero_()
        flush.zero_()
        g.device_barrier()
        graph.replay()
        torch.cuda.synchronize()
        m = marks.cpu().numpy().astype(np.int64)
        d0, d1 = span(tr_d)
        c0, c1 = span(tr_c)
        if rep:
            rows.append([d0 - m[0], d1 - d0, m[1] - d1, c0 - m[1], c1 - c0, m[2] - c1, m[2] - m[0]])
    if rank == 0:
        r = np.array(rows) / 1e3
        names = ["stamp0->disp CTA0", "disp CTA span", "disp end->stamp1", "stamp1->comb CTA0",
                 "comb CTA span", "comb end->stamp2", "stamp0->stamp2"]
        print(f"== {world} rank(s), {a.tokens} tokens, {a.reps} reps (us, median [min..max])")
        for i, n in enumerate(names):
            print(f"  {n:20s} {np.median(r[:, i]):7.2f}  [{r[:, i].min():6.2f} .. {r[:, i].max():6.2f}]")


if __name__ == "__main__":
    main()
