"""Diagnostics: where the host wall time of an HT create_handle goes, N=1.

    python tools/ht_handle_profile.py

Times EpGroup.create_handle + destroy at the bench's C3 shape (E=256, K=8,
H=7168, 4096 tokens) back to back and after an idle gap (as bench.py times
it), then prints a torch.profiler table (host ops and the device kernels).
"""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import paper_2603_13606_b200 as ep
    from oracle import workload as owl
    torch.cuda.set_device(0)
    for strict in (False, True):
        cfg = ep.EpConfig(ep.Algorithm.HT, 1, 1, 256, 8, 7168, 4096, ep.Dtype.BF16, expert_out_window=True)
        g = bench.make_group(1, 0, cfg, strict=strict)
        wl = owl.make_workload(256, 1, 4096, 8, 7168, 7)
        topk = torch.from_numpy(wl.routing[0]).cuda()

        def handle():
            h = g.create_handle(topk)
            h.destroy()

        for _ in range(20):
            handle()
        torch.cuda.synchronize()
        ts = []
        for _ in range(100):
            t0 = time.perf_counter()
            h = g.create_handle(topk)
            ts.append(time.perf_counter() - t0)
            h.destroy()
        ts.sort()
        print(f"strict={strict} back-to-back create_handle: median {ts[50] * 1e6:.1f} us, min {ts[0] * 1e6:.1f}")
        ts = []
        for _ in range(30):
            torch.cuda.synchronize()
            time.sleep(0.002)
            t0 = time.perf_counter()
            h = g.create_handle(topk)
            ts.append(time.perf_counter() - t0)
            h.destroy()
        ts.sort()
        print(f"strict={strict} after 2 ms idle: median {ts[15] * 1e6:.1f} us, min {ts[0] * 1e6:.1f}")
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for _ in range(20):
                handle()
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=20))
        print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=12))
        if not strict:
            import ctypes

            import numpy as np

            from paper_2603_13606_b200 import _lib
            tr = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
            # checkpoints of ht_open_kernel (csrc/ht.cu OPEN_STAMP, block_hist8 / block_rank8)
            labels = ["start", "histograms", "barrier", "bases", "meta-sent", "ranked+", "meta-wait", "meta-recv",
                      "end", "", "pass1", "", "scanned", "ranked"]
            for rep in range(3):
                tr.zero_()
                torch.cuda.synchronize()
                time.sleep(0.002)
                _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(tr.data_ptr()))
                h = g.create_handle(topk)
                _lib.call("epb_group_set_trace", g._g, ctypes.c_void_p(0))
                h.destroy()
                t = tr.cpu().numpy().reshape(-1, 16)
                t0 = t[:, 0][t[:, 0] > 0].min()
                print(f"-- ht_open stamps, rep {rep} (us after the first CTA start: min / med / max over CTAs)")
                for i, lab in enumerate(labels):
                    col = t[:, i][t[:, i] > 0]
                    if len(col):
                        d = (col - t0) / 1e3
                        print(f"  {i} {lab:10s} n={len(col):3d} {d.min():7.2f} {np.median(d):7.2f} {d.max():7.2f}")
        g.destroy()


if __name__ == "__main__":
    main()
