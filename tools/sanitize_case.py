"""A small workload for compute-sanitizer (racecheck / synccheck): LL
(fast path, general path, legacy layout, staged) and HT rounds on ranks
emulated on one GPU (N=1 and N=2), checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import workload as owl  # noqa: E402
from tests.gpu_util import make_cfg, run_ht, run_ll  # noqa: E402
from tests.test_gpu_parity import _check_ll, _ll_oracle  # noqa: E402


def main():
    os.environ.setdefault("EPB_TIMEOUT_MS", "120000")
    for n in (1, 2):
        # fast path (K <= 8, FP8 + scales), general path (K = 10), legacy layout
        for (e, k, h, b, dt, sc, layout) in ((16, 4, 256, 8, "fp8", True, "optimized"),
                                              (24, 10, 64, 6, "bf16", False, "optimized"),
                                              (16, 4, 128, 8, "bf16", False, "legacy")):
            cfg = make_cfg("ll", n, n, e, b, k, h, dt, sc)
            wl = owl.make_workload(e, n, b, k, h, seed=n + k)
            res = run_ll(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale, staged=(n == 2),
                         layout=layout)
            d, comb = _ll_oracle(cfg, wl, owl.expert_scale)
            _check_ll(cfg, res, d, comb)
            print(f"ll n={n} k={k} {dt} {layout}: ok", flush=True)
        cfg = make_cfg("ht", n, n, 16, 32, 4, 256, "bf16")
        wl = owl.make_workload(16, n, 32, 4, 256, seed=3)
        run_ht(cfg, wl.tokens, wl.routing, wl.weights, owl.expert_scale)
        print(f"ht n={n}: ok", flush=True)
    print("sanitize_case: ok")


if __name__ == "__main__":
    main()
