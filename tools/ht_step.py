"""Run only the HT leg of bench.py (profiling helper).

    python tools/ht_step.py [--ht-tokens 4096] [--ht-steps 3]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ht-tokens", type=int, default=4096)
    ap.add_argument("--ht-steps", type=int, default=3)
    a = ap.parse_args()
    world, rank = bench.init_dist()
    res = bench.run_ht(a, world, rank)
    if rank == 0:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
