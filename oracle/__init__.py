"""CPU oracle for the EP dispatch/combine hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in vectorised numpy, the algorithm of the reference
simulator `epsim` (arxiv 2603.13606 "NCCL EP" desk-scale model, mounted at
/root/reference/pkg/src/epsim) for exactly the functions on the hot path:

  codecs    E4M3 table/encoder/block quantisation, bf16/f16 codecs  (core.py:84-178)
  layout    MoeShape ownership, region sizes, footprints, header codec (layout.py, ll.py:58-121, ht.py:78-174)
  workload  seeded synthetic inputs                                  (oracle.py:32-45)
  ll        LL dispatch (counts, slot order, expert-major output, plan)
            and LL combine (wire rounding, ascending-k f32 sum)       (ll.py:227-507)
  ht        HT metadata, sorted 2D dispatch, hierarchical combine     (ht.py:291-740)

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU baseline.  The product path (`paper_2603_13606_b200`) never
imports it and fails loudly when its CUDA library is missing.

Parity pinning: `tests/golden/make_golden.py` runs the reference `epsim`
engines (importable in the build container) and stores their outputs as
fixtures under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against every fixture bit-for-bit, so parity is pinned.
"""

from . import codecs, layout, workload, ll, ht  # noqa: F401
