"""Test driver: run `fn(rank)` for every emulated rank of a single-GPU
`Fabric` concurrently, one worker thread per rank (the reference tests'
threads-as-ranks model, epsim harness.py:20-67, re-expressed on a thread
pool).  The first failing rank shuts the fabric down so every other rank's
blocking collective raises TransportClosed instead of hanging; the root
cause (not those secondary errors) is re-raised."""

from __future__ import annotations

import concurrent.futures as cf

import torch

import paper_2603_13606_b200 as ep


def run_ranks(num_ranks: int, fn, on_error=None, join_timeout: float = 300.0) -> list:
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None

    def on_rank(rank):
        if dev is not None:
            torch.cuda.set_device(dev)
        return fn(rank)

    pool = cf.ThreadPoolExecutor(max_workers=num_ranks, thread_name_prefix="rank")
    futs = {pool.submit(on_rank, r): r for r in range(num_ranks)}
    failures = []
    try:
        for fut in cf.as_completed(futs, timeout=join_timeout):
            if fut.exception() is not None:
                if not failures and on_error is not None:
                    on_error()
                failures.append(fut.exception())
    except cf.TimeoutError:
        if on_error is not None:
            on_error()
        hung = sorted(r for f, r in futs.items() if not f.done())
        raise RuntimeError(f"rank threads hung: {hung}") from None
    finally:
        pool.shutdown(wait=False)
    if failures:
        def secondary(e):
            return isinstance(e, ep.EpError) and e.code == ep.ErrorCode.TRANSPORT_CLOSED
        raise next((e for e in failures if not secondary(e)), failures[0])
    return [futs_r.result() for futs_r in sorted(futs, key=futs.get)]
