"""Threads-as-ranks driver for emulated groups (epsim harness.py:20-67):
run fn(rank) on one host thread per rank over a single-GPU `Fabric`."""

from __future__ import annotations

import threading
import time

import torch

from .core import EpError, ErrorCode


def run_ranks(num_ranks: int, fn, on_error=None, join_timeout: float = 300.0):
    results = [None] * num_ranks
    errors = []
    lock = threading.Lock()
    device = torch.cuda.current_device() if torch.cuda.is_available() else None

    def body(rank):
        try:
            if device is not None:
                torch.cuda.set_device(device)
            results[rank] = fn(rank)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            with lock:
                first = not errors
                errors.append((rank, exc))
            if first and on_error is not None:
                on_error()

    threads = [threading.Thread(target=body, args=(r,), daemon=True, name=f"rank-{r}")
               for r in range(num_ranks)]
    for t in threads:
        t.start()
    deadline = time.monotonic() + join_timeout
    for t in threads:
        t.join(timeout=max(0.0, deadline - time.monotonic()))
    if any(t.is_alive() for t in threads):
        if on_error is not None:
            on_error()
        raise RuntimeError("rank threads hung: " + ", ".join(t.name for t in threads if t.is_alive()))
    if errors:
        real = [e for _, e in errors
                if not (isinstance(e, EpError) and e.code == ErrorCode.TRANSPORT_CLOSED)]
        raise (real[0] if real else errors[0][1])
    return results
