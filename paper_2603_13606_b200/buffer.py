"""Buffer-style wrapper (PAPER.md §"Common Backend
Architecture", Table "Buffer operations"):

    recv_x, recv_i, recv_w, h, ev = buf.dispatch(x, topk_idx, topk_weights, handle)
    out, out_w, ev                = buf.combine(x, h, topk_weights)
    buf.get_tokens_per_expert_list(); buf.get_comm_stream(); buf.capture()
    buf.destroy_handle(h)

It adapts framework tensors to the tagged-tensor API (api.py) and owns what a
framework integration needs around it:

* the group window comes from the PyTorch caching allocator through the
  allocation hooks (api.py:43-55), kept in a map until release;
* outputs stay in the wire dtype (bf16 / FP8 + block scales for LL, bf16 for
  HT) and live in caching-allocator memory — no f32 widening copies; the
  expert output goes back to combine as bf16;
* per-expert token counts land in pinned, GPU-mapped host memory written by
  the dispatch kernel itself (LL) or from the metadata round (HT), so
  get_tokens_per_expert_list() needs no device-to-host copy;
* communication runs on a dedicated stream ordered after `previous_event`
  (default: the caller's current stream); each call returns an event on that
  stream and, unless async_finish, makes the caller's stream wait on it.

Cached dispatch (a training backward pass): pass an existing handle; LL
reuses its routing snapshot, HT opens a fresh metadata round for it.

Zero-copy HT combine: get_expert_out_buffer(handle) hands out the expert
output tensor inside the registered window; a combine on it is pulled by the
token owners over NVLink instead of pushed.
"""

from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import api
from .core import FP8_BLOCK, Algorithm, Dtype, EpConfig, EpError, ErrorCode, TensorTag, tensor_from_torch

_TORCH_TO_DTYPE = {torch.float32: Dtype.F32, torch.bfloat16: Dtype.BF16, torch.float16: Dtype.F16,
                   torch.uint8: Dtype.FP8}


class Buffer:
    """One rank's EP communication buffer over an EpGroup."""

    def __init__(self, fabric, rank: int, config: EpConfig, layout: str = "optimized", strict: bool = False,
                 zero_copy_combine: bool = True):
        if config.algorithm is Algorithm.HT and zero_copy_combine and not config.expert_out_window \
                and config.hidden % 8 == 0:
            config = dataclasses.replace(config, expert_out_window=True)
        self.config = config
        self.rank = rank
        self._allocs: dict = {}
        hooks = api.AllocationHooks(allocate=self._allocate, release=self._release)
        self.group = api.create_group(fabric, rank, config, hooks=hooks, layout=layout, strict=strict)
        dev = self.group.device
        # emulated ranks share the fabric's stream (cross-rank ordering on one
        # GPU); one process per GPU gets its own communication stream
        shared = getattr(fabric, "_stream", None)
        self._comm = shared if shared is not None else torch.cuda.Stream(device=dev)
        ell, n = config.experts_per_rank, config.num_ranks
        # pinned host memory is device-mapped under UVA: the dispatch kernel
        # stores the counts straight into it
        self._counts_host = torch.zeros((ell, n), dtype=torch.float32).pin_memory()
        self._last_handle: Optional[api.EpHandle] = None
        self._last_event: Optional[torch.cuda.Event] = None

    # -- allocator callbacks (PyTorch caching allocator) -------------------------
    def _allocate(self, nbytes: int, alignment: int):
        t = torch.empty(nbytes + alignment, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
        off = (-t.data_ptr()) % alignment
        view = t[off:off + nbytes]
        self._allocs[view.data_ptr()] = t
        return view

    def _release(self, buf) -> None:
        self._allocs.pop(buf.data_ptr() if isinstance(buf, torch.Tensor) else int(buf), None)

    # -- streams / events ---------------------------------------------------------
    def get_comm_stream(self) -> torch.cuda.Stream:
        return self._comm

    def capture(self) -> torch.cuda.Event:
        """An event recorded on the communication stream now."""
        ev = torch.cuda.Event()
        ev.record(self._comm)
        return ev

    def _enter(self, previous_event):
        if previous_event is not None:
            self._comm.wait_event(previous_event)
        else:
            self._comm.wait_stream(torch.cuda.current_stream())

    def _guard(self, inputs, outputs) -> None:
        """Caching-allocator stream bookkeeping: inputs made on the caller's
        stream are read on the communication stream, outputs allocated on
        the communication stream are consumed on the caller's stream — each
        must not be recycled before the other stream is done with it."""
        cur = torch.cuda.current_stream()
        if cur == self._comm:
            return
        for t in inputs:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(self._comm)
        for t in outputs:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(cur)

    def _leave(self, async_finish: bool) -> torch.cuda.Event:
        ev = self.capture()
        if not async_finish:
            torch.cuda.current_stream().wait_event(ev)
        return ev

    # -- dispatch / combine -----------------------------------------------------------
    def dispatch(self, x, topk_idx, topk_weights=None, handle: Optional[api.EpHandle] = None,
                 previous_event=None, async_finish: bool = False, x_scales=None):
        """Returns (recv_x, recv_i, recv_w, handle, event).

        LL: recv_x = [L, N*B, H] in the wire dtype — for FP8 with scales a
        tuple (codes uint8, scales f32 [L, N*B, H/128]); rows of (local
        expert l, source r) are recv_x[l, r*B : r*B + recv_i[l, r]];
        recv_i = counts int32 [L, N]; recv_w = None (LL weights are given at
        combine, api.py:489-491).  `x` may be bf16/f16/f32 (quantised in the
        kernel under an FP8 config) or uint8 FP8 codes with `x_scales`.
        HT: recv_x = [recv_total, H] sorted by (local expert, source, token);
        recv_i = expert id per row (int32); recv_w = weight per row (f32).
        """
        cfg = self.config
        g = self.group
        ht = cfg.algorithm is Algorithm.HT
        if ht and topk_weights is None:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "HT dispatch needs topk_weights")
        self._enter(previous_event)
        with torch.cuda.stream(self._comm):
            if handle is None:
                handle = g.create_handle(topk_idx)
            elif handle.state is api.HandleState.DESTROYED:
                raise EpError(ErrorCode.HANDLE_STATE_ERROR, "cached dispatch on a destroyed handle")
            dt = _TORCH_TO_DTYPE.get(x.dtype)
            if dt is None:
                raise EpError(ErrorCode.TAG_MISMATCH, f"dispatch x dtype {x.dtype}")
            inputs = [tensor_from_torch(x, TensorTag.TOKENS)]
            if x_scales is not None:
                inputs.append(tensor_from_torch(x_scales, TensorTag.SCALES))
            ell, n, h = cfg.experts_per_rank, cfg.num_ranks, cfg.hidden
            dev = g.device
            wire_t = cfg.token_dtype.torch_dtype
            if ht:
                w = topk_weights if topk_weights.dtype == torch.float32 else topk_weights.float()
                inputs.append(tensor_from_torch(w, TensorTag.TOPK_WEIGHTS))
                # a reused handle opens a fresh metadata round inside
                # dispatch; same routing, same receive count
                total = handle.get_num_recv_tokens()
                recv = torch.empty((total, h), dtype=wire_t, device=dev)
                outputs = [tensor_from_torch(recv, TensorTag.TOKENS),
                           tensor_from_torch(self._counts_host, TensorTag.TOKENS_PER_EXPERTS)]
                handle.dispatch(inputs, outputs)
                res = handle.dispatch_result
                recv_i = res.origin[:, 0].contiguous()
                recv_w = res.origin_w
                recv_x = recv
            else:
                bmax = cfg.max_tokens_per_rank
                recv = torch.empty((ell, n * bmax, h), dtype=wire_t, device=dev)
                outputs = [tensor_from_torch(recv, TensorTag.TOKENS),
                           tensor_from_torch(self._counts_host, TensorTag.RECV_EXPERT_COUNTER_HOST)]
                scales = None
                if cfg.with_scales:
                    scales = torch.empty((ell, n * bmax, h // FP8_BLOCK), dtype=torch.float32, device=dev)
                    outputs.append(tensor_from_torch(scales, TensorTag.SCALES))
                handle.dispatch(inputs, outputs)
                res = handle.dispatch_result
                recv_x = (recv, scales) if scales is not None else recv
                recv_i = res.counts
                recv_w = None
        self._guard((x, x_scales, topk_idx, topk_weights),
                    (recv_x if isinstance(recv_x, tuple) else (recv_x,)) + (recv_i, recv_w))
        self._last_handle = handle
        ev = self._leave(async_finish)
        self._last_event = ev
        return recv_x, recv_i, recv_w, handle, ev

    def combine(self, x, handle: api.EpHandle, topk_weights, previous_event=None, async_finish: bool = False,
                out_dtype=None):
        """Returns (out [b, H], out_w, event).  `x` is the expert output in
        the dispatch layout (LL [L, N*B, H], HT [recv_total, H]), bf16 or
        f32; `topk_weights` [b, K] (HT: must equal the dispatched weights,
        ht.py:605-609).  out_dtype defaults to x's dtype (bf16 or f32)."""
        cfg = self.config
        self._enter(previous_event)
        with torch.cuda.stream(self._comm):
            w = topk_weights if topk_weights.dtype == torch.float32 else topk_weights.float()
            odt = out_dtype or (x.dtype if x.dtype in (torch.bfloat16, torch.float32) else torch.float32)
            out = torch.empty((w.shape[0], cfg.hidden), dtype=odt, device=self.group.device)
            handle.combine([tensor_from_torch(x, TensorTag.TOKENS), tensor_from_torch(w, TensorTag.TOPK_WEIGHTS)],
                           [tensor_from_torch(out, TensorTag.TOKENS)])
        self._guard((x, topk_weights, w), (out,))
        ev = self._leave(async_finish)
        self._last_event = ev
        return out, topk_weights, ev

    def get_expert_out_buffer(self, handle: api.EpHandle) -> torch.Tensor:
        """HT: [recv_total, H] bf16 tensor in the registered window for the
        handle's expert outputs; combine(x=this tensor) is zero-copy."""
        return handle.expert_out_buffer()

    # -- counts --------------------------------------------------------------------------
    def get_tokens_per_expert_list(self) -> list:
        """Tokens received per local expert by the last dispatch (summed over
        sources), read from pinned mapped host memory after the dispatch's
        event completes — no device-to-host copy."""
        if self._last_handle is None:
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "no dispatch yet")
        if self._last_event is not None:
            self._last_event.synchronize()
        if self.config.algorithm is Algorithm.HT:
            m = self._last_handle.dispatch_result.meta_m
            ell = self.config.experts_per_rank
            lo = self.rank * ell
            hi = min(lo + ell, self.config.num_experts)
            out = np.zeros(ell, np.int64)
            out[:hi - lo] = m[:, lo:hi].sum(axis=0)
            return out.tolist()
        return self._counts_host.numpy().sum(axis=1).astype(np.int64).tolist()

    # -- lifetime -------------------------------------------------------------------------
    def destroy_handle(self, handle: api.EpHandle) -> None:
        if handle.state in (api.HandleState.DISPATCHED,):
            raise EpError(ErrorCode.HANDLE_STATE_ERROR, "combine before destroying a dispatched handle")
        handle.destroy()
        if self._last_handle is handle:
            self._last_handle = None

    def destroy(self) -> None:
        torch.cuda.current_stream().wait_stream(self._comm)
        self.group.destroy()
