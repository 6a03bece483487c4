"""Domain types of the reference API (epsim core.py), B200 edition.

Mirrors epsim.core name-for-name: Dtype, TensorTag, NDTensor, tensor_create,
tensor_from_f32, EpConfig, Algorithm, EpError, ErrorCode, quantize_block,
dequantize_block.  Differences are storage and placement only:

* NDTensor storage is a torch tensor, on the GPU by default (host tensors and
  numpy buffers are accepted; they are staged to the device by the API).
* every dtype conversion (read_f32 / write_f32, FP8 block quantisation) runs
  in the CUDA library (libepb200.so), bit-exact with the reference codecs
  (core.py:84-178); there is no host arithmetic path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib

FP8_BLOCK = 128
FP8_MAX = 448.0


class ErrorCode(Enum):
    INVALID_ARGUMENT = "InvalidArgument"
    SHAPE_MISMATCH = "ShapeMismatch"
    TAG_MISMATCH = "TagMismatch"
    CONFIG_MISMATCH = "ConfigMismatch"
    CAPACITY_EXCEEDED = "CapacityExceeded"
    HANDLE_STATE_ERROR = "HandleStateError"
    TRANSPORT_CLOSED = "TransportClosed"


_STATUS = [None, ErrorCode.INVALID_ARGUMENT, ErrorCode.SHAPE_MISMATCH, ErrorCode.TAG_MISMATCH,
           ErrorCode.CONFIG_MISMATCH, ErrorCode.CAPACITY_EXCEEDED, ErrorCode.HANDLE_STATE_ERROR,
           ErrorCode.TRANSPORT_CLOSED]


class EpError(Exception):
    """The single error type every public operation raises (core.py:31-42)."""

    def __init__(self, code: ErrorCode, detail: str):
        super().__init__(f"{code.value}: {detail}")
        self.code = code
        self.detail = detail


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libepb200 (not an API misuse)."""


def raise_status(rc: int, detail: str):
    if 1 <= rc < len(_STATUS):
        raise EpError(_STATUS[rc], detail)
    raise CudaError(detail)


class Dtype(Enum):
    F32 = "f32"
    BF16 = "bf16"
    F16 = "f16"
    FP8 = "fp8"

    @property
    def byte_width(self) -> int:
        return _WIDTH[self]

    @property
    def code(self) -> int:
        return _CODE[self]

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH[self]


_WIDTH = {Dtype.F32: 4, Dtype.BF16: 2, Dtype.F16: 2, Dtype.FP8: 1}
_CODE = {Dtype.F32: _lib.F32, Dtype.BF16: _lib.BF16, Dtype.F16: _lib.F16, Dtype.FP8: _lib.FP8}
# bf16 keeps its own torch dtype (same bits as the reference's uint16 storage);
# fp8 storage is raw E4M3 code bytes as in the reference
_TORCH = {Dtype.F32: torch.float32, Dtype.BF16: torch.bfloat16, Dtype.F16: torch.float16,
          Dtype.FP8: torch.uint8}
_NUMPY = {Dtype.F32: np.float32, Dtype.BF16: np.uint16, Dtype.F16: np.float16, Dtype.FP8: np.uint8}


class TensorTag(Enum):
    TOKENS = "TOKENS"
    TOPK_IDX = "TOPK_IDX"
    TOPK_WEIGHTS = "TOPK_WEIGHTS"
    SCALES = "SCALES"
    RECV_EXPERT_COUNTER_DEVICE = "RECV_EXPERT_COUNTER_DEVICE"
    RECV_EXPERT_COUNTER_HOST = "RECV_EXPERT_COUNTER_HOST"
    NONE = "NONE"
    TOKENS_PER_EXPERTS = "TOKENS_PER_EXPERTS"


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryMissing("no CUDA device: the EP path runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------
# device codecs (all arithmetic inside libepb200)
# ---------------------------------------------------------------------------


def to_device_f32(values, device=None) -> torch.Tensor:
    dev = device or default_device()
    if isinstance(values, torch.Tensor):
        return values.to(device=dev, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(dev)


def encode_f32(x: torch.Tensor, dtype: Dtype) -> torch.Tensor:
    """f32 device tensor -> storage of `dtype` (NDTensor.write_f32 codecs)."""
    x = x.contiguous()
    if dtype is Dtype.F32:
        return x.clone()
    out = torch.empty(x.shape, dtype=dtype.torch_dtype, device=x.device)
    _lib.call("epb_convert", x.data_ptr(), _lib.F32, out.data_ptr(), dtype.code, x.numel(),
              _stream_ptr())
    return out


def decode_f32(x: torch.Tensor, dtype: Dtype) -> torch.Tensor:
    """storage of `dtype` (device) -> f32 (NDTensor.read_f32 codecs)."""
    x = x.contiguous()
    if dtype is Dtype.F32:
        return x.clone()
    out = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    _lib.call("epb_convert", x.data_ptr(), dtype.code, out.data_ptr(), _lib.F32, x.numel(),
              _stream_ptr())
    return out


def _finite_or_raise(x: torch.Tensor):
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.call("epb_check_finite", x.data_ptr(), x.numel(), flag.data_ptr(), _stream_ptr())
    if int(flag.item()):
        raise EpError(ErrorCode.INVALID_ARGUMENT, "non-finite input to quantize_block")


def quantize_block(row):
    """Block-128 FP8 quantisation on the GPU (core.py:127-150).

    Accepts numpy or torch (f32/bf16/f16); returns (codes u8, scales f32) as
    torch tensors on the device, bit-exact with the reference."""
    x = row if isinstance(row, torch.Tensor) else to_device_f32(row)
    if not x.is_cuda:
        x = x.to(default_device())
    h = x.shape[-1]
    if h % FP8_BLOCK:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"hidden size {h} not divisible by {FP8_BLOCK}")
    x = x.contiguous()
    code = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}[x.dtype]
    if x.dtype == torch.float32:
        _finite_or_raise(x)
    rows = x.numel() // h
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scales = torch.empty(x.shape[:-1] + (h // FP8_BLOCK,), dtype=torch.float32, device=x.device)
    _lib.call("epb_fp8_quantize", x.data_ptr(), code, rows, h, codes.data_ptr(), scales.data_ptr(),
              _stream_ptr())
    return codes, scales


def dequantize_block(codes, scales):
    """Inverse of quantize_block (core.py:153-162), on the GPU."""
    dev = default_device()
    c = codes if isinstance(codes, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(codes, np.uint8))
    s = scales if isinstance(scales, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(scales, np.float32))
    c = c.to(dev).contiguous()
    s = s.to(dev, torch.float32).contiguous()
    if c.shape[-1] != FP8_BLOCK * s.shape[-1]:
        raise EpError(ErrorCode.INVALID_ARGUMENT,
                      f"{c.shape[-1]} codes vs {s.shape[-1]} scales (need {FP8_BLOCK} codes per scale)")
    out = torch.empty(c.shape, dtype=torch.float32, device=dev)
    h = c.shape[-1]
    _lib.call("epb_fp8_dequantize", c.data_ptr(), s.data_ptr(), c.numel() // max(h, 1), h,
              out.data_ptr(), _stream_ptr())
    return out


# ---------------------------------------------------------------------------
# tensors
# ---------------------------------------------------------------------------


def _row_major_strides(shape):
    strides, acc = [], 1
    for extent in reversed(shape):
        strides.append(acc)
        acc *= extent
    return tuple(reversed(strides))


@dataclass
class NDTensor:
    """Typed, strided N-D descriptor over a flat torch storage tensor
    (epsim NDTensor, core.py:186-241).  `data` is 1-D in the dtype's storage
    type (float32 / bfloat16 / float16 / uint8 codes); `offset` is in
    elements."""

    shape: tuple
    strides: tuple
    dtype: Dtype
    tag: TensorTag
    data: torch.Tensor
    offset: int = 0

    @property
    def num_elements(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    @property
    def device(self) -> torch.device:
        return self.data.device

    def view(self) -> torch.Tensor:
        """The typed torch view (no copy), built once per descriptor."""
        # storage_offset is absolute in the storage: a `data` that is itself a
        # view (a slice of a larger tensor) contributes its own offset
        key = (self.data.data_ptr(), self.shape, self.strides, self.offset)
        cached = self.__dict__.get("_view")
        if cached is None or cached[0] != key:
            cached = (key, torch.as_strided(self.data, self.shape, self.strides,
                                            self.data.storage_offset() + self.offset))
            self.__dict__["_view"] = cached
        return cached[1]

    def is_contiguous_view(self) -> bool:
        return self.strides == _row_major_strides(self.shape)

    def read_f32(self) -> np.ndarray:
        """Materialise as a host float32 ndarray (conversion on the GPU)."""
        v = self.view()
        if self.dtype is Dtype.F32:
            return v.detach().to("cpu").contiguous().numpy().copy()
        dev = v.device if v.is_cuda else default_device()
        return decode_f32(v.to(dev), self.dtype).cpu().numpy()

    def read_f32_device(self) -> torch.Tensor:
        v = self.view()
        dev = v.device if v.is_cuda else default_device()
        return decode_f32(v.to(dev), self.dtype)

    def write_f32(self, values) -> None:
        """Store f32 values converted to the tensor dtype (GPU codecs)."""
        if isinstance(values, torch.Tensor):
            shp = tuple(values.shape)
        else:
            values = np.asarray(values, dtype=np.float32)
            shp = values.shape
        if tuple(shp) != tuple(self.shape):
            raise EpError(ErrorCode.SHAPE_MISMATCH, f"write of {tuple(shp)} into tensor {self.shape}")
        dev = self.data.device if self.data.is_cuda else default_device()
        enc = encode_f32(to_device_f32(values, dev), self.dtype)
        self.view().copy_(enc.to(self.data.device))

    def raw(self) -> np.ndarray:
        """Stored elements (bit patterns for bf16/fp8) as a host ndarray."""
        v = self.view().detach().to("cpu").contiguous()
        if self.dtype is Dtype.BF16:
            v = v.view(torch.int16)
            return v.numpy().view(np.uint16).copy()
        return v.numpy().copy()

    def write_raw(self, values) -> None:
        if isinstance(values, torch.Tensor):
            t = values
        else:
            arr = np.ascontiguousarray(values, dtype=_NUMPY[self.dtype]).reshape(self.shape)
            t = torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16) if self.dtype is Dtype.BF16 \
                else torch.from_numpy(arr)
        self.view().copy_(t.reshape(self.shape).to(self.data.device))


def _storage_from_buffer(buffer, dtype: Dtype, count: int, shape) -> torch.Tensor:
    needed = count * dtype.byte_width
    if isinstance(buffer, torch.Tensor):
        flat = buffer.reshape(-1) if buffer.is_contiguous() else None
        if flat is None:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "buffer tensor must be contiguous")
        if flat.dtype == dtype.torch_dtype:
            if flat.numel() < count:
                raise EpError(ErrorCode.INVALID_ARGUMENT, f"buffer too small for {shape} {dtype.value}")
            return flat[:count]
        if flat.dtype == torch.uint8:
            if flat.numel() < needed:
                raise EpError(ErrorCode.INVALID_ARGUMENT,
                              f"buffer of {flat.numel()} B too small for {shape} {dtype.value} ({needed} B)")
            return flat[:needed].view(dtype.torch_dtype)
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"buffer dtype {flat.dtype} incompatible with {dtype.value}")
    if isinstance(buffer, np.ndarray):
        flat = buffer.reshape(-1)
        if flat.dtype == np.uint8:
            if flat.nbytes < needed:
                raise EpError(ErrorCode.INVALID_ARGUMENT,
                              f"buffer of {flat.nbytes} B too small for {shape} {dtype.value} ({needed} B)")
            t = torch.from_numpy(flat[:needed])
            return t.view(dtype.torch_dtype)
        if flat.dtype != _NUMPY[dtype]:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"buffer dtype {flat.dtype} incompatible with {dtype.value}")
        if flat.size < count:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"buffer too small for {shape} {dtype.value}")
        t = torch.from_numpy(flat[:count])
        return t.view(torch.bfloat16) if dtype is Dtype.BF16 else t
    raw = memoryview(buffer).cast("B")
    if raw.nbytes < needed:
        raise EpError(ErrorCode.INVALID_ARGUMENT,
                      f"buffer of {raw.nbytes} B too small for {shape} {dtype.value} ({needed} B)")
    t = torch.frombuffer(raw, dtype=torch.uint8, count=needed)
    return t.view(dtype.torch_dtype)


def tensor_create(shape, dtype: Dtype, tag: TensorTag, buffer=None, device=None) -> NDTensor:
    """Create a contiguous row-major tensor descriptor (core.py:252-304).

    Without `buffer` the storage is allocated zeroed on `device` (default:
    the current CUDA device).  `buffer` may be a torch tensor (any device),
    a numpy array, or a bytes-like object, viewed without copying."""
    shape = tuple(int(s) for s in shape)
    if len(shape) == 0:
        raise EpError(ErrorCode.INVALID_ARGUMENT, "empty shape")
    if any(s < 0 for s in shape):
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"negative extent in {shape}")
    count = int(np.prod(shape))
    if buffer is None:
        dev = device if device is not None else default_device()
        data = torch.zeros(count, dtype=dtype.torch_dtype, device=dev)
    else:
        data = _storage_from_buffer(buffer, dtype, count, shape)
    return NDTensor(shape, _row_major_strides(shape), dtype, tag, data)


def tensor_from_f32(values, dtype: Dtype, tag: TensorTag, device=None) -> NDTensor:
    """Allocate a tensor of `dtype` holding the given f32 values."""
    shape = tuple(values.shape)
    t = tensor_create(shape, dtype, tag, device=device)
    t.write_f32(values)
    return t


def tensor_from_torch(t: torch.Tensor, tag: TensorTag) -> NDTensor:
    """Wrap an existing torch tensor (zero-copy)."""
    dt = {torch.float32: Dtype.F32, torch.bfloat16: Dtype.BF16, torch.float16: Dtype.F16,
          torch.uint8: Dtype.FP8}.get(t.dtype)
    if dt is None:
        raise EpError(ErrorCode.INVALID_ARGUMENT, f"unsupported torch dtype {t.dtype}")
    if not t.is_contiguous():
        raise EpError(ErrorCode.INVALID_ARGUMENT, "tensor must be contiguous")
    return NDTensor(tuple(t.shape), _row_major_strides(tuple(t.shape)), dt, tag, t.reshape(-1))


# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------


class Algorithm(Enum):
    LL = "ll"
    HT = "ht"


@dataclass(frozen=True)
class EpConfig:
    """Static, rank-identical configuration (core.py:325-383)."""

    algorithm: Algorithm
    num_ranks: int
    ranks_per_node: int
    num_experts: int
    top_k: int
    hidden: int
    max_tokens_per_rank: int
    token_dtype: Dtype = Dtype.F32
    with_scales: bool = False
    ht_chunk_tokens: int = 4
    ht_fifo_depth: int = 8
    # extension: LL combine wire dtype (None = token_dtype, the reference's
    # ll.py:437-438); C2 "FP8 dispatch + bf16 combine" sets Dtype.BF16
    combine_dtype: "Dtype | None" = None
    # extension: HT registered expert-output region in the window; a combine
    # whose expert rows live there is pulled by the home ranks over NVLink
    # (EpHandle.expert_out_buffer / Buffer.get_expert_out_buffer)
    expert_out_window: bool = False

    def __post_init__(self):
        n, e, k = self.num_ranks, self.num_experts, self.top_k
        if n < 1:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"num_ranks {n} < 1")
        if not (1 <= k <= e):
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"top_k {k} outside [1, {e}]")
        if self.ranks_per_node < 1 or n % self.ranks_per_node != 0:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          f"ranks_per_node {self.ranks_per_node} must divide num_ranks {n}")
        if e < n:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"num_experts {e} < num_ranks {n}")
        if self.hidden < 1:
            raise EpError(ErrorCode.INVALID_ARGUMENT, f"hidden {self.hidden} < 1")
        if self.max_tokens_per_rank < 1:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          f"max_tokens_per_rank {self.max_tokens_per_rank} < 1")
        if self.with_scales:
            if self.token_dtype is not Dtype.FP8:
                raise EpError(ErrorCode.INVALID_ARGUMENT, "with_scales requires token_dtype fp8")
            if self.hidden % FP8_BLOCK != 0:
                raise EpError(ErrorCode.INVALID_ARGUMENT,
                              f"with_scales requires hidden divisible by {FP8_BLOCK}")
        if self.algorithm is Algorithm.HT and self.token_dtype is Dtype.FP8:
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          "fp8 token dtype is not supported by the HT algorithm")
        if self.ht_chunk_tokens < 1 or self.ht_fifo_depth < 1:
            raise EpError(ErrorCode.INVALID_ARGUMENT, "ht_chunk_tokens and ht_fifo_depth must be >= 1")
        # limits of the GPU implementation (flags pack 20-bit counts, rank masks are 64-bit)
        if n > 64 or k > 32 or self.max_tokens_per_rank >= (1 << 20):
            raise EpError(ErrorCode.INVALID_ARGUMENT,
                          "GPU path supports num_ranks <= 64, top_k <= 32, max_tokens_per_rank < 2^20")

    @property
    def experts_per_rank(self) -> int:
        return math.ceil(self.num_experts / self.num_ranks)

    def fingerprint(self) -> bytes:
        parts = (self.algorithm.value, self.num_ranks, self.ranks_per_node, self.num_experts,
                 self.top_k, self.hidden, self.max_tokens_per_rank, self.token_dtype.value,
                 int(self.with_scales), self.ht_chunk_tokens, self.ht_fifo_depth)
        fp = "|".join(str(p) for p in parts)
        if self.combine_dtype is not None:
            fp += "|c=" + self.combine_dtype.value
        if self.expert_out_window:
            fp += "|yout"
        return fp.encode()

    @property
    def combine_wire(self) -> "Dtype":
        return self.token_dtype if self.combine_dtype is None else self.combine_dtype

    def to_c(self, layout: str = "optimized") -> _lib.Config:
        c = _lib.Config()
        c.algorithm = _lib.LL if self.algorithm is Algorithm.LL else _lib.HT
        c.num_ranks, c.ranks_per_node = self.num_ranks, self.ranks_per_node
        c.num_experts, c.top_k, c.hidden = self.num_experts, self.top_k, self.hidden
        c.max_tokens_per_rank = self.max_tokens_per_rank
        c.token_dtype = self.token_dtype.code
        c.with_scales = int(self.with_scales)
        c.layout = 0 if layout == "optimized" else 1
        c.ht_chunk_tokens, c.ht_fifo_depth = self.ht_chunk_tokens, self.ht_fifo_depth
        c.combine_dtype = -1 if self.combine_dtype is None else self.combine_dtype.code
        c.expert_out_window = int(self.expert_out_window)
        return c
