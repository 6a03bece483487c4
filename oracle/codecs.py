"""Wire numerics restated from epsim core.py (test infrastructure only).

* E4M3 code -> value table, NaN codes (S.1111.111) decode to 0     core.py:84-101
* nearest-E4M3 encoder, |x| clamped to 448, exact midpoints go to the
  SMALLER magnitude, sign taken from signbit (so -0.0 -> 0x80)      core.py:106-120
* block-128 quantisation: scale = f32(absmax / 448), zero block ->
  scale 0 and codes 0, codes = enc(f32(x / scale))                 core.py:127-150
* dequantisation: f32(value(code) * scale)                         core.py:153-162
* bf16: widen = bits << 16; narrow = RNE on the top 16 bits         core.py:170-178
"""

from __future__ import annotations

import numpy as np

FP8_BLOCK = 128
FP8_MAX = np.float32(448.0)


class OracleError(ValueError):
    """Raised where the reference raises EpError(InvalidArgument)."""


def _e4m3_value(code: int) -> float:
    sign = -1.0 if code & 0x80 else 1.0
    exp, man = (code >> 3) & 0xF, code & 0x7
    if exp == 0xF and man == 0x7:
        return 0.0                      # NaN code; never produced
    if exp == 0:
        return sign * man * 2.0 ** -9   # subnormal: man/8 * 2^-6
    return sign * (8 + man) * 2.0 ** (exp - 10)


E4M3 = np.array([_e4m3_value(c) for c in range(256)], dtype=np.float32)

# ascending positive magnitudes of codes 0x00..0x7E and the f64 midpoints
_MAG = E4M3[:0x7F].astype(np.float64)
_MID = 0.5 * (_MAG[:-1] + _MAG[1:])


def encode_e4m3(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    mag = np.minimum(np.abs(x.astype(np.float64)), 448.0)
    # number of midpoints strictly below |x|: a tie stays on the lower code
    code = np.searchsorted(_MID, mag, side="left").astype(np.uint8)
    return np.where(np.signbit(x), code | np.uint8(0x80), code).astype(np.uint8)


def decode_e4m3(codes) -> np.ndarray:
    return E4M3[np.asarray(codes, dtype=np.uint8)]


def quantize_block(x) -> tuple[np.ndarray, np.ndarray]:
    x = np.asarray(x, dtype=np.float32)
    h = x.shape[-1]
    if h % FP8_BLOCK:
        raise OracleError(f"hidden {h} not a multiple of {FP8_BLOCK}")
    if not np.isfinite(x).all():
        raise OracleError("non-finite input")
    blk = x.reshape(x.shape[:-1] + (h // FP8_BLOCK, FP8_BLOCK))
    scale = (np.abs(blk).max(axis=-1) / FP8_MAX).astype(np.float32)
    div = np.where(scale > 0, scale, np.float32(1.0)).astype(np.float32)
    codes = encode_e4m3((blk / div[..., None]).astype(np.float32))
    return codes.reshape(x.shape), scale


def dequantize_block(codes, scales) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint8)
    scales = np.asarray(scales, dtype=np.float32)
    nb = scales.shape[-1]
    if codes.shape[-1] != nb * FP8_BLOCK:
        raise OracleError("codes/scales mismatch")
    v = decode_e4m3(codes).reshape(codes.shape[:-1] + (nb, FP8_BLOCK))
    return (v * scales[..., None]).astype(np.float32).reshape(codes.shape)


def bf16_to_f32(bits) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x) -> np.ndarray:
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32)
    return ((u + np.uint32(0x7FFF) + ((u >> 16) & np.uint32(1))) >> 16).astype(np.uint16)


def wire_roundtrip(x, dtype: str, with_scales: bool) -> np.ndarray:
    """f32 value of a row after one wire hop in `dtype` (oracle.py:48-64)."""
    x = np.asarray(x, dtype=np.float32)
    if dtype == "f32":
        return x.copy()
    if dtype == "bf16":
        return bf16_to_f32(f32_to_bf16(x))
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "fp8":
        if with_scales:
            return dequantize_block(*quantize_block(x))
        return decode_e4m3(encode_e4m3(x))
    raise OracleError(f"dtype {dtype}")


def to_storage(x, dtype: str) -> np.ndarray:
    """f32 -> raw storage of a tensor of `dtype` (NDTensor.write_f32, core.py:222-234)."""
    x = np.asarray(x, dtype=np.float32)
    if dtype == "f32":
        return x.copy()
    if dtype == "bf16":
        return f32_to_bf16(x)
    if dtype == "f16":
        return x.astype(np.float16)
    if dtype == "fp8":
        return encode_e4m3(x)
    raise OracleError(dtype)


def from_storage(raw, dtype: str) -> np.ndarray:
    """raw storage -> f32 (NDTensor.read_f32, core.py:213-220)."""
    if dtype == "bf16":
        return bf16_to_f32(raw)
    if dtype == "fp8":
        return decode_e4m3(raw)
    return np.asarray(raw).astype(np.float32)
