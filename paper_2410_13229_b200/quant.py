"""Quantization primitives -- mirror of the reference's `ssmq.quant` API
(pkg/src/ssmq/quant.py) with the tensor op on the GPU.

`quantize` runs in libqmb's kernel (clip(rint(x / f32(s)), +-qmax), quant.py:142-155).
Scale computation (`compute_scale_*`, `nearest_rank`) is offline calibration
arithmetic on host statistics and keeps the reference's exact formulas.

QTensor.values may be a numpy array (reference-compatible drop-in: results
come back as numpy) or a CUDA torch tensor (device-resident fast path).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

import numpy as np
import torch

from . import _device, _lib

SCALE_FLOOR = 1e-8            # quant.py:20
DEFAULT_PERCENTILE = 99.999   # quant.py:24


class SchemeKind(str, Enum):
    STATIC_SYMMETRIC_MAX = "static_symmetric_max"
    STATIC_SYMMETRIC_PERCENTILE = "static_symmetric_percentile"
    DYNAMIC_SYMMETRIC_MAX = "dynamic_symmetric_max"
    STATIC_LOG2 = "static_log2"
    STATIC_ASYMMETRIC_PERCENTILE = "static_asymmetric_percentile"


_PERCENTILE_KINDS = (SchemeKind.STATIC_SYMMETRIC_PERCENTILE, SchemeKind.STATIC_ASYMMETRIC_PERCENTILE)


@dataclass(frozen=True)
class QuantScheme:
    """quant.py:41-57"""

    kind: SchemeKind
    p: float | None = None

    def __post_init__(self):
        if self.kind in _PERCENTILE_KINDS:
            if self.p is None or not (0.0 < self.p <= 100.0):
                raise ValueError(f"percentile scheme requires p in (0, 100], got {self.p}")
        elif self.p is not None:
            raise ValueError(f"scheme {self.kind.value} does not take a percentile")

    @property
    def symmetric(self) -> bool:
        return self.kind != SchemeKind.STATIC_ASYMMETRIC_PERCENTILE


def qmax(bit_width: int) -> int:
    return 2 ** (bit_width - 1) - 1


def qmin(bit_width: int) -> int:
    return -(2 ** (bit_width - 1))


def is_device(v) -> bool:
    return isinstance(v, torch.Tensor) and v.is_cuda


@dataclass(frozen=True)
class QTensor:
    """Integer tensor with a static scale (quant.py:76-98)."""

    values: object
    scale: float
    zero_point: int = 0
    bit_width: int = 8

    def __post_init__(self):
        if self.bit_width < 2:
            raise ValueError(f"bit width must be >= 2, got {self.bit_width}")
        if not (self.scale > 0.0):
            raise ValueError(f"scale must be positive, got {self.scale}")
        v = self.values
        if isinstance(v, torch.Tensor):
            if v.dtype.is_floating_point or v.dtype == torch.bool:
                raise ValueError("QTensor values must be integers")
        elif not np.issubdtype(np.asarray(v).dtype, np.integer):
            raise ValueError("QTensor values must be integers")
        lo, hi = qmin(self.bit_width), qmax(self.bit_width)
        if not isinstance(v, torch.Tensor):
            arr = np.asarray(v)
            if arr.size and (arr.min() < lo or arr.max() > hi):
                raise ValueError(f"values outside representable range [{lo}, {hi}]")

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.values.shape)


def compute_scale_absmax(x, bit_width: int = 8) -> float:
    """quant.py:101-111"""
    arr = np.asarray(x, dtype=np.float64)
    if arr.size == 0:
        raise ValueError("empty calibration tensor")
    if bit_width < 2:
        raise ValueError("bit width must be >= 2")
    m = float(np.max(np.abs(arr)))
    if m == 0.0:
        return SCALE_FLOOR
    return m / qmax(bit_width)


def nearest_rank(values, p: float) -> float:
    """quant.py:114-128: sorted(values)[ceil(p/100 * n) - 1], exact rational rank."""
    arr = np.sort(np.asarray(values, dtype=np.float64), axis=None)
    n = arr.size
    if n == 0:
        raise ValueError("empty calibration tensor")
    if not (0.0 < p <= 100.0):
        raise ValueError(f"percentile must lie in (0, 100], got {p}")
    rank = math.ceil(Fraction(p) * n / 100)
    idx = min(max(rank - 1, 0), n - 1)
    return float(arr[idx])


def compute_scale_percentile(pooled_abs, p: float, bit_width: int = 8) -> float:
    """quant.py:131-139"""
    v = nearest_rank(pooled_abs, p)
    if v < 0.0:
        raise ValueError("pooled absolute values must be non-negative")
    if v == 0.0:
        return SCALE_FLOOR
    return v / qmax(bit_width)


def quantize(x, scale: float, bit_width: int = 8, check: bool = True) -> QTensor:
    """quant.py:142-155 on the GPU.  numpy in -> numpy values out; CUDA tensor in
    -> CUDA tensor out.  Raises ValueError on non-finite input (checked at a sync
    point unless check=False, in which case the caller owns the error word)."""
    if not (scale > 0.0):
        raise ValueError(f"scale must be positive, got {scale}")
    as_numpy = not is_device(x)
    if as_numpy:
        arr = np.asarray(x)
        f64 = arr.dtype == np.float64  # numpy keeps f64 / f64 (e.g. Hadamard-fused weights)
        xt = _device.to_device(arr.astype(np.float64 if f64 else np.float32, copy=False))
    else:
        f64 = x.dtype == torch.float64
        xt = _device.to_device(x, torch.float64 if f64 else torch.float32)
    out = torch.empty(xt.shape, dtype=torch.int8, device=xt.device)
    err = _device.err_flag()
    _lib.call("qmb_quantize_f64" if f64 else "qmb_quantize", xt.data_ptr(), xt.numel(), float(scale),
              int(bit_width), out.data_ptr(), err.ptr, _device.stream_ptr())
    if check or as_numpy:
        err.raise_if_set()
    vals = out.cpu().numpy() if as_numpy else out
    return QTensor(vals, float(scale), 0, bit_width)


def dequantize(q: QTensor, dtype=np.float32):
    """quant.py:158-163: (values - zp) * scale computed in float64, cast."""
    v = q.values
    if isinstance(v, torch.Tensor):
        vals = v.to(torch.float64)
        if q.zero_point:
            vals = vals - q.zero_point
        tdt = torch.float32 if dtype in (np.float32, torch.float32) else torch.float64
        return (vals * q.scale).to(tdt)
    vals = np.asarray(v).astype(np.float64)
    if q.zero_point:
        vals = vals - q.zero_point
    return (vals * q.scale).astype(dtype)
