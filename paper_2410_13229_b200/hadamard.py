"""Walsh-Hadamard plans and the fused Hadamard+quantize op -- mirror of
`ssmq.hadamard` (pkg/src/ssmq/hadamard.py) with the transform on the GPU.

n = 2^p * m with m in {1, 12, 20}; the base matrices are the symmetric
Paley-II Hadamard matrices built from the conference matrices over GF(5) and
GF(9) = GF(3)[i]/(i^2+1) (element a + b*i at index a + 3b) with each entry
c -> c*[[1,1],[1,-1]] and 0 -> [[1,-1],[-1,-1]]; this reproduces the
reference's tables (hadamard.py:24-61) exactly (checked in tests against the
golden fixture).  The size limit is the kernel's (one row in shared memory),
not the reference's MAX_TRANSFORM_DIM=4096 (hadamard.py:19), which excludes
the 2.8B shape (d_inner=5120).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .quant import QTensor, is_device

MAX_TRANSFORM_DIM = 32768


def _paley2(q: int, elems, sub, chi) -> np.ndarray:
    n = q + 1
    C = np.zeros((n, n), dtype=np.int64)
    for i in range(n):
        for j in range(n):
            if i == j:
                C[i, j] = 0
            elif i == 0 or j == 0:
                C[i, j] = 1
            else:
                C[i, j] = chi(sub(elems[i - 1], elems[j - 1]))
    A = np.array([[1, 1], [1, -1]])
    Z = np.array([[1, -1], [-1, -1]])
    H = np.zeros((2 * n, 2 * n), dtype=np.int8)
    for i in range(n):
        for j in range(n):
            H[2 * i:2 * i + 2, 2 * j:2 * j + 2] = Z if C[i, j] == 0 else C[i, j] * A
    return H


def _base12() -> np.ndarray:
    squares = {(x * x) % 5 for x in range(1, 5)}
    return _paley2(5, list(range(5)), lambda a, b: (a - b) % 5,
                   lambda v: 0 if v == 0 else (1 if v in squares else -1))


def _base20() -> np.ndarray:
    def mul(u, v):  # (a + b i)(c + d i), i^2 = -1 over GF(3)
        return ((u[0] * v[0] - u[1] * v[1]) % 3, (u[0] * v[1] + u[1] * v[0]) % 3)

    elems = [(a, b) for b in range(3) for a in range(3)]
    squares = {mul(e, e) for e in elems if e != (0, 0)}
    return _paley2(9, elems, lambda u, v: ((u[0] - v[0]) % 3, (u[1] - v[1]) % 3),
                   lambda v: 0 if v == (0, 0) else (1 if v in squares else -1))


_BASES = {1: np.ones((1, 1), dtype=np.int8), 12: _base12(), 20: _base20()}
BASE_SIZES = (1, 12, 20)


def _base_matrix(m: int) -> np.ndarray:
    return _BASES[m].copy()


def build_walsh(k: int) -> np.ndarray:
    """Sylvester Walsh-Hadamard matrix of order 2^k (hadamard.py:66-76)."""
    if k < 0:
        raise ValueError("k must be non-negative")
    if 2**k > MAX_TRANSFORM_DIM:
        raise ValueError(f"2^{k} exceeds the size limit {MAX_TRANSFORM_DIM}")
    h2 = np.array([[1, 1], [1, -1]], dtype=np.int32)
    h = np.ones((1, 1), dtype=np.int32)
    for _ in range(k):
        h = np.kron(h2, h)
    return h


@dataclass(frozen=True)
class HadamardPlan:
    """n = 2^p * m (hadamard.py:79-106)."""

    n: int
    p: int
    m: int
    base: np.ndarray

    def __post_init__(self):
        if self.n != (1 << self.p) * self.m:
            raise ValueError("plan factorization is inconsistent")
        if self.base.shape != (self.m, self.m):
            raise ValueError("base matrix shape mismatch")
        if not np.isin(self.base, (-1, 1)).all():
            raise ValueError("base entries must be +/-1")
        gram = self.base.astype(np.int64) @ self.base.astype(np.int64).T
        if not np.array_equal(gram, self.m * np.eye(self.m, dtype=np.int64)):
            raise ValueError("base matrix is not Hadamard")
        self.base.setflags(write=False)


def plan_for_dim(n: int) -> HadamardPlan:
    """Maximal p with n = 2^p * m, m a known base size (hadamard.py:109-120)."""
    if n < 1:
        raise ValueError("transform dimension must be positive")
    if n > MAX_TRANSFORM_DIM:
        raise ValueError(f"dimension {n} exceeds the size limit {MAX_TRANSFORM_DIM}")
    for p in range(n.bit_length() - 1, -1, -1):
        step = 1 << p
        if n % step == 0 and n // step in BASE_SIZES:
            m = n // step
            return HadamardPlan(n, p, m, _base_matrix(m))
    raise ValueError(f"no Hadamard factorization available for n={n}")


def dense_matrix(plan: HadamardPlan) -> np.ndarray:
    return np.kron(build_walsh(plan.p), plan.base.astype(np.int32))


def _run(plan, y, scale: float, bit_width: int, want_f32: bool):
    as_numpy = not is_device(y)
    arr = np.asarray(y, dtype=np.float32) if as_numpy else y
    if arr.shape[-1] != plan.n:
        raise ValueError(f"length mismatch: expected {plan.n}, got {arr.shape[-1]}")
    yt = _device.to_device(arr, torch.float32)
    rows = yt.numel() // plan.n
    out = torch.empty(yt.shape, dtype=torch.int8, device=yt.device)
    yh = torch.empty(yt.shape, dtype=torch.float32, device=yt.device) if want_f32 else None
    base = np.ascontiguousarray(np.asarray(plan.base, dtype=np.int8))
    err = _device.err_flag()
    _lib.call("qmb_hadamard_quantize", yt.data_ptr(), rows, int(plan.p), int(plan.m), base.ctypes.data,
              float(scale), int(bit_width), out.data_ptr(), _device.ptr(yh), err.ptr, _device.stream_ptr())
    return out, yh, err, as_numpy


def apply_hadamard(plan: HadamardPlan, x):
    """H_n x along the last axis (hadamard.py:128-149), float32 on the GPU."""
    out, yh, err, as_numpy = _run(plan, x, 1.0, 8, True)
    err.t.zero_()  # the byproduct quantization may flag huge values; the transform itself never raises
    return yh.cpu().numpy() if as_numpy else yh


def hadamard_quantize(y, scale: float, plan: HadamardPlan, bit_width: int = 8) -> QTensor:
    """quantize(H_n y, scale) fused in one kernel (hadamard.py:164-166)."""
    if not (scale > 0.0):
        raise ValueError(f"scale must be positive, got {scale}")
    out, _, err, as_numpy = _run(plan, y, scale, bit_width, False)
    err.raise_if_set()
    return QTensor(out.cpu().numpy() if as_numpy else out, float(scale), 0, bit_width)


def fuse_inverse_into_weights(w_out: np.ndarray, plan: HadamardPlan) -> np.ndarray:
    """W^H = H_n W on the feature axis (hadamard.py:152-161): offline weight
    preparation in float64 on the host, same operation order as the reference
    (per m-chunk +/-1 base product, then the butterfly with h ascending)."""
    w = np.asarray(w_out, dtype=np.float64)
    if w.ndim != 2 or w.shape[0] != plan.n:
        raise ValueError(f"dimension mismatch: weight feature axis must be {plan.n}")
    blocks = 1 << plan.p
    v = np.array(w.T, dtype=np.float64)  # rows = output features, transform along axis 1
    if plan.m > 1:
        v = v.reshape(v.shape[0], blocks, plan.m) @ plan.base.T.astype(np.float64)
        v = v.reshape(v.shape[0], plan.n)
    v = v.reshape(v.shape[0], blocks, plan.m)
    h = 1
    while h < blocks:
        v4 = v.reshape(v.shape[0], blocks // (2 * h), 2, h, plan.m)
        s = v4[:, :, 0] + v4[:, :, 1]
        d = v4[:, :, 0] - v4[:, :, 1]
        v4[:, :, 0] = s
        v4[:, :, 1] = d
        h *= 2
    return np.ascontiguousarray(v.reshape(v.shape[0], plan.n).T)
