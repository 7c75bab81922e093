"""Device plumbing: torch tensors as memory, the current CUDA stream, the
error-flag word and workspace caching.  No arithmetic happens here."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_DEVICE = None


def device() -> torch.device:
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise _lib.QmbError("paper_2410_13229_b200 requires a CUDA GPU (sm_100a); no CPU fallback exists")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def to_device(arr, dtype=None) -> torch.Tensor:
    """Upload a numpy array (or pass through a CUDA tensor), contiguous."""
    if isinstance(arr, torch.Tensor):
        t = arr if arr.is_cuda else arr.to(device())
    else:
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device())
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class ErrFlag:
    """A device uint32 error word (QMB_ERR_* bits) checked at sync points."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=device())

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def reset(self) -> None:
        self.t.zero_()

    def raise_if_set(self) -> None:
        v = int(self.t.item())
        if v:
            self.t.zero_()
            if v & _lib.QMB_ERR_SCAN:
                raise FloatingPointError("scan divergence: non-finite intermediate")
            raise ValueError("non-finite activation")


_err = None


def err_flag() -> ErrFlag:
    global _err
    if _err is None:
        _err = ErrFlag()
    return _err


class Workspace:
    """Grow-only device scratch buffer."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())
        return self.buf


_ws = Workspace()


def workspace(nbytes: int) -> torch.Tensor:
    return _ws.get(nbytes)


def c_ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)
