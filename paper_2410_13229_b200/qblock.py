"""Quantized block -- mirror of `ssmq.qblock` (pkg/src/ssmq/qblock.py) whose
operators run in libqmb's sm_100a kernels.

Drop-in contract: every function accepts the reference's own objects
(QTensor / QuantizedBlock / HadamardPlan from `ssmq`, duck-typed) as well as
this package's mirrors, and returns numpy when given numpy (same semantics and
error types as the reference) or CUDA tensors when given CUDA tensors.
Integer outputs are bit-exact with the reference; see DESIGN.md.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _device, _lib
from .hadamard import HadamardPlan, fuse_inverse_into_weights, hadamard_quantize  # noqa: F401  (API mirror)
from .quant import QTensor, QuantScheme, SchemeKind, compute_scale_absmax, dequantize, is_device, quantize
from .ssm import BlockConfig, SSMParams

MAX_ACC_DIM = 2**15  # qblock.py:29


class Mode(str, Enum):
    """qblock.py:32-44"""

    NAIVE = "naive"
    IN_PERCENTILE = "in_percentile"
    OUT_HADAMARD = "out_hadamard"
    FULL = "full"

    @property
    def percentile_input(self) -> bool:
        return self in (Mode.IN_PERCENTILE, Mode.FULL)

    @property
    def hadamard_output(self) -> bool:
        return self in (Mode.OUT_HADAMARD, Mode.FULL)


MODE_TAGS = {"naive": Mode.NAIVE, "in-per": Mode.IN_PERCENTILE, "out-had": Mode.OUT_HADAMARD, "quamba": Mode.FULL}
TAG_FOR_MODE = {mode: tag for tag, mode in MODE_TAGS.items()}
ACT_SITES = ("in", "conv_in", "conv_out", "x", "b", "c", "dt_r", "dt", "y", "y_had")
_MODE_CODE = {"naive": 0, "in_percentile": 1, "out_hadamard": 2, "full": 3}


@dataclass(frozen=True)
class ScaleEntry:
    """qblock.py:60-72"""

    scale: float
    zero_point: int
    scheme: QuantScheme

    def __post_init__(self):
        if not (self.scale > 0.0):
            raise ValueError(f"scale must be positive, got {self.scale}")
        if self.scheme.symmetric and self.zero_point != 0:
            raise ValueError("symmetric scheme requires zero_point = 0")


@dataclass(eq=False)
class QuantizedBlock:
    """qblock.py:75-95"""

    cfg: BlockConfig
    mode: Mode
    weights: dict
    act: dict
    plan: HadamardPlan

    def __post_init__(self):
        missing = [s for s in ACT_SITES if s not in self.act]
        if missing:
            raise ValueError(f"missing activation scales: {missing}")
        if self.mode.percentile_input:
            if self.act["x"].scheme.kind is not SchemeKind.STATIC_SYMMETRIC_PERCENTILE and \
                    getattr(self.act["x"].scheme.kind, "value", None) != SchemeKind.STATIC_SYMMETRIC_PERCENTILE.value:
                raise ValueError(f"mode {self.mode.value} requires a percentile scan-input scale")
        if self.mode.hadamard_output != ("w_out_h" in self.weights):
            raise ValueError("fused output weights must be present exactly in Hadamard modes")

    @property
    def bit_width(self) -> int:
        return self.weights["w_in"].bit_width


# --------------------------------------------------------------------------- device handle
def _host_i8(qt) -> np.ndarray:
    v = qt.values
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(v).astype(np.int8))


def _mode_value(mode) -> str:
    return mode.value if hasattr(mode, "value") else str(mode)


class DeviceBlock:
    """An uploaded QuantizedBlock: one libqmb handle (int8 weights repacked
    K-major, f32 epilogue constants, dequant and expf tables) living in HBM."""

    def __init__(self, qb, d_inner: int | None = None):
        """d_inner: override for a channel slice of a block (tensor parallelism, tp.py)."""
        _device.device()
        lib = _lib.load()
        cfg = qb.cfg
        mode = _mode_value(qb.mode)
        self.d_model, self.d_inner = int(cfg.d_model), int(d_inner if d_inner is not None else cfg.d_inner)
        self.d_state, self.d_conv, self.dt_rank = int(cfg.d_state), int(cfg.d_conv), int(cfg.dt_rank)
        self.bit_width = int(qb.weights["w_in"].bit_width)
        self.act_in = float(qb.act["in"].scale)
        desc = _lib.BlockDesc()
        desc.d_model, desc.d_inner, desc.d_state = self.d_model, self.d_inner, self.d_state
        desc.d_conv, desc.dt_rank = self.d_conv, self.dt_rank
        desc.bit_width = self.bit_width
        desc.mode = _MODE_CODE[mode]
        for i, site in enumerate(ACT_SITES):
            desc.act[i] = float(qb.act[site].scale)
        keep = []
        for name in ("a", "d", "w_in", "conv_w", "conv_b", "w_b", "w_c", "w_dt_rank", "w_dt", "dt_bias", "w_out",
                     "w_out_h"):
            if name not in qb.weights:
                continue
            if name == "w_out" and "w_out_h" in qb.weights and qb.mode.hadamard_output:
                continue  # the handle runs the fused w_out_h (container loads never page w_out in)
            w = qb.weights[name]
            if w.zero_point:
                raise ValueError("qlinear requires symmetric operands")
            arr = _host_i8(w)
            keep.append(arr)
            setattr(desc, name, _lib.QWeight(arr.ctypes.data, float(w.scale)))
        base = np.ascontiguousarray(np.asarray(qb.plan.base, dtype=np.int8))
        keep.append(base)
        desc.had_p, desc.had_m, desc.had_base = int(qb.plan.p), int(qb.plan.m), base.ctypes.data
        h = ctypes.c_void_p()
        _lib.check(lib.qmb_block_create(ctypes.byref(desc), ctypes.byref(h)), "qmb_block_create")
        self.handle = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.qmb_block_destroy(h)
            self.handle = None

    def workspace_bytes(self, rows: int) -> int:
        return int(self._lib.qmb_block_workspace_bytes(self.handle, int(rows)))

    def workspace_layout(self, rows: int) -> dict:
        offs = (ctypes.c_size_t * len(_lib.WS_SLOTS))()
        _lib.check(self._lib.qmb_block_workspace_layout(self.handle, int(rows), offs))
        return {name: int(offs[i]) for i, name in enumerate(_lib.WS_SLOTS)}

    def prefill(self, u_q: torch.Tensor, B: int, T: int, out: torch.Tensor, *, u_scale: float | None = None,
                conv_state_out=None, ssm_state_out=None, scan_exp: int = 0, workspace=None, err=None,
                stream: int | None = None, accumulate: bool = False) -> torch.Tensor:
        """block_forward_q over B sequences; accumulate=True adds the block output
        into `out` (the residual stream) instead of overwriting it."""
        M = B * T
        ws = workspace if workspace is not None else _device.workspace(self.workspace_bytes(M))
        e = err if err is not None else _device.err_flag()
        fn = self._lib.qmb_block_prefill_accum if accumulate else self._lib.qmb_block_prefill
        _lib.check(fn(
            self.handle, u_q.data_ptr(), float(u_scale or 0.0), int(B), int(T), out.data_ptr(),
            _device.ptr(conv_state_out), _device.ptr(ssm_state_out), int(scan_exp), ws.data_ptr(), ws.numel(),
            e.ptr, stream if stream is not None else _device.stream_ptr()), "qmb_block_prefill")
        return out

    def decode(self, u_q: torch.Tensor, conv_state: torch.Tensor, ssm_state: torch.Tensor, out: torch.Tensor, *,
               u_scale: float | None = None, workspace=None, err=None, stream: int | None = None,
               accumulate: bool = False) -> torch.Tensor:
        B = u_q.shape[0]
        ws = workspace if workspace is not None else _device.workspace(self.workspace_bytes(B))
        e = err if err is not None else _device.err_flag()
        fn = self._lib.qmb_block_decode_accum if accumulate else self._lib.qmb_block_decode
        _lib.check(fn(
            self.handle, u_q.data_ptr(), float(u_scale or 0.0), int(B), conv_state.data_ptr(),
            ssm_state.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), e.ptr,
            stream if stream is not None else _device.stream_ptr()), "qmb_block_decode")
        return out

    def new_state(self, B: int):
        dev = _device.device()
        conv = torch.zeros((B, max(self.d_conv - 1, 0), self.d_inner), dtype=torch.int8, device=dev)
        h = torch.zeros((B, self.d_inner, self.d_state), dtype=torch.float32, device=dev)
        return conv, h


def _block_fingerprint(qb) -> tuple:
    """Identity of what a device handle was built from: the weight arrays (object
    ids and buffer addresses) and every weight / activation scale.  The reference's
    QuantizedBlock is a mutable dataclass (qblock.py:75-95): re-calibrating it or
    swapping a weight changes this, and the next call rebuilds the handle."""
    w = tuple((k, id(v), id(getattr(v, "values", None)), float(v.scale)) for k, v in sorted(qb.weights.items()))
    a = tuple((k, float(v.scale)) for k, v in sorted(qb.act.items()))
    return w, a, _mode_value(qb.mode), id(qb.plan)


def device_block(qb) -> DeviceBlock:
    """The device handle of a QuantizedBlock (reference or mirror object), cached
    on the object and rebuilt when its weights or scales change."""
    dev = qb.__dict__.get("_qmb_device")
    fp = _block_fingerprint(qb)
    if dev is None or qb.__dict__.get("_qmb_device_fp") != fp:
        dev = DeviceBlock(qb)
        qb.__dict__["_qmb_device"] = dev
        qb.__dict__["_qmb_device_fp"] = fp
    return dev


# --------------------------------------------------------------------------- operator mirrors
def _finish(t: torch.Tensor, as_numpy: bool):
    _device.err_flag().raise_if_set()
    return t.cpu().numpy() if as_numpy else t


def qlinear(x_q, w_q, bias_q=None, s_out: float | None = None, extra_scale: float = 1.0, *, path: int = 0):
    """qblock.py:98-123 on the tensor cores (path 1) or the dp4a GEMV kernel (path 2);
    path 0 picks by shape."""
    if x_q.zero_point or w_q.zero_point:
        raise ValueError("qlinear requires symmetric operands")
    d_in = w_q.values.shape[0]
    if x_q.values.shape[-1] != d_in:
        raise ValueError("qlinear inner dimensions do not match")
    if d_in > MAX_ACC_DIM:
        raise ValueError(f"inner dimension {d_in} exceeds the int32 accumulation bound")
    as_numpy = not is_device(x_q.values)
    x = _device.to_device(x_q.values, torch.int8)
    w = _device.to_device(w_q.values, torch.int8)
    lead = tuple(x.shape[:-1])
    M = int(np.prod(lead)) if lead else 1
    N = int(w.shape[1])
    b = _device.to_device(bias_q.values, torch.int8) if bias_q is not None else None
    quant_out = s_out is not None
    out = torch.empty(lead + (N,), dtype=torch.int8 if quant_out else torch.float32, device=x.device)
    lib = _lib.load()
    wsb = int(lib.qmb_qlinear_workspace_bytes(M, int(d_in), N))
    ws = _device.workspace(wsb)
    err = _device.err_flag()
    _lib.check(lib.qmb_qlinear(x.data_ptr(), M, int(d_in), float(x_q.scale), w.data_ptr(), N, float(w_q.scale),
                               _device.ptr(b), float(bias_q.scale) if bias_q is not None else 0.0,
                               float(s_out) if quant_out else 0.0, float(extra_scale), int(x_q.bit_width),
                               out.data_ptr(), ws.data_ptr(), ws.numel(), int(path), err.ptr, _device.stream_ptr()),
               "qmb_qlinear")
    vals = _finish(out, as_numpy)
    if not quant_out:
        return vals
    return QTensor(vals, float(s_out), 0, x_q.bit_width)


def fused_qconv(x_q, w_q, bias_q, s_out: float):
    """qblock.py:126-143: x_q (T, C) or (B, T, C)."""
    if x_q.zero_point or w_q.zero_point:
        raise ValueError("fused conv requires symmetric operands")
    as_numpy = not is_device(x_q.values)
    x = _device.to_device(x_q.values, torch.int8)
    if x.dim() == 2:
        B, (T, C) = 1, x.shape
    else:
        B, T, C = x.shape
    K = int(w_q.values.shape[0])
    if w_q.values.shape[1] != C:
        raise ValueError("conv channel mismatch")
    w = _device.to_device(w_q.values, torch.int8)
    b = _device.to_device(bias_q.values, torch.int8) if bias_q is not None else None
    out = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    err = _device.err_flag()
    _lib.call("qmb_fused_qconv", x.data_ptr(), int(B), int(T), int(C), float(x_q.scale), w.data_ptr(), K,
              float(w_q.scale), _device.ptr(b), float(bias_q.scale) if bias_q is not None else 0.0, float(s_out),
              int(x_q.bit_width), out.data_ptr(), err.ptr, _device.stream_ptr())
    return QTensor(_finish(out, as_numpy), float(s_out), 0, x_q.bit_width)


def quantized_selective_scan(a_q, b_q, c_q, d_q, dt_q, x_q, h0=None, return_state: bool = False):
    """qblock.py:146-167 (dequantize-on-read scan).  Extension: optional carried
    state h0 (D, N) / (B, D, N) and return of the final state, as scan_core
    offers (kernels.py:69-99)."""
    as_numpy = not is_device(x_q.values)
    x = _device.to_device(x_q.values, torch.int8)
    batched = x.dim() == 3
    B = x.shape[0] if batched else 1
    T, D = (x.shape[1], x.shape[2]) if batched else (x.shape[0], x.shape[1])
    N = int(a_q.values.shape[1])
    dt = _device.to_device(dt_q.values, torch.int8)
    bq = _device.to_device(b_q.values, torch.int8)
    cq = _device.to_device(c_q.values, torch.int8)
    if tuple(dt.shape) != tuple(x.shape) or bq.shape[-1] != N or cq.shape[-1] != N or bq.shape[-2] != T:
        raise ValueError("scan argument shapes are inconsistent")
    if tuple(a_q.values.shape) != (D, N) or tuple(d_q.values.shape) != (D,):
        raise ValueError("scan parameter shapes are inconsistent")
    a = _device.to_device(a_q.values, torch.int8)
    dd = _device.to_device(d_q.values, torch.int8)
    y = torch.empty((B * T, D), dtype=torch.float32, device=x.device)
    need_h = h0 is not None or return_state
    h = None
    if need_h:
        if h0 is not None:
            h = _device.to_device(np.asarray(h0, dtype=np.float32) if not is_device(h0) else h0,
                                  torch.float32).clone().reshape(B, D, N)
        else:
            h = torch.zeros((B, D, N), dtype=torch.float32, device=x.device)
    err = _device.err_flag()
    nws = _lib.load().qmb_selective_scan_workspace_bytes(int(D), int(N))
    ws = torch.empty(max(int(nws), 1), dtype=torch.uint8, device=x.device)
    _lib.call("qmb_selective_scan", a.data_ptr(), float(a_q.scale), bq.data_ptr(), float(b_q.scale), cq.data_ptr(),
              float(c_q.scale), dd.data_ptr(), float(d_q.scale), dt.data_ptr(), float(dt_q.scale), x.data_ptr(),
              float(x_q.scale), int(B), int(T), int(D), int(N), _device.ptr(h), int(h0 is not None),
              y.data_ptr(), ws.data_ptr(), ws.numel(), err.ptr, _device.stream_ptr())
    y = y.reshape(x.shape)
    yv = _finish(y, as_numpy)
    if not return_state:
        return yv
    hv = h if batched else h[0]
    return yv, (hv.cpu().numpy() if as_numpy else hv)


def fused_rmsnorm_quant(x_out, x_res, gain, s_out: float, bit_width: int = 8):
    """qblock.py:170-182: (quantize(rmsnorm(x_out + x_res, gain), s_out), x_out + x_res)."""
    as_numpy = not is_device(x_out)
    xo = _device.to_device(np.asarray(x_out, dtype=np.float32) if as_numpy else x_out, torch.float32)
    xr = _device.to_device(np.asarray(x_res, dtype=np.float32) if not is_device(x_res) else x_res, torch.float32)
    g = _device.to_device(np.asarray(gain, dtype=np.float32) if not is_device(gain) else gain, torch.float32)
    D = xo.shape[-1]
    M = xo.numel() // D
    if M > 0 and not bool(torch.isfinite(g).all()):
        # a non-finite gain makes that column of every normalized row non-finite:
        # the reference's quantize raises (quant.py:149-150)
        raise ValueError("non-finite activation")
    res = torch.empty_like(xo)
    u = torch.empty(xo.shape, dtype=torch.int8, device=xo.device)
    err = _device.err_flag()
    _lib.call("qmb_rmsnorm_residual_quant", xo.data_ptr(), xr.data_ptr(), res.data_ptr(), g.data_ptr(), M, int(D),
              float(s_out), int(bit_width), u.data_ptr(), None, err.ptr, _device.stream_ptr())
    uq = _finish(u, as_numpy)
    return QTensor(uq, float(s_out), 0, bit_width), (res.cpu().numpy() if as_numpy else res)


def block_forward_q(u_q, qb):
    """qblock.py:185-215 on the GPU.  u_q.values: (T, d_model) like the reference,
    or (B, T, d_model) for independent sequences (batched extension)."""
    as_numpy = not is_device(u_q.values)
    dev = device_block(qb)
    u = _device.to_device(u_q.values, torch.int8)
    if u.shape[-1] != dev.d_model:
        raise ValueError("qlinear inner dimensions do not match")
    if u.dim() == 2:
        B, T = 1, u.shape[0]
    else:
        B, T = u.shape[0], u.shape[1]
    out = torch.empty(tuple(u.shape[:-1]) + (dev.d_model,), dtype=torch.float32, device=u.device)
    dev.prefill(u, B, T, out, u_scale=float(u_q.scale))
    return _finish(out, as_numpy)


def quantize_weight(w, bit_width: int = 8) -> QTensor:
    """qblock.py:218-220: per-tensor abs-max (host scale) + GPU quantize."""
    return quantize(w, compute_scale_absmax(w, bit_width), bit_width)


def quantize_block(params: SSMParams, cfg: BlockConfig, act: dict, mode: Mode, plan: HadamardPlan,
                   bit_width: int = 8) -> QuantizedBlock:
    """qblock.py:223-240"""
    weights = {name: quantize_weight(getattr(params, name), bit_width) for name in params.tensor_names()}
    if mode.hadamard_output:
        weights["w_out_h"] = quantize_weight(fuse_inverse_into_weights(params.w_out.astype(np.float64), plan),
                                             bit_width)
    return QuantizedBlock(cfg=cfg, mode=mode, weights=weights, act=act, plan=plan)
