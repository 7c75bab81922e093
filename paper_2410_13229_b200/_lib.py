"""ctypes binding of libqmb.so (include/qmb.h).

There is no fallback: if the CUDA library or a GPU is missing, every entry
point raises.  Device memory and streams come from torch (plumbing only);
all compute runs in the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# QMB_LIB: an alternative in-tree build of the same ABI (A/B timing of kernel variants, tools/ab_lib.sh)
LIB_PATH = Path(os.environ["QMB_LIB"]) if os.environ.get("QMB_LIB") else PKG / "libqmb.so"

c_i8p = ctypes.c_void_p
c_vp = ctypes.c_void_p
c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_dbl = ctypes.c_double
c_sz = ctypes.c_size_t

QMB_ERR_NONFINITE = 1
QMB_ERR_SCAN = 2
QMB_NUM_ACT = 10
WS_SLOTS = ("UPAD", "XQ", "Z", "SCANX", "B", "C", "DTR", "DELTA", "YQ", "BCF", "ACC32")


class QWeight(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("scale", c_dbl)]


class BlockDesc(ctypes.Structure):
    _fields_ = [
        ("d_model", c_int), ("d_inner", c_int), ("d_state", c_int), ("d_conv", c_int), ("dt_rank", c_int),
        ("bit_width", c_int), ("mode", c_int),
        ("act", c_dbl * QMB_NUM_ACT),
        ("a", QWeight), ("d", QWeight), ("w_in", QWeight), ("conv_w", QWeight), ("conv_b", QWeight),
        ("w_b", QWeight), ("w_c", QWeight), ("w_dt_rank", QWeight), ("w_dt", QWeight), ("dt_bias", QWeight),
        ("w_out", QWeight), ("w_out_h", QWeight),
        ("had_p", c_int), ("had_m", c_int), ("had_base", ctypes.c_void_p),
    ]


class TpArgs(ctypes.Structure):  # qmb_tp_args
    _fields_ = [("stage", c_int), ("xacc", ctypes.c_void_p), ("y_local", ctypes.c_void_p),
                ("y_full", ctypes.c_void_p), ("yq_full", ctypes.c_void_p), ("e_full", ctypes.c_longlong),
                ("e0", c_int), ("had_p", c_int), ("had_m", c_int), ("had_base", ctypes.c_void_p),
                ("oacc", ctypes.c_void_p)]


# name -> (restype, argtypes); must match include/qmb.h exactly
PROTOTYPES = {
    "qmb_abi_version": (c_int, []),
    "qmb_last_error": (ctypes.c_char_p, []),
    "qmb_block_create": (c_int, [ctypes.POINTER(BlockDesc), ctypes.POINTER(c_vp)]),
    "qmb_block_destroy": (None, [c_vp]),
    "qmb_block_workspace_bytes": (c_sz, [c_vp, c_ll]),
    "qmb_block_workspace_layout": (c_int, [c_vp, c_ll, ctypes.POINTER(c_sz)]),
    "qmb_block_prefill": (c_int, [c_vp, c_i8p, c_dbl, c_int, c_int, c_vp, c_i8p, c_vp, c_int, c_vp, c_sz, c_vp, c_vp]),
    "qmb_block_decode": (c_int, [c_vp, c_i8p, c_dbl, c_int, c_i8p, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "qmb_block_prefill_accum": (c_int, [c_vp, c_i8p, c_dbl, c_int, c_int, c_vp, c_i8p, c_vp, c_int, c_vp, c_sz, c_vp,
                                        c_vp]),
    "qmb_block_decode_accum": (c_int, [c_vp, c_i8p, c_dbl, c_int, c_i8p, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "qmb_block_prefill_profiled": (c_int, [c_vp, c_i8p, c_dbl, c_int, c_int, c_vp, c_int, c_vp, c_sz, c_vp, c_vp,
                                           ctypes.POINTER(ctypes.c_float)]),
    "qmb_rmsnorm_residual_quant":(c_int, [c_vp, c_vp, c_vp, c_vp, c_ll, c_int, c_dbl, c_int, c_i8p, c_vp, c_vp,
                                           c_vp]),
    "qmb_quantize": (c_int, [c_vp, c_ll, c_dbl, c_int, c_i8p, c_vp, c_vp]),
    "qmb_quantize_f64": (c_int, [c_vp, c_ll, c_dbl, c_int, c_i8p, c_vp, c_vp]),
    "qmb_qlinear_workspace_bytes":(c_sz, [c_ll, c_int, c_int]),
    "qmb_qlinear": (c_int, [c_i8p, c_ll, c_int, c_dbl, c_i8p, c_int, c_dbl, c_i8p, c_dbl, c_dbl, c_dbl, c_int,
                            c_vp, c_vp, c_sz, c_int, c_vp, c_vp]),
    "qmb_fused_qconv": (c_int, [c_i8p, c_int, c_int, c_int, c_dbl, c_i8p, c_int, c_dbl, c_i8p, c_dbl, c_dbl, c_int,
                                c_i8p, c_vp, c_vp]),
    "qmb_selective_scan": (c_int, [c_i8p, c_dbl, c_i8p, c_dbl, c_i8p, c_dbl, c_i8p, c_dbl, c_i8p, c_dbl, c_i8p,
                                   c_dbl, c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "qmb_selective_scan_workspace_bytes": (c_sz, [c_int, c_int]),
    "qmb_block_tp_stage": (c_int, [c_vp, ctypes.POINTER(TpArgs), c_vp, c_dbl, c_int, c_int, c_int, c_vp, c_vp, c_vp,
                                   c_int, c_vp, c_sz, c_vp, c_vp]),
    "qmb_hadamard_quantize": (c_int, [c_vp, c_ll, c_int, c_int, c_i8p, c_dbl, c_int, c_i8p, c_vp, c_vp, c_vp]),
    "qmb_measure_i8_peak": (c_int, [c_int, ctypes.POINTER(c_dbl)]),
    "qmb_gemm_bench": (c_int, [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(ctypes.c_float)]),
    "qmb_eval_math":(c_int, [c_int, c_vp, c_vp, c_ll, c_vp]),
    "qmb_verify_math":(c_int, [c_int, c_int, c_vp, c_vp, c_vp]),
    "qmb_embed_gather": (c_int, [c_vp, c_vp, c_ll, c_int, c_vp, c_vp]),
    "qmb_lm_head": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_vp, c_vp]),
    "qmb_lm_split16": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp]),
    "qmb_argmax": (c_int, [c_vp, c_int, c_int, c_ll, c_vp, c_vp]),
    "qmb_lm_combine16": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_vp, c_vp]),
}

_lib = None


class QmbError(RuntimeError):
    pass


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libqmb.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise QmbError(f"libqmb.so not built at {p}; run __graft_entry__.build()")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.qmb_abi_version() != 1:
        raise QmbError("libqmb ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = _lib.qmb_last_error().decode() if _lib is not None else ""
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise NotImplementedError(msg)
    if rc == -3:
        raise MemoryError(msg)
    raise QmbError(f"{what}: CUDA error {rc}: {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)
