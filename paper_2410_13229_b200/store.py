"""Container -> device loader.

Reads the reference's model container -- a UTF-8 JSON manifest line, then a raw
little-endian tensor payload with contiguous offsets (`ssmq/store.py:55-73`
`model_to_bytes`, read back by `:82-173`) -- without materializing the payload:
the file is memory-mapped, every tensor is a zero-copy view of it, and
`load_device_model` hands the int8 views straight to `qmb_block_create`, which
repacks them into the layer's device handle.  In Hadamard-output modes the runtime
needs only the fused `w_out_h`, so `w_out` is never paged in.

Validation follows the reference's reader, with its ValueError texts
(`store.py:82-134`, `calibration.py:142-149`).  Float containers (the reference's
calibration-side FloatModel) are outside this hot path and are refused.
"""
from __future__ import annotations

import json
import os
from pathlib import Path

import numpy as np

from .hadamard import plan_for_dim
from .model import ModelConfig, QuantizedLayer, QuantizedModel
from .qblock import ACT_SITES, MODE_TAGS, QuantizedBlock, ScaleEntry
from .quant import QTensor, QuantScheme, SchemeKind

CONTAINER_VERSION = 1  # store.py:24
SCALESET_VERSION = 1   # calibration.py:112

_DTYPES = {"f32": np.dtype("<f4"), "i8": np.dtype("i1")}  # store.py:26
_SSM_TENSORS = ("a", "d", "w_in", "conv_w", "conv_b", "w_b", "w_c", "w_dt_rank", "w_dt", "dt_bias", "w_out")


class ScaleSet:
    """Mirror of `ssmq.calibration.ScaleSet` (calibration.py:109-153): named static
    scales, read from a container manifest."""

    def __init__(self, bit_width: int = 8):
        self.bit_width = bit_width
        self.entries: dict[str, ScaleEntry] = {}

    def __contains__(self, site: str) -> bool:
        return site in self.entries

    def __getitem__(self, site: str) -> ScaleEntry:
        return self.entries[site]

    def set(self, site: str, entry: ScaleEntry) -> None:
        self.entries[site] = entry

    def to_dict(self) -> dict:
        sites = {name: {"scale": e.scale, "zero_point": e.zero_point, "scheme": e.scheme.kind.value,
                        "p": e.scheme.p} for name, e in self.entries.items()}
        return {"version": SCALESET_VERSION, "bit_width": self.bit_width, "sites": sites}

    @classmethod
    def from_dict(cls, doc: dict) -> "ScaleSet":
        if doc.get("version") != SCALESET_VERSION:
            raise ValueError(f"unsupported scale-set version {doc.get('version')}")
        ss = cls(bit_width=int(doc["bit_width"]))
        for name, rec in doc["sites"].items():
            scheme = QuantScheme(SchemeKind(rec["scheme"]), rec.get("p"))
            ss.set(name, ScaleEntry(float(rec["scale"]), int(rec["zero_point"]), scheme))
        return ss


def _split(path_or_bytes):
    """(manifest dict, payload as a uint8 array): a memory map for a path."""
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        raw = bytes(path_or_bytes)
        head, sep, payload = raw.partition(b"\n")
        if not sep:
            raise ValueError("missing manifest delimiter")
        return json.loads(head.decode("utf-8")), np.frombuffer(payload, dtype=np.uint8)
    path = Path(path_or_bytes)
    with open(path, "rb") as f:
        head = f.readline()
    if not head.endswith(b"\n"):
        raise ValueError("missing manifest delimiter")
    manifest = json.loads(head[:-1].decode("utf-8"))
    size = os.path.getsize(path) - len(head)
    payload = (np.memmap(path, dtype=np.uint8, mode="r", offset=len(head), shape=(size,)) if size > 0
               else np.zeros(0, dtype=np.uint8))
    return manifest, payload


def _views(manifest: dict, payload: np.ndarray) -> dict:
    """store.py:82-103 `_read_tensors`, as zero-copy views of the payload."""
    expected = 0
    out = {}
    for rec in manifest["tensors"]:
        dtype = rec["dtype"]
        if dtype not in _DTYPES:
            raise ValueError(f"unknown dtype {dtype!r} in manifest")
        if rec["byte_offset"] != expected:
            raise ValueError("tensor offsets are not contiguous")
        shape = tuple(rec["shape"])
        np_dtype = _DTYPES[dtype]
        nbytes = int(np.prod(shape, dtype=np.int64)) * np_dtype.itemsize if shape else np_dtype.itemsize
        if nbytes != rec["byte_length"]:
            raise ValueError(f"tensor {rec['name']} length does not match its shape")
        expected += rec["byte_length"]
        if expected > payload.shape[0]:
            raise ValueError("payload length mismatch")
        out[rec["name"]] = payload[rec["byte_offset"]:expected].view(np_dtype).reshape(shape)
    if expected != payload.shape[0]:
        raise ValueError("payload length mismatch")
    return out


def _tensor(tensors: dict, name: str) -> np.ndarray:
    if name not in tensors:
        raise ValueError(f"container is missing tensor {name!r}")
    return tensors[name]


def load_model(path_or_bytes, runtime_only: bool = False) -> QuantizedModel:
    """store.py:106-123 `model_from_bytes` / `load_model` for quantized containers:
    the reference's QuantizedModel structure, tensors as views of the mapped file.
    runtime_only: leave out `w_out` in Hadamard-output modes (the device handle runs
    the fused `w_out_h`), so its bytes are never read."""
    manifest, payload = _split(path_or_bytes)
    if manifest.get("version") != CONTAINER_VERSION:
        raise ValueError(f"unsupported container version {manifest.get('version')}")
    config = ModelConfig(**manifest["config"])
    tensors = _views(manifest, payload)
    tag = manifest["mode"]
    if tag == "float":
        raise ValueError("float containers are the calibration model, not the quantized runtime")
    if tag not in MODE_TAGS:
        raise ValueError(f"unknown mode tag {tag!r}")
    mode = MODE_TAGS[tag]
    scales = ScaleSet.from_dict(manifest["scales"])
    plan = plan_for_dim(config.d_inner)
    bits = config.bit_width
    layers = []
    for idx in range(config.n_layers):  # store.py:151-166 `_build_quantized`
        prefix = f"layers.{idx}."
        names = list(_SSM_TENSORS) + (["w_out_h"] if mode.hadamard_output else [])
        if runtime_only and mode.hadamard_output:
            names.remove("w_out")
        weights = {}
        for name in names:
            entry = scales[prefix + name]
            weights[name] = QTensor(_tensor(tensors, prefix + name), entry.scale, entry.zero_point, bits)
        act = {site: scales[prefix + site] for site in ACT_SITES}
        block = QuantizedBlock(cfg=config.block, mode=mode, weights=weights, act=act, plan=plan)
        layers.append(QuantizedLayer(norm_weight=_tensor(tensors, prefix + "norm_weight"), block=block))
    return QuantizedModel(config=config, mode=mode, embedding=_tensor(tensors, "embedding"), layers=layers,
                          final_norm=_tensor(tensors, "final_norm"), scales=scales)


def load_device_model(path_or_bytes):
    """The container straight into a DeviceModel (one libqmb handle per layer, the
    embedding and norms in HBM)."""
    from .model import device_model

    return device_model(load_model(path_or_bytes, runtime_only=True))
