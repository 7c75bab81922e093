"""GPU calibration: mirror of `ssmq/calibration.py:33-250`.

Static scale collection with the activations, pools and reductions on the GPU:

* `CalibrationStats` / `SiteStats` (calibration.py:33-90): per-site abs-max (a
  max is exact in any order) and the pooled |x| values, kept on the device while
  the pool is below POOL_CAP; beyond the cap the reference's seeded reservoir
  (calibration.py:50-62) replaces slots with probability cap/seen.  Its draws are
  the reference's exact sequence of scalar `rng.integers(0, base + i + 1)` calls
  (numpy's bounded-integer generator is not vectorizable without changing the
  stream), made on the host; the pool itself and the slot writes stay on the GPU.
* `finalize_scales` (calibration.py:156-175): abs-max / qmax, or the nearest-rank
  percentile (quant.py:114-139, exact rational rank) as a k-th order statistic of
  the device pool -- the same float64 value numpy's sort returns.
* `run_calibration` (calibration.py:188-211) over `forward_fp` below: the float
  model (model.py:232-259, ssm.py:149-180) on the GPU with the reference's
  observation sites.  Every elementwise step is the library's bit-exact
  restatement (RMSNorm with numpy's pairwise mean, silu via np.exp, softplus via
  glibc expf / log1pf, the scan's expf, the Hadamard transform in the reference's
  f32 operation order, the conv and scan in the reference's loop order); only the
  four matmuls (OpenBLAS sgemm on the host) sum in a different order, so scales
  agree within a relative tolerance (tests/test_calibration.py), not bit for bit.
  Given the same activations the statistics and scales are bit-identical.
* `quantize_model` (calibration.py:214-250): per-tensor abs-max weights with the
  host-exact `qblock.quantize_block`, as the reference does.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _device, _lib
from .hadamard import plan_for_dim
from .model import ModelConfig, QuantizedLayer, QuantizedModel
from .qblock import ACT_SITES, Mode, ScaleEntry, quantize_block
from .quant import DEFAULT_PERCENTILE, SCALE_FLOOR, QuantScheme, SchemeKind, qmax
from .ssm import SSMParams
from .store import ScaleSet

POOL_CAP = 2 ** 22  # calibration.py:30

_ABSMAX = QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX)


def _dev_abs64(activation) -> torch.Tensor:
    t = activation if isinstance(activation, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(activation))
    return t.to(device=_device.device(), dtype=torch.float64).abs().reshape(-1)


class SiteStats:
    """calibration.py:33-67, with the pool on the device."""

    def __init__(self):
        self.absmax = 0.0
        self.count = 0
        self.seen = 0
        self.pool: list[torch.Tensor] = []
        self.pooled = 0

    def add(self, values: torch.Tensor, rng: np.random.Generator) -> None:
        n = int(values.numel())
        self.absmax = max(self.absmax, float(values.max()) if n else 0.0)
        self.count += 1
        self.seen += n
        if self.pooled + n <= POOL_CAP:
            self.pool.append(values)
            self.pooled += n
            return
        flat = torch.cat(self.pool) if self.pool else values.new_empty(0)
        if flat.numel() < POOL_CAP:
            take = POOL_CAP - flat.numel()
            flat = torch.cat([flat, values[:take]])
            values = values[take:]
        nv = int(values.numel())
        base = self.seen - nv
        # the reference's draws, one scalar call per element (calibration.py:57-60)
        js = np.fromiter((rng.integers(0, base + i + 1) for i in range(nv)), dtype=np.int64, count=nv)
        src = np.nonzero(js < POOL_CAP)[0]
        if src.size:
            dst = js[src]
            # sequential semantics: the last element written to a slot wins
            _, last = np.unique(dst[::-1], return_index=True)
            keep = src.size - 1 - last
            flat[torch.from_numpy(dst[keep]).to(flat.device)] = values[torch.from_numpy(src[keep]).to(flat.device)]
        self.pool = [flat]
        self.pooled = int(flat.numel())

    def pooled_values(self) -> torch.Tensor:
        if not self.pool:
            return torch.empty(0, dtype=torch.float64, device=_device.device())
        return torch.sort(torch.cat(self.pool)).values


class CalibrationStats:
    """calibration.py:70-90: per-site statistics accumulated over calibration runs."""

    def __init__(self, seed: int = 0):
        self.sites: dict[str, SiteStats] = {}
        self._rng = np.random.default_rng(seed)

    def observe(self, site: str, activation) -> None:
        self.sites.setdefault(site, SiteStats()).add(_dev_abs64(activation), self._rng)

    def merge(self, other: "CalibrationStats") -> "CalibrationStats":
        """Deterministic shard merge: abs-max by max, pools by concatenation."""
        for site, stats in other.sites.items():
            mine = self.sites.setdefault(site, SiteStats())
            mine.absmax = max(mine.absmax, stats.absmax)
            mine.count += stats.count
            mine.seen += stats.seen
            mine.pool = mine.pool + [t.clone() for t in stats.pool]
            mine.pooled += stats.pooled
        return self


def default_schemes(n_layers: int, p: float = DEFAULT_PERCENTILE) -> dict[str, QuantScheme]:
    """calibration.py:96-106: percentile at every scan input, abs-max elsewhere."""
    schemes = {}
    for layer in range(n_layers):
        for site in ACT_SITES:
            name = f"layers.{layer}.{site}"
            schemes[name] = QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, p) if site == "x" else _ABSMAX
    return schemes


def _percentile_scale(st: SiteStats, p: float, bit_width: int) -> float:
    """quant.py:114-139 on the device pool: sorted(values)[ceil(p n / 100) - 1]."""
    vals = torch.cat(st.pool) if st.pool else None
    n = 0 if vals is None else int(vals.numel())
    if n == 0:
        raise ValueError("empty calibration tensor")
    if not (0.0 < p <= 100.0):
        raise ValueError(f"percentile must lie in (0, 100], got {p}")
    rank = math.ceil(Fraction(p) * n / 100)
    idx = min(max(rank - 1, 0), n - 1)
    v = float(torch.kthvalue(vals, idx + 1).values)
    if v < 0.0:
        raise ValueError("pooled absolute values must be non-negative")
    return SCALE_FLOOR if v == 0.0 else v / qmax(bit_width)


def finalize_scales(stats: CalibrationStats, schemes: dict, bit_width: int = 8) -> ScaleSet:
    """calibration.py:156-175: resolve per-site scales; every assigned site must
    have been visited."""
    ss = ScaleSet(bit_width=bit_width)
    for site in sorted(schemes):
        scheme = schemes[site]
        if site not in stats.sites or stats.sites[site].count == 0:
            raise ValueError(f"site {site} was never observed during calibration")
        st = stats.sites[site]
        kind = getattr(scheme.kind, "value", scheme.kind)
        if kind == SchemeKind.STATIC_SYMMETRIC_MAX.value:
            scale = st.absmax / qmax(bit_width) if st.absmax > 0 else SCALE_FLOOR
        elif kind == SchemeKind.STATIC_SYMMETRIC_PERCENTILE.value:
            scale = _percentile_scale(st, scheme.p, bit_width)
        else:
            raise ValueError(f"scheme {kind} is not a static calibration scheme")
        ss.set(site, ScaleEntry(scale, 0, QuantScheme(SchemeKind(kind), scheme.p)))
    return ss


def sample_corpus(corpus, num_samples: int, seed: int):
    """calibration.py:178-185: seeded sampling without replacement."""
    if not corpus:
        raise ValueError("empty corpus")
    rng = np.random.default_rng(seed)
    n = min(num_samples, len(corpus))
    idx = rng.choice(len(corpus), size=n, replace=False)
    return [corpus[i] for i in idx]


# --------------------------------------------------------------------------- float model on the device
@dataclass
class LayerParams:
    norm_weight: np.ndarray
    ssm: SSMParams


@dataclass(eq=False)
class FloatModel:
    """model.py:75-93 (the calibration-side float model)."""

    config: ModelConfig
    embedding: np.ndarray
    layers: list
    final_norm: np.ndarray

    @property
    def plan(self):
        return plan_for_dim(self.config.d_inner)


def _f32(a) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(device=_device.device(), dtype=torch.float32).contiguous()


def _math(fn: int, x: torch.Tensor) -> torch.Tensor:
    """qmb_eval_math: the library's bit-exact restatements (1 glibc expf, 3 softplus, 5 silu)."""
    x = x.contiguous()
    y = torch.empty_like(x)
    _lib.call("qmb_eval_math", fn, x.data_ptr(), y.data_ptr(), x.numel(), _device.stream_ptr())
    return y


def _rmsnorm(x: torch.Tensor, gain: torch.Tensor) -> torch.Tensor:
    """ssm.py:104-107 (numpy pairwise mean, IEEE sqrt / div) through the norm kernel."""
    M, D = x.shape
    y = torch.empty_like(x)
    err = _device.err_flag()
    _lib.call("qmb_rmsnorm_residual_quant", x.data_ptr(), None, None, gain.data_ptr(), M, D, 1.0, 8, None,
              y.data_ptr(), err.ptr, _device.stream_ptr())
    return y


def _hadamard_f32(plan, y: torch.Tensor) -> torch.Tensor:
    """apply_hadamard (hadamard.py:128-149) in the reference's f32 order (the kernel's y_h)."""
    M, n = y.shape
    base = np.ascontiguousarray(np.asarray(plan.base, dtype=np.int8))
    yh = torch.empty_like(y)
    q = torch.empty((M, n), dtype=torch.int8, device=y.device)
    err = _device.err_flag()
    _lib.call("qmb_hadamard_quantize", y.data_ptr(), M, int(plan.p), int(plan.m), base.ctypes.data, 1.0, 8,
              q.data_ptr(), yh.data_ptr(), err.ptr, _device.stream_ptr())
    return yh


def _mm(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    return torch.matmul(a, b)  # (TF32 off: _device sets allow_tf32 = False)


def block_forward_fp(u: torch.Tensor, p: dict, plan, observer=None) -> torch.Tensor:
    """ssm.py:149-180 on the device; `observer(site, tensor)` as in the reference."""
    ob = observer if observer is not None else (lambda site, t: t)
    E = p["w_out"].shape[0]
    xz = _mm(u, p["w_in"])
    x_branch = ob("conv_in", xz[:, :E].contiguous())
    z_branch = xz[:, E:].contiguous()
    # causal_conv (_core.pyx:31-43): acc = bias; acc = acc + w[k] * x[t - K + 1 + k]
    T, K = x_branch.shape[0], p["conv_w"].shape[0]
    xp = torch.cat([x_branch.new_zeros(K - 1, E), x_branch])
    acc = p["conv_b"].expand(T, E).clone()
    for k in range(K):
        acc = acc + p["conv_w"][k] * xp[k:k + T]
    x = _math(5, acc)  # silu (ssm.py:98-101)
    x = ob("conv_out", x)
    x = ob("x", x)
    b = ob("b", _mm(x, p["w_b"]))
    c = ob("c", _mm(x, p["w_c"]))
    dt_r = ob("dt_r", _mm(x, p["w_dt_rank"]))
    delta = ob("dt", _math(3, _mm(dt_r, p["w_dt"]) + p["dt_bias"]))  # softplus (ssm.py:93-95)
    # scan_core (_core.pyx:46-65): per t: h = h * expf(dt a) + (dt x) b; acc += h c (j in order)
    ea = _math(1, delta[:, :, None] * p["a"][None])
    h = torch.zeros_like(p["a"])
    N = p["a"].shape[1]
    ys = []
    for t in range(T):
        dbx = delta[t] * x[t]
        h = h * ea[t] + dbx[:, None] * b[t][None, :]
        yt = torch.zeros_like(dbx)
        for j in range(N):
            yt = yt + h[:, j] * c[t, j]
        ys.append(yt + p["d"] * x[t])
    y = torch.stack(ys)
    gated = ob("y", y * _math(5, z_branch))  # gate (ssm.py:110-111)
    if plan is not None and observer is not None:
        ob("y_had", _hadamard_f32(plan, gated))
    return _mm(gated, p["w_out"])


def _device_layers(model):
    cached = model.__dict__.get("_qmb_float_layers")
    if cached is None:
        cached = [dict(norm=_f32(l.norm_weight), **{k: _f32(getattr(l.ssm, k)) for k in
                                                   ("a", "d", "w_in", "conv_w", "conv_b", "w_b", "w_c",
                                                    "w_dt_rank", "w_dt", "dt_bias", "w_out")})
                  for l in model.layers]
        model.__dict__["_qmb_float_layers"] = cached
        model.__dict__["_qmb_float_emb"] = _f32(model.embedding)
    return cached, model.__dict__["_qmb_float_emb"]


def forward_fp(model, tokens, observer=None) -> torch.Tensor:
    """model.py:232-243 up to the final norm: the float residual stream through every
    layer with the observation hooks (the logits are not needed for calibration)."""
    layers, emb = _device_layers(model)
    tok = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=emb.device)
    res = emb[tok]
    plan = plan_for_dim(model.config.d_inner)
    for idx, p in enumerate(layers):
        u = _rmsnorm(res, p["norm"])
        if observer is not None:
            u = observer(f"layers.{idx}.in", u)
        scoped = (lambda i: (lambda site, t: observer(f"layers.{i}." + site, t)))(idx) if observer else None
        res = res + block_forward_fp(u, p, plan, scoped)
    _device.err_flag().raise_if_set()
    return res


def run_calibration(model, corpus, num_samples: int = 512, p: float = DEFAULT_PERCENTILE, seed: int = 42,
                    schemes: dict | None = None) -> ScaleSet:
    """calibration.py:188-211 with the float forward and the statistics on the GPU."""
    stats = CalibrationStats(seed=seed)

    def hook(site, tensor):
        stats.observe(site, tensor)
        return tensor

    for seq in sample_corpus(corpus, num_samples, seed):
        forward_fp(model, seq, observer=hook)
    if schemes is None:
        schemes = default_schemes(model.config.n_layers, p)
    return finalize_scales(stats, schemes, model.config.bit_width)


def quantize_model(model, scales: ScaleSet, mode: Mode) -> QuantizedModel:
    """calibration.py:214-250: per-tensor abs-max weights (host-exact, like the
    reference) and the activation scales bound per mode."""
    cfg = model.config
    bits = cfg.bit_width
    out_scales = ScaleSet(bit_width=bits)
    for name, entry in scales.entries.items():
        out_scales.set(name, entry)
    plan = plan_for_dim(cfg.d_inner)
    qlayers = []
    for idx, layer in enumerate(model.layers):
        prefix = f"layers.{idx}."
        act = {site: scales[prefix + site] for site in ACT_SITES}
        if not mode.percentile_input:
            e = scales[prefix + "conv_out"]
            act["x"] = ScaleEntry(e.scale, 0, _ABSMAX)
            out_scales.set(prefix + "x", act["x"])
        block = quantize_block(layer.ssm, cfg.block, act, mode, plan, bits)
        for wname, wq in block.weights.items():
            out_scales.set(prefix + wname, ScaleEntry(wq.scale, 0, _ABSMAX))
        qlayers.append(QuantizedLayer(norm_weight=np.array(layer.norm_weight, copy=True), block=block))
    return QuantizedModel(config=cfg, mode=mode, embedding=np.array(model.embedding, copy=True), layers=qlayers,
                          final_norm=np.array(model.final_norm, copy=True), scales=out_scales)
