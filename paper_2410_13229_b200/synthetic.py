"""Synthetic random-init W8A8 models for benchmarking at the paper's shapes.

Weights follow the reference's init convention (ssm.py:183-210; model.py:111-124)
but are drawn on the GPU (torch RNG), so a 2.8B-shape model builds in seconds.
Static activation scales come from an offline float calibration pass over a
short synthetic corpus, observed at the reference's sites (ssm.py:149-180;
calibration.py:96-106: percentile at the scan input, abs-max elsewhere).  This
calibration forward is torch float32 (TF32 off): offline tooling, not the
benchmarked path.  Weight quantization (quantize, quantize_f64) runs in libqmb.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import torch

from . import _device, _lib
from .hadamard import plan_for_dim
from .model import ModelConfig, QuantizedLayer, QuantizedModel
from .qblock import ACT_SITES, Mode, QuantizedBlock, ScaleEntry
from .quant import DEFAULT_PERCENTILE, SCALE_FLOOR, QTensor, QuantScheme, SchemeKind

ABSMAX = QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX)

# Mamba-1 reference shapes
CONFIGS = {
    "tiny": ModelConfig(vocab_size=256, d_model=256, n_layers=4, d_state=16, dt_rank=16),
    "130m": ModelConfig(vocab_size=50280, d_model=768, n_layers=24, d_state=16, dt_rank=48),
    "2.8b": ModelConfig(vocab_size=50280, d_model=2560, n_layers=64, d_state=16, dt_rank=160),
}


def _uniform(shape, lo, hi, gen):
    return torch.empty(shape, dtype=torch.float64, device=_device.device()).uniform_(lo, hi, generator=gen)


def _init_block(cfg: ModelConfig, gen) -> dict:
    D, E, N, K, R = cfg.d_model, cfg.d_inner, cfg.d_state, cfg.d_conv, cfg.dt_rank

    def proj(fan_in, shape):
        lim = 1.0 / math.sqrt(fan_in)
        return _uniform(shape, -lim, lim, gen).float()

    a = -torch.exp(_uniform((E, N), 0.0, math.log(N), gen)).float()
    dt_bias = torch.log(torch.expm1(_uniform((E,), 1e-3, 1e-1, gen))).float()
    return dict(a=a, d=torch.ones(E, device=a.device), w_in=proj(D, (D, 2 * E)), conv_w=proj(K, (K, E)),
                conv_b=proj(K, (E,)), w_b=proj(E, (E, N)), w_c=proj(E, (E, N)), w_dt_rank=proj(E, (E, R)),
                w_dt=proj(R, (R, E)), dt_bias=dt_bias, w_out=proj(E, (E, D)))


def _fp32_mm(a, b):
    return torch.matmul(a, b)


def _silu(x):
    return x / (1.0 + torch.exp(-x))


def _rmsnorm(x, g, eps=1e-6):
    return x / torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + eps) * g


def _hadamard_f64(plan, x):
    """H_n x along the last axis in float64 (weight fusion / y_had observation)."""
    base = torch.as_tensor(np.asarray(plan.base, dtype=np.float64), device=x.device)
    blocks = 1 << plan.p
    v = x.to(torch.float64).reshape(-1, blocks, plan.m)
    if plan.m > 1:
        v = v @ base.T
    h = 1
    while h < blocks:
        v4 = v.reshape(v.shape[0], blocks // (2 * h), 2, h, plan.m)
        s = v4[:, :, 0] + v4[:, :, 1]
        d = v4[:, :, 0] - v4[:, :, 1]
        v = torch.stack([s, d], dim=2).reshape(v.shape[0], blocks, plan.m)
        h *= 2
    return v.reshape(x.shape)


def _float_block(u, p, plan, obs):
    """Float block forward with observers (ssm.py:149-180), one sequence u (T, D)."""
    E = p["w_out"].shape[0]
    xz = _fp32_mm(u, p["w_in"])
    x_in, z = xz[:, :E], xz[:, E:]
    obs("conv_in", x_in)
    K = p["conv_w"].shape[0]
    xp = torch.cat([torch.zeros(K - 1, E, device=u.device), x_in])
    conv = p["conv_b"].clone().expand_as(x_in).clone()
    for k in range(K):
        conv = conv + p["conv_w"][k] * xp[k:k + x_in.shape[0]]
    x = _silu(conv)
    obs("conv_out", x)
    obs("x", x)
    b = _fp32_mm(x, p["w_b"])
    c = _fp32_mm(x, p["w_c"])
    dtr = _fp32_mm(x, p["w_dt_rank"])
    obs("b", b)
    obs("c", c)
    obs("dt_r", dtr)
    delta = torch.nn.functional.softplus(_fp32_mm(dtr, p["w_dt"]) + p["dt_bias"])
    obs("dt", delta)
    T = u.shape[0]
    h = torch.zeros_like(p["a"])
    ys = []
    for t in range(T):
        h = h * torch.exp(delta[t][:, None] * p["a"]) + (delta[t] * x[t])[:, None] * b[t][None, :]
        ys.append(h @ c[t] + p["d"] * x[t])
    y = torch.stack(ys)
    gated = y * _silu(z)
    obs("y", gated)
    obs("y_had", _hadamard_f64(plan, gated))
    return _fp32_mm(gated, p["w_out"])


class _Site:
    def __init__(self):
        self.absmax = 0.0
        self.pool = []

    def add(self, t, keep):
        a = t.detach().abs().to(torch.float64).reshape(-1)
        self.absmax = max(self.absmax, float(a.max()))
        if keep:
            self.pool.append(a)

    def percentile(self, p):
        vals = torch.cat(self.pool)
        n = vals.numel()
        rank = math.ceil(Fraction(p) * n / 100)
        idx = min(max(rank - 1, 0), n - 1)
        v = float(torch.kthvalue(vals, idx + 1).values)
        return SCALE_FLOOR if v == 0.0 else v / 127


def _quantize_dev(w: torch.Tensor, bits: int = 8) -> QTensor:
    """Per-tensor abs-max weight quantization (qblock.py:218-220) in libqmb."""
    m = float(w.abs().max().to(torch.float64))
    s = SCALE_FLOOR if m == 0.0 else m / (2 ** (bits - 1) - 1)
    out = torch.empty(w.shape, dtype=torch.int8, device=w.device)
    err = _device.err_flag()
    f64 = w.dtype == torch.float64
    _lib.call("qmb_quantize_f64" if f64 else "qmb_quantize", w.contiguous().data_ptr(), w.numel(), s, bits,
              out.data_ptr(), err.ptr, _device.stream_ptr())
    err.raise_if_set()
    return QTensor(out, s, 0, bits)


@torch.no_grad()
def build_model(cfg: ModelConfig, seed: int = 0, calib_tokens: int = 256, mode: Mode = Mode.FULL,
                p: float = DEFAULT_PERCENTILE) -> QuantizedModel:
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dev = _device.device()
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        lim = 1.0 / math.sqrt(cfg.d_model)
        emb = _uniform((cfg.vocab_size, cfg.d_model), -lim, lim, gen).float()
        plan = plan_for_dim(cfg.d_inner)
        tok = torch.randint(0, cfg.vocab_size, (calib_tokens,), device=dev, generator=gen)
        res = emb[tok]
        layers = []
        for _ in range(cfg.n_layers):
            params = _init_block(cfg, gen)
            norm = torch.ones(cfg.d_model, device=dev)
            sites = {s: _Site() for s in ACT_SITES}
            u = _rmsnorm(res, norm)
            sites["in"].add(u, False)
            out = _float_block(u, params, plan, lambda s, t: sites[s].add(t, s == "x"))
            res = res + out
            act = {}
            for s in ACT_SITES:
                st = sites[s]
                if s == "x" and mode.percentile_input:
                    act[s] = ScaleEntry(st.percentile(p), 0, QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, p))
                else:
                    act[s] = ScaleEntry(st.absmax / 127 if st.absmax > 0 else SCALE_FLOOR, 0, ABSMAX)
            if not mode.percentile_input:
                act["x"] = ScaleEntry(act["conv_out"].scale, 0, ABSMAX)
            weights = {k: _quantize_dev(v, cfg.bit_width) for k, v in params.items()}
            if mode.hadamard_output:
                wh = _hadamard_f64(plan, params["w_out"].to(torch.float64).T.contiguous()).T.contiguous()
                weights["w_out_h"] = _quantize_dev(wh, cfg.bit_width)
            blk = QuantizedBlock(cfg=cfg.block, mode=mode, weights=weights, act=act, plan=plan)
            layers.append(QuantizedLayer(norm_weight=norm, block=blk))
            del params
        return QuantizedModel(config=cfg, mode=mode, embedding=emb, layers=layers,
                              final_norm=torch.ones(cfg.d_model, device=dev))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
