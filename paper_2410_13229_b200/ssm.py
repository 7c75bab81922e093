"""Block configuration and float parameters -- mirror of the config/parameter
part of `ssmq.ssm` (pkg/src/ssmq/ssm.py:18-90, 183-210).  The float block
forward itself is not part of the B200 path (it is the reference's
calibration/oracle model)."""
from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

from .hadamard import plan_for_dim

RMSNORM_EPS = 1e-6  # ssm.py:18


@dataclass(frozen=True)
class BlockConfig:
    d_model: int
    expand: int = 2
    d_state: int = 16
    d_conv: int = 4
    dt_rank: int = 4

    def __post_init__(self):
        for f in fields(self):
            if getattr(self, f.name) <= 0:
                raise ValueError(f"{f.name} must be positive")
        plan_for_dim(self.d_inner)

    @property
    def d_inner(self) -> int:
        return self.expand * self.d_model


@dataclass
class SSMParams:
    """All float weights of one block (shapes as ssm.py:43-54)."""

    a: np.ndarray
    d: np.ndarray
    w_in: np.ndarray
    conv_w: np.ndarray
    conv_b: np.ndarray
    w_b: np.ndarray
    w_c: np.ndarray
    w_dt_rank: np.ndarray
    w_dt: np.ndarray
    dt_bias: np.ndarray
    w_out: np.ndarray

    def tensor_names(self) -> list[str]:
        return [f.name for f in fields(self)]

    def validate(self, cfg: BlockConfig) -> None:
        di, ds = cfg.d_inner, cfg.d_state
        expected = {
            "a": (di, ds), "d": (di,), "w_in": (cfg.d_model, 2 * di), "conv_w": (cfg.d_conv, di),
            "conv_b": (di,), "w_b": (di, ds), "w_c": (di, ds), "w_dt_rank": (di, cfg.dt_rank),
            "w_dt": (cfg.dt_rank, di), "dt_bias": (di,), "w_out": (di, cfg.d_model),
        }
        for name, shape in expected.items():
            got = getattr(self, name).shape
            if got != shape:
                raise ValueError(f"{name} has shape {got}, expected {shape}")
        if not (self.a < 0).all():
            raise ValueError("state transition entries must be strictly negative")


def init_block_params(cfg: BlockConfig, rng: np.random.Generator) -> SSMParams:
    """Seeded synthetic weights with the reference's init convention (ssm.py:183-210):
    a = -exp(U[0, ln N]), dt_bias = softplus^-1(U[1e-3, 1e-1]), projections
    U[+-1/sqrt(fan_in)], d = 1.  Draw order matches the reference so a given seed
    gives the same weights."""

    def proj(fan_in, shape):
        lim = 1.0 / np.sqrt(fan_in)
        return rng.uniform(-lim, lim, size=shape).astype(np.float32)

    di, ds = cfg.d_inner, cfg.d_state
    a = -np.exp(rng.uniform(0.0, np.log(ds), size=(di, ds))).astype(np.float32)
    dt_target = rng.uniform(1e-3, 1e-1, size=di)
    dt_bias = np.log(np.expm1(dt_target)).astype(np.float32)
    return SSMParams(
        a=a,
        d=np.ones(di, dtype=np.float32),
        w_in=proj(cfg.d_model, (cfg.d_model, 2 * di)),
        conv_w=proj(cfg.d_conv, (cfg.d_conv, di)),
        conv_b=proj(cfg.d_conv, (di,)),
        w_b=proj(di, (di, ds)),
        w_c=proj(di, (di, ds)),
        w_dt_rank=proj(di, (di, cfg.dt_rank)),
        w_dt=proj(cfg.dt_rank, (cfg.dt_rank, di)),
        dt_bias=dt_bias,
        w_out=proj(di, (di, cfg.d_model)),
    )
