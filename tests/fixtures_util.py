"""Build oracle / product blocks and models from the golden fixtures."""
from __future__ import annotations

import hashlib
import json

import numpy as np

from conftest import load_npz

WEIGHT_NAMES = ("a", "d", "w_in", "conv_w", "conv_b", "w_b", "w_c", "w_dt_rank", "w_dt", "dt_bias", "w_out")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _absmax_scale(w) -> float:
    m = float(np.max(np.abs(np.asarray(w, dtype=np.float64))))
    return 1e-8 if m == 0.0 else m / 127


def regen_block_weights(meta) -> dict:
    """Regenerate a block's int8 weights from its seed (reference init convention,
    ssm.py:183-210; per-tensor abs-max, qblock.py:218-240) on the host."""
    from oracle import oracle as o
    from paper_2410_13229_b200.hadamard import fuse_inverse_into_weights, plan_for_dim
    from paper_2410_13229_b200.ssm import BlockConfig, init_block_params

    c = meta["cfg"]
    cfg = BlockConfig(d_model=c["d_model"], expand=c["expand"], d_state=c["d_state"], d_conv=c["d_conv"],
                      dt_rank=c["dt_rank"])
    params = init_block_params(cfg, np.random.default_rng(meta["seed"]))
    if meta.get("outliers"):
        params.a[1, :] = -0.005
        params.w_in[:, 3] *= 8.0
    out = {}
    for name in WEIGHT_NAMES:
        w = getattr(params, name)
        s = _absmax_scale(w)
        out[name] = (o.quantize(w, s), s)
    if meta["mode"] in ("out_hadamard", "full"):
        wh = fuse_inverse_into_weights(params.w_out.astype(np.float64), plan_for_dim(cfg.d_inner))
        s = _absmax_scale(wh)
        out["w_out_h"] = (o.quantize(wh, s), s)
    return out


def block_weights(z, meta) -> dict:
    if meta.get("weights_stored", True):
        return {k: (z[f"w_{k}"], meta["w_scale"][k]) for k in meta["w_scale"]}
    return regen_block_weights(meta)


def oracle_block(z, meta, weights=None):
    from oracle import oracle as o

    w = weights or block_weights(z, meta)
    cfg = dict(meta["cfg"], bit_width=meta["bit_width"])
    return o.Block(cfg, meta["mode"], w, dict(meta["act"]), (meta["plan"]["p"], meta["plan"]["m"], z["plan_base"]))


def mirror_block(z, meta, weights=None):
    """The product's QuantizedBlock mirror built from fixture data (numpy values)."""
    from paper_2410_13229_b200 import hadamard as H
    from paper_2410_13229_b200.qblock import Mode, QuantizedBlock, ScaleEntry
    from paper_2410_13229_b200.quant import QTensor, QuantScheme, SchemeKind
    from paper_2410_13229_b200.ssm import BlockConfig

    w = weights or block_weights(z, meta)
    c = meta["cfg"]
    cfg = BlockConfig(d_model=c["d_model"], expand=c["expand"], d_state=c["d_state"], d_conv=c["d_conv"],
                      dt_rank=c["dt_rank"])
    act = {}
    for site, s in meta["act"].items():
        kind, p = meta["act_scheme"][site]
        act[site] = ScaleEntry(s, 0, QuantScheme(SchemeKind(kind), p))
    weights_q = {k: QTensor(v, float(s), 0, meta["bit_width"]) for k, (v, s) in w.items()}
    plan = H.HadamardPlan(meta["plan"]["n"], meta["plan"]["p"], meta["plan"]["m"], np.array(z["plan_base"]))
    return QuantizedBlock(cfg=cfg, mode=Mode(meta["mode"]), weights=weights_q, act=act, plan=plan)


BLOCK_FIXTURES = ["tiny_full", "m12_full", "m20_full", "p2_naive", "p2_outhad", "p2_inper", "s130m", "s2p8b"]
SMALL_BLOCKS = BLOCK_FIXTURES[:6]


def load_block(name):
    return load_npz(f"block_{name}.npz")


# ----------------------------------------------------------------------------- models
def regen_model(meta):
    """Regenerate a float toy model with the reference convention (model.py:111-124)
    and quantize it with the fixture's ScaleSet (calibration.py:214-250)."""
    from paper_2410_13229_b200.hadamard import fuse_inverse_into_weights, plan_for_dim
    from paper_2410_13229_b200.ssm import BlockConfig, init_block_params
    from oracle import oracle as o

    c = meta["config"]
    rng = np.random.default_rng(meta["seed"])
    lim = 1.0 / np.sqrt(c["d_model"])
    emb = rng.uniform(-lim, lim, size=(c["vocab_size"], c["d_model"])).astype(np.float32)
    cfg = BlockConfig(d_model=c["d_model"], expand=c["expand"], d_state=c["d_state"], d_conv=c["d_conv"],
                      dt_rank=c["dt_rank"])
    plan = plan_for_dim(cfg.d_inner)
    layers = []
    for _ in range(c["n_layers"]):
        params = init_block_params(cfg, rng)
        layers.append(params)
    assert not meta["outliers"], "outlier models are stored with weights"
    blocks = []
    for i, params in enumerate(layers):
        w = {}
        for name in WEIGHT_NAMES:
            arr = getattr(params, name)
            s = _absmax_scale(arr)
            w[name] = (o.quantize(arr, s), s)
        wh = fuse_inverse_into_weights(params.w_out.astype(np.float64), plan)
        s = _absmax_scale(wh)
        w["w_out_h"] = (o.quantize(wh, s), s)
        blocks.append(w)
    norms = [np.ones(c["d_model"], np.float32) for _ in range(c["n_layers"])]
    return emb, norms, np.ones(c["d_model"], np.float32), blocks


def model_parts(z, meta):
    c = meta["config"]
    if meta.get("weights_stored", True):
        emb = z["embedding"]
        norms = [z[f"l{i}_norm"] for i in range(c["n_layers"])]
        final = z["final_norm"]
        blocks = []
        for i in range(c["n_layers"]):
            w = {}
            for k in list(WEIGHT_NAMES) + ["w_out_h"]:
                key = f"l{i}_w_{k}"
                if key in z.files:
                    w[k] = (z[key], meta["scales"]["sites"][f"layers.{i}.{k}"]["scale"])
            blocks.append(w)
        return emb, norms, final, blocks
    return regen_model(meta)


def layer_act(meta, i) -> dict:
    sites = meta["scales"]["sites"]
    return {s: sites[f"layers.{i}.{s}"]["scale"] for s in
            ("in", "conv_in", "conv_out", "x", "b", "c", "dt_r", "dt", "y", "y_had")}


def oracle_model(z, meta):
    from oracle import oracle as o

    emb, norms, final, blocks = model_parts(z, meta)
    c = meta["config"]
    cfg = dict(d_model=c["d_model"], d_inner=c["d_model"] * c["expand"], d_state=c["d_state"], d_conv=c["d_conv"],
               dt_rank=c["dt_rank"], bit_width=c["bit_width"])
    ob = [o.Block(cfg, "full", w, layer_act(meta, i), (meta["plan"]["p"], meta["plan"]["m"], z["plan_base"]))
          for i, w in enumerate(blocks)]
    return o.Model(emb, norms, ob, final, c["bit_width"])


def mirror_model(z, meta):
    from paper_2410_13229_b200 import hadamard as H
    from paper_2410_13229_b200.model import ModelConfig, QuantizedLayer, QuantizedModel
    from paper_2410_13229_b200.qblock import Mode, QuantizedBlock, ScaleEntry
    from paper_2410_13229_b200.quant import QTensor, QuantScheme, SchemeKind

    emb, norms, final, blocks = model_parts(z, meta)
    c = meta["config"]
    mcfg = ModelConfig(**c)
    plan = H.HadamardPlan(mcfg.d_inner, meta["plan"]["p"], meta["plan"]["m"], np.array(z["plan_base"]))
    sites = meta["scales"]["sites"]
    layers = []
    for i, w in enumerate(blocks):
        act = {}
        for s in ("in", "conv_in", "conv_out", "x", "b", "c", "dt_r", "dt", "y", "y_had"):
            rec = sites[f"layers.{i}.{s}"]
            act[s] = ScaleEntry(rec["scale"], 0, QuantScheme(SchemeKind(rec["scheme"]), rec["p"]))
        wq = {k: QTensor(v, float(s), 0, c["bit_width"]) for k, (v, s) in w.items()}
        qb = QuantizedBlock(cfg=mcfg.block, mode=Mode.FULL, weights=wq, act=act, plan=plan)
        layers.append(QuantizedLayer(norm_weight=norms[i], block=qb))
    return QuantizedModel(config=mcfg, mode=Mode.FULL, embedding=emb, layers=layers, final_norm=final)


def json_meta(meta):
    return json.dumps(meta)[:200]
