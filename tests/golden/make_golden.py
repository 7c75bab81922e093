"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container (the reference is not available on the GPU box):

    cp -r /root/reference/pkg /tmp/ref/pkg && (cd /tmp/ref/pkg && python setup.py build_ext --inplace)
    SSMQ_REF=/tmp/ref/pkg/src python tests/golden/make_golden.py

Every fixture records the reference's own outputs for its own public
functions (block stage replay per qblock.py:185-215, forward_q per
model.py:246-258), with the compiled Cython backend asserted.  Large weights
are not stored: they are regenerated from the recorded seed with the
reference's init convention and pinned by SHA-256 of the reference's int8
bytes.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("SSMQ_REF", "/tmp/ref/pkg/src")
sys.path.insert(0, REF)

import ssmq.hadamard as H  # noqa: E402

H.MAX_TRANSFORM_DIM = 8192  # the 2.8B shape (d_inner 5120) needs the limit raised

from ssmq import kernels  # noqa: E402
from ssmq.calibration import quantize_model, run_calibration  # noqa: E402
from ssmq.hadamard import apply_hadamard, plan_for_dim  # noqa: E402
from ssmq.model import ModelConfig, forward_q, init_toy_model, inject_outliers, make_corpus  # noqa: E402
from ssmq.qblock import (ACT_SITES, Mode, ScaleEntry, fused_qconv, fused_rmsnorm_quant, qlinear,  # noqa: E402
                         quantize_block, quantized_selective_scan)
from ssmq.quant import QTensor, QuantScheme, SchemeKind, compute_scale_absmax, dequantize, quantize  # noqa: E402
from ssmq.ssm import BlockConfig, block_forward_fp, gate, init_block_params, scan_core, softplus  # noqa: E402

assert kernels.backend_name() == "compiled", "build the reference's Cython core first"

OUT = Path(__file__).resolve().parent
ABSMAX = QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def stage_replay(u_q, qb) -> dict:
    """Reference functions called in the order of block_forward_q (qblock.py:192-215)."""
    n_bits = qb.bit_width
    w_in = qb.weights["w_in"]
    acc = u_q.values.astype(np.int32) @ w_in.values.astype(np.int32)
    s_lin = np.float32(u_q.scale * w_in.scale)
    E = qb.cfg.d_inner
    x_real = acc[:, :E].astype(np.float32) * s_lin
    z = acc[:, E:].astype(np.float32) * s_lin
    x_q = quantize(x_real, qb.act["conv_in"].scale, n_bits)
    scan_x = fused_qconv(x_q, qb.weights["conv_w"], qb.weights["conv_b"], qb.act["x"].scale)
    b_q = qlinear(scan_x, qb.weights["w_b"], s_out=qb.act["b"].scale)
    c_q = qlinear(scan_x, qb.weights["w_c"], s_out=qb.act["c"].scale)
    dtr_q = qlinear(scan_x, qb.weights["w_dt_rank"], s_out=qb.act["dt_r"].scale)
    dt_real = qlinear(dtr_q, qb.weights["w_dt"], bias_q=qb.weights["dt_bias"])
    delta_q = quantize(softplus(dt_real), qb.act["dt"].scale, n_bits)
    y = quantized_selective_scan(qb.weights["a"], b_q, c_q, qb.weights["d"], delta_q, scan_x)
    _, h = scan_core(dequantize(scan_x), dequantize(delta_q), dequantize(b_q), dequantize(c_q),
                     dequantize(qb.weights["a"]), dequantize(qb.weights["d"]))
    gated = gate(y, z)
    if qb.mode.hadamard_output:
        from ssmq.hadamard import hadamard_quantize
        y_q = hadamard_quantize(gated, qb.act["y_had"].scale, qb.plan, n_bits)
        out = qlinear(y_q, qb.weights["w_out_h"], extra_scale=1.0 / qb.plan.n)
    else:
        y_q = quantize(gated, qb.act["y"].scale, n_bits)
        out = qlinear(y_q, qb.weights["w_out"])
    from ssmq.qblock import block_forward_q
    ref_out = block_forward_q(u_q, qb)
    assert np.array_equal(ref_out, out), "stage replay must equal block_forward_q"
    return dict(x_q=x_q.values, z=z, scan_x=scan_x.values, b_q=b_q.values, c_q=c_q.values, dtr_q=dtr_q.values,
                dt_real=dt_real, delta_q=delta_q.values, y=y, h=h, gated=gated, y_q=y_q.values, out=out)


def calibrated_block(cfg, seed, mode, T, p=99.9, outliers=False, u_seed=None):
    params = init_block_params(cfg, np.random.default_rng(seed))
    if outliers:
        params.a[1, :] = -0.005
        params.w_in[:, 3] *= 8.0
    rng = np.random.default_rng(seed + 1000 if u_seed is None else u_seed)
    u = rng.uniform(-1, 1, size=(T, cfg.d_model)).astype(np.float32)
    plan = plan_for_dim(cfg.d_inner)
    observed = {}

    def ob(site, t):
        observed.setdefault(site, []).append(np.asarray(t))
        return t

    block_forward_fp(u, params, plan=plan, observer=ob)
    s_in = compute_scale_absmax(u)
    act = {"in": ScaleEntry(s_in, 0, ABSMAX)}
    for site in ACT_SITES[1:]:
        vals = np.concatenate([np.abs(v).ravel() for v in observed[site]])
        if site == "x" and mode.percentile_input:
            from ssmq.quant import compute_scale_percentile
            act[site] = ScaleEntry(compute_scale_percentile(vals, p), 0,
                                   QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, p))
        else:
            act[site] = ScaleEntry(compute_scale_absmax(vals), 0, ABSMAX)
    qb = quantize_block(params, cfg, act, mode, plan)
    u_q = quantize(u, s_in, 8)
    return params, qb, u_q


def block_meta(name, cfg, qb, u_q, seed, extra=None):
    meta = dict(
        name=name, seed=seed,
        cfg=dict(d_model=cfg.d_model, expand=cfg.expand, d_state=cfg.d_state, d_conv=cfg.d_conv,
                 dt_rank=cfg.dt_rank, d_inner=cfg.d_inner),
        mode=qb.mode.value, bit_width=qb.bit_width,
        act={k: v.scale for k, v in qb.act.items()},
        act_scheme={k: [v.scheme.kind.value, v.scheme.p] for k, v in qb.act.items()},
        w_scale={k: v.scale for k, v in qb.weights.items()},
        w_sha={k: sha(v.values) for k, v in qb.weights.items()},
        plan=dict(n=qb.plan.n, p=qb.plan.p, m=qb.plan.m), u_scale=u_q.scale,
    )
    if extra:
        meta.update(extra)
    return meta


def save_block(name, cfg, seed, mode, T, store_weights=True, **kw):
    params, qb, u_q = calibrated_block(cfg, seed, mode, T, **kw)
    st = stage_replay(u_q, qb)
    arrays = {f"st_{k}": v for k, v in st.items()}
    arrays["u_q"] = u_q.values
    arrays["plan_base"] = np.asarray(qb.plan.base, np.int8)
    if store_weights:
        for k, v in qb.weights.items():
            arrays[f"w_{k}"] = v.values
    meta = block_meta(name, cfg, qb, u_q, seed, dict(weights_stored=store_weights, outliers=kw.get("outliers", False)))
    np.savez_compressed(OUT / f"block_{name}.npz", meta=np.array(json.dumps(meta)), **arrays)
    print("block", name, {k: v.shape for k, v in st.items() if hasattr(v, "shape")}["out"])


def model_case(name, mcfg, seed, n_seq, T, outliers, tokens_T, calib_T=None, store_weights=True):
    fm = init_toy_model(mcfg, seed=seed)
    info = None
    if outliers:
        info = inject_outliers(fm, np.random.default_rng((seed, 1)))
    corpus = make_corpus(mcfg.vocab_size, n_seq, calib_T or T, seed=(seed, 2),
                         spike_tokens=info["spike_tokens"] if info else ())
    scales = run_calibration(fm, corpus, num_samples=n_seq, p=99.999, seed=42)
    qm = quantize_model(fm, scales, Mode.FULL)
    tokens = make_corpus(mcfg.vocab_size, 1, tokens_T, seed=(seed, 3))[0]
    logits = forward_q(qm, tokens)
    # per-layer u_q / out via the reference's own ops (model.py:249-258)
    x_out = qm.embedding[tokens]
    x_res = np.zeros_like(x_out)
    layer_arrays = {}
    from ssmq.qblock import block_forward_q
    for i, layer in enumerate(qm.layers):
        u_q, x_res = fused_rmsnorm_quant(x_out, x_res, layer.norm_weight, layer.block.act["in"].scale, 8)
        x_out = block_forward_q(u_q, layer.block)
        layer_arrays[f"l{i}_u_q"] = u_q.values
        layer_arrays[f"l{i}_out"] = x_out
        layer_arrays[f"l{i}_res"] = x_res
    arrays = dict(tokens=tokens, logits=logits, **layer_arrays)
    if store_weights:
        arrays["embedding"] = qm.embedding
        arrays["final_norm"] = qm.final_norm
        for i, layer in enumerate(qm.layers):
            arrays[f"l{i}_norm"] = layer.norm_weight
            for k, v in layer.block.weights.items():
                arrays[f"l{i}_w_{k}"] = v.values
    meta = dict(name=name, seed=seed, config=mcfg.to_dict(), mode="full", outliers=outliers, info=info,
                scales=json.loads(qm.scales.to_json_bytes().decode()),
                w_sha=[{k: sha(v.values) for k, v in layer.block.weights.items()} for layer in qm.layers],
                emb_sha=sha(qm.embedding), plan=dict(p=qm.layers[0].block.plan.p, m=qm.layers[0].block.plan.m),
                weights_stored=store_weights)
    arrays["plan_base"] = np.asarray(qm.layers[0].block.plan.base, np.int8)
    np.savez_compressed(OUT / f"model_{name}.npz", meta=np.array(json.dumps(meta)), **arrays)
    print("model", name, logits.shape)


def transcendental_vectors():
    """Known-answer vectors of the numpy/libm primitives at hard inputs."""
    rng = np.random.default_rng(123)
    x = np.concatenate([
        rng.uniform(-110, 95, 20000), rng.uniform(-20, 20, 20000), rng.uniform(-1, 1, 5000),
        np.array([0.0, -0.0, 1e-30, -1e-30, 88.72283935546875, 88.7228, 88.73, -103.97, -104.0, -87.3, -87.5,
                  np.inf, -np.inf, 1e-8, -1e-8, 0.5, -0.5, 1.0, -1.0]),
    ]).astype(np.float32)
    with np.errstate(all="ignore"):
        exp = np.exp(x)
        sp = softplus(x)
        sil = x / (np.float32(1.0) + np.exp(-x))
    ms = np.random.default_rng(5).standard_normal((64, 2560)).astype(np.float32) * np.float32(3.0)
    mean = np.mean(np.square(ms), axis=-1, keepdims=True)
    np.savez_compressed(OUT / "transcendentals.npz", x=x, np_exp=exp, softplus=sp, silu=sil, ms_rows=ms,
                        ms_mean=mean)


def hadamard_vectors():
    rng = np.random.default_rng(77)
    out = {}
    for n in (16, 96, 160, 512, 1536, 5120):
        plan = plan_for_dim(n)
        y = rng.standard_normal((5, n)).astype(np.float32)
        y[:, 3] *= 100.0
        out[f"y{n}"] = y
        out[f"h{n}"] = apply_hadamard(plan, y)
    out["base12"] = np.asarray(plan_for_dim(96).base, np.int8)
    out["base20"] = np.asarray(plan_for_dim(160).base, np.int8)
    np.savez_compressed(OUT / "hadamard.npz", **out)


def main():
    transcendental_vectors()
    hadamard_vectors()
    save_block("tiny_full", BlockConfig(d_model=8, expand=2, d_state=4, d_conv=3, dt_rank=2), 9, Mode.FULL, 12)
    save_block("m12_full", BlockConfig(d_model=48, d_state=16, d_conv=4, dt_rank=8), 21, Mode.FULL, 40)
    save_block("m20_full", BlockConfig(d_model=80, d_state=16, d_conv=4, dt_rank=6), 22, Mode.FULL, 33,
               outliers=True)
    save_block("p2_naive", BlockConfig(d_model=64, d_state=16, d_conv=4, dt_rank=4), 23, Mode.NAIVE, 50)
    save_block("p2_outhad", BlockConfig(d_model=32, d_state=8, d_conv=4, dt_rank=4), 24, Mode.OUT_HADAMARD, 29)
    save_block("p2_inper", BlockConfig(d_model=32, d_state=16, d_conv=2, dt_rank=3), 25, Mode.IN_PERCENTILE, 31)
    save_block("s130m", BlockConfig(d_model=768, d_state=16, d_conv=4, dt_rank=48), 31, Mode.FULL, 64,
               store_weights=False)
    save_block("s2p8b", BlockConfig(d_model=2560, d_state=16, d_conv=4, dt_rank=160), 32, Mode.FULL, 16,
               store_weights=False)
    model_case("tiny2", ModelConfig(vocab_size=256, d_model=64, n_layers=2, d_state=16, dt_rank=4), 0, 8, 64,
               True, 48)
    model_case("config1", ModelConfig(vocab_size=256, d_model=256, n_layers=4, d_state=16, dt_rank=16), 0, 2, 512,
               False, 512, store_weights=False)


if __name__ == "__main__":
    main()
