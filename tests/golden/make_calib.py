"""Golden calibration fixtures from the REAL reference (ssmq/calibration.py).

    bash oracle/build_ref.sh && PYTHONPATH=oracle/_ref python tests/golden/make_calib.py

1. stats: seeded activations observed in a fixed order by the reference's
   CalibrationStats (one site overflows POOL_CAP, so the seeded reservoir runs),
   finalized with percentile and abs-max schemes -> the ScaleSet.
2. tiny2 end to end: the float tiny2 model (with injected outliers), its
   calibration corpus and run_calibration's ScaleSet.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from calib_plan import stats_activations  # noqa: E402
from ssmq import kernels  # noqa: E402
from ssmq.calibration import CalibrationStats, finalize_scales, run_calibration  # noqa: E402
from ssmq.model import ModelConfig, init_toy_model, inject_outliers, make_corpus  # noqa: E402
from ssmq.quant import QuantScheme, SchemeKind  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    assert kernels.backend_name() == "compiled", kernels.backend_name()
    stats = CalibrationStats(seed=7)
    for site, a in stats_activations():
        stats.observe(site, a)
    pooled = sum(a.size for s, a in stats_activations() if s == "layers.0.x")
    assert pooled > 2 ** 22, pooled  # the reservoir path runs
    schemes = {"layers.0.in": QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX),
               "layers.0.x": QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, 99.999),
               "layers.0.b": QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, 99.0),
               "layers.0.dt": QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, 100.0),
               "layers.0.y": QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX)}
    ss = finalize_scales(stats, schemes, 8)
    out = {"stats_scales": json.dumps(ss.to_dict())}

    mcfg = ModelConfig(vocab_size=256, d_model=64, n_layers=2, d_state=16, dt_rank=4)
    fm = init_toy_model(mcfg, seed=0)
    inject_outliers(fm, np.random.default_rng((0, 1)))  # (the weights recorded below are post-injection)
    corpus = make_corpus(mcfg.vocab_size, 8, 64, seed=(0, 2))
    scales = run_calibration(fm, corpus, num_samples=8, p=99.999, seed=42)
    out["tiny2_scales"] = json.dumps(scales.to_dict())
    out["tiny2_config"] = json.dumps(mcfg.to_dict())
    arrays = {"embedding": fm.embedding, "final_norm": fm.final_norm}
    for i, layer in enumerate(fm.layers):
        arrays[f"l{i}_norm"] = layer.norm_weight
        for k in ("a", "d", "w_in", "conv_w", "conv_b", "w_b", "w_c", "w_dt_rank", "w_dt", "dt_bias", "w_out"):
            arrays[f"l{i}_{k}"] = getattr(layer.ssm, k)
    for j, seq in enumerate(corpus):
        arrays[f"corpus{j}"] = seq
    np.savez_compressed(OUT / "calib.npz", meta=np.array(json.dumps(out)), **arrays)
    print("stats sites", sorted(ss.entries), "tiny2 sites", len(scales.entries))


if __name__ == "__main__":
    main()
