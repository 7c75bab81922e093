"""Reference model containers (ssmq/store.py:55-73 `model_to_bytes`) for the
container -> device loader tests, produced by the REAL reference package.

    bash oracle/build_ref.sh && PYTHONPATH=oracle/_ref python tests/golden/make_containers.py

tiny2 (FULL mode, the same calibration as model_tiny2.npz) and its NAIVE-mode
quantization (no fused w_out_h), with the reference's forward_q logits on a fixed
token sequence for each."""
from __future__ import annotations

from pathlib import Path

import numpy as np
from ssmq import kernels
from ssmq.calibration import quantize_model, run_calibration
from ssmq.model import ModelConfig, forward_q, init_toy_model, inject_outliers, make_corpus
from ssmq.qblock import Mode
from ssmq.store import model_to_bytes

OUT = Path(__file__).resolve().parent


def main():
    assert kernels.backend_name() == "compiled", kernels.backend_name()
    mcfg = ModelConfig(vocab_size=256, d_model=64, n_layers=2, d_state=16, dt_rank=4)
    fm = init_toy_model(mcfg, seed=0)
    info = inject_outliers(fm, np.random.default_rng((0, 1)))
    corpus = make_corpus(mcfg.vocab_size, 8, 64, seed=(0, 2), spike_tokens=info["spike_tokens"])
    scales = run_calibration(fm, corpus, num_samples=8, p=99.999, seed=42)
    tokens = make_corpus(mcfg.vocab_size, 1, 48, seed=(0, 3))[0]
    arrays = {"tokens": tokens}
    for tag, mode in (("full", Mode.FULL), ("naive", Mode.NAIVE)):
        qm = quantize_model(fm, scales, mode)
        raw = model_to_bytes(qm)
        assert model_to_bytes(load_model_bytes(raw)) == raw  # the reference's own round trip
        (OUT / f"container_tiny2_{tag}.ssmq").write_bytes(raw)
        arrays[f"logits_{tag}"] = forward_q(qm, tokens)
        print(tag, len(raw), "bytes")
    np.savez_compressed(OUT / "container_tiny2_logits.npz", **arrays)


def load_model_bytes(raw):
    from ssmq.store import model_from_bytes
    return model_from_bytes(raw)


if __name__ == "__main__":
    main()
