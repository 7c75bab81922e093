"""Container -> device loader: the reference's own containers
(tests/golden/make_containers.py) parsed without copies, validated with the
reference's errors (ssmq/store.py:82-134), and run on the device."""
import json
from pathlib import Path

import numpy as np
import pytest

from fixtures_util import load_npz

GOLD = Path(__file__).resolve().parent / "golden"


def _fixture_model():
    z, meta = load_npz("model_tiny2.npz")
    return z, meta


@pytest.mark.parametrize("tag", ["full", "naive"])
def test_container_tensors_and_scales_match_reference(tag):
    from paper_2410_13229_b200.store import load_model

    qm = load_model(GOLD / f"container_tiny2_{tag}.ssmq")
    z, meta = _fixture_model()
    assert qm.config.to_dict() == meta["config"]
    assert np.array_equal(qm.embedding, z["embedding"]) and np.array_equal(qm.final_norm, z["final_norm"])
    sites = meta["scales"]["sites"]
    for i, layer in enumerate(qm.layers):
        assert np.array_equal(layer.norm_weight, z[f"l{i}_norm"])
        for k, w in layer.block.weights.items():  # (both modes quantize with the same scales)
            assert w.scale == sites[f"layers.{i}.{k}"]["scale"]
            assert np.array_equal(np.asarray(w.values), z[f"l{i}_w_{k}"]), (i, k)
        for site, e in layer.block.act.items():
            assert e.scale == sites[f"layers.{i}.{site}"]["scale"]
    assert ("w_out_h" in qm.layers[0].block.weights) == (tag == "full")


def test_container_runtime_only_skips_unfused_out_proj():
    from paper_2410_13229_b200.store import load_model

    qm = load_model(GOLD / "container_tiny2_full.ssmq", runtime_only=True)
    assert "w_out" not in qm.layers[0].block.weights and "w_out_h" in qm.layers[0].block.weights


def _corrupt(raw: bytes, fn) -> bytes:
    head, _, payload = raw.partition(b"\n")
    man = json.loads(head)
    payload = fn(man, payload)
    return json.dumps(man).encode() + b"\n" + payload


@pytest.mark.parametrize("case,msg", [
    ("no_delim", "missing manifest delimiter"),
    ("version", "unsupported container version 2"),
    ("dtype", "unknown dtype 'f16' in manifest"),
    ("offset", "tensor offsets are not contiguous"),
    ("length", "length does not match its shape"),
    ("truncated", "payload length mismatch"),
    ("trailing", "payload length mismatch"),
    ("mode", "unknown mode tag 'bogus'"),
    ("scales", "unsupported scale-set version 7"),
    ("missing", "container is missing tensor 'layers.1.w_c'"),
])
def test_container_validation_errors(case, msg):
    from paper_2410_13229_b200.store import load_model

    raw = (GOLD / "container_tiny2_full.ssmq").read_bytes()
    if case == "no_delim":
        bad = raw.partition(b"\n")[0]
    else:
        def edit(man, payload):
            t = man["tensors"]
            if case == "version":
                man["version"] = 2
            elif case == "dtype":
                t[0]["dtype"] = "f16"
            elif case == "offset":
                t[1]["byte_offset"] += 4
            elif case == "length":
                t[0]["byte_length"] += 4
            elif case == "truncated":
                payload = payload[:-1]
            elif case == "trailing":
                payload = payload + b"\0"
            elif case == "mode":
                man["mode"] = "bogus"
            elif case == "scales":
                man["scales"]["version"] = 7
            elif case == "missing":
                i = next(k for k, r in enumerate(t) if r["name"] == "layers.1.w_c")
                n = t[i]["byte_length"]
                del t[i]
                for r in t[i:]:
                    r["byte_offset"] -= n
                off = sum(r["byte_length"] for r in t[:i])
                payload = payload[:off] + payload[off + n:]
            return payload
        bad = _corrupt(raw, edit)
    with pytest.raises(ValueError, match=msg):
        load_model(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["full", "naive"])
def test_container_device_model_logits(cuda, tag):
    """load_device_model -> forward: hidden states bit-exact with the same model
    built from the fixture arrays; logits within the LM-head tolerance of the
    reference's forward_q on the same container."""
    import torch

    from paper_2410_13229_b200.store import load_device_model

    ref = np.load(GOLD / "container_tiny2_logits.npz")
    dm = load_device_model(GOLD / f"container_tiny2_{tag}.ssmq")
    tok = torch.from_numpy(ref["tokens"].astype(np.int64)).cuda()[None]
    logits = dm.forward(tok)[0].cpu().numpy()
    want = ref[f"logits_{tag}"]
    assert logits.shape == want.shape
    assert np.max(np.abs(logits - want)) <= 1e-5 * np.max(np.abs(want))
    assert np.array_equal(logits.argmax(-1), want.argmax(-1))
