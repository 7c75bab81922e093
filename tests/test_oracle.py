"""Pin the CPU oracle (oracle/) against the reference: golden fixtures produced
by the real reference package (tests/golden/make_golden.py), the reference
tests' hand-derived known answers, and the host's live numpy / libm."""
import numpy as np
import pytest

from conftest import load_npz
from fixtures_util import (BLOCK_FIXTURES, block_weights, layer_act, load_block, model_parts, oracle_block,
                           oracle_model, sha)

STAGES = ("x_q", "z", "scan_x", "b_q", "c_q", "dtr_q", "dt_real", "delta_q", "y", "h", "gated", "y_q", "out")


# ----------------------------------------------------------------- transcendentals
def test_np_exp_restatement_matches_live_numpy(oracle):
    bits = np.arange(0, 1 << 32, 997, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    with np.errstate(all="ignore"):
        ref = np.exp(x)
    got = oracle.np_exp(x)
    bad = (got.view(np.uint32) != ref.view(np.uint32)) & ~(np.isnan(got) & np.isnan(ref))
    assert bad.sum() == 0


def test_glibc_expf_log1pf_restatements_match_libm(oracle):
    L = oracle.lib()
    assert L.oracle_count_expf_mismatch(0, 1 << 32, 997) == 0
    assert L.oracle_count_log1pf_mismatch(0, 1 << 32, 997) == 0


def test_softplus_silu_match_numpy(oracle):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-40, 40, 200000), rng.uniform(-1, 1, 50000)]).astype(np.float32)
    with np.errstate(all="ignore"):
        sp = np.logaddexp(x, np.float32(0))
        si = x / (np.float32(1.0) + np.exp(-x))
    assert np.array_equal(oracle.softplus(x).view(np.uint32), sp.view(np.uint32))
    assert np.array_equal(oracle.silu(x).view(np.uint32), si.view(np.uint32))


def test_transcendental_golden_vectors(oracle):
    z, _ = load_npz("transcendentals.npz")
    x = z["x"]
    for name, fn in (("np_exp", oracle.np_exp), ("softplus", oracle.softplus), ("silu", oracle.silu)):
        got, ref = fn(x), z[name]
        same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
        assert same.all(), name


def test_pairwise_mean_matches_numpy(oracle):
    z, _ = load_npz("transcendentals.npz")
    rows = z["ms_rows"]
    g = np.ones(rows.shape[1], np.float32)
    # rmsnorm(x, 1) = x / sqrt(mean + eps): equal iff the means are equal
    ref = rows / np.sqrt(z["ms_mean"] + 1e-6) * g
    assert np.array_equal(oracle.rmsnorm(rows, g), ref)
    rng = np.random.default_rng(3)
    for n in (1, 5, 8, 13, 64, 127, 128, 129, 200, 256, 768, 1000, 2560, 4096, 5120):
        x = (rng.standard_normal((7, n)) * rng.uniform(0.01, 100, (7, 1))).astype(np.float32)
        gain = rng.uniform(0.5, 1.5, n).astype(np.float32)
        from numpy import sqrt
        ms = np.mean(np.square(x), axis=-1, keepdims=True)
        ref = x / sqrt(ms + 1e-6) * gain
        assert np.array_equal(oracle.rmsnorm(x, gain), ref), n


# ----------------------------------------------------------------- known answers (reference tests)
def test_quantize_known_answers(oracle):
    # test_quant.py:103-124
    assert oracle.quantize(np.array([0.5, -1.0, 2.54], np.float32), 0.02).tolist() == [25, -50, 127]
    assert oracle.quantize(np.array([0.03]), 0.02).tolist() == [2]  # half-to-even tie
    with pytest.raises(ValueError, match="non-finite"):
        oracle.quantize(np.array([1.0, np.nan], np.float32), 0.1)


def test_qlinear_scalar_known_answer(oracle):
    # test_qblock.py:40-42
    out = oracle.qlinear(np.array([[1]], np.int8), 0.5, np.array([[2]], np.int8), 0.25)
    assert out[0, 0] == np.float32(0.25)


def test_scan_near_ln2(oracle):
    # test_qblock.py:165-176 (exact-grid scalar system)
    dt_q = oracle.quantize(np.array([[np.log(2.0)]]), 0.0078125)
    x_q = oracle.quantize(np.array([[1.0]]), 0.0625)
    y, _ = oracle.quantized_scan(np.array([[-1]], np.int8), 1.0, np.array([[1]], np.int8), 1.0,
                                 np.array([[1]], np.int8), 1.0, np.array([0], np.int8), 1.0, dt_q, 0.0078125,
                                 x_q, 0.0625)
    assert abs(float(y[0, 0]) - np.log(2.0)) <= 0.0625


def test_hadamard_spike_is_flat(oracle):
    # test_hadamard.py:199-206: a spike transforms to a flat vector
    from paper_2410_13229_b200.hadamard import plan_for_dim

    plan = plan_for_dim(4)
    y = np.array([[64.0, 0, 0, 0]], np.float32)
    assert oracle.hadamard(y, plan.p, plan.m, plan.base).tolist() == [[64.0, 64.0, 64.0, 64.0]]


def test_hadamard_golden(oracle):
    z, _ = load_npz("hadamard.npz")
    from paper_2410_13229_b200.hadamard import plan_for_dim

    for n in (16, 96, 160, 512, 1536, 5120):
        plan = plan_for_dim(n)
        assert np.array_equal(oracle.hadamard(z[f"y{n}"], plan.p, plan.m, plan.base), z[f"h{n}"]), n


def test_scan_carried_state_equals_one_shot(oracle):
    # test_formats.py:76-94
    rng = np.random.default_rng(0)
    T, d, n = 12, 3, 2
    x = rng.standard_normal((T, d)).astype(np.float32)
    delta = np.exp(rng.uniform(-3, -1, (T, d))).astype(np.float32)
    a = (-np.exp(rng.uniform(-1, 1, (d, n)))).astype(np.float32)
    b = rng.standard_normal((T, n)).astype(np.float32)
    c = rng.standard_normal((T, n)).astype(np.float32)
    dv = rng.standard_normal(d).astype(np.float32)
    full, h_full = oracle.scan(x, delta, b, c, a, dv)
    h = None
    ys = []
    for t in range(T):
        y, h = oracle.scan(x[t:t + 1], delta[t:t + 1], b[t:t + 1], c[t:t + 1], a, dv, h)
        ys.append(y)
    assert np.array_equal(np.concatenate(ys), full) and np.array_equal(h, h_full)


# ----------------------------------------------------------------- golden block / model replays
@pytest.mark.parametrize("name", BLOCK_FIXTURES)
def test_block_stage_replay_matches_reference(oracle, name):
    z, meta = load_block(name)
    w = block_weights(z, meta)
    for k, (v, s) in w.items():
        assert sha(v) == meta["w_sha"][k], f"weight prep differs from the reference: {k}"
        assert s == meta["w_scale"][k], k
    blk = oracle_block(z, meta, w)
    st = oracle.block_stages(z["u_q"], meta["u_scale"], blk)
    for k in STAGES:
        got, ref = st[k], z[f"st_{k}"]
        assert got.dtype == ref.dtype and np.array_equal(got, ref), f"{name}: stage {k}"


def test_model_forward_matches_reference(oracle):
    z, meta = load_npz("model_tiny2.npz")
    m = oracle_model(z, meta)
    collect = []
    logits = oracle.forward_q(m, z["tokens"], collect)
    for i, st in enumerate(collect):
        assert np.array_equal(st["u_q"], z[f"l{i}_u_q"]), i
        assert np.array_equal(st["out"], z[f"l{i}_out"]), i
        assert np.array_equal(st["res"], z[f"l{i}_res"]), i
    ref = z["logits"]
    assert np.max(np.abs(logits - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_config1_forward_matches_reference(oracle):
    z, meta = load_npz("model_config1.npz")
    emb, norms, final, blocks = model_parts(z, meta)
    assert sha(emb) == meta["emb_sha"]
    for i, w in enumerate(blocks):
        for k, (v, _) in w.items():
            assert sha(v) == meta["w_sha"][i][k], (i, k)
    m = oracle_model(z, meta)
    collect = []
    logits = oracle.forward_q(m, z["tokens"], collect)
    for i, st in enumerate(collect):
        assert np.array_equal(st["u_q"], z[f"l{i}_u_q"]), i
        assert np.array_equal(st["out"], z[f"l{i}_out"]), i
    ref = z["logits"]
    assert np.max(np.abs(logits - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_composed_decode_equals_prefix_prefill(oracle):
    """The quantized decode oracle (carried conv window + h) reproduces the
    one-shot forward row by row: hidden states bit-exact."""
    z, meta = load_npz("model_tiny2.npz")
    m = oracle_model(z, meta)
    tokens = z["tokens"][:20]
    full = oracle.forward_hidden(m, tokens)
    states = oracle.decode_states(m, tokens[:12])
    for t in range(12, 20):
        x_out = m.embedding[np.asarray([tokens[t]])]
        x_res = np.zeros_like(x_out)
        new = []
        for gain, blk, (cs, h) in zip(m.norms, m.blocks, states):
            u_q, x_res = oracle.fused_rmsnorm_quant(x_out, x_res, gain, blk.act["in"], m.bits)
            x_out, cs, h = oracle.block_decode_step(u_q, blk.act["in"], blk, cs, h)
            new.append((cs, h))
        states = new
        hidden = oracle.rmsnorm(x_out + x_res, m.final_norm)
        assert np.array_equal(hidden[0], full[t]), t
