"""GPU block parity: every intermediate of block_forward_q, bit-exact against
the reference's golden stage replay (tests/golden) and the oracle."""
import numpy as np
import pytest
import torch

from fixtures_util import BLOCK_FIXTURES, SMALL_BLOCKS, block_weights, load_block, mirror_block, oracle_block

pytestmark = pytest.mark.gpu


def _ws_views(dev, ws, M, meta):
    lay = dev.workspace_layout(M)
    E = meta["cfg"]["d_inner"]
    N = meta["cfg"]["d_state"]
    R = meta["cfg"]["dt_rank"]
    Ep = (E + 15) // 16 * 16
    Rp = (R + 15) // 16 * 16

    def view(slot, dtype, cols, ld):
        nbytes = torch.tensor([], dtype=dtype).element_size()
        t = ws[lay[slot]:lay[slot] + M * ld * nbytes].view(dtype).reshape(M, ld)[:, :cols]
        return t.cpu().numpy()

    return dict(x_q=lambda: view("XQ", torch.int8, E, E), gated=lambda: view("Z", torch.float32, E, E),
                scan_x=lambda: view("SCANX", torch.int8, E, Ep), b_q=lambda: view("B", torch.int8, N, N),
                c_q=lambda: view("C", torch.int8, N, N), dtr_q=lambda: view("DTR", torch.int8, R, Rp),
                delta_q=lambda: view("DELTA", torch.int8, E, E), y_q=lambda: view("YQ", torch.int8, E, Ep))


@pytest.mark.parametrize("scan_exp", [0, 1])
@pytest.mark.parametrize("name", BLOCK_FIXTURES)
def test_block_prefill_stages_bit_exact(cuda, name, scan_exp):
    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block(name)
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    dev = device_block(qb)
    u = torch.from_numpy(z["u_q"]).cuda()
    T = u.shape[0]
    out = torch.empty((T, meta["cfg"]["d_model"]), dtype=torch.float32, device="cuda")
    ws = torch.zeros(dev.workspace_bytes(T), dtype=torch.uint8, device="cuda")
    E, N = meta["cfg"]["d_inner"], meta["cfg"]["d_state"]
    K = meta["cfg"]["d_conv"]
    conv_state = torch.zeros((1, K - 1, E), dtype=torch.int8, device="cuda")
    h = torch.zeros((1, E, N), dtype=torch.float32, device="cuda")
    dev.prefill(u, 1, T, out, u_scale=meta["u_scale"], conv_state_out=conv_state, ssm_state_out=h,
                scan_exp=scan_exp, workspace=ws)
    _device.err_flag().raise_if_set()
    views = _ws_views(dev, ws, T, meta)
    for stage in ("x_q", "scan_x", "b_q", "c_q", "dtr_q", "delta_q", "gated", "y_q"):
        got = views[stage]()
        ref = z[f"st_{stage}"]
        if got.dtype.kind == "f":
            ok = np.array_equal(got.view(np.uint32), ref.view(np.uint32))
        else:
            ok = np.array_equal(got, ref)
        assert ok, f"{name}: first mismatching stage {stage}: {np.count_nonzero(got != ref)} of {ref.size}"
    assert np.array_equal(out.cpu().numpy().view(np.uint32), z["st_out"].view(np.uint32)), f"{name}: out"
    assert np.array_equal(h[0].cpu().numpy().view(np.uint32), z["st_h"].view(np.uint32)), f"{name}: final h"
    ob = oracle_block(z, meta, w)
    from oracle import oracle as o
    st = o.block_stages(z["u_q"], meta["u_scale"], ob)
    assert np.array_equal(conv_state[0].cpu().numpy(), st["conv_state"])


@pytest.mark.parametrize("name", SMALL_BLOCKS)
def test_block_forward_q_dropin_numpy(cuda, name):
    """block_forward_q with numpy QTensors (the reference's calling convention)."""
    from paper_2410_13229_b200 import QTensor, block_forward_q

    z, meta = load_block(name)
    qb = mirror_block(z, meta)
    out = block_forward_q(QTensor(z["u_q"], meta["u_scale"]), qb)
    assert isinstance(out, np.ndarray) and np.array_equal(out, z["st_out"])


@pytest.mark.parametrize("name", ["m20_full", "p2_naive", "s130m"])
def test_block_batched_sequences(cuda, oracle, name):
    """B independent sequences in one launch equal B separate oracle runs."""
    from paper_2410_13229_b200 import QTensor, block_forward_q

    z, meta = load_block(name)
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    ob = oracle_block(z, meta, w)
    rng = np.random.default_rng(5)
    B, T, D = 3, 21, meta["cfg"]["d_model"]
    u = rng.integers(-127, 128, size=(B, T, D)).astype(np.int8)
    got = block_forward_q(QTensor(u, meta["u_scale"]), qb)
    for b in range(B):
        ref = oracle.block_forward_q(u[b], meta["u_scale"], ob)
        assert np.array_equal(got[b], ref), b


@pytest.mark.parametrize("name,B,T", [("m12_full", 20, 13), ("m20_full", 37, 9), ("s130m", 33, 17)])
def test_block_many_sequences_bit_exact(cuda, oracle, name, B, T):
    """Large batches take the batch-tiled scan (8 channels x 32 sequences per
    CTA); ragged B / T / channel tails included.  Final states checked too."""
    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block(name)
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    ob = oracle_block(z, meta, w)
    dev = device_block(qb)
    D, E, N = meta["cfg"]["d_model"], meta["cfg"]["d_inner"], meta["cfg"]["d_state"]
    rng = np.random.default_rng(B * 100 + T)
    u = rng.integers(-127, 128, size=(B, T, D)).astype(np.int8)
    out = torch.empty((B * T, D), dtype=torch.float32, device="cuda")
    conv, h = dev.new_state(B)
    dev.prefill(torch.from_numpy(u).cuda().reshape(B * T, D), B, T, out, u_scale=meta["u_scale"],
                conv_state_out=conv, ssm_state_out=h)
    _device.err_flag().raise_if_set()
    got = out.reshape(B, T, D).cpu().numpy()
    hs = h.cpu().numpy()
    for b in range(B):
        st = oracle.block_stages(u[b], meta["u_scale"], ob)
        assert np.array_equal(got[b].view(np.uint32), st["out"].view(np.uint32)), b
        assert np.array_equal(hs[b].view(np.uint32), st["h"].view(np.uint32)), b


@pytest.mark.parametrize("name,B,T", [("m12_full", 1, 1), ("m12_full", 2, 2), ("m20_full", 3, 3), ("m20_full", 5, 47),
                                      ("m20_full", 2, 1000), ("p2_naive", 4, 16), ("p2_inper", 7, 33),
                                      ("s130m", 1, 100), ("s130m", 1, 2048), ("s130m", 15, 21), ("s2p8b", 2, 40),
                                      ("s2p8b", 4, 17)])
def test_block_small_batch_bit_exact(cuda, oracle, name, B, T):
    """B < 16 takes the state-split scan (2 lanes per channel, 4 for a single
    sequence, skewed 4 steps apart, the in-order acc sum handed lane to lane): ragged
    T (shorter than the skew, not a multiple of the 16-step chunk, 1000 steps, the
    130M shape at BASELINE config 2's 2K tokens) and partial sequence groups; outputs
    and final states bit-exact against the oracle."""
    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block(name)
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    ob = oracle_block(z, meta, w)
    dev = device_block(qb)
    D = meta["cfg"]["d_model"]
    rng = np.random.default_rng(B * 1000 + T)
    u = rng.integers(-127, 128, size=(B, T, D)).astype(np.int8)
    out = torch.empty((B * T, D), dtype=torch.float32, device="cuda")
    conv, h = dev.new_state(B)
    dev.prefill(torch.from_numpy(u).cuda().reshape(B * T, D), B, T, out, u_scale=meta["u_scale"],
                conv_state_out=conv, ssm_state_out=h)
    _device.err_flag().raise_if_set()
    got = out.reshape(B, T, D).cpu().numpy()
    hs = h.cpu().numpy()
    for b in range(B):
        st = oracle.block_stages(u[b], meta["u_scale"], ob)
        assert np.array_equal(got[b].view(np.uint32), st["out"].view(np.uint32)), b
        assert np.array_equal(hs[b].view(np.uint32), st["h"].view(np.uint32)), b


@pytest.mark.parametrize("name,B", [("tiny_full", 2), ("m12_full", 2), ("p2_inper", 2), ("s2p8b", 2), ("s2p8b", 37),
                                    ("s130m", 5), ("m20_full", 64)])
def test_block_decode_equals_prefill(cuda, name, B):
    """Prefill k tokens (exporting state), then decode the rest one by one: every
    decoded row and the final state equal the one-shot prefill bit-for-bit."""
    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block(name)
    qb = mirror_block(z, meta)
    dev = device_block(qb)
    u = torch.from_numpy(z["u_q"]).cuda()
    T, D = u.shape
    ub = u[None].repeat(B, 1, 1).contiguous()
    k = T // 2
    conv, h = dev.new_state(B)
    pre = torch.empty((B * k, D), dtype=torch.float32, device="cuda")
    dev.prefill(ub[:, :k].contiguous().reshape(B * k, D), B, k, pre, u_scale=meta["u_scale"], conv_state_out=conv,
                ssm_state_out=h)
    rows = [pre.reshape(B, k, D)]
    for t in range(k, T):
        o = torch.empty((B, D), dtype=torch.float32, device="cuda")
        dev.decode(ub[:, t].contiguous(), conv, h, o, u_scale=meta["u_scale"])
        rows.append(o[:, None])
    _device.err_flag().raise_if_set()
    got = torch.cat(rows, dim=1).cpu().numpy()
    for b in range(B):
        assert np.array_equal(got[b].view(np.uint32), z["st_out"].view(np.uint32)), b
    assert np.array_equal(h[0].cpu().numpy().view(np.uint32), z["st_h"].view(np.uint32))


@pytest.mark.parametrize("name", ["m20_full", "p2_naive", "s130m"])
def test_block_accumulate_is_the_residual_add(cuda, name):
    """qmb_block_prefill_accum / qmb_block_decode_accum add the block output into a
    residual buffer in out_proj's epilogue: bit-identical to the f32 add
    `x_out + x_res` that the next fused_rmsnorm_quant performs (qblock.py:181)."""
    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block(name)
    qb = mirror_block(z, meta)
    dev = device_block(qb)
    rng = np.random.default_rng(11)
    B, T, D = 3, 9, meta["cfg"]["d_model"]
    u = torch.from_numpy(rng.integers(-127, 128, size=(B * T, D)).astype(np.int8)).cuda()
    res0 = rng.standard_normal((B * T, D)).astype(np.float32)
    out = torch.empty((B * T, D), dtype=torch.float32, device="cuda")
    dev.prefill(u, B, T, out, u_scale=meta["u_scale"])
    res = torch.from_numpy(res0).cuda()
    dev.prefill(u, B, T, res, u_scale=meta["u_scale"], accumulate=True)
    _device.err_flag().raise_if_set()
    ref = out.cpu().numpy() + res0
    assert np.array_equal(res.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    # decode: one step from a fresh state, plain vs accumulated
    conv, h = dev.new_state(B)
    conv2, h2 = dev.new_state(B)
    row = torch.empty((B, D), dtype=torch.float32, device="cuda")
    dev.decode(u[:B].contiguous(), conv, h, row, u_scale=meta["u_scale"])
    acc = torch.from_numpy(res0[:B].copy()).cuda()
    dev.decode(u[:B].contiguous(), conv2, h2, acc, u_scale=meta["u_scale"], accumulate=True)
    _device.err_flag().raise_if_set()
    assert np.array_equal(acc.cpu().numpy().view(np.uint32), (row.cpu().numpy() + res0[:B]).view(np.uint32))


def test_handle_rebuilt_when_block_is_recalibrated(cuda, oracle):
    """The device handle cached on a QuantizedBlock is rebuilt when its scales change
    (the reference's QuantizedBlock is a mutable dataclass, qblock.py:75-95)."""
    from paper_2410_13229_b200 import QTensor, block_forward_q
    from paper_2410_13229_b200.qblock import ScaleEntry

    z, meta = load_block("m20_full")
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    u = QTensor(z["u_q"], meta["u_scale"])
    first = block_forward_q(u, qb)
    assert np.array_equal(first.view(np.uint32), z["st_out"].view(np.uint32))
    # re-calibrate one site in place, as run_calibration + quantize_block would
    old = qb.act["y_had"]
    qb.act["y_had"] = ScaleEntry(old.scale * 1.5, old.zero_point, old.scheme)
    meta2 = dict(meta, act=dict(meta["act"], y_had=old.scale * 1.5))
    ob2 = oracle_block(z, meta2, w)
    ref2 = oracle.block_forward_q(z["u_q"], meta["u_scale"], ob2)
    second = block_forward_q(u, qb)
    assert np.array_equal(second.view(np.uint32), ref2.view(np.uint32))
    assert not np.array_equal(second, first)


def test_nonfinite_gain_raises(cuda):
    from paper_2410_13229_b200 import fused_rmsnorm_quant

    x = np.ones((3, 16), dtype=np.float32)
    g = np.ones(16, dtype=np.float32)
    g[5] = np.nan
    with pytest.raises(ValueError, match="non-finite activation"):
        fused_rmsnorm_quant(x, np.zeros_like(x), g, 0.05)


def test_block_empty_and_single_token_edges(cuda, oracle):
    """Empty inputs (B = 0, T = 0) are no-ops like the reference's zero-length
    arrays; T = 1 prefill equals the reference's one-row block (conv window of
    zeros, h0 = 0); a 0-sequence decode is a no-op."""
    from paper_2410_13229_b200 import QTensor, block_forward_q
    from paper_2410_13229_b200.qblock import device_block

    z, meta = load_block("m20_full")
    w = block_weights(z, meta)
    qb = mirror_block(z, meta, w)
    ob = oracle_block(z, meta, w)
    dev = device_block(qb)
    D = meta["cfg"]["d_model"]
    for B, T in ((0, 5), (3, 0)):
        out = torch.full((max(B * T, 1), D), 7.0, device="cuda")
        dev.prefill(torch.zeros((max(B * T, 1), D), dtype=torch.int8, device="cuda"), B, T, out,
                    u_scale=meta["u_scale"])
        assert bool((out == 7.0).all())
    one = block_forward_q(QTensor(z["u_q"][:1], meta["u_scale"]), qb)
    assert np.array_equal(one.view(np.uint32), oracle.block_forward_q(z["u_q"][:1], meta["u_scale"], ob).view(np.uint32))
    conv, h = dev.new_state(1)
    row = torch.full((1, D), 3.0, device="cuda")
    dev.decode(torch.zeros((1, D), dtype=torch.int8, device="cuda")[:0], conv[:0], h[:0], row[:0],
               u_scale=meta["u_scale"])
    assert bool((row == 3.0).all())
