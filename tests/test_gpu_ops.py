"""GPU parity of the individual kernels (through the C ABI) against the oracle."""
import numpy as np
import pytest
import torch

from conftest import load_npz

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint32), b.view(np.uint32)) or \
            bool(((a.view(np.uint32) == b.view(np.uint32)) | (np.isnan(a) & np.isnan(b))).all())
    return np.array_equal(a, b)


@pytest.mark.parametrize("fn,name", [(0, "np_exp"), (1, "glibc_expf"), (2, "glibc_log1pf"), (3, "softplus"),
                                     (4, "silu")])
def test_transcendentals_bit_exact(cuda, oracle, fn, name):
    from paper_2410_13229_b200 import _device, _lib

    bits = np.arange(0, 1 << 32, 4099, dtype=np.uint64).astype(np.uint32)
    x = np.concatenate([bits.view(np.float32),
                        np.random.default_rng(fn).uniform(-30, 30, 400000).astype(np.float32)])
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty_like(xt)
    _lib.call("qmb_eval_math", fn, xt.data_ptr(), yt.data_ptr(), xt.numel(), _device.stream_ptr())
    got = yt.cpu().numpy()
    ref = getattr(oracle, name)(x)
    same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
    assert same.all(), f"{name}: {np.count_nonzero(~same)} mismatches, e.g. x={x[~same][:5]}"


@pytest.mark.parametrize("fa,fb", [(4, 5), (4, 6), (4, 7)])
def test_hot_path_math_exhaustive(cuda, fa, fb):
    """Hot-path restatements equal the reference restatement on ALL 2^32 inputs."""
    from paper_2410_13229_b200 import _device, _lib

    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("qmb_verify_math", fa, fb, bad.data_ptr(), first.data_ptr(), _device.stream_ptr())
    torch.cuda.synchronize()
    n, f = int(bad.item()), int(first.item()) & 0xFFFFFFFF
    x = np.array([f], np.uint32).view(np.float32)[0]
    assert n == 0, f"{n} mismatches, first at bits {f:#010x} (x={x!r})"


def test_quantize_known_answers(cuda):
    from paper_2410_13229_b200 import quantize

    # test_quant.py:103-124
    assert quantize(np.array([0.5, -1.0, 2.54], np.float32), 0.02).values.tolist() == [25, -50, 127]
    assert quantize(np.array([0.03]), 0.02).values.tolist() == [2]
    with pytest.raises(ValueError, match="non-finite"):
        quantize(np.array([1.0, np.inf], np.float32), 0.1)


def test_quantize_random_bit_exact(cuda, oracle):
    from paper_2410_13229_b200 import quantize

    rng = np.random.default_rng(1)
    for s in (1e-4, 0.0123, 0.5, 3.7):
        x = (rng.standard_normal(100000) * s * 60).astype(np.float32)
        x[:1000] = (np.round(x[:1000] / np.float32(s)) + 0.5).astype(np.float32) * np.float32(s)  # ties
        assert np.array_equal(quantize(x, s).values, oracle.quantize(x, s))
        assert np.array_equal(quantize(x, s, 4).values, oracle.quantize(x, s, 4))


@pytest.mark.parametrize("path", [0, 1, 2, 3])
@pytest.mark.parametrize("M,K,N", [(1, 1, 1), (5, 7, 3), (16, 16, 16), (37, 200, 50), (130, 256, 300), (64, 2560, 1000),
                                   (64, 320, 9600), (7, 2560, 10240), (1, 2560, 10240), (2, 5120, 192),
                                   (3, 160, 5120), (8, 5120, 2560), (5, 768, 3072), (1, 48, 1536),
                                   (64, 160, 5120), (33, 5120, 192),
                                   (256, 2560, 192), (300, 160, 640), (129, 5120, 96), (4100, 400, 1300),
                                   (2600, 2560, 2100)])
def test_qlinear_bit_exact(cuda, oracle, path, M, K, N):
    """path 1: tcgen05 tiles (split-K below 129 rows), 2: SIMT, 3: the decode GEMV
    (M <= 8, K a multiple of 16; other shapes are refused)."""
    from paper_2410_13229_b200 import QTensor, qlinear

    if path == 3 and not (M <= 8 and K % 16 == 0):
        pytest.skip("GEMV path covers M <= 8, K % 16 == 0")

    rng = np.random.default_rng(M * 1000 + K + N)
    xq = rng.integers(-127, 128, size=(M, K)).astype(np.int8)
    wq = rng.integers(-127, 128, size=(K, N)).astype(np.int8)
    bq = rng.integers(-127, 128, size=(N,)).astype(np.int8)
    x, w, b = QTensor(xq, 0.031), QTensor(wq, 0.007), QTensor(bq, 0.01)
    got = qlinear(x, w, path=path)
    assert _bits_equal(got, oracle.qlinear(xq, 0.031, wq, 0.007))
    got = qlinear(x, w, bias_q=b, s_out=0.9, path=path)
    assert np.array_equal(got.values, oracle.qlinear(xq, 0.031, wq, 0.007, bias=(bq, 0.01), s_out=0.9))
    got = qlinear(x, w, extra_scale=1.0 / 96, path=path)
    assert _bits_equal(got, oracle.qlinear(xq, 0.031, wq, 0.007, extra=1.0 / 96))


def test_qlinear_known_answers(cuda):
    from paper_2410_13229_b200 import QTensor, qlinear

    # test_qblock.py:40-47
    out = qlinear(QTensor(np.array([[1]], np.int8), 0.5), QTensor(np.array([[2]], np.int8), 0.25))
    assert out.shape == (1, 1) and out[0, 0] == np.float32(0.25)
    out = qlinear(QTensor(np.array([[3, -7]], np.int8), 0.5), QTensor(np.zeros((2, 1), np.int8), 0.25))
    assert not out.any()
    with pytest.raises(ValueError, match="int32 accumulation"):
        qlinear(QTensor(np.zeros((1, 2**15 + 1), np.int8), 1.0), QTensor(np.zeros((2**15 + 1, 1), np.int8), 1.0))


@pytest.mark.parametrize("T,C,K", [(12, 6, 4), (5, 2, 3), (64, 96, 4), (33, 160, 4), (7, 48, 2), (200, 512, 4),
                                   (37, 64, 3), (3, 32, 4), (1, 16, 4), (21, 32, 5)])
def test_fused_qconv_bit_exact(cuda, oracle, T, C, K):
    from paper_2410_13229_b200 import QTensor, fused_qconv

    rng = np.random.default_rng(T * C + K)
    xq = rng.integers(-127, 128, size=(T, C)).astype(np.int8)
    wq = rng.integers(-127, 128, size=(K, C)).astype(np.int8)
    bq = rng.integers(-127, 128, size=(C,)).astype(np.int8)
    got = fused_qconv(QTensor(xq, 0.02), QTensor(wq, 0.01), QTensor(bq, 0.003), 0.015)
    assert np.array_equal(got.values, oracle.fused_qconv(xq, 0.02, wq, 0.01, (bq, 0.003), 0.015))
    got = fused_qconv(QTensor(xq, 0.02), QTensor(wq, 0.01), None, 0.015)
    assert np.array_equal(got.values, oracle.fused_qconv(xq, 0.02, wq, 0.01, None, 0.015))


def test_fused_qconv_zero_input_gives_bias_rows(cuda, oracle):
    from paper_2410_13229_b200 import QTensor, fused_qconv, quantize_weight

    # test_qblock.py:86-94
    bias_q = quantize_weight(np.array([0.8, -0.4], np.float32))
    out = fused_qconv(QTensor(np.zeros((5, 2), np.int8), 0.1), QTensor(np.ones((3, 2), np.int8), 0.05), bias_q,
                      0.01)
    exp = oracle.quantize(oracle.silu(oracle.dequantize(bias_q.values, bias_q.scale)), 0.01)
    assert np.array_equal(out.values, np.tile(exp, (5, 1)))


@pytest.mark.parametrize("T,D,N", [(1, 1, 1), (11, 8, 5), (40, 96, 16), (64, 130, 16), (17, 33, 4), (9, 20, 32)])
def test_selective_scan_bit_exact(cuda, oracle, T, D, N):
    from paper_2410_13229_b200 import QTensor, quantize_weight, quantized_selective_scan

    rng = np.random.default_rng(T * 100 + D * 10 + N)
    a_q = quantize_weight((-np.exp(rng.uniform(-1, 1, size=(D, N)))).astype(np.float32))
    d_q = quantize_weight(rng.standard_normal(D).astype(np.float32))
    b_q = QTensor(rng.integers(-127, 128, size=(T, N)).astype(np.int8), 0.01)
    c_q = QTensor(rng.integers(-127, 128, size=(T, N)).astype(np.int8), 0.012)
    dt_q = QTensor(rng.integers(0, 128, size=(T, D)).astype(np.int8), 0.001)
    x_q = QTensor(rng.integers(-127, 128, size=(T, D)).astype(np.int8), 0.02)
    y, h = quantized_selective_scan(a_q, b_q, c_q, d_q, dt_q, x_q, return_state=True)
    ry, rh = oracle.quantized_scan(a_q.values, a_q.scale, b_q.values, 0.01, c_q.values, 0.012, d_q.values, d_q.scale,
                                   dt_q.values, 0.001, x_q.values, 0.02)
    assert _bits_equal(y, ry) and _bits_equal(h, rh)
    # carried state: two halves == one shot (test_formats.py:76-94)
    k = T // 2
    sl = lambda q, a, b: QTensor(q.values[a:b], q.scale)  # noqa: E731
    y1, h1 = quantized_selective_scan(a_q, sl(b_q, 0, k), sl(c_q, 0, k), d_q, sl(dt_q, 0, k), sl(x_q, 0, k),
                                      return_state=True)
    y2, h2 = quantized_selective_scan(a_q, sl(b_q, k, T), sl(c_q, k, T), d_q, sl(dt_q, k, T), sl(x_q, k, T), h0=h1,
                                      return_state=True)
    assert _bits_equal(np.concatenate([y1, y2]), ry) and _bits_equal(h2, rh)


def test_scan_divergence_raises(cuda):
    from paper_2410_13229_b200 import QTensor, quantized_selective_scan

    a_q = QTensor(np.full((2, 2), 100, np.int8), 1.0)  # exp(dt*a) explodes
    ones = QTensor(np.full((50, 2), 100, np.int8), 1.0)
    with pytest.raises(FloatingPointError):
        quantized_selective_scan(a_q, ones, ones, QTensor(np.ones(2, np.int8), 1.0), QTensor(np.full((50, 2), 100,
                                 np.int8), 1.0), QTensor(np.full((50, 2), 100, np.int8), 1.0))


def test_hadamard_golden_and_quant(cuda, oracle):
    from paper_2410_13229_b200 import apply_hadamard, hadamard_quantize, plan_for_dim

    z, _ = load_npz("hadamard.npz")
    for n in (16, 96, 160, 512, 1536, 5120):
        plan = plan_for_dim(n)
        got = apply_hadamard(plan, z[f"y{n}"])
        assert _bits_equal(got, z[f"h{n}"]), n
        s = float(np.abs(z[f"h{n}"]).max() / 127)
        assert np.array_equal(hadamard_quantize(z[f"y{n}"], s, plan).values, oracle.quantize(z[f"h{n}"], s))
    # test_hadamard.py:199-206
    plan = plan_for_dim(4)
    assert hadamard_quantize(np.array([[64.0, 0, 0, 0]], np.float32), 1.0, plan).values.tolist() == [[64] * 4]


@pytest.mark.parametrize("n", [1024, 2048, 3072, 4096])
def test_hadamard_family_dims_bit_exact(cuda, oracle, n):
    """The packed kernels at the other Mamba d_inner sizes (2^10..2^12 run the
    butterfly alone, hadamard.py:145; 3072 = 12 x 2^8) against the oracle, which
    the n = 512 / 16 / 96 / 1536 / 5120 goldens pin to the reference."""
    from paper_2410_13229_b200 import apply_hadamard, plan_for_dim

    plan = plan_for_dim(n)
    y = (np.random.default_rng(n).standard_normal((9, n)) * 3).astype(np.float32)
    y[1, ::5] = -0.0
    got = apply_hadamard(plan, y)
    assert _bits_equal(got, oracle.hadamard(y, plan.p, plan.m, plan.base)), n


@pytest.mark.parametrize("n", [1536, 5120, 3072, 2048, 4096])
def test_hadamard_quant_ties_clamps_and_nonfinite(cuda, oracle, n):
    """The packed quantize of the fast Hadamard kernels: exact .5 ties (scalar
    fallback), values far beyond +-qmax, near-zero rows and a non-finite row."""
    from paper_2410_13229_b200 import apply_hadamard, hadamard_quantize, plan_for_dim

    plan = plan_for_dim(n)
    rng = np.random.default_rng(n)
    y = (rng.standard_normal((6, n)) * 4).astype(np.float32)
    y[0] = 0.0
    y[0, 0] = 2.5                      # every output is +-2.5: all ties
    y[1] = np.float32(0.5) * rng.integers(-9, 10, n).astype(np.float32) / np.float32(np.sqrt(n))
    y[2] *= np.float32(1e4)            # clamps
    y[3] *= np.float32(1e-30)          # rounds to 0
    y[4, ::7] = -0.0
    h = apply_hadamard(plan, y)
    for s in (1.0, 0.37, float(np.abs(h[5]).max() / 127)):
        assert np.array_equal(hadamard_quantize(y, s, plan).values, oracle.quantize(h, s)), s
    bad = y.copy()
    bad[5, 17] = np.inf
    with pytest.raises(ValueError):
        hadamard_quantize(bad, 1.0, plan)


@pytest.mark.parametrize("M,D", [(700, 2560), (1300, 768)])
def test_rmsnorm_single_stream_bit_exact(cuda, oracle, M, D):
    """The model's layers >= 1 (out_proj already accumulated into the stream) and its
    final norm: rmsnorm of one stream -> int8 codes, or -> f32 (persistent kernel)."""
    from paper_2410_13229_b200 import _device, _lib

    lib = _lib.load()
    rng = np.random.default_rng(M)
    x = (rng.standard_normal((M, D)) * 3).astype(np.float32)
    x[1, ::3] = -0.0
    x[2] *= np.float32(1e-20)
    x[3, :5] = np.float32(3e-38)
    x[4] *= np.float32(1e15)
    x[5, :] = 0.0
    gain = rng.uniform(0.5, 1.5, D).astype(np.float32)
    xd, gd = torch.from_numpy(x).cuda(), torch.from_numpy(gain).cuda()
    u = torch.empty((M, D), dtype=torch.int8, device="cuda")
    y = torch.empty((M, D), dtype=torch.float32, device="cuda")
    err = _device.err_flag()
    st = _device.stream_ptr()
    for s_out in (0.02, 0.005):
        _lib.check(lib.qmb_rmsnorm_residual_quant(xd.data_ptr(), None, None, gd.data_ptr(), M, D, s_out, 8,
                                                  u.data_ptr(), None, err.ptr, st), "rmsnorm")
        err.raise_if_set()
        assert np.array_equal(u.cpu().numpy(), oracle.quantize(oracle.rmsnorm(x, gain), s_out)), s_out
    _lib.check(lib.qmb_rmsnorm_residual_quant(xd.data_ptr(), None, None, gd.data_ptr(), M, D, 1.0, 8, None,
                                              y.data_ptr(), err.ptr, st), "rmsnorm")
    err.raise_if_set()
    assert _bits_equal(y.cpu().numpy(), oracle.rmsnorm(x, gain))


@pytest.mark.parametrize("M,D", [(3, 8), (6, 16), (33, 64), (50, 768), (17, 2560), (9, 1000),
                                 (700, 2560), (640, 768), (1200, 64), (600, 1000)])
def test_rmsnorm_residual_quant_bit_exact(cuda, oracle, M, D):
    """Small M: CTA-per-row kernel; M >= 592: warp-per-row kernels (balanced pairwise
    tree for 2^k equal leaves, generic plan otherwise), incl. rows that take the
    exact-division fallback (zeros, -0, tiny and huge magnitudes)."""
    from paper_2410_13229_b200 import fused_rmsnorm_quant

    rng = np.random.default_rng(M + D)
    x_out = (rng.standard_normal((M, D)) * 3).astype(np.float32)
    x_res = (rng.standard_normal((M, D)) * 2).astype(np.float32)
    if M >= 600:
        x_out[1, ::3] = 0.0
        x_res[1, ::3] = -0.0
        x_out[2] *= np.float32(1e-20)
        x_res[2] *= np.float32(1e-20)
        x_out[3, :5] = np.float32(3e-38)
        x_res[3, :5] = 0.0
        x_out[4] *= np.float32(1e15)
        x_res[4] *= np.float32(1e15)
    gain = rng.uniform(0.5, 1.5, D).astype(np.float32)
    q, res = fused_rmsnorm_quant(x_out, x_res, gain, 0.02)
    rq, rres = oracle.fused_rmsnorm_quant(x_out, x_res, gain, 0.02)
    assert np.array_equal(q.values, rq) and np.array_equal(res, rres)
    # test_qblock.py:187-192: cancellation gives exact zeros
    q, res = fused_rmsnorm_quant(x_out, -x_out, gain, 0.05)
    assert not q.values.any() and not res.any()


@pytest.mark.parametrize("M,K,V", [(1, 2560, 50280), (64, 2560, 50280), (3, 768, 1000), (65, 100, 130), (7, 37, 5)])
def test_lm_head_tolerance(cuda, M, K, V):
    """The tied f32 LM head (model.py:257-258) against an f64 product: within the
    logit tolerance of SURVEY §8c (1e-5 of the largest |logit|)."""
    from paper_2410_13229_b200 import _device, _lib

    g = torch.Generator(device="cuda").manual_seed(M * 7 + V)
    x = torch.randn((M, K), generator=g, device="cuda")
    emb = torch.randn((V, K), generator=g, device="cuda") * 0.05
    out = torch.empty((M, V), dtype=torch.float32, device="cuda")
    _lib.call("qmb_lm_head", x.data_ptr(), M, K, emb.data_ptr(), V, out.data_ptr(), _device.stream_ptr())
    ref = (x.double() @ emb.double().T)
    err = float((out.double() - ref).abs().max())
    assert err <= 1e-5 * float(ref.abs().max()), err


@pytest.mark.parametrize("M,K,V", [(64, 2560, 50280), (9, 768, 1000), (130, 100, 130)])
def test_lm_head_split16_tolerance(cuda, M, K, V):
    """The LM head above 8 rows (fp16-split tensor-core product, model.lm_head_split16)
    against an f64 product: within 1e-5 of the largest |logit|, on rows of very
    different magnitudes (the per-row power-of-two scaling), zero rows and tiny /
    huge weights."""
    from paper_2410_13229_b200.model import lm_head_split16, split16_weights

    g = torch.Generator(device="cuda").manual_seed(M + K)
    x = torch.randn((M, K), generator=g, device="cuda")
    x[1] *= 1e4
    x[2] *= 1e-6
    x[3] = 0.0
    emb = torch.randn((V, K), generator=g, device="cuda") * 0.05
    emb[0] *= 1e-7
    emb[1, :7] = 3.0
    out = lm_head_split16(x, *split16_weights(emb))
    ref = x.double() @ emb.double().T
    for r in range(M):  # per row: the tolerance is relative to that row's largest logit
        err = float((out[r].double() - ref[r]).abs().max())
        assert err <= 1e-5 * float(ref[r].abs().max()) + 1e-30, (r, err)
    assert not out[3].any()


def test_argmax_numpy_semantics(cuda):
    """qmb_argmax == numpy.argmax per row: first index of the maximum (ties), a NaN
    wins (first NaN), all -inf rows, strided rows."""
    from paper_2410_13229_b200.model import DeviceModel

    rng = np.random.default_rng(3)
    x = rng.standard_normal((9, 50280)).astype(np.float32)
    x[1, [5, 17, 40000]] = 9.0          # ties: first index
    x[2, [100, 30000]] = np.nan         # first NaN
    x[3, :] = -np.inf
    x[4, :] = 0.0
    x[5, -1] = 1e30                     # last column
    x[6, 7] = np.inf
    dm = DeviceModel.__new__(DeviceModel)
    from paper_2410_13229_b200 import _lib
    dm._lib = _lib.load()
    xt = torch.from_numpy(x).cuda()
    got = dm.argmax(xt).cpu().numpy()
    assert np.array_equal(got, np.argmax(x, axis=-1)), (got, np.argmax(x, axis=-1))
    big = torch.from_numpy(np.concatenate([x, x], axis=1)).cuda()[:, :50280]  # strided rows
    assert np.array_equal(dm.argmax(big).cpu().numpy(), np.argmax(x, axis=-1))
