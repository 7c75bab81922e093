"""Quantized model loop -- mirror of `ssmq.model.forward_q` (pkg/src/ssmq/model.py:246-258)
plus the batched, state-carrying prefill/decode engine the B200 path adds.

The per-layer work (fused residual+RMSNorm+quant, block forward) runs in
libqmb; the tied f32 LM head (libqmb's GEMV up to 8 rows, cuBLAS f32 above)
is tolerance-checked only.
"""
from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .qblock import DeviceBlock, Mode, QuantizedBlock, device_block
from .quant import is_device
from .ssm import BlockConfig


@dataclass(frozen=True)
class ModelConfig:
    """model.py:32-72"""

    vocab_size: int = 256
    d_model: int = 64
    n_layers: int = 2
    expand: int = 2
    d_state: int = 16
    d_conv: int = 4
    dt_rank: int = 4
    bit_width: int = 8

    def __post_init__(self):
        if self.vocab_size <= 0 or self.n_layers <= 0:
            raise ValueError("vocab_size and n_layers must be positive")
        self.block

    @property
    def block(self) -> BlockConfig:
        return BlockConfig(d_model=self.d_model, expand=self.expand, d_state=self.d_state, d_conv=self.d_conv,
                           dt_rank=self.dt_rank)

    @property
    def d_inner(self) -> int:
        return self.expand * self.d_model

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("vocab_size", "d_model", "n_layers", "expand", "d_state", "d_conv",
                                              "dt_rank", "bit_width")}


@dataclass
class QuantizedLayer:
    norm_weight: object
    block: QuantizedBlock


@dataclass(eq=False)
class QuantizedModel:
    config: ModelConfig
    mode: Mode
    embedding: object
    layers: list
    final_norm: object
    scales: object = None


def _f32_dev(a) -> torch.Tensor:
    return _device.to_device(a if is_device(a) else np.asarray(a, dtype=np.float32), torch.float32)


class DeviceModel:
    """Device-resident quantized model: embedding, norms and one libqmb block
    handle per layer; batched prefill with optional state export, single-token
    decode with carried (conv window, h) state, greedy generation."""

    def __init__(self, model):
        cfg = model.config
        self.cfg = cfg
        self.D = int(cfg.d_model)
        self.V = int(cfg.vocab_size)
        self.bits = int(cfg.bit_width)
        self.embedding = _f32_dev(model.embedding)
        self.final_norm = _f32_dev(model.final_norm)
        self.norms = [_f32_dev(l.norm_weight) for l in model.layers]
        # the norm kernels range-check their input, not gain: a non-finite gain would make
        # every forward's quantize raise in the reference (quant.py:149-150), so refuse it here
        self.gains_finite = all(bool(torch.isfinite(g).all()) for g in self.norms + [self.final_norm])
        self.s_in = [float(l.block.act["in"].scale) for l in model.layers]
        self.blocks: list[DeviceBlock] = [device_block(l.block) for l in model.layers]
        self._lib = _lib.load()

    # ---------------------------------------------------------------- pieces
    def _rmsnorm(self, x_out, x_res, res_out, gain, s_out, u_q, y_out, M, err, stream):
        if not self.gains_finite and M > 0:
            raise ValueError("non-finite activation")
        _lib.check(self._lib.qmb_rmsnorm_residual_quant(
            x_out.data_ptr(), _device.ptr(x_res), _device.ptr(res_out), gain.data_ptr(), int(M), self.D,
            float(s_out), self.bits, _device.ptr(u_q), _device.ptr(y_out), err.ptr, stream), "rmsnorm")

    def embed(self, tokens: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        tok = tokens.reshape(-1).to(torch.int64)
        out = out if out is not None else torch.empty((tok.numel(), self.D), dtype=torch.float32,
                                                      device=tok.device)
        _lib.check(self._lib.qmb_embed_gather(self.embedding.data_ptr(), tok.data_ptr(), tok.numel(), self.D,
                                              out.data_ptr(), _device.stream_ptr()), "embed")
        return out

    def lm_head(self, final: torch.Tensor) -> torch.Tensor:
        """Tied f32 logits final @ embedding^T (model.py:257-258); tolerance-only
        against the reference's BLAS summation order.  Up to 8 rows: libqmb's
        streaming f32 GEMV (the embedding read once); more rows: the split-fp16
        tensor-core product (lm_head_split16) -- cuBLAS's f32 SIMT GEMM took 347 us
        at B = 64, libqmb's FFMA2 tile kernel (qmb_lm_head) 464 us."""
        x = final.reshape(-1, self.D).contiguous()
        M = x.shape[0]
        if M <= 8:
            out = torch.empty((M, self.V), dtype=torch.float32, device=x.device)
            _lib.check(self._lib.qmb_lm_head(x.data_ptr(), int(M), self.D, self.embedding.data_ptr(), self.V,
                                             out.data_ptr(), _device.stream_ptr()), "lm_head")
            return out.reshape(tuple(final.shape[:-1]) + (self.V,))
        if getattr(self, "_emb16", None) is None:
            self._emb16 = split16_weights(self.embedding)
        return lm_head_split16(x, *self._emb16).reshape(tuple(final.shape[:-1]) + (self.V,))

    # ---------------------------------------------------------------- prefill
    def forward_hidden(self, tokens: torch.Tensor, *, states=None, scan_exp: int = 0, err=None):
        """tokens [B, T] -> final-normed hidden [B*T, D] f32.  If `states` is a
        list (one (conv, h) pair per layer, shaped for B), the prefill writes
        the carried decode state into it."""
        B, T = tokens.shape
        groups = prefill_groups(B, T)
        if groups > 1 and states is None:
            return self._forward_hidden_groups(tokens, groups, scan_exp, err)
        return self._forward_hidden_one(tokens, states=states, scan_exp=scan_exp, err=err)

    def _forward_hidden_groups(self, tokens, groups, scan_exp, err):
        """Sequences are independent (model.py:306-320): the batch runs as `groups`
        contiguous row groups, each through all layers on its own CUDA stream with
        its own workspace, so one group's kernels fill the SMs another group's
        kernel leaves idle in its last wave.  Each group's rows are computed by the
        same kernels as a lone prefill of those sequences: bit-identical."""
        B, T = tokens.shape
        err = err if err is not None else _device.err_flag()
        main = torch.cuda.current_stream()
        if getattr(self, "_pf_streams", None) is None or len(self._pf_streams) < groups:
            self._pf_streams = [torch.cuda.Stream() for _ in range(groups)]
            self._pf_ws = [None] * groups
        final = torch.empty((B * T, self.D), dtype=torch.float32, device=tokens.device)
        bounds = [(g * B) // groups for g in range(groups + 1)]
        for g in range(groups):
            s = self._pf_streams[g]
            s.wait_stream(main)
            with torch.cuda.stream(s):
                rows = tokens[bounds[g]:bounds[g + 1]]
                need = max(b.workspace_bytes(rows.shape[0] * T) for b in self.blocks)
                if self._pf_ws[g] is None or self._pf_ws[g].numel() < need:
                    self._pf_ws[g] = torch.empty(need, dtype=torch.uint8, device=tokens.device)
                self._forward_hidden_one(rows, scan_exp=scan_exp, err=err, ws=self._pf_ws[g],
                                         out=final[bounds[g] * T:bounds[g + 1] * T])
        for g in range(groups):
            main.wait_stream(self._pf_streams[g])
        final.record_stream(main)
        return final

    def _forward_hidden_one(self, tokens, *, states=None, scan_exp=0, err=None, ws=None, out=None):
        B, T = tokens.shape
        M = B * T
        stream = _device.stream_ptr()
        err = err if err is not None else _device.err_flag()
        x_out = self.embed(tokens)
        x_res = torch.zeros_like(x_out)
        u_q = torch.empty((M, self.D), dtype=torch.int8, device=x_out.device)
        if ws is None:
            ws = _device.workspace(max(b.workspace_bytes(M) for b in self.blocks))
        # The residual stream lives in x_res: layer 0 forms res = emb + 0 (model.py:249-253);
        # every block then adds its output into x_res in out_proj's epilogue, which is the
        # next fused_rmsnorm_quant's `x_out + x_res` (qblock.py:181) - so later norms read
        # the stream directly.
        for li, blk in enumerate(self.blocks):
            if li == 0:
                self._rmsnorm(x_out, x_res, x_res, self.norms[li], self.s_in[li], u_q, None, M, err, stream)
            else:
                self._rmsnorm(x_res, None, None, self.norms[li], self.s_in[li], u_q, None, M, err, stream)
            conv, h = states[li] if states is not None else (None, None)
            blk.prefill(u_q, B, T, x_res, conv_state_out=conv, ssm_state_out=h, scan_exp=scan_exp, workspace=ws,
                        err=err, stream=stream, accumulate=True)
        final = out if out is not None else torch.empty_like(x_out)
        self._rmsnorm(x_res, None, None, self.final_norm, 1.0, None, final, M, err, stream)
        return final

    def forward(self, tokens: torch.Tensor, *, last_only: bool = False, scan_exp: int = 0) -> torch.Tensor:
        """Logits [B, T, V] (or [B, V] for the last position only)."""
        B, T = tokens.shape
        final = self.forward_hidden(tokens, scan_exp=scan_exp)
        if last_only:
            final = final.reshape(B, T, self.D)[:, -1]
            return self.lm_head(final)
        return self.lm_head(final).reshape(B, T, self.V)

    # ---------------------------------------------------------------- decode
    def new_states(self, B: int):
        return [blk.new_state(B) for blk in self.blocks]

    def prefill(self, tokens: torch.Tensor, states=None):
        """Prompt prefill that also exports the decode state; returns
        (last-position logits [B, V], states)."""
        B, T = tokens.shape
        states = states if states is not None else self.new_states(B)
        final = self.forward_hidden(tokens, states=states)
        return self.lm_head(final.reshape(B, T, self.D)[:, -1]), states

    def decode_step(self, tokens: torch.Tensor, states, *, err=None, bufs=None) -> torch.Tensor:
        """One token per sequence: tokens [B] -> logits [B, V]; states updated in place."""
        B = tokens.shape[0]
        stream = _device.stream_ptr()
        err = err if err is not None else _device.err_flag()
        if bufs is None:
            bufs = self.decode_buffers(B)
        x_out, x_res, u_q, final, ws = bufs
        self.embed(tokens, out=x_out)
        x_res.zero_()
        for li, blk in enumerate(self.blocks):  # residual stream in x_res, as in forward_hidden
            if li == 0:
                self._rmsnorm(x_out, x_res, x_res, self.norms[li], self.s_in[li], u_q, None, B, err, stream)
            else:
                self._rmsnorm(x_res, None, None, self.norms[li], self.s_in[li], u_q, None, B, err, stream)
            conv, h = states[li]
            blk.decode(u_q, conv, h, x_res, workspace=ws, err=err, stream=stream, accumulate=True)
        self._rmsnorm(x_res, None, None, self.final_norm, 1.0, None, final, B, err, stream)
        return self.lm_head(final)

    def decode_buffers(self, B: int):
        dev = _device.device()
        x_out = torch.empty((B, self.D), dtype=torch.float32, device=dev)
        x_res = torch.empty_like(x_out)
        u_q = torch.empty((B, self.D), dtype=torch.int8, device=dev)
        final = torch.empty_like(x_out)
        ws = torch.empty(max(b.workspace_bytes(B) for b in self.blocks), dtype=torch.uint8, device=dev)
        return x_out, x_res, u_q, final, ws

    def capture_decode(self, states):
        """Capture one decode step over all layers (embed, 64 x (norm + 7 block
        kernels), final norm, LM head) into a CUDA graph bound to `states`.
        Returns (graph, token_in [B] int64, logits_out [B, V]); replay after
        writing the next tokens into token_in."""
        B = states[0][1].shape[0]
        dev = _device.device()
        bufs = self.decode_buffers(B)
        tok = torch.zeros(B, dtype=torch.int64, device=dev)
        scratch = self.new_states(B)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # lazy init (kernel attributes, cuBLAS) outside the capture
            self.decode_step(tok, scratch, bufs=bufs)
            self.decode_step(tok, scratch, bufs=bufs)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        _device.err_flag().reset()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            logits = self.decode_step(tok, states, bufs=bufs)
        graph._qmb_keep = (bufs, scratch)  # keep captured buffers alive with the graph
        return graph, tok, logits

    def argmax(self, logits: torch.Tensor) -> torch.Tensor:
        """Greedy next tokens on the device (numpy.argmax semantics: first index of
        the maximum, NaN wins): [..., V] f32 -> [...] int64."""
        x = logits.reshape(-1, logits.shape[-1])
        if x.stride(-1) != 1:
            x = x.contiguous()
        out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
        _lib.check(self._lib.qmb_argmax(x.data_ptr(), int(x.shape[0]), int(x.shape[1]), int(x.stride(0)),
                                        out.data_ptr(), _device.stream_ptr()), "argmax")
        return out.reshape(logits.shape[:-1])

    def greedy_generate(self, prompt: torch.Tensor, steps: int, use_graph: bool = True) -> torch.Tensor:
        """Greedy decoding with carried state (quantized analogue of
        model.greedy_decode, model.py:364-379).  prompt [B, T] -> [B, T+steps].
        Decode steps replay one captured CUDA graph."""
        logits, states = self.prefill(prompt)
        out = [prompt]
        if use_graph and steps > 1:
            graph, tok, glogits = self.capture_decode(states)
        else:
            bufs = self.decode_buffers(prompt.shape[0])
        for s in range(steps):
            nxt = self.argmax(logits)
            out.append(nxt[:, None])
            if s + 1 < steps:
                if use_graph and steps > 1:
                    tok.copy_(nxt)
                    graph.replay()
                    logits = glogits
                else:
                    logits = self.decode_step(nxt, states, bufs=bufs)
        _device.err_flag().raise_if_set()
        return torch.cat(out, dim=1)


def prefill_groups(B: int, T: int) -> int:
    """Row groups (CUDA streams) of a batched prefill.  Default: 2 from 32 sequences
    (2.8B, B = 64 x T = 1024, 16 layers: 5.49-5.55 vs 5.54-5.61 ms per layer over three
    interleaved pairs, `tools/prefill_streams.py`; 3-4 groups are slower: the
    persistent GEMMs' CTAs that start late on SMs held by the other groups' kernels
    stretch their static tile schedule); QMB_PREFILL_STREAMS overrides."""
    env = os.environ.get("QMB_PREFILL_STREAMS")
    g = int(env) if env else (2 if B >= 32 else 1)
    return max(1, min(g, B))


def split16_weights(w: torch.Tensor):
    """(w_hi, w_lo, k): w * 2^k = w_hi + w_lo + O(2^-22 |w|) with fp16 halves, 2^k a
    power of two putting max |w| in [2^13, 2^14) (exact scaling, no fp16 overflow)."""
    amax = float(w.abs().max()) if w.numel() else 0.0
    k = 0 if not (amax > 0.0) or not torch.isfinite(torch.tensor(amax)) else 14 - int(torch.frexp(
        torch.tensor(amax, dtype=torch.float64))[1])
    ws = w.float() * (2.0 ** k)
    hi = ws.half()
    lo = (ws - hi.float()).half()
    return hi.contiguous(), lo.contiguous(), k


def lm_head_split16(x: torch.Tensor, w_hi: torch.Tensor, w_lo: torch.Tensor, k: int) -> torch.Tensor:
    """f32 x [M, K] @ W^T [K, V] on the fp16 tensor cores: each row of x scaled by a
    power of two below 2^14 and split x = x_hi + x_lo (fp16, libqmb qmb_lm_split16);
    then x W^T ~ x_hi W_hi + x_lo W_hi + x_hi W_lo with f32 accumulation (cuBLAS, two
    GEMMs over the weights: [x_hi; x_lo] W_hi^T and x_hi W_lo^T), combined and
    unscaled by qmb_lm_combine16.  The dropped x_lo W_lo and the halves' own rounding
    are ~2^-22 relative per product -- well inside the LM head's f32 tolerance
    (1e-5 of the largest |logit|, tests/test_gpu_ops.py)."""
    lib = _lib.load()
    x = x.contiguous()
    M, K = x.shape
    V = w_hi.shape[0]
    st = _device.stream_ptr()
    x16 = torch.empty((2 * M, K), dtype=torch.float16, device=x.device)
    inv = torch.empty((M,), dtype=torch.float32, device=x.device)
    _lib.check(lib.qmb_lm_split16(x.data_ptr(), int(M), int(K), x16.data_ptr(), inv.data_ptr(), st), "lm_split16")
    prev = torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    try:
        p = torch.mm(x16, w_hi.T, out_dtype=torch.float32)
        q = torch.mm(x16[:M], w_lo.T, out_dtype=torch.float32)
    finally:
        torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = prev
    out = torch.empty((M, V), dtype=torch.float32, device=x.device)
    _lib.check(lib.qmb_lm_combine16(p.data_ptr(), q.data_ptr(), inv.data_ptr(), int(M), int(V), int(k),
                                    out.data_ptr(), st), "lm_combine16")
    return out


def device_model(model) -> DeviceModel:
    """The device mirror of a QuantizedModel, cached on the object; rebuilt when the
    embedding / norm arrays are replaced (each block's handle revalidates itself)."""
    dm = model.__dict__.get("_qmb_device_model")
    fp = (id(model.embedding), id(model.final_norm), tuple(id(l.norm_weight) for l in model.layers),
          tuple(id(l.block) for l in model.layers))
    if dm is None or model.__dict__.get("_qmb_device_model_fp") != fp:
        dm = DeviceModel(model)
        model.__dict__["_qmb_device_model"] = dm
        model.__dict__["_qmb_device_model_fp"] = fp
    else:
        dm.blocks = [device_block(l.block) for l in model.layers]
    return dm


def forward_q(model, tokens):
    """model.py:246-258: tokens (T,) -> logits (T, vocab) f32 (numpy in, numpy out)."""
    as_numpy = not is_device(tokens)
    tok = _device.to_device(np.asarray(tokens, dtype=np.int64) if as_numpy else tokens, torch.int64)
    squeeze = tok.dim() == 1
    if squeeze:
        tok = tok[None]
    logits = device_model(model).forward(tok)
    _device.err_flag().raise_if_set()
    if squeeze:
        logits = logits[0]
    return logits.cpu().numpy() if as_numpy else logits


def forward(model, tokens, observer=None):
    """model.py:261-266 (quantized models only on this path)."""
    if observer is not None:
        raise ValueError("observers attach to the float path only")
    return forward_q(model, tokens)
