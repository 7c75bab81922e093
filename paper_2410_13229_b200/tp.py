"""Tensor-parallel E-sharding of the quantized block.

For batch-1 latency at the 2.8B shape the channels (d_inner) of every block are
split over G ranks, rank r owning the contiguous range [r E/G, (r+1) E/G).  Its
block handle is an ordinary libqmb handle built from that slice of the weights
(`w_in`'s x and z columns, the conv taps, a, d, dt_bias and `w_dt`'s columns of
those channels; the rows of `w_b`, `w_c`, `w_dt_rank` and `w_out(_h)` as K-slices;
every per-tensor scale unchanged), run through `qmb_block_tp_stage` in four
stages around three collectives (qblock.py:185-215):

  1  in_proj, conv, x_proj over the local K-slice    -> int32 [M, 2N+R]   all-reduce SUM
  2  x_proj requant, dt_proj, scan, gate              -> f32 y [M, E/G]   all-gather (channels)
  3  Hadamard of the gathered y (full plan), out_proj over the local K-slice
                                                      -> int32 [M, D]     all-reduce SUM
  4  out_proj epilogue

x_proj and out_proj partial products are exchanged as int32 accumulators, exact
and order-independent, so every rank's output is bit-identical to the unsharded
block.  The Hadamard couples all channels; instead of exchanging the top
log2(G) butterfly stages pairwise, each rank gathers the gated y once and runs the
whole transform (its cost is small next to the weight streaming TP divides).

Collectives: `torch.distributed` (NCCL on B200s, gloo in the CPU-host tests) via
`DistComm`, or `VirtualComm`, which runs all G shards in one process on one GPU
(the single-GPU parity tests of the decomposition).
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from . import _device, _lib
from .hadamard import plan_for_dim
from .qblock import DeviceBlock
from .quant import QTensor


def shard_block(qb, rank: int, world: int):
    """The channel slice of a QuantizedBlock owned by `rank` (a block-like object)."""
    E = int(qb.cfg.d_inner)
    if E % world or (E // world) % 16:
        raise ValueError(f"d_inner {E} does not split into {world} slices of whole 16-channel groups")
    El = E // world
    e0 = rank * El
    sl = slice(e0, e0 + El)
    W = {k: (v.values.detach().cpu().numpy() if isinstance(v.values, torch.Tensor) else np.asarray(v.values))
         for k, v in qb.weights.items()}
    parts = {
        "w_in": np.concatenate([W["w_in"][:, sl], W["w_in"][:, E + e0:E + e0 + El]], axis=1),
        "conv_w": W["conv_w"][:, sl], "conv_b": W["conv_b"][sl], "a": W["a"][sl], "d": W["d"][sl],
        "dt_bias": W["dt_bias"][sl], "w_b": W["w_b"][sl], "w_c": W["w_c"][sl], "w_dt_rank": W["w_dt_rank"][sl],
        "w_dt": W["w_dt"][:, sl], "w_out": W["w_out"][sl],
    }
    if "w_out_h" in W:
        parts["w_out_h"] = W["w_out_h"][sl]
    weights = {k: QTensor(np.ascontiguousarray(v), qb.weights[k].scale, qb.weights[k].zero_point,
                          qb.weights[k].bit_width) for k, v in parts.items()}
    local = SimpleNamespace(cfg=qb.cfg, mode=qb.mode, weights=weights, act=qb.act, plan=plan_for_dim(El))
    return local, e0, El


class TPBlock:
    """One rank's shard of a quantized block."""

    def __init__(self, qb, rank: int, world: int):
        local, self.e0, self.El = shard_block(qb, rank, world)
        self.E = int(qb.cfg.d_inner)
        self.D = int(qb.cfg.d_model)
        self.N, self.R = int(qb.cfg.d_state), int(qb.cfg.dt_rank)
        self.Nx = 2 * self.N + self.R
        self.dev = DeviceBlock(local, d_inner=self.El)
        self.full_plan = qb.plan
        self._base = np.ascontiguousarray(np.asarray(qb.plan.base, dtype=np.int8))
        self.act_in = float(qb.act["in"].scale)

    def new_state(self, B: int):
        return self.dev.new_state(B)

    def buffers(self, M: int) -> dict:
        dev = _device.device()
        return dict(xacc=torch.empty((M, self.Nx), dtype=torch.int32, device=dev),
                    y_local=torch.empty((M, self.El), dtype=torch.float32, device=dev),
                    yq_full=torch.empty((M, self.E), dtype=torch.int8, device=dev),
                    oacc=torch.empty((M, self.D), dtype=torch.int32, device=dev),
                    ws=torch.empty(self.dev.workspace_bytes(M), dtype=torch.uint8, device=dev))

    def stage(self, k: int, bufs: dict, u_q, B: int, T: int, *, y_full=None, decode=False, conv=None, h=None,
              out=None, accumulate=False, err=None, u_scale=None):
        a = _lib.TpArgs()
        a.stage = k
        a.xacc = bufs["xacc"].data_ptr()
        a.y_local = bufs["y_local"].data_ptr()
        a.y_full = y_full.data_ptr() if y_full is not None else None
        a.yq_full = bufs["yq_full"].data_ptr()
        a.e_full, a.e0 = self.E, self.e0
        a.had_p, a.had_m, a.had_base = int(self.full_plan.p), int(self.full_plan.m), self._base.ctypes.data
        a.oacc = bufs["oacc"].data_ptr()
        e = err if err is not None else _device.err_flag()
        ws = bufs["ws"]
        _lib.check(_lib.load().qmb_block_tp_stage(
            self.dev.handle, a, _device.ptr(u_q), float(u_scale or 0.0), int(B), int(T), int(decode),
            _device.ptr(conv), _device.ptr(h), _device.ptr(out), int(accumulate), ws.data_ptr(), ws.numel(), e.ptr,
            _device.stream_ptr()), f"qmb_block_tp_stage({k})")


class VirtualComm:
    """All G shards in one process (single-GPU tests): the collectives are sums /
    concatenations of the shards' buffers."""

    def __init__(self, world: int):
        self.world = world

    def all_reduce_sum(self, ts: list):
        s = ts[0].clone()
        for t in ts[1:]:
            s += t
        for t in ts:
            t.copy_(s)

    def all_gather_cols(self, ts: list) -> list:
        full = torch.cat(ts, dim=1).contiguous()
        return [full] * len(ts)


class DistComm:
    """torch.distributed collectives (one process per GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)

    def all_reduce_sum(self, ts: list):
        self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.SUM, group=self.group)

    def all_gather_cols(self, ts: list) -> list:
        y = ts[0].contiguous()
        M, El = y.shape
        flat = torch.empty((self.world * M, El), dtype=y.dtype, device=y.device)
        self.dist.all_gather_into_tensor(flat, y, group=self.group)  # (one buffer: CUDA-graph capturable)
        return [flat.view(self.world, M, El).permute(1, 0, 2).reshape(M, self.world * El).contiguous()]


def tp_block_forward(shards: list, comm, u_q, B: int, T: int, outs: list, *, decode=False, states=None,
                     accumulate=False, bufs=None, u_scale=None):
    """One layer over the local shards (all G for VirtualComm, this rank's one for
    DistComm): out[r] <- the block output (or += with accumulate), states (conv, h)
    per shard carried (decode) or exported (prefill)."""
    M = B * T
    bufs = bufs or [s.buffers(M) for s in shards]
    st = states or [(None, None)] * len(shards)
    for s, b, (cv, hh) in zip(shards, bufs, st):
        s.stage(1, b, u_q, B, T, decode=decode, conv=cv, h=hh, u_scale=u_scale)
    comm.all_reduce_sum([b["xacc"] for b in bufs])
    for s, b, (cv, hh) in zip(shards, bufs, st):
        s.stage(2, b, u_q, B, T, decode=decode, conv=cv, h=hh, u_scale=u_scale)
    y_full = comm.all_gather_cols([b["y_local"] for b in bufs])
    for s, b, y in zip(shards, bufs, y_full):
        s.stage(3, b, None, B, T, y_full=y)
    comm.all_reduce_sum([b["oacc"] for b in bufs])
    for s, b, o in zip(shards, bufs, outs):
        s.stage(4, b, None, B, T, out=o, accumulate=accumulate)
    return outs


class TPModel:
    """The quantized model loop (model.py:246-258) over tensor-parallel blocks:
    embedding, norms and LM head replicated, each block split into channel shards.
    `shard_ids`: the shards this process holds -- [rank] with DistComm, all of
    range(world) with VirtualComm.  Bit-identical to DeviceModel."""

    def __init__(self, model, comm, shard_ids: list, world: int):
        from .model import DeviceModel

        self.comm, self.world, self.ids = comm, world, list(shard_ids)
        base = DeviceModel.__new__(DeviceModel)  # embedding / norm / LM-head helpers only
        cfg = model.config
        base.cfg, base.D, base.V, base.bits = cfg, int(cfg.d_model), int(cfg.vocab_size), int(cfg.bit_width)
        from .model import _f32_dev

        base.embedding = _f32_dev(model.embedding)
        base.final_norm = _f32_dev(model.final_norm)
        base.norms = [_f32_dev(l.norm_weight) for l in model.layers]
        base.s_in = [float(l.block.act["in"].scale) for l in model.layers]
        base.gains_finite = all(bool(torch.isfinite(g).all()) for g in base.norms + [base.final_norm])
        base._lib = _lib.load()
        self.base = base
        self.layers = [[TPBlock(l.block, r, world) for r in self.ids] for l in model.layers]

    def new_states(self, B: int):
        return [[s.new_state(B) for s in shards] for shards in self.layers]

    def _run(self, tokens: torch.Tensor, B: int, T: int, states, decode: bool):
        M = B * T
        base, stream, err = self.base, _device.stream_ptr(), _device.err_flag()
        x_out = base.embed(tokens)
        res = [torch.zeros_like(x_out) for _ in self.ids]
        u_q = torch.empty((M, base.D), dtype=torch.int8, device=x_out.device)
        bufs = [s.buffers(M) for s in self.layers[0]]
        for li, shards in enumerate(self.layers):
            if li == 0:
                base._rmsnorm(x_out, res[0], res[0], base.norms[li], base.s_in[li], u_q, None, M, err, stream)
                for r in res[1:]:
                    r.copy_(res[0])
            else:
                base._rmsnorm(res[0], None, None, base.norms[li], base.s_in[li], u_q, None, M, err, stream)
            tp_block_forward(shards, self.comm, u_q, B, T, res, decode=decode,
                             states=states[li] if states is not None else None, accumulate=True, bufs=bufs)
        final = torch.empty_like(x_out)
        base._rmsnorm(res[0], None, None, base.final_norm, 1.0, None, final, M, err, stream)
        return final

    def forward_hidden(self, tokens: torch.Tensor, states=None) -> torch.Tensor:
        B, T = tokens.shape
        return self._run(tokens, B, T, states, False)

    def prefill(self, tokens: torch.Tensor, states=None):
        B, T = tokens.shape
        states = states if states is not None else self.new_states(B)
        final = self._run(tokens, B, T, states, False)
        return self.base.lm_head(final.reshape(B, T, self.base.D)[:, -1]), states

    def decode_step(self, tokens: torch.Tensor, states) -> torch.Tensor:
        B = tokens.shape[0]
        return self.base.lm_head(self._run(tokens, B, 1, states, True))

    def capture_decode(self, states):
        """One decode step (every layer's four stages and three collectives, norms,
        LM head) captured as a CUDA graph bound to `states`, as DeviceModel.capture_decode:
        returns (graph, token_in [B] int64, logits_out [B, V]).  With DistComm the NCCL
        collectives are captured too (warmed up first, outside the capture)."""
        B = states[0][0][1].shape[0]
        dev = _device.device()
        tok = torch.zeros(B, dtype=torch.int64, device=dev)
        scratch = self.new_states(B)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # lazy init (communicators, kernel attributes) outside the capture
            self.decode_step(tok, scratch)
            self.decode_step(tok, scratch)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        _device.err_flag().reset()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            logits = self.decode_step(tok, states)
        graph._qmb_keep = scratch
        return graph, tok, logits
