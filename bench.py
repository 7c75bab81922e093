#!/usr/bin/env python
"""Benchmark: W8A8 Mamba-2.8B-shape prefill (1K tokens) + decode on B200.

Our arm (default): one step = batched prefill of B sequences x T tokens through
all 64 layers (embedding, fused residual+RMSNorm+quant, the seven-kernel
block, final norm, last-position tied LM head, greedy argmax) on device-resident
inputs.  `e2e` is the same step through the public API with the tokens copied
from pinned host memory and the last-position logits copied back.  Decode
(carried state, one token per sequence) is measured after it.
Reference arm (--impl reference): the reference itself (ssmq with its compiled
Cython backend, built into oracle/_ref by oracle/build_ref.sh) timed on all
host cores, one 2.8B layer per process on a bounded token sample, extrapolated
linearly to 64 layers; the oracle port stands in only if oracle/_ref is absent.

Multi-GPU: one process per GPU; `--gpus N` starts the N ranks itself
(torch.distributed.run) unless already under torchrun; sequences are
batch-sharded (weak scaling: B per GPU); the only collective is an all_gather
of the generated token ids (NCCL over NVLink).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "W8A8 Mamba-2.8B tokens/s (1K prefill, decode) and scan/FWHT HBM GB/s vs peak"
UNIT = "tokens/s"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ============================================================== CPU reference arm
REF_DIR = ROOT / "oracle" / "_ref"   # the real reference, built by oracle/build_ref.sh (git-ignored)
SHAPE_2P8B = dict(d_model=2560, d_inner=5120, d_state=16, d_conv=4, dt_rank=160)


def _have_ref() -> bool:
    return (REF_DIR / "ssmq").is_dir()


def _ref_layer_sample(args):
    """Time one 2.8B-shape layer of the UNMODIFIED reference (ssmq, compiled
    Cython backend): fused_rmsnorm_quant (qblock.py:170) + block_forward_q
    (qblock.py:185) on T tokens, exactly the per-layer body of forward_q
    (model.py:251-256).  Returns seconds.  Weights follow the reference's own
    init + quantize_block (ssm.py:183-210, qblock.py:223-240)."""
    T, seed = args
    import sys as _s
    _s.path.insert(0, str(REF_DIR))
    import numpy as np
    import ssmq.hadamard as rh
    from ssmq import kernels
    from ssmq.qblock import ACT_SITES, Mode, ScaleEntry, block_forward_q, fused_rmsnorm_quant, quantize_block
    from ssmq.quant import QuantScheme, SchemeKind
    from ssmq.ssm import BlockConfig, init_block_params

    assert kernels.backend_name() == "compiled"
    rh.MAX_TRANSFORM_DIM = 8192  # the 2.8B shape needs the patched transform bound
    c = SHAPE_2P8B
    cfg = BlockConfig(d_model=c["d_model"], expand=2, d_state=c["d_state"], d_conv=c["d_conv"], dt_rank=c["dt_rank"])
    rng = np.random.default_rng(seed)
    params = init_block_params(cfg, rng)
    sch = QuantScheme(SchemeKind.STATIC_SYMMETRIC_MAX)
    scales = {"in": 0.03, "conv_in": 0.02, "conv_out": 0.01, "x": 0.01, "b": 0.01, "c": 0.01, "dt_r": 0.01,
              "dt": 0.1 / 127, "y": 0.01, "y_had": 0.2}
    act = {k: ScaleEntry(scales[k], 0, sch) for k in ACT_SITES}
    act["x"] = ScaleEntry(scales["x"], 0, QuantScheme(SchemeKind.STATIC_SYMMETRIC_PERCENTILE, 99.999))
    blk = quantize_block(params, cfg, act, Mode.FULL, rh.plan_for_dim(cfg.d_inner))
    x = rng.standard_normal((T, c["d_model"])).astype(np.float32)
    gain = np.ones(c["d_model"], np.float32)
    t0 = time.perf_counter()
    u_q, res = fused_rmsnorm_quant(x, np.zeros_like(x), gain, 0.03)
    block_forward_q(u_q, blk)
    return time.perf_counter() - t0


def _oracle_layer_sample(args):
    """Fallback when the reference was not built: the CPU oracle port (oracle/),
    same per-layer work.  Returns seconds."""
    T, seed = args
    import numpy as np
    from oracle import oracle as o
    from paper_2410_13229_b200.hadamard import plan_for_dim

    D, E, N, K, R = 2560, 5120, 16, 4, 160
    rng = np.random.default_rng(seed)

    def w(shape, s):
        return rng.integers(-127, 128, size=shape).astype(np.int8), s

    plan = plan_for_dim(E)
    weights = {"a": (rng.integers(-127, -8, size=(E, N)).astype(np.int8), 16 / 127), "d": w((E,), 1 / 127),
               "w_in": w((D, 2 * E), 0.02 / 127), "conv_w": w((K, E), 0.5 / 127), "conv_b": w((E,), 0.5 / 127),
               "w_b": w((E, N), 0.014 / 127), "w_c": w((E, N), 0.014 / 127), "w_dt_rank": w((E, R), 0.014 / 127),
               "w_dt": w((R, E), 0.08 / 127), "dt_bias": w((E,), 4.6 / 127), "w_out_h": w((E, D), 1.0 / 127)}
    act = {s: 0.05 for s in o.ACT_SITES}
    act["dt"] = 0.1 / 127
    blk = o.Block(dict(d_model=D, d_inner=E, d_state=N, d_conv=K, dt_rank=R, bit_width=8), "full", weights, act,
                  (plan.p, plan.m, plan.base))
    x = rng.standard_normal((T, D)).astype(np.float32)
    gain = np.ones(D, np.float32)
    t0 = time.perf_counter()
    u_q, res = o.fused_rmsnorm_quant(x, np.zeros_like(x), gain, 0.03)
    o.block_forward_q(u_q, 0.03, blk)
    return time.perf_counter() - t0


def cpu_baseline(T: int = 8, procs: int = 1, layers: int = 64, pool=None):
    """The reference's CPU path on the host: the real ssmq when oracle/_ref was
    built (kind "reference"), else the oracle port (kind "port").  One 2.8B
    layer at T tokens per process (`procs` independent sequences in parallel,
    SPEC.md:393), extrapolated linearly x layers (linear in T, L)."""
    ref = _have_ref()
    fn = _ref_layer_sample if ref else _oracle_layer_sample
    if pool is None:
        secs = [fn((T, 0))]
        procs = 1
    else:
        secs = pool.map(fn, [(T, i) for i in range(procs)])
    t = max(secs)
    value = procs * T / (t * layers)
    what = ("ssmq (the reference, compiled Cython backend, oracle/_ref) fused_rmsnorm_quant + block_forward_q"
            if ref else "oracle/ CPU restatement (numpy int32 matmul via f64 BLAS + C scan)")
    return {"value": value, "unit": UNIT, "cores": procs, "kind": "reference" if ref else "port",
            "sample": f"{procs} process(es) x 1 layer of the 2.8B shape (D=2560,E=5120,N=16,R=160) at T={T} "
                      f"tokens each, {t:.2f} s/layer, extrapolated x{layers} layers; {what}"}


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    from multiprocessing import get_context

    procs = max(1, (os.cpu_count() or 1))
    T = args.ref_tokens
    with get_context("spawn").Pool(procs) as pool:
        for _ in range(min(args.warmup, 1)):  # imports + first-touch outside the timed samples
            cpu_baseline(T=1, procs=procs, pool=pool)
        t0 = time.perf_counter()
        vals = []
        cb = None
        for _ in range(args.steps):
            cb = cpu_baseline(T=T, procs=procs, pool=pool)
            vals.append(cb["value"])
        elapsed = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8/int32/f32", "data": "synthetic",
            "config": {"workload": f"Mamba-2.8b-shape W8A8 prefill (reference CPU path, bounded sample)",
                       "d_model": 2560, "n_layers": 64, "d_state": 16, "dt_rank": 160,
                       "tokens_per_layer_sample": T, "same_config": False},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": cb["kind"], "sample": cb["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ============================================================== GPU arm
def _timed(fn, n, stream, world, dev):
    """CUDA-event time of n calls on `stream` (barrier + synchronize on both
    sides), max over ranks.  Returns ms per call."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / n
    if world > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def _decode_bytes(cfg, B: int) -> float:
    """Algorithmic HBM bytes of one decode step: every int8 weight
    once, the f32 state h read + written and the int8 conv window read +
    written per sequence and layer, the f32 tied embedding once (LM head)."""
    D, E, N, K, R, L, V = cfg.d_model, cfg.d_inner, cfg.d_state, cfg.d_conv, cfg.dt_rank, cfg.n_layers, cfg.vocab_size
    w = D * 2 * E + E * (2 * N + R) + R * E + E * D + K * E + E * N + 3 * E
    state = B * (E * N * 4 * 2 + (K - 1) * E * 2)
    return float(L * (w + state) + V * D * 4)


def _decode_line(dm, cfg, tokens, B, steps, stream, world, dev, hbm):
    """Decode with carried state: prefill 16 tokens, capture one CUDA graph of a
    full decode step (all layers + LM head), time its replay."""
    _, states = dm.prefill(tokens[:B, :16].contiguous())
    graph, tok_in, _ = dm.capture_decode(states)
    tok_in.copy_(tokens[:B, 0])
    for _ in range(3):
        graph.replay()
    ms = _timed(graph.replay, steps, stream, world, dev)
    nbytes = _decode_bytes(cfg, B)
    ach = nbytes / (ms * 1e-3) / 1e9
    del graph, states
    return {"value": world * B / (ms * 1e-3), "unit": "tokens/s", "batch_per_gpu": B, "ms_per_token": ms,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "algorithmic_bytes_per_step": nbytes},
            "note": "one token per sequence per step, carried (conv window, h) state, CUDA-graph replay"}


def _prefill_line(dm, tokens, steps, stream, world, dev):
    B, T = tokens.shape
    dm.forward(tokens, last_only=True)
    ms = _timed(lambda: dm.forward(tokens, last_only=True), steps, stream, world, dev)
    return {"value": world * B * T / (ms * 1e-3), "unit": "tokens/s", "batch_per_gpu": B, "seq_len": T,
            "ms_per_step": ms}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch through torchrun or let "
                         f"bench.py spawn the ranks)")
    ndev = torch.cuda.device_count()
    shared = False
    if ndev < world:
        if not args.shared_gpu_dry_run:
            raise SystemExit(f"bench.py: --gpus {world} needs {world} GPUs, this node has {ndev}")
        shared = True  # plumbing dry run: ranks share the GPU(s); NCCL refuses that, so gloo
    torch.cuda.set_device(local % max(ndev, 1))
    backend = None
    if world > 1:
        backend = "gloo" if shared else "nccl"
        dist.init_process_group(backend)
        assert dist.get_world_size() == world
    from paper_2410_13229_b200 import _device, _lib
    from paper_2410_13229_b200.model import device_model, prefill_groups
    from paper_2410_13229_b200.synthetic import CONFIGS, build_model

    lib = _lib.load()
    cfg = CONFIGS[args.config]
    B, T = args.batch, args.seq
    t_build = time.perf_counter()
    qm = build_model(cfg, seed=args.seed, calib_tokens=args.calib_tokens)
    dm = device_model(qm)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    dev = _device.device()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    tokens = torch.randint(0, cfg.vocab_size, (B, T), device=dev, generator=gen)
    stream = torch.cuda.current_stream()
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))

    gathered = torch.empty((world * B,), dtype=torch.int64, device=dev)

    def step(tok):
        logits = dm.forward(tok, last_only=True)
        nxt = dm.argmax(logits)
        if world > 1:
            if shared:  # gloo dry run: host copies
                parts = [torch.empty_like(nxt, device="cpu") for _ in range(world)]
                dist.all_gather(parts, nxt.cpu())
            else:
                dist.all_gather_into_tensor(gathered, nxt)
        return logits, nxt

    for _ in range(args.warmup):
        step(tokens)
    torch.cuda.synchronize()
    _device.err_flag().raise_if_set()
    if args.ncu:
        # one profiled step between cudaProfilerStart/Stop (ncu --profile-from-start off)
        torch.cuda.profiler.start()
        step(tokens)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_step": "done", "config": args.config, "batch": B, "seq": T}), flush=True)
        return

    with ClockSampler(local % max(ndev, 1)) as clk:
        ms = _timed(lambda: step(tokens), args.steps, stream, world, dev)
    value = world * B * T / (ms * 1e-3)

    # ---------------------------------------------------------- e2e through the public API
    host_tok = torch.empty((B, T), dtype=torch.int64).pin_memory()
    host_tok.copy_(tokens.cpu())
    host_logits = torch.empty((B, cfg.vocab_size), dtype=torch.float32).pin_memory()

    def e2e_step():
        tok = host_tok.to(dev, non_blocking=True)
        logits, _ = step(tok)
        host_logits.copy_(logits, non_blocking=True)

    e2e_step()
    ms_e2e = _timed(e2e_step, max(1, args.steps), stream, world, dev)
    e2e = {"value": world * B * T / (ms_e2e * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": host_tok.numel() * 8, "d2h_bytes_per_step": host_logits.numel() * 4}

    # ---------------------------------------------------------- decode (carried state), B and 1
    decode = _decode_line(dm, cfg, tokens, B, max(10, args.steps * 8), stream, world, dev, hbm)
    extras = {}
    if not args.no_extras:
        # BASELINE config 3, batch 1: prefill 1K tokens of one sequence + decode at B = 1
        extras["batch1_prefill"] = _prefill_line(dm, tokens[:1].contiguous(), max(3, args.steps), stream, world, dev)
        extras["batch1_decode"] = _decode_line(dm, cfg, tokens, 1, max(20, args.steps * 8), stream, world, dev, hbm)
        # BASELINE config 4 per-GPU shard: 32 sequences x 16K tokens over 8 GPUs = 4 x 16K per GPU
        Tl = 16384
        ltok = torch.randint(0, cfg.vocab_size, (4, Tl), device=dev, generator=gen)
        extras["long_context_4x16k"] = _prefill_line(dm, ltok, 2, stream, world, dev)
        del ltok
        torch.cuda.empty_cache()
    if world > 1 and not args.no_extras:
        # batch-1 latency over all N GPUs: tensor-parallel E-sharding --
        # each rank streams 1/N of every block's weights; three collectives per layer
        # (int32 all-reduces of the x_proj / out_proj partials, a gather of the gated y)
        from paper_2410_13229_b200.tp import DistComm, TPModel

        tpm = TPModel(qm, DistComm(), [rank], world)
        tstates = tpm.new_states(1)
        tpm.prefill(tokens[:1, :16].contiguous(), tstates)
        cur = tokens[:1, 0].contiguous()
        for _ in range(3):
            tpm.decode_step(cur, tstates)
        mode = "eager"
        step = lambda: tpm.decode_step(cur, tstates)  # noqa: E731
        if backend == "nccl":  # the whole step (collectives included) as one CUDA graph
            try:
                tgraph, ttok, _ = tpm.capture_decode(tstates)
                ttok.copy_(cur)
                step, mode = tgraph.replay, "CUDA graph"
            except Exception as exc:  # (fall back to eager timing, say so)
                mode = f"eager (graph capture failed: {type(exc).__name__})"
        ms_tp = _timed(step, max(10, args.steps * 4), stream, world, dev)
        extras["tp_batch1_decode"] = {
            "value": 1.0 / (ms_tp * 1e-3), "unit": "tokens/s", "batch": 1, "tensor_parallel": world,
            "ms_per_token": ms_tp,
            "note": "one sequence served by all N GPUs (channel-sharded blocks, %s, %s collectives)" % (mode, backend)}
        del tpm, tstates
        torch.cuda.empty_cache()

    # ---------------------------------------------------------- roofline of the dominant kernel
    import ctypes
    blk = dm.blocks[0]
    M = B * T
    u = torch.randint(-127, 128, (M, cfg.d_model), dtype=torch.int8, device=dev)
    out = torch.empty((M, cfg.d_model), dtype=torch.float32, device=dev)
    ws = _device.workspace(blk.workspace_bytes(M))
    stage_ms = (ctypes.c_float * 7)()
    acc = [0.0] * 7
    reps = 3
    for r in range(reps + 1):
        _lib.check(lib.qmb_block_prefill_profiled(blk.handle, u.data_ptr(), 0.0, B, T, out.data_ptr(), 0,
                                                  ws.data_ptr(), ws.numel(), _device.err_flag().ptr,
                                                  stream.cuda_stream, stage_ms))
        if r:
            acc = [a + s / reps for a, s in zip(acc, stage_ms)]
    del u, out
    names = ["in_proj", "conv", "x_proj", "dt_proj", "scan", "hadamard_quant", "out_proj"]
    D, E, N, R = cfg.d_model, cfg.d_inner, cfg.d_state, cfg.dt_rank
    peak_i8 = ctypes.c_double()
    _lib.check(lib.qmb_measure_i8_peak(2000, ctypes.byref(peak_i8)))
    # algorithmic work per launch.  x_proj / dt_proj are skinny GEMMs whose
    # binding roofline is HBM: activation bytes in + out.
    work = {
        "in_proj": ("tensor", 2.0 * M * D * 2 * E / 1e12, "TFLOP/s"),
        "out_proj": ("tensor", 2.0 * M * E * D / 1e12, "TFLOP/s"),
        "x_proj": ("hbm", (M * E + M * (2 * N + R) + E * (2 * N + R)) / 1e9, "GB/s"),
        "dt_proj": ("hbm", (M * R + M * E + R * E) / 1e9, "GB/s"),
        "conv": ("hbm", M * E * 2 / 1e9, "GB/s"),
        "scan": ("hbm", M * E * (1 + 1 + 4 + 4) / 1e9 + M * 2 * N / 1e9, "GB/s"),
        "hadamard_quant": ("hbm", M * E * 5 / 1e9, "GB/s"),
    }
    per = {}
    for i, n in enumerate(names):
        bound, amt, unit = work[n]
        t = acc[i] * 1e-3
        ach = amt / t
        peak = peak_i8.value if bound == "tensor" else hbm
        per[n] = {"ms": round(acc[i], 4), "bound": bound, "achieved": ach, "unit": unit, "frac": ach / peak}
    dom = max(per, key=lambda k: per[k]["ms"])
    d = per[dom]
    # measured DRAM traffic per launch (ncu --set full, tools/ncu_layer.sh -> profiles/), in the same
    # unit as `achieved` x seconds: bytes for HBM-bound kernels
    traffic = None
    co_bounds = None
    try:
        tr = json.loads((ROOT / "profiles" / "dram_traffic.json").read_text())
        if dom in tr.get("kernels", {}):
            k = tr["kernels"][dom]
            traffic = k["dram_bytes"]
            # what else bounds it (same ncu capture): shared-memory wavefronts per SM-cycle
            # (1 / clk / SM peak; the exact scan's expf table), issue slots, SMs active
            if k.get("elapsed_cycles"):
                sms = torch.cuda.get_device_properties(0).multi_processor_count
                wf = k.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
                co_bounds = {
                    "shared_wavefront_frac": (wf / (sms * k["elapsed_cycles"]) if wf else None),
                    "issue_slots_busy_frac": (k["issue_slots_busy_pct"] / 100 if "issue_slots_busy_pct" in k else None),
                    "sm_active_frac": (k["sm_active_cycles"] / k["elapsed_cycles"] if "sm_active_cycles" in k else None),
                    "source": "ncu --set full of one launch (profiles/dram_traffic.json, tools/ncu_layer.sh)"}
    except Exception:
        pass
    roofline = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"],
                "peak": peak_i8.value if d["bound"] == "tensor" else hbm, "unit": d["unit"], "frac": d["frac"],
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
                "co_bounds": co_bounds,
                "algorithmic_bytes": (work[dom][1] * 1e9 if d["bound"] == "hbm" else None),
                "peak_source": ("measured tcgen05 kind::i8 probe (qmb_measure_i8_peak)" if d["bound"] == "tensor"
                                else "MEASURED_PEAKS.json hbm_gbs"),
                "per_kernel": per}

    # ---------------------------------------------------------- BASELINE config 2: 130M shape
    if not args.no_extras and args.config == "2.8b":
        del dm, qm
        torch.cuda.empty_cache()
        c130 = CONFIGS["130m"]
        qm130 = build_model(c130, seed=args.seed, calib_tokens=args.calib_tokens)
        dm130 = device_model(qm130)
        tok130 = torch.randint(0, c130.vocab_size, (1, 2048), device=dev, generator=gen)
        extras["130m_prefill_2k"] = _prefill_line(dm130, tok130, max(3, args.steps), stream, world, dev)
        extras["130m_decode_b1"] = _decode_line(dm130, c130, tok130, 1, 128, stream, world, dev, hbm)
        extras["130m_decode_b1"]["note"] = "128 greedy-decode-shaped steps at batch 1 (CUDA-graph replay)"

    cpu = cpu_baseline(T=8) if (rank == 0 and world == 1 and not args.no_cpu) else None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int8 x int8 -> int32 GEMMs; f32 scan/norm (W8A8)",
                "data": "synthetic tokens, random-init weights (reference init convention), GPU float calibration",
                "config": {"workload": f"Mamba-{args.config}-shape W8A8 prefill {T} tokens x batch {B}/GPU "
                                       f"(+ decode batch {B}/GPU)",
                           "d_model": cfg.d_model, "n_layers": cfg.n_layers, "d_state": cfg.d_state,
                           "dt_rank": cfg.dt_rank, "vocab": cfg.vocab_size, "batch_per_gpu": B, "seq_len": T,
                           "parallelism": f"dp{world} (batch-sharded, all_gather of next tokens)",
                           "l2": "inputs larger than L2 (per-layer activations >= 1.3 GB)",
                           "step": "embed + 64x(rmsnorm+block) + final norm + last-position LM head + argmax"},
                "e2e": e2e, "decode": decode, "extras": extras, "roofline": roofline, "cpu_baseline": cpu,
                "comm": {"backend": backend, "world_size": world,
                         "dry_run_shared_gpu": shared, "collective": "all_gather_into_tensor of next-token ids"},
                # ours per step: per prefill row group (model.prefill_groups) embed + L x (rmsnorm, in_proj,
                # conv, x_proj, dt_proj, bc_dequant, scan, hadamard, out_proj) + final norm; then LM-head
                # split / combine (or the f32 GEMV at <= 8 rows) + argmax (the LM head's two cuBLAS GEMMs
                # are not counted)
                "clocks": clk.summary(),
                "gpu_launches": prefill_groups(B, T) * (2 + 9 * cfg.n_layers) + (2 if B > 8 else 1) + 1,
                "gpu_launches_unit": "per step",
                "int8_peak_tops": peak_i8.value, "build_s": round(t_build, 1)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="2.8b", choices=["tiny", "130m", "2.8b"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--calib-tokens", type=int, default=256)
    ap.add_argument("--ref-tokens", type=int, default=8, help="reference arm: tokens per layer sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip batch-1 / long-context / 130M lines")
    ap.add_argument("--shared-gpu-dry-run", action="store_true",
                    help="let N ranks share fewer GPUs (gloo) to exercise the multi-rank path; not a measurement")
    ap.add_argument("--ncu", action="store_true", help="profile one prefill step (ncu --profile-from-start off)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
