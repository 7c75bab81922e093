#!/usr/bin/env python
"""BASELINE config 5: the quantized selective scan and the fused Hadamard + int8
quantize over the Mamba family's d_inner (1536 .. 5120) and sequence lengths
1 .. 32K, against the HBM roofline (the reference's kernel benchmark,
pkg/benchmarks/bench_kernels.py, times the same two kernels on the CPU).

Each point is one layer of a synthetic W8A8 block (random init, GPU-calibrated
scales) prefilled at B x T tokens through `qmb_block_prefill_profiled`, which
times every stage with CUDA events on the launching stream; the scan and
Hadamard times are the means over --reps runs.  B = min(64, 65536 / T), so each
point up to T = 1024 is a batch of 64 sequences and the long ones hold ~64K
tokens.  The inputs are the producer stages' fresh outputs (warm in L2 when a
stage's working set is under the 126 MB L2, as inside a real layer).

Algorithmic bytes: scan = M E (x 1 + dt 1 + z 4 + y 4) + M 2N (b | c codes);
Hadamard = M E (f32 in + int8 out).  Roofline: MEASURED_PEAKS.json hbm_gbs.
"""
from __future__ import annotations

import argparse
import ctypes
import dataclasses
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d-model", type=int, nargs="*", default=[768, 1024, 1536, 2048, 2560])
    ap.add_argument("--seq", type=int, nargs="*", default=[1, 128, 1024, 4096, 16384, 32768])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batch", type=int, nargs="*", default=None, help="batch sizes (default: min(64, 65536 / T))")
    ap.add_argument("--out", default="gpurun_out/kernel_sweep.json")
    args = ap.parse_args()
    import torch

    from paper_2410_13229_b200 import _device, _lib
    from paper_2410_13229_b200.model import ModelConfig, device_model
    from paper_2410_13229_b200.synthetic import build_model

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6465.8))
    lib = _lib.load()
    dev = _device.device()
    rows = []
    for D in args.d_model:
        cfg = ModelConfig(vocab_size=1024, d_model=D, n_layers=1, d_state=16, dt_rank=math.ceil(D / 16))
        dm = device_model(build_model(cfg, seed=0, calib_tokens=128))
        blk = dm.blocks[0]
        E, N = 2 * D, 16
        for T, B in [(T, B) for T in args.seq for B in (args.batch or [min(64, max(1, 65536 // T))])]:
            M = B * T
            u = torch.randint(-127, 128, (M, D), dtype=torch.int8, device=dev)
            out = torch.empty((M, D), dtype=torch.float32, device=dev)
            ws = _device.workspace(blk.workspace_bytes(M))
            ms = (ctypes.c_float * 7)()
            acc = [0.0] * 7
            for r in range(args.reps + 1):
                _lib.check(lib.qmb_block_prefill_profiled(blk.handle, u.data_ptr(), 0.0, B, T, out.data_ptr(), 0,
                                                          ws.data_ptr(), ws.numel(), _device.err_flag().ptr,
                                                          torch.cuda.current_stream().cuda_stream, ms))
                if r:
                    acc = [a + m / args.reps for a, m in zip(acc, ms)]
            _device.err_flag().raise_if_set()
            scan_b = M * E * 10 + M * 2 * N
            had_b = M * E * 5
            scan_ms, had_ms = acc[4], acc[5]
            row = {"d_model": D, "d_inner": E, "B": B, "T": T, "M": M,
                   "scan_ms": round(scan_ms, 4), "scan_gbs": round(scan_b / scan_ms / 1e6, 1),
                   "scan_frac": round(scan_b / scan_ms / 1e6 / hbm, 3),
                   "hadamard_ms": round(had_ms, 4), "hadamard_gbs": round(had_b / had_ms / 1e6, 1),
                   "hadamard_frac": round(had_b / had_ms / 1e6 / hbm, 3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del u, out, ws
        del dm, blk
        torch.cuda.empty_cache()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"hbm_gbs": hbm, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
