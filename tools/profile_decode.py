#!/usr/bin/env python
"""Decode-step profiling on a synthetic 2-layer 2.8B-shape model: per-launch
device times of one decode step (run under `ncu --profile-from-start off` for
the launch list), plus CUDA-event time of eager vs graph-replayed steps."""
import argparse
import dataclasses
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--layers", type=int, default=2)
    args = ap.parse_args()
    import torch

    from paper_2410_13229_b200 import _device
    from paper_2410_13229_b200.model import device_model
    from paper_2410_13229_b200.synthetic import CONFIGS, build_model

    cfg = dataclasses.replace(CONFIGS["2.8b"], n_layers=args.layers)
    dm = device_model(build_model(cfg, seed=0, calib_tokens=64))
    dev = _device.device()
    B = args.batch
    tokens = torch.randint(0, cfg.vocab_size, (B, 8), device=dev)
    _, states = dm.prefill(tokens)
    bufs = dm.decode_buffers(B)
    cur = tokens[:, 0].contiguous()
    for _ in range(3):
        dm.decode_step(cur, states, bufs=bufs)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    dm.decode_step(cur, states, bufs=bufs)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        dm.decode_step(cur, states, bufs=bufs)
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / n
    host = (time.perf_counter() - t0) / n * 1e3
    graph, tok, _ = dm.capture_decode(states)
    tok.copy_(cur)
    graph.replay()
    e0.record()
    for _ in range(n):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"layers": args.layers, "batch": B, "eager_ms": eager, "eager_host_ms": host,
                      "graph_ms": e0.elapsed_time(e1) / n}))


if __name__ == "__main__":
    main()
