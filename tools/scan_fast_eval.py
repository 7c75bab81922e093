#!/usr/bin/env python
"""Fast-mode scan (scan_exp = 2) against the exact scan on one synthetic
Mamba-2.8B-shape layer at the headline size (B = 64 x T = 1024 unless given):
the same block input run both ways, compared stage by stage from the workspace
(gated y: max |d| / max |y|, relative L2; y_q: the fraction of int8 codes that
differ; the final state h; the block output), plus CUDA-event times of the two
scans (qmb_block_prefill_profiled)."""
from __future__ import annotations

import argparse
import ctypes
import dataclasses
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=1024)
    args = ap.parse_args()
    import torch

    from paper_2410_13229_b200 import _device, _lib
    from paper_2410_13229_b200.model import device_model
    from paper_2410_13229_b200.synthetic import CONFIGS, build_model

    cfg = dataclasses.replace(CONFIGS["2.8b"], n_layers=1, vocab_size=1024)
    dm = device_model(build_model(cfg, seed=0, calib_tokens=128))
    blk = dm.blocks[0]
    dev = _device.device()
    B, T = args.batch, args.seq
    M, D, E, N = B * T, cfg.d_model, 2 * cfg.d_model, 16
    # a realistic block input: the first layer's normalized, quantized embeddings
    tokens = torch.randint(0, cfg.vocab_size, (B, T), device=dev)
    x = dm.embed(tokens)
    u = torch.empty((M, D), dtype=torch.int8, device=dev)
    dm._rmsnorm(x, None, None, dm.norms[0], dm.s_in[0], u, None, M, _device.err_flag(), _device.stream_ptr())
    lay = blk.workspace_layout(M)
    runs = {}
    for se in (0, 2):
        ws = torch.zeros(blk.workspace_bytes(M), dtype=torch.uint8, device=dev)
        out = torch.empty((M, D), dtype=torch.float32, device=dev)
        conv, h = blk.new_state(B)
        blk.prefill(u, B, T, out, conv_state_out=conv, ssm_state_out=h, scan_exp=se, workspace=ws)
        _device.err_flag().raise_if_set()
        Ep = (E + 15) // 16 * 16
        gated = ws[lay["Z"]:lay["Z"] + M * E * 4].view(torch.float32).reshape(M, E).clone()
        yq = ws[lay["YQ"]:lay["YQ"] + M * Ep].view(torch.int8).reshape(M, Ep)[:, :E].clone()
        runs[se] = dict(gated=gated, yq=yq, h=h.clone(), out=out.clone())
    ex, fa = runs[0], runs[2]

    def rel(a, b):
        d = (a.double() - b.double())
        return dict(max_abs_over_max=float(d.abs().max() / b.double().abs().max()),
                    rel_l2=float(d.norm() / b.double().norm()))

    res = {"B": B, "T": T, "gated": rel(fa["gated"], ex["gated"]), "h": rel(fa["h"], ex["h"]),
           "out": rel(fa["out"], ex["out"]),
           "y_q_flip_rate": float((fa["yq"] != ex["yq"]).double().mean()),
           "y_q_max_code_diff": int((fa["yq"].int() - ex["yq"].int()).abs().max())}
    lib = _lib.load()
    ms = (ctypes.c_float * 7)()
    out = torch.empty((M, D), dtype=torch.float32, device=dev)
    ws = _device.workspace(blk.workspace_bytes(M))
    for se in (0, 2, 0, 2):
        _lib.check(lib.qmb_block_prefill_profiled(blk.handle, u.data_ptr(), 0.0, B, T, out.data_ptr(), se,
                                                  ws.data_ptr(), ws.numel(), _device.err_flag().ptr,
                                                  torch.cuda.current_stream().cuda_stream, ms))
        res[f"scan_ms_{'exact' if se == 0 else 'fast'}"] = round(ms[4], 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
