"""Batched prefill as row groups on separate CUDA streams (QMB_PREFILL_STREAMS):
time forward_hidden at the headline shape (2.8B shape, B x T, n layers) per group
count and check the final hidden states are bit-identical to one group."""
import argparse
import dataclasses
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2410_13229_b200.model import device_model  # noqa: E402
from paper_2410_13229_b200.synthetic import CONFIGS, build_model  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--groups", default="1,2,4,1,2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS["2.8b"], n_layers=a.layers)
    dm = device_model(build_model(cfg, seed=0))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    tok = torch.randint(0, cfg.vocab_size, (a.batch, a.seq), device="cuda", generator=gen)
    ref = None
    res = []
    for g in [int(x) for x in a.groups.split(",")]:
        os.environ["QMB_PREFILL_STREAMS"] = str(g)
        out = dm.forward_hidden(tok)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        del out
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            dm.forward_hidden(tok)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        r = {"groups": g, "ms": round(ms, 3), "ms_per_layer": round(ms / a.layers, 4),
             "tok_s_64l": round(a.batch * a.seq / (ms / a.layers * 64) * 1e3, 1), "bit_identical": same}
        print(json.dumps(r), flush=True)
        res.append(r)


if __name__ == "__main__":
    main()
