#!/usr/bin/env python
"""Decode-shape (M = batch) int8 GEMM timings per path: tensor-core, SIMT GEMV,
tensor-core with split-K (qmb_gemm_bench; operands L2-resident across iterations)."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch  # noqa: F401
    from paper_2410_13229_b200 import _lib

    lib = _lib.load()
    ms = ctypes.c_float()
    res = {}
    for M in [int(a) for a in (sys.argv[1:] or ["64", "1"])]:
        shapes = {"in_proj": (10240, 2560, 3), "out_proj": (2560, 5120, 0), "x_proj": (192, 5120, 1),
                  "dt_proj": (5120, 160, 4)}
        for name, (n, k, mode) in shapes.items():
            for tag, off in (("tc", 0), ("simt", 10), ("tc_splitk", 20), ("tc_cold", 120), ("simt_cold", 110)):
                rc = lib.qmb_gemm_bench(M, n, k, mode + off, 20, ctypes.byref(ms))
                key = f"M{M}/{name}/{tag}"
                if rc != 0:
                    res[key] = "err: " + lib.qmb_last_error().decode()
                else:
                    res[key] = {"us": round(ms.value * 1e3, 2), "GB/s_weights": round(n * k / (ms.value * 1e-3) / 1e9, 1)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
