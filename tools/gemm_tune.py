#!/usr/bin/env python
"""Time the tcgen05 int8 GEMM at the 2.8B layer shapes with each epilogue mode
(qmb_gemm_bench) and print achieved TOP/s vs the measured int8 peak."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch  # noqa: F401  (CUDA context)
    from paper_2410_13229_b200 import _lib

    lib = _lib.load()
    peak = ctypes.c_double()
    _lib.check(lib.qmb_measure_i8_peak(2000, ctypes.byref(peak)))
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    shapes = {"in_proj": (M, 10240, 2560), "out_proj": (M, 2560, 5120), "x_proj": (M, 192, 5120),
              "dt_proj": (M, 5120, 160)}
    res = {"int8_peak_tops": peak.value}
    ms = ctypes.c_float()
    for name, (m, n, k) in shapes.items():
        for mode in (0, 1, 2, 3, 4):
            if lib.qmb_gemm_bench(m, n, k, mode, 5, ctypes.byref(ms)) != 0:
                res[f"{name}/m{mode}"] = "err: " + lib.qmb_last_error().decode()
                continue
            tops = 2.0 * m * n * k / (ms.value * 1e-3) / 1e12
            res[f"{name}/m{mode}"] = {"ms": round(ms.value, 4), "tops": round(tops, 1),
                                      "frac": round(tops / peak.value, 3)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
