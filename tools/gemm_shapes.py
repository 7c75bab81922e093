"""Prefill GEMM shapes of the 2.8B layer through qmb_gemm_bench (ms per launch, warm L2).
mode +1000: random operands.  mode 0: f32 out, 1: int8 out, 3: int8 | f32 halves, 5: int8 | silu f32 halves (in_proj), 4: softplus int8."""
import ctypes, json, sys
sys.path.insert(0, '.')
from paper_2410_13229_b200 import _lib
lib = _lib.load()
ms = ctypes.c_float()
res = {}
for (M, N, K, modes) in ((65536, 10240, 2560, (0, 1, 3, 5, 1000, 1001, 1003, 1005)), (65536, 2560, 5120, (0, 1, 1000)), (65536, 5120, 160, (4, 1, 1004))):
    for mode in modes:
        rc = lib.qmb_gemm_bench(M, N, K, mode, 10, ctypes.byref(ms))
        t = ms.value
        res[f"M{M} N{N} K{K} mode{mode}"] = {"ms": round(t, 4), "TOPS": round(2 * M * N * K / t / 1e9, 1)} if rc == 0 else lib.qmb_last_error().decode()
print(json.dumps(res, indent=1))
