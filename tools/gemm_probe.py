import ctypes, json, sys
sys.path.insert(0, '.')
import torch
from paper_2410_13229_b200 import _lib
lib = _lib.load()
ms = ctypes.c_float()
res = {}
for mode in (0, 1, 3, 5, 103, 105, 123, 125):
    rc = lib.qmb_gemm_bench(64, 10240, 2560, mode, 20, ctypes.byref(ms))
    res[f"M64 N10240 K2560 mode{mode}"] = round(ms.value * 1e3, 2) if rc == 0 else lib.qmb_last_error().decode()
for mode in (3, 103):
    rc = lib.qmb_gemm_bench(128, 10240, 2560, mode, 20, ctypes.byref(ms))
    res[f"M128 mode{mode}"] = round(ms.value * 1e3, 2)
    rc = lib.qmb_gemm_bench(64, 9472, 2560, mode, 20, ctypes.byref(ms))
    res[f"M64 N9472(148 tiles) mode{mode}"] = round(ms.value * 1e3, 2)
print(json.dumps(res, indent=1))
