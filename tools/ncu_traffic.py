#!/usr/bin/env python
"""Per-launch DRAM traffic of the layer kernels from the `ncu --page raw` exports
of tools/ncu_layer.sh -> profiles/dram_traffic.json (read by bench.py for the
roofline `traffic` field).  usage: tools/ncu_traffic.py gpurun_out/ncu profiles/dram_traffic.json"""
import csv
import json
import sys
from pathlib import Path

STAGE = {"gemm_i8_tc_kernel_0": "in_proj", "gemm_i8_tc_kernel_1": "x_proj", "gemm_i8_tc_kernel_2": "dt_proj",
         "gemm_i8_tc_kernel_3": "out_proj", "scan_p2_0": "scan", "scan_c1_0": "scan", "conv_silu_quant_0": "conv",
         "hadamard_0": "hadamard_quant", "rmsnorm_0": "rmsnorm_residual_layer0", "rmsnorm_1": "rmsnorm_final", "bc_dequant_0": "bc_dequant"}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, units, data = rows[hi], rows[hi + 1], rows[hi + 2:]
    out = {}
    for r in data[:1]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        out["kernel"] = d.get("Kernel Name", "")[:120]

        def val(k, scale_units):
            if k not in d:
                return None
            v = float(d[k].replace(",", ""))
            return v * scale_units.get(u.get(k, ""), 1.0)

        byte_units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        rd = val("dram__bytes_read.sum", byte_units)
        wr = val("dram__bytes_write.sum", byte_units)
        t = val("gpu__time_duration.sum", {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                                           "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0})
        out.update(dram_read=rd, dram_write=wr, dram_bytes=(rd or 0) + (wr or 0), seconds_under_ncu=t)
        for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
            if k in d:
                out[k] = float(d[k].replace(",", ""))
    return out


def parse_details(path):
    """Elapsed / SM-active cycles and issue-slot utilisation from the details export:
    what bounds a kernel that is neither at its DRAM nor its tensor roofline."""
    want = {"Elapsed Cycles": "elapsed_cycles", "SM Active Cycles": "sm_active_cycles",
            "Issue Slots Busy": "issue_slots_busy_pct", "SM Frequency": "sm_ghz"}
    out = {}
    rows = list(csv.reader(open(path)))
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = want.get(d.get("Metric Name"))
        if k and k not in out:
            try:
                out[k] = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                pass
    return out


def main(src, dst):
    res = {}
    for p in sorted(Path(src).glob("*.raw.csv")):
        key = STAGE.get(p.name[: -len(".raw.csv")])
        if not key:
            continue
        try:
            res[key] = parse(p)
            det = p.with_name(p.name[: -len(".raw.csv")] + ".details.csv")
            if det.exists():
                res[key].update(parse_details(det))
        except Exception as e:  # noqa: BLE001
            print(f"skip {p}: {e}", file=sys.stderr)
    Path(dst).write_text(json.dumps({"source": "ncu --set full --clock-control none, one launch per kernel "
                                               "(tools/ncu_layer.sh on tools/profile_layer.py, 2.8B shape, "
                                               "M = 65,536 rows)", "kernels": res}, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
