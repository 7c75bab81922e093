#!/usr/bin/env python
"""Opcode histogram and top stall lines from `ncu --page source --csv --print-source sass` exports."""
import collections
import csv
import gzip
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    i = next(k for k, r in enumerate(rows) if "Source" in r and "Address" in r)
    return rows[i], rows[i + 1:]


def main(path, top=30):
    h, data = load(path)
    si = h.index("Source")
    wi = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    tot = sum(int(r[wi] or 0) for r in data if len(r) > wi)
    totE = sum(int(r[ei] or 0) for r in data if len(r) > ei)
    print("stall samples", tot, "warp instructions", totE)
    opx = collections.Counter()
    st = collections.Counter()
    for r in data:
        if len(r) <= ei:
            continue
        toks = r[si].strip().split()
        if not toks:
            continue
        o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        o = o.split(".")[0]
        opx[o] += int(r[ei] or 0)
        st[o] += int(r[wi] or 0)
    for o, c in opx.most_common(22):
        print(f"  {o:10s} exec {100 * c / max(totE, 1):5.1f}%  stall {100 * st[o] / max(tot, 1):5.1f}%")
    reasons = collections.Counter()
    for c in h:
        if c.startswith("stall_") and "Not Issued" not in c:
            k = h.index(c)
            reasons[c[6:]] = sum(int(r[k] or 0) for r in data if len(r) > k)
    print("stall reasons:", ", ".join(f"{k} {100 * v / max(tot, 1):.1f}%" for k, v in reasons.most_common(8)))
    if "L1 Wavefronts Shared" in h:
        k1, k2 = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
        w = sum(int(r[k1] or 0) for r in data if len(r) > k1)
        wi_ = sum(int(r[k2] or 0) for r in data if len(r) > k2)
        print(f"shared wavefronts {w} (ideal {wi_}), per warp instr {w / max(totE, 1):.3f}")
    print("top stall instructions:")
    for r in sorted([r for r in data if len(r) > wi], key=lambda r: -int(r[wi] or 0))[:top]:
        print(f"  {r[wi]:>7} {r[ei]:>10}  {r[si][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
