"""pytest plugin: run the REFERENCE's own test suite with its quantized block
operators rebound to this library (the drop-in of SURVEY.md §8b).

Loaded with `-p dropin_plugin` before collection, so the reference test modules'
`from ssmq.qblock import block_forward_q, ...` bind the B200 implementations.
Rebound (reference file:line of each original):
  ssmq.qblock.block_forward_q       qblock.py:185   (also ssmq.model's global, model.py:14)
  ssmq.qblock.fused_rmsnorm_quant   qblock.py:170   (also ssmq.model's global)
  ssmq.qblock.qlinear               qblock.py:98
  ssmq.qblock.fused_qconv           qblock.py:126
  ssmq.qblock.quantized_selective_scan qblock.py:146
  ssmq.hadamard.hadamard_quantize   hadamard.py:164
  ssmq.model.forward_q              model.py:246    (forward / evaluate look it up at call time)
Every call is counted; the counts are written to $QMB_DROPIN_COUNTS at exit so the
outer test can prove the B200 path ran.  Test infrastructure only.
"""
from __future__ import annotations

import atexit
import json
import os
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import ssmq.hadamard as _rh  # noqa: E402
import ssmq.model as _rm  # noqa: E402
import ssmq.qblock as _rq  # noqa: E402
from ssmq import kernels as _rk  # noqa: E402

import paper_2410_13229_b200 as _ours  # noqa: E402
from paper_2410_13229_b200 import _lib  # noqa: E402

assert _rk.backend_name() == "compiled", "reference must run its compiled backend"
_lib.load()  # fail loudly: no library -> no drop-in

COUNTS: Counter = Counter()


def _counted(name, fn):
    def wrapper(*a, **k):
        COUNTS[name] += 1
        return fn(*a, **k)

    wrapper.__name__ = name
    wrapper.__doc__ = fn.__doc__
    return wrapper


_REBIND = {
    (_rq, "block_forward_q"): _ours.block_forward_q,
    (_rq, "fused_rmsnorm_quant"): _ours.fused_rmsnorm_quant,
    (_rq, "qlinear"): _ours.qlinear,
    (_rq, "fused_qconv"): _ours.fused_qconv,
    (_rq, "quantized_selective_scan"): _ours.quantized_selective_scan,
    (_rh, "hadamard_quantize"): _ours.hadamard_quantize,
    (_rm, "block_forward_q"): _ours.block_forward_q,
    (_rm, "fused_rmsnorm_quant"): _ours.fused_rmsnorm_quant,
    (_rm, "forward_q"): _ours.forward_q,
}
for (mod, name), fn in _REBIND.items():
    setattr(mod, name, _counted(f"{mod.__name__}.{name}", fn))


def _dump():
    out = os.environ.get("QMB_DROPIN_COUNTS")
    if out:
        Path(out).write_text(json.dumps(dict(COUNTS)))


atexit.register(_dump)
