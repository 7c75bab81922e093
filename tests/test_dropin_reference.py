"""The reference's OWN tests (pkg/tests/test_qblock.py, test_model.py, built into
oracle/_ref by oracle/build_ref.sh) run against this library: the quantized
block operators and forward_q are rebound to the B200 implementations by
tests/dropin_plugin.py (SURVEY.md §8b "rebinding helpers let the reference tests
run on B200 unchanged").  Asserts the suite passes AND that the rebound
operators were actually called."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", ["test_qblock.py", "test_model.py"])
def test_reference_suite_through_dropin(cuda, tmp_path, suite):
    if not (REF / "ssmq").is_dir() or not (REF / "tests" / suite).exists():
        pytest.skip("oracle/_ref not built (bash oracle/build_ref.sh)")
    counts = tmp_path / "counts.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(REF / "tests"), str(ROOT / "tests"), str(ROOT)]),
               QMB_DROPIN_COUNTS=str(counts))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin", "-p", "no:cacheprovider",
                        "--rootdir", str(REF / "tests"), str(REF / "tests" / suite)],
                       cwd=str(REF / "tests"), env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    n = json.loads(counts.read_text())
    assert sum(n.values()) > 0, n
    if suite == "test_qblock.py":
        assert n.get("ssmq.qblock.block_forward_q", 0) > 0 and n.get("ssmq.qblock.fused_rmsnorm_quant", 0) > 0, n
    else:
        assert n.get("ssmq.model.forward_q", 0) > 0, n
