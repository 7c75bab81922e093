#!/bin/bash
# Build the REAL reference package (ssmq, Cython backend) into oracle/_ref/ --
# test infrastructure: the drop-in tests rebind its operators to this library,
# and bench.py --impl reference times its block_forward_q on the host cores.
# /root/reference is read-only, so the build runs on a copy under /tmp; only the
# installed package (oracle/_ref/ssmq, git-ignored, shipped to the GPU box with
# the snapshot) lands in the repo.  No reference source is committed.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=${REF_SRC:-/root/reference/pkg}
if [ ! -d "$SRC" ]; then echo "reference not present ($SRC); keeping prebuilt oracle/_ref" >&2; exit 0; fi
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from ssmq import kernels
assert kernels.backend_name() == "compiled", kernels.backend_name()
print("oracle/_ref: ssmq built, backend", kernels.backend_name())
PY
# the reference's own test suite (run against this library by tests/test_dropin_reference.py)
rm -rf "$HERE/_ref/tests"
cp -r "$SRC/tests" "$HERE/_ref/tests"
