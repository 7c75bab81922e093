"""CPU checks of the drop-in boundary: libqmb.so loads without a GPU and exports
every entry point include/qmb.h declares; the ctypes prototypes cover them."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "qmb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qmb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_13229_b200 import _build

    _build.build_library()
    return ctypes.CDLL(str(ROOT / "paper_2410_13229_b200" / "libqmb.so"))


def test_header_declares_entry_points():
    names = _declared()
    assert "qmb_block_prefill" in names and "qmb_block_decode" in names and len(names) >= 15


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_prototypes_match_header():
    from paper_2410_13229_b200 import _lib

    assert sorted(_lib.PROTOTYPES) == _declared()


def test_abi_version_and_error_text(lib):
    from paper_2410_13229_b200 import _lib

    L = _lib.load()
    assert L.qmb_abi_version() == 1
    # argument validation runs on the host, before any CUDA call
    rc = L.qmb_quantize(None, 4, -1.0, 8, None, None, None)
    assert rc == -1 and b"scale must be positive" in L.qmb_last_error()
    rc = L.qmb_qlinear(None, 1, 40000, 1.0, None, 1, 1.0, None, 0.0, 0.0, 1.0, 8, None, None, 0, 0, None, None)
    assert rc == -1 and b"int32 accumulation" in L.qmb_last_error()


def test_block_create_validates_like_the_reference(lib):
    from paper_2410_13229_b200 import _lib

    L = _lib.load()
    d = _lib.BlockDesc()
    h = ctypes.c_void_p()
    assert L.qmb_block_create(ctypes.byref(d), ctypes.byref(h)) == -1  # zero dims
    d.d_model, d.d_inner, d.d_state, d.d_conv, d.dt_rank, d.bit_width, d.mode = 8, 16, 4, 3, 2, 8, 3
    for i in range(10):
        d.act[i] = 0.05
    assert L.qmb_block_create(ctypes.byref(d), ctypes.byref(h)) == -1  # weights missing
    assert b"missing weight" in L.qmb_last_error()
