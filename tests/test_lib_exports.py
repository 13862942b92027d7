"""The C-ABI library loads without a GPU and exports every symbol that
include/hsweep.h declares (no compute calls here)."""

import ctypes
import re

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "hsweep.h").read_text()
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = _declared()
    for must in ("hs_stencil_apply", "hs_jacobi", "hs_restrict_residual", "hs_prolong_add",
                 "hs_sweep_create", "hs_sweep_apply", "hs_vcycle", "hs_block_dot",
                 "hs_block_update", "hs_lincomb"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1412_0464_b200 import build as b
    lib_path = b.build()
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.hs_version() == 1


def test_ctypes_signatures_cover_header():
    from paper_1412_0464_b200._lib import SIGNATURES
    assert set(_declared()) == set(SIGNATURES)
