"""The C-ABI library loads and exports every symbol include/bgp.h declares
(no GPU needed: nothing here launches a kernel)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bgp.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(bgp_\w+)\s*\(", text, re.M)))


def test_header_declares_the_path():
    names = _declared()
    for must in ("bgp_construct", "bgp_potrf", "bgp_trsv", "bgp_trsm_rect", "bgp_logdet",
                 "bgp_sumsq", "bgp_xprod_mat_vec", "bgp_xprod_self", "bgp_xprod_self_diag",
                 "bgp_pack", "bgp_unpack", "bgp_init", "bgp_finalize"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1305_4886_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    # every declared symbol has a ctypes prototype in the binding
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    from paper_1305_4886_b200 import _lib
    assert b"sm_100a" in _lib.load().bgp_version()
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_generator_struct_layout_matches_header():
    from paper_1305_4886_b200._lib import Generator
    # 4 ints + 8 + 2 doubles
    assert ctypes.sizeof(Generator) == 4 * 4 + 11 * 8  # include/bgp.h bgp_generator


def test_missing_library_fails_loudly(tmp_path):
    from paper_1305_4886_b200 import _lib
    from paper_1305_4886_b200.errors import BackendUnavailable
    with pytest.raises(BackendUnavailable):
        _lib.load(str(tmp_path / "libbgp.so"))
