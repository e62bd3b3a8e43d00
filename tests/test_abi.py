"""The C-ABI library loads and exports every symbol include/hd.h declares (no compute)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "hd.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void\*|const char\*)\s+(hd_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    from paper_2211_16718_b200 import _lib

    assert sorted(_lib.EXPORTS) == _declared()


def test_library_exports_every_symbol():
    from paper_2211_16718_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhd.so not built (run __graft_entry__.build())")
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(L, s)]
    assert not missing
    lib = _lib.load()
    assert lib.hd_abi_version() == 3
    assert lib.hd_status_string(-4) == b"unsupported configuration"


def test_workspace_size_is_host_only():
    from paper_2211_16718_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhd.so not built")
    lib = _lib.load()
    g = _lib.HdGeom()
    for d in range(3):
        g.n[d] = 16
        g.length[d] = 1.0
        g.periodic[d] = 1
    g.ghost = 3
    nbytes = lib.hd_workspace_bytes(ctypes.byref(g))
    assert nbytes >= 38 * 22 ** 3 * 8  # 33 work fields + the peer-mode state (5)
    g.ghost = 2
    assert lib.hd_workspace_bytes(ctypes.byref(g)) == -1


def test_product_fails_loudly_without_gpu():
    import torch

    import paper_2211_16718_b200 as hd

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hd.NativeUnavailable):
        hd.get_plan(hd.GridSpec((8, 8, 8)))
