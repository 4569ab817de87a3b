"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU needed)."""

import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        names += re.findall(r"KCG_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt)
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2204_08057_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_north_star_entry_points():
    names = _declared()
    for n in ("kron_cg_create", "kron_cg_solve", "sylvester_solve", "kron_cg_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n


def test_binding_names_match_header(lib):
    from paper_2204_08057_b200 import kroncg
    assert sorted(kroncg.EXPORTS) == sorted(_declared())


def test_host_logic_without_gpu(lib):
    # workspace sizing and descriptor validation run on the host only
    from paper_2204_08057_b200 import kroncg as K
    d = K.kcg_desc(10, 9, 4, 12, 0, 0, 0, 0, 0)
    ws = K.kron_cg_workspace_size(ctypes.byref(d))
    vec = 12 * 4 * 4 ** 10 * 8
    assert 4 * vec <= ws <= 4 * vec + 64 * 2 ** 20
    d2 = K.kcg_desc(10, 9, 4, 12, 0, 0, 0, 1, 0)
    ws2 = K.kron_cg_workspace_size(ctypes.byref(d2))
    assert ws2 - ws >= 12 * (9 + 4) * 4 ** 10 * 8
    for bad in [K.kcg_desc(13, 9, 4, 1, 0, 0, 0, 0, 0), K.kcg_desc(5, 9, 9, 1, 0, 0, 0, 0, 0),
                K.kcg_desc(5, 2, 3, 1, 0, 0, 0, 0, 0), K.kcg_desc(5, 9, 3, 0, 0, 0, 0, 0, 0)]:
        assert K.kron_cg_workspace_size(ctypes.byref(bad)) == 0
    # the textbook-CG variant (reading R9) reserves its CTA partial sums; unknown variants are rejected
    dh = K.kcg_desc(10, 9, 4, 12, 0, 0, 0, 0, 0, 0, 0, K.KCG_CG_HS)
    wsh = K.kron_cg_workspace_size(ctypes.byref(dh))
    assert wsh - ws >= 2 * 1024 * 12 * 4 * 3 * 8
    assert K.kron_cg_workspace_size(ctypes.byref(K.kcg_desc(10, 9, 4, 12, 0, 0, 0, 0, 0, 0, 0, 2))) == 0
    assert K.kcg_status_string(6) == b"KCG_E_BREAKDOWN"
    # create rejects a bad descriptor before touching the GPU
    ctx = ctypes.c_void_p()
    st = K.kron_cg_create(ctypes.byref(K.kcg_desc(13, 9, 4, 1, 0, 0, 0, 0, 0)), None, None, None,
                          None, None, None, 0, None, ctypes.byref(ctx))
    assert st == K.KCG_E_SHAPE
    assert b"level" in K.kcg_last_error(ctx)
    K.kron_cg_destroy(ctx)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2204_08057_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True) + \
            glob.glob(os.path.join(pkg, "csrc", "*")):
        txt = open(f).read()
        assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
        assert "oracle/" not in txt, f
