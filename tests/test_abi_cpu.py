"""Host-side checks of the C ABI that need no GPU: the library loads, exports every
symbol include/dcnn.h declares, and rejects bad calls with status codes."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dcnn.h")).read()
    return sorted(set(re.findall(r"^DCNN_API [^(]*?\b(dcnn_[a-z_]+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2203_03996_b200 import load_library, LIB_PATH
    lib = load_library()
    names = _declared()
    assert "dcnn_create_net" in names and "dcnn_process_frame" in names
    for n in names:
        assert hasattr(lib, n), n
    # only the C ABI is exported (hidden visibility for everything else)
    out = os.popen(f"nm -D --defined-only {LIB_PATH}").read()
    exported = set(re.findall(r" T (dcnn_\w+)", out))
    assert exported == set(names), exported ^ set(names)


def test_null_and_bad_arguments_fail_with_status():
    from paper_2203_03996_b200 import load_library
    from paper_2203_03996_b200._lib import dcnn_net_desc
    lib = load_library()
    h = C.c_void_p()
    assert lib.dcnn_create_net(None, C.byref(h)) == 1                 # DCNN_ERR_ARG
    d = dcnn_net_desc()
    d.in_h = 0
    assert lib.dcnn_create_net(C.byref(d), C.byref(h)) == 2           # DCNN_ERR_SHAPE
    assert b"positive" in lib.dcnn_last_error()
    assert lib.dcnn_set_threshold(None, 0, 0.1) == 1
    assert lib.dcnn_reset(None, 0) == 1
    assert lib.dcnn_process_frame(None, None, None, None) == 1


def test_binding_fails_loudly_without_library(tmp_path):
    import paper_2203_03996_b200._lib as L
    saved = L._lib
    try:
        L._lib = None
        with pytest.raises(ImportError):
            L.load_library(str(tmp_path / "missing.so"))
    finally:
        L._lib = saved
