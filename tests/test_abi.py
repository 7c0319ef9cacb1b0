"""The C ABI library loads and exports every symbol include/tsvd.h declares;
calls that need a device fail with a status (no crash, no CPU fallback).
CPU only (-m "not gpu")."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "tsvd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tsvd_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def built():
    from paper_2403_06218_b200.build import build
    return build()


def test_header_symbols_exported(built):
    import paper_2403_06218_b200 as t
    names = _header_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tsvd_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert sorted(t.EXPORTS) == names
    L = t.lib()
    for n in names:
        assert getattr(L, n) is not None


def test_no_device_fails_loudly(built):
    import numpy as np
    import paper_2403_06218_b200 as t
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    L = t.lib()
    h = C.c_void_p()
    A = np.ones((4, 3))
    st = L.tsvd_create_dense(C.byref(h), 4, 3, A.ctypes.data, 3, t.TSVD_ROW_MAJOR, t.TSVD_HOST)
    assert st == t.TSVD_ECUDA
    with pytest.raises(t.TsvdError):
        t.TruncatedSVD(A)
    assert L.tsvd_strerror(t.TSVD_ESHAPE) == b"invalid shape"


def test_shape_validation_before_device(built):
    import numpy as np
    import paper_2403_06218_b200 as t
    L = t.lib()
    h = C.c_void_p()
    A = np.ones((3, 4))      # m < n -> ESHAPE, checked before any CUDA call
    assert L.tsvd_create_dense(C.byref(h), 3, 4, A.ctypes.data, 4, 0, 0) == t.TSVD_ESHAPE
    assert L.tsvd_create_dense(C.byref(h), 3, 4, None, 4, 0, 0) == t.TSVD_EINVAL
