"""C-ABI boundary checks that need no GPU: the library loads and exports every
function include/gmpgr.h declares; errors map to the reference's exception classes."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "gmpgr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gr_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_surface():
    from paper_2502_11490_b200 import _lib

    assert header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_header_symbol():
    from paper_2502_11490_b200 import _lib

    lib = _lib.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.gr_abi_version() == 1
    assert lib.gr_device_count() >= 0


def test_error_mapping():
    from paper_2502_11490_b200 import _lib
    from paper_2502_11490_b200.errors import InvalidArgumentError

    h = ctypes.c_void_p()
    # null dims -> GR_EINVAL before any device work
    rc = _lib.lib().gr_model_create(0, 1, None, None, None, None, 1, ctypes.byref(h))
    assert rc == _lib.GR_EINVAL
    with pytest.raises(InvalidArgumentError):
        _lib.check(rc)
    assert b"null" in _lib.lib().gr_last_error()


def test_no_cpu_fallback_without_device():
    from paper_2502_11490_b200 import _lib
    import paper_2502_11490_b200 as P

    if _lib.lib().gr_device_count() > 0:
        pytest.skip("a GPU is visible")
    m = P.create_model(d_x=4, d_h=4, z_dim=2, hidden=(8,), seed=0)
    import numpy as np

    with pytest.raises(P.DeviceError):
        P.relevance_batch(m.metric, np.ones((1, 4), np.float32), np.ones((1, 4), np.float32))
