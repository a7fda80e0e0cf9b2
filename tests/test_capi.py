"""The C-ABI library loads and exports every symbol include/toep_b200.h
declares; argument validation happens before any CUDA call, so the
DataError paths are exercised here without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1502_03162_b200 import _lib
from paper_1502_03162_b200.errors import DataError

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "toep_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(toep_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.load_library()
    for name in declared_functions():
        assert hasattr(L, name), name


def test_abi_version():
    assert _lib.load_library().toep_abi_version() == 1


def _create(rows, length, row_ptr, idx, vals):
    L = _lib.load_library()
    h = ctypes.c_void_p()
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ix = np.ascontiguousarray(idx if len(idx) else [0], np.int64)
    vv = np.ascontiguousarray(vals if len(vals) else [0], np.float32)
    rc = L.toep_taps_create(rows, length, rp.ctypes.data_as(_lib._i64p), ix.ctypes.data_as(_lib._i64p),
                            vv.ctypes.data_as(_lib._fp), ctypes.byref(h))
    return rc, L.toep_last_error().decode()


@pytest.mark.parametrize("args,msg", [
    ((1, 4, [0, 2], [1, 1], [1.0, 2.0]), "strictly increasing"),       # sparsify.py:81-82
    ((1, 4, [0, 2], [3, 1], [1.0, 2.0]), "strictly increasing"),
    ((1, 4, [0, 1], [4], [1.0]), "indices must lie in"),                # sparsify.py:83-84
    ((1, 4, [0, 1], [-1], [1.0]), "indices must lie in"),
    ((1, 4, [0, 1], [0], [float("nan")]), "finite"),
    ((1, 0, [0, 0], [], []), "length must be at least 1"),              # sparsify.py:87-88
    ((0, 4, [0], [], []), "at least one filter row"),
    ((2, 4, [0, 2, 1], [0, 1], [1.0, 1.0]), "non-decreasing"),
])
def test_taps_validation_without_gpu(args, msg):
    rc, err = _create(*args)
    assert rc == _lib.TOEP_ERR_INVALID
    assert msg in err


def test_check_maps_codes_to_exceptions():
    _lib.load_library()
    with pytest.raises(DataError):
        _lib.check(_lib.TOEP_ERR_INVALID)
    with pytest.raises(DataError):
        _lib.check(_lib.TOEP_ERR_UNSUPPORTED)
    with pytest.raises(_lib.NativeError):
        _lib.check(_lib.TOEP_ERR_CUDA)
    _lib.check(_lib.TOEP_OK)


def test_null_handles_rejected():
    L = _lib.load_library()
    assert L.toep_taps_destroy(None) == 0
    assert L.toep_renderer_destroy(None) == 0
    assert L.toep_renderer_render(None, None, 0, None, 0, None) == _lib.TOEP_ERR_INVALID
    assert L.toep_mixer_partial(None, None, 0, 0, 0, None, 0, None) == _lib.TOEP_ERR_INVALID
    assert L.toep_streamer_step(None, None, 0, None, 0, None) == _lib.TOEP_ERR_INVALID
    assert L.toep_renderer_out_len(None, 10) == -1
