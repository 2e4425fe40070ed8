"""C-ABI checks that need no GPU: the library builds/loads, exports every symbol
include/ht.h declares, and validates arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1710_08538_b200 as ht

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "ht.h")).read()
    return sorted(set(re.findall(r"HT_API\s+[\w\s\*]+?\b(ht_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    assert declared_symbols() == sorted(ht.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(ht.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_version_and_strerror():
    assert ht.ht_version() >= 100
    for code in list(ht.ERRORS) + [0]:
        assert isinstance(ht.ht_strerror(code), str) and ht.ht_strerror(code)


def test_argument_errors_before_any_write():
    lib = ht.load_library()
    A = np.asfortranarray(np.arange(16.0).reshape(4, 4))
    keep = A.copy()
    assert lib.ht_reduce(-1, A.ctypes.data, A.ctypes.data, None, None, 0, 0, 0) == -1
    assert lib.ht_reduce(4, None, A.ctypes.data, None, None, 0, 0, 0) == -2
    assert lib.ht_reduce(4, A.ctypes.data, None, None, None, 0, 0, 0) == -3
    assert lib.ht_reduce(4, A.ctypes.data, A.ctypes.data, None, None, 1, 0, 0) == -4
    assert lib.ht_reduce(4, A.ctypes.data, A.ctypes.data, None, None, 0, 1, 0) == -5
    assert lib.ht_reduce(4, A.ctypes.data, A.ctypes.data, A.ctypes.data, None, 2, 0, 0) == -6
    assert lib.ht_reduce(4, A.ctypes.data, A.ctypes.data, None, A.ctypes.data, 0, 3, 0) == -7
    assert np.array_equal(A, keep)
    assert lib.ht_reduce(0, None, None, None, None, 1, 1, 0) == 0
    # out-of-place host entry point: inputs, then outputs
    p = A.ctypes.data
    assert lib.ht_reduce_host(-1, p, p, p, p, None, None, 0, 0, 0) == -1
    assert lib.ht_reduce_host(4, None, p, p, p, None, None, 0, 0, 0) == -2
    assert lib.ht_reduce_host(4, p, None, p, p, None, None, 0, 0, 0) == -3
    assert lib.ht_reduce_host(4, p, p, None, p, None, None, 0, 0, 0) == -2
    assert lib.ht_reduce_host(4, p, p, p, None, None, None, 0, 0, 0) == -3
    assert lib.ht_reduce_host(4, p, p, p, p, None, None, 1, 0, 0) == -4
    assert np.array_equal(A, keep)
    assert lib.ht_reduce_host(0, None, None, None, None, None, None, 1, 1, 0) == 0


def test_ex_option_errors_before_any_write():
    lib = ht.load_library()
    A = np.asfortranarray(np.arange(16.0).reshape(4, 4))
    keep = A.copy()
    p = A.ctypes.data
    rep = ht.HTReport()
    opt = ht.make_options(nb=1 << 21)
    assert lib.ht_reduce_ex(4, p, 4, p, 4, None, 4, None, 4, 0, 0, ctypes.byref(opt), ctypes.byref(rep)) == -8
    opt = ht.make_options(row_range=(3, 1))
    assert lib.ht_reduce_ex(4, p, 4, p, 4, None, 4, None, 4, 0, 0, ctypes.byref(opt), ctypes.byref(rep)) == -9
    assert np.array_equal(A, keep)


def test_report_layout_matches_header():
    """ht_report / ht_options field order in the binding follows include/ht.h."""
    txt = open(os.path.join(ROOT, "include", "ht.h")).read()
    body = txt[txt.index("typedef struct {", txt.index("Statistics of one reduction")):txt.index("} ht_report;")]
    names = re.findall(r"\b(?:double|int64_t)\s+(\w+)\s*;", body)
    assert names == [f for f, _ in ht.HTReport._fields_]


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(ht.HTError) as e:
        ht.ht_reduce(np.eye(5), np.eye(5))
    assert e.value.code == 2  # HT_ECUDA
