"""CPU: the C-ABI library loads and exports every symbol include/*.h declares."""

import ctypes
import os
import re

from conftest import REPO

HEADER = os.path.join(REPO, "include", "nld_b200.h")
LIB = os.path.join(REPO, "paper_2407_06834_b200", "libnld_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return re.findall(r"NLD_API\s+(?:const\s+)?\w+\s*\*?\s*(nld_\w+)\s*\(", text)


def test_header_declares_entry_points():
    names = declared_symbols()
    for required in ("nld_op_create", "nld_op_apply", "nld_op_degree",
                     "nld_cg_solve", "nld_op_destroy", "nld_last_error",
                     "nld_op_stats", "nld_basis_apply"):
        assert required in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version_and_error_channel():
    lib = ctypes.CDLL(LIB)
    lib.nld_abi_version.restype = ctypes.c_int
    assert lib.nld_abi_version() == 1
    lib.nld_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.nld_last_error(), bytes)


def test_python_binding_matches_header():
    from paper_2407_06834_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_create_rejects_bad_windows_without_gpu():
    # validation happens before any device work and maps onto the
    # reference's exception classes
    from paper_2407_06834_b200 import _lib
    handle = ctypes.c_void_p()
    idx = (ctypes.c_int32 * 4)(0, 1, 2, 3)
    off = (ctypes.c_int32 * 2)(0, 4)
    params = _lib.Params(32, 4, 2.0, 0.21875, 1e-8, 0, 0, 5000)
    st = _lib.lib.nld_op_create(None, 10, 4, idx, off, 1, 0.1,
                                ctypes.byref(params), None, ctypes.byref(handle))
    assert st == _lib.ERR_WINDOW
    assert b"one to three" in _lib.lib.nld_last_error()
    off2 = (ctypes.c_int32 * 2)(0, 2)
    idx2 = (ctypes.c_int32 * 2)(0, 9)
    st = _lib.lib.nld_op_create(None, 10, 4, idx2, off2, 1, 0.1,
                                ctypes.byref(params), None, ctypes.byref(handle))
    assert st == _lib.ERR_DIMENSION
    st = _lib.lib.nld_op_create(None, 10, 4, idx2, off2, 1, -1.0,
                                ctypes.byref(params), None, ctypes.byref(handle))
    assert st == _lib.ERR_VALUE
