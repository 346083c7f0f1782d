"""Loader for the sm_100a library (libupy_cuda.so, built in-tree by
`__graft_entry__.build()` / `python -m paper_2403_13839_b200.build`).

There is deliberately no fallback: if the library or a CUDA device is missing
the product path raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UPY_LIB") or os.path.join(HERE, "libupy_cuda.so")
_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    for sym in _abi.EXPORTS:
        if not hasattr(lib, sym):
            raise NativeLibraryMissing(f"{LIB_PATH} does not export {sym}")
    _abi.check_layout(lib)
    lib.upy_abi_version.restype = C.c_int
    lib.upy_last_error.restype = C.c_char_p
    lib.upy_launch_count.restype = C.c_uint64
    lib.upy_query_workspace.restype = C.c_int
    lib.upy_query_workspace.argtypes = [C.POINTER(_abi.UpyArena), C.POINTER(_abi.UpyOptions),
                                        C.POINTER(C.c_size_t)]
    lib.upy_decompile_batch.restype = C.c_int
    lib.upy_decompile_batch.argtypes = [C.POINTER(_abi.UpyArena), C.POINTER(_abi.UpyOptions),
                                        C.POINTER(_abi.UpyOut), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.upy_decode_batch.restype = C.c_int
    lib.upy_decode_batch.argtypes = [C.POINTER(_abi.UpyArena), C.c_void_p, C.c_void_p, C.c_void_p]
    lib.upy_stackscan_batch.restype = C.c_int
    lib.upy_stackscan_batch.argtypes = [C.POINTER(_abi.UpyArena), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
    lib.upy_pyc_load.restype = C.c_int
    lib.upy_pyc_load.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.c_int64, C.c_int, C.c_int,
                                 C.POINTER(C.POINTER(_abi.UpyPycBatch))]
    lib.upy_pyc_write_image.restype = C.c_int
    lib.upy_pyc_write_image.argtypes = [C.POINTER(_abi.UpyPycBatch), C.c_void_p, C.c_uint64]
    lib.upy_pyc_free.restype = None
    lib.upy_pyc_free.argtypes = [C.POINTER(_abi.UpyPycBatch)]
    _lib = lib
    return lib


def check(rc, what):
    if rc != 0:
        msg = _lib.upy_last_error().decode(errors="replace") if _lib is not None else ""
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")
