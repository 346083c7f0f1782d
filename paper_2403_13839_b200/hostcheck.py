"""TEST-ONLY: run the decompiler's C++ sources compiled for the host
(build/libupy_host.so, built from tools/hostcheck.cpp) on a packed arena.

This exists so the device code's logic can be checked against the reference
without a GPU.  The product path (`api.decompile_many`) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import _abi
from .arena import DECODED_DTYPE
from .errors import make_exception

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "build", "libupy_host.so")
_lib = None


def build(force=False, opt="-O2"):
    srcs = [os.path.join(ROOT, "tools", "hostcheck.cpp")]
    csrc = os.path.join(ROOT, "paper_2403_13839_b200", "csrc")
    deps = srcs + [os.path.join(csrc, f) for f in os.listdir(csrc)]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["g++", opt, "-g", "-std=c++17", "-shared", "-fPIC", "-o", LIB + ".tmp", srcs[0]])
    os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        _lib.upyh_decompile.restype = C.c_int
    return _lib


def run(arena, style=None, arena_bytes=256 << 20, text_cap=None, function_tree=False, output=0):
    """Decompile every root of `arena` on the host; returns list of (status, text, aux)."""
    L = lib()
    blob = arena.blob
    base = blob.ctypes.data
    A = _abi.arena_struct(arena, base)
    n = arena.n_roots
    cap = text_cap or max(1 << 20, arena.code_bytes * 16)
    text = np.zeros(cap, dtype=np.uint8)
    off = np.zeros(n, dtype=np.uint64)
    ln = np.zeros(n, dtype=np.uint32)
    st = np.zeros(n, dtype=np.int32)
    aux = np.zeros(2 * n, dtype=np.int64)
    dec = np.zeros(arena.n_objs, dtype=DECODED_DTYPE)
    indent = ("    " if style is None else style.indent).encode("utf-8", "surrogatepass")
    tool = ("unpyre" if style is None else style.tool).encode("utf-8", "surrogatepass")
    header = 1 if (style is not None and style.header) else 0
    L.upyh_decompile(C.byref(A), header, indent, len(indent), tool, len(tool), C.c_uint64(arena_bytes),
                     text.ctypes.data_as(C.c_void_p), C.c_uint64(cap), off.ctypes.data_as(C.c_void_p),
                     ln.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                     aux.ctypes.data_as(C.c_void_p), dec.ctypes.data_as(C.c_void_p), 1 if function_tree else 0, output)
    out = []
    tb = text.tobytes()
    for i in range(n):
        s = tb[int(off[i]):int(off[i]) + int(ln[i])].decode("utf-8", "surrogatepass")
        out.append((int(st[i]), s, (int(aux[2 * i]), int(aux[2 * i + 1]))))
    return out


def decode(arena):
    """decode_scalar on the host for every object: (records, decoded) arrays laid
    out like the device workspace (records at code_off/2)."""
    from .arena import INS_DTYPE

    L = lib()
    A = _abi.arena_struct(arena, arena.blob.ctypes.data)
    ins = np.zeros(arena.total_code_units + 1, dtype=INS_DTYPE)
    dec = np.zeros(arena.n_objs, dtype=DECODED_DTYPE)
    L.upyh_decode(C.byref(A), ins.ctypes.data_as(C.c_void_p), dec.ctypes.data_as(C.c_void_p))
    return ins, dec


def decompile_many(codes, style=None, function_tree=False):
    from .arena import pack
    res = run(pack(codes), style, function_tree=function_tree)
    return [s if st == 0 else make_exception(st, s, aux) for st, s, aux in res]


def stackscan(arena):
    """Stack-depth scan on the host (csrc/stackscan.h, after decode_scalar):
    (records laid out like the device's, per-object summaries)."""
    from .arena import STACKINFO_DTYPE, STACKREC_DTYPE

    L = lib()
    A = _abi.arena_struct(arena, arena.blob.ctypes.data)
    out = np.zeros(arena.total_code_units + 1, dtype=STACKREC_DTYPE)
    info = np.zeros(arena.n_objs, dtype=STACKINFO_DTYPE)
    L.upyh_stackscan(C.byref(A), out.ctypes.data_as(C.c_void_p), info.ctypes.data_as(C.c_void_p))
    return out, info
