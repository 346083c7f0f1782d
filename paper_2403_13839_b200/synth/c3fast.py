"""C3 corpus straight into an arena: `c3_arena(n, minor)` is
byte-identical to `arena.pack([corpus.c3(i, minor) for i in range(first, first + n)])`
but built in about a second per million objects (co_code from the native
generator synth/c3gen.cpp on every host core, the pools laid out with numpy
exactly as `_Packer` orders them).  Benchmark input generation only.

Layout facts `pack` produces for these objects (arena.py:84-283): strings are
interned in first-use order -- the 6 names, the 6 varnames, then per object its
name (which is also its qualname) and, once, the filename "<synth>"; every
object gets its own const rows (None first, then the ints 1..3 in first-use
order, one 32-bit limb each) and its own refs rows (consts, names, varnames);
exception and line tables are empty.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .. import arena as A
from .._optables import BY_NAME, TABLES

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "build", "libc3gen.so")
SRC = os.path.join(HERE, "c3gen.cpp")
OPS = ("LOAD_FAST", "LOAD_CONST", "BINARY_MULTIPLY", "BINARY_ADD", "BINARY_SUBTRACT", "BINARY_OP", "STORE_FAST",
       "LOAD_GLOBAL", "LOAD_ATTR", "PRECALL", "CALL", "CALL_FUNCTION", "LOAD_METHOD", "CALL_METHOD",
       "BINARY_SUBSCR", "STORE_ATTR", "RETURN_VALUE", "RESUME")
NAMES = ("g", "h", "attr", "m", "n", "k")
LOCALS = ("a", "b", "c", "d", "e", "f")
N_STMTS = 33
_lib = None


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-o", LIB + ".tmp", SRC])
    os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.c3gen.restype = C.c_int
        _lib.c3gen.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.c3names.restype = C.c_int
        _lib.c3names.argtypes = [C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
    return _lib


def _optab(minor):
    t = np.zeros((len(OPS), 3), dtype=np.int32)
    names = BY_NAME[minor]
    for i, op in enumerate(OPS):
        if op in names:
            code = names[op]
            _name, has_arg, _kind, cache = TABLES[minor][code]
            t[i] = (code, 1 if has_arg else 0, cache)
    return t


def c3_arena(n, minor=10, first=0, threads=0):
    lib = _load()
    lens = np.zeros(n, dtype=np.uint32)
    kv = np.zeros((n, 4), dtype=np.uint8)
    nk = np.zeros(n, dtype=np.uint8)
    tab = _optab(minor)
    lib.c3gen(minor, first, n, N_STMTS, tab.ctypes.data, None, None, lens.ctypes.data, kv.ctypes.data,
              nk.ctypes.data, threads)
    nk64 = nk.astype(np.int64)

    # ---- byte pool: 16-aligned code segments, then the strings (tables are empty)
    seg = (lens.astype(np.int64) + 15) & ~15
    code_off = np.zeros(n, dtype=np.uint64)
    if n:
        code_off[1:] = np.cumsum(seg)[:-1]
    code_end = int(seg.sum())
    fixed = b"".join(s.encode() for s in NAMES + LOCALS)
    fixed_len = [len(s) for s in NAMES + LOCALS]
    seeds = first + np.arange(n, dtype=np.int64)
    name_len = np.full(n, 4, dtype=np.int64)  # "c3_" + decimal digits
    for k in range(1, 20):
        name_len += seeds >= 10 ** k
    # interned order: 12 fixed, name_0, "<synth>", name_1, ..., name_{n-1}
    str_len = np.concatenate([fixed_len, name_len[:1], [len(b"<synth>")], name_len[1:]]).astype(np.int64)
    str_off = code_end + np.concatenate([[0], np.cumsum(str_len)[:-1]]).astype(np.int64)
    n_bytes = code_end + int(str_len.sum())
    order_n = len(str_len)

    n_consts = int(nk64.sum())
    n_ints = n_consts - n  # every pool holds None + its ints
    n_refs = n_consts + 12 * n
    counts = {"objs": n, "consts": n_consts, "strs": order_n, "refs": n_refs, "limbs": n_ints,
              "bytes": n_bytes, "roots": n}
    sizes = {"objs": A.OBJ_DTYPE.itemsize, "consts": A.CONST_DTYPE.itemsize, "strs": A.STR_DTYPE.itemsize,
             "refs": 4, "limbs": 4, "bytes": 1, "roots": 4}
    offsets, total = {}, 0
    for s in A.SECTIONS:
        offsets[s] = total
        total = A._align(total + counts[s] * sizes[s], A.ALIGN)
    blob = np.zeros(max(total, A.ALIGN), dtype=np.uint8)
    ar = A.Arena(blob, offsets, counts, int(lens.max()) if n else 0, (code_end + 1) // 2)

    # ---- consts + limbs: object i's pool is rows [cbase_i, cbase_i + nk_i)
    cbase = np.concatenate([[0], np.cumsum(nk64)[:-1]])
    flat_vals = kv[np.arange(4)[None, :] < nk64[:, None]]          # pool values, pool order
    consts = ar.section("consts")
    is_int = flat_vals != 0
    consts["kind"] = np.where(is_int, A.KIND_ID["int"], A.KIND_ID["none"])
    consts["ival"] = is_int.astype(np.int32)
    consts["n"] = is_int.astype(np.uint32)
    consts["off"][is_int] = np.arange(n_ints, dtype=np.uint64)
    ar.section("limbs")[:] = flat_vals[is_int].astype(np.uint32)

    # ---- refs: per object [const ids][names 0..5][varnames 6..11]
    rbase = cbase + 12 * np.arange(n, dtype=np.int64)
    refs = ar.section("refs")
    per = nk64 + 12
    pos = np.arange(n_refs) - np.repeat(rbase, per)
    is_c = pos < np.repeat(nk64, per)
    refs[is_c] = (np.repeat(cbase, per) + pos)[is_c]
    refs[~is_c] = (pos - np.repeat(nk64, per))[~is_c]

    objs = ar.section("objs")
    objs["argcount"] = 2
    objs["nlocals"] = 6
    objs["stacksize"] = 16
    objs["flags"] = 0x43
    objs["firstlineno"] = 1
    objs["code_off"] = code_off
    objs["exc_off"] = code_end
    objs["lnt_off"] = code_end
    objs["code_len"] = lens
    objs["consts_off"] = rbase
    objs["n_consts"] = nk
    objs["names_off"] = rbase + nk64
    objs["n_names"] = 6
    objs["varnames_off"] = rbase + nk64 + 6
    objs["n_varnames"] = 6
    objs["freevars_off"] = rbase + nk64 + 12
    objs["cellvars_off"] = rbase + nk64 + 12
    sid = np.where(np.arange(n) == 0, 12, 13 + np.arange(n))
    objs["name"] = sid
    objs["qualname"] = sid
    objs["filename"] = 13
    objs["minor"] = minor

    strs = ar.section("strs")
    strs["off"] = str_off
    strs["len"] = str_len
    by = ar.section("bytes")
    lib.c3gen(minor, first, n, N_STMTS, tab.ctypes.data, by.ctypes.data, code_off.ctypes.data, lens.ctypes.data,
              kv.ctypes.data, nk.ctypes.data, threads)
    by[code_end:code_end + len(fixed)] = np.frombuffer(fixed, dtype=np.uint8)
    synth_at = int(str_off[13])
    by[synth_at:synth_at + 7] = np.frombuffer(b"<synth>", dtype=np.uint8)
    name_off = np.concatenate([str_off[12:13], str_off[14:]]).astype(np.uint64)
    lib.c3names(first, n, by.ctypes.data, name_off.ctypes.data, threads)
    ar.section("roots")[:] = np.arange(n, dtype=np.int32)
    return ar
