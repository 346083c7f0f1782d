"""Pack CodeObject trees into the flat struct-of-arrays arena the device reads
(include/upy.h: upy_obj / upy_const / upy_str / refs / limbs / bytes / roots),
and unpack an arena back into CodeObject trees.

The arena is ONE contiguous byte image (sections 256-byte aligned) so a batch
moves host->device in a single copy.  Code segments come first in the byte
pool, each 16-byte aligned, so the decode kernel can issue aligned 128-bit
loads and the decoded record of unit u of object o lives at code_off/2 + u.

Input objects may be this package's `model.CodeObject` or any object with the
same attributes (the reference's `unpyre.CodeObject`, code_model.py:101-123).
"""
from __future__ import annotations

import numpy as np

from .model import CodeObject, Const, VersionTag

OBJ_DTYPE = np.dtype([
    ("argcount", "<i8"), ("posonlyargcount", "<i8"), ("kwonlyargcount", "<i8"),
    ("nlocals", "<i8"), ("stacksize", "<i8"), ("flags", "<i8"), ("firstlineno", "<i8"),
    ("code_off", "<u8"), ("exc_off", "<u8"), ("lnt_off", "<u8"),
    ("code_len", "<u4"), ("exc_len", "<u4"), ("lnt_len", "<u4"),
    ("consts_off", "<u4"), ("n_consts", "<u4"),
    ("names_off", "<u4"), ("n_names", "<u4"),
    ("varnames_off", "<u4"), ("n_varnames", "<u4"),
    ("freevars_off", "<u4"), ("n_freevars", "<u4"),
    ("cellvars_off", "<u4"), ("n_cellvars", "<u4"),
    ("name", "<u4"), ("filename", "<u4"), ("qualname", "<u4"),
    ("minor", "<u4"), ("pad", "<u4"),
], align=True)
CONST_DTYPE = np.dtype([("kind", "<u4"), ("ival", "<i4"), ("n", "<u4"), ("pad", "<u4"),
                        ("off", "<u8"), ("re", "<f8"), ("im", "<f8")], align=True)
STR_DTYPE = np.dtype([("off", "<u8"), ("len", "<u4"), ("pad", "<u4")], align=True)
INS_DTYPE = np.dtype([("offset", "<u4"), ("arg", "<u4"), ("opcode", "u1"), ("n_prefixes", "u1"),
                      ("cache_units", "u1"), ("flags", "u1")], align=True)
DECODED_DTYPE = np.dtype([("status", "<i4"), ("n_instrs", "<i4"), ("aux0", "<i8"), ("aux1", "<i8")],
                         align=True)
STACKREC_DTYPE = np.dtype([("depth", "<i2"), ("flags", "u1"), ("pad", "u1")])
STACKINFO_DTYPE = np.dtype([("status", "<i4"), ("n_segments", "<i4"), ("max_depth", "<i4"), ("min_depth", "<i4"),
                            ("n_pushes", "<i4"), ("n_unknown", "<i4")])
assert STACKREC_DTYPE.itemsize == 4 and STACKINFO_DTYPE.itemsize == 24
assert OBJ_DTYPE.itemsize == 152 and CONST_DTYPE.itemsize == 40 and STR_DTYPE.itemsize == 16
assert INS_DTYPE.itemsize == 12 and DECODED_DTYPE.itemsize == 24

KIND_ID = {"none": 0, "bool": 1, "int": 2, "float": 3, "complex": 4, "str": 5, "bytes": 6,
           "tuple": 7, "frozenset": 8, "code": 9, "ellipsis": 10}
KIND_NAME = {v: k for k, v in KIND_ID.items()}
SECTIONS = ("objs", "consts", "strs", "refs", "limbs", "bytes", "roots")
ALIGN = 256


def _enc(s):
    return s.encode("utf-8", "surrogatepass")


class Arena:
    """A packed batch: `blob` (uint8) plus section offsets/counts."""

    def __init__(self, blob, offsets, counts, max_code_len, total_code_units):
        self.blob = blob
        self.offsets = offsets          # section -> byte offset in blob
        self.counts = counts            # section -> element count
        self.max_code_len = int(max_code_len)
        self.total_code_units = int(total_code_units)
        self.pinned = None               # optional page-locked torch view of blob

    def section(self, name):
        dt = {"objs": OBJ_DTYPE, "consts": CONST_DTYPE, "strs": STR_DTYPE, "refs": np.dtype("<u4"),
              "limbs": np.dtype("<u4"), "bytes": np.dtype("u1"), "roots": np.dtype("<i4")}[name]
        off, n = self.offsets[name], self.counts[name]
        return self.blob[off:off + n * dt.itemsize].view(dt)

    @property
    def n_roots(self):
        return self.counts["roots"]

    @property
    def n_objs(self):
        return self.counts["objs"]

    @property
    def code_bytes(self):
        """Sum of |co_code| over every object (roots and nested)."""
        return int(self.section("objs")["code_len"].sum())


class _Packer:
    def __init__(self):
        self.objs = []          # dict rows
        self.obj_index = {}     # id(code) -> index
        self.consts = []        # tuples (kind, ival, n, off, re, im)
        self.strs = []          # (bytes_off placeholder index)
        self.str_index = {}
        self.str_bytes = []     # list of bytes for strings
        self.refs = []
        self.limbs = []
        self.nlimbs = 0
        self.codes = []         # raw code bytes per object
        self.excs = []
        self.lnts = []
        self.blobs = []         # bytes/str const payloads: list of bytes
        self.blob_len = 0

    def sid(self, s):
        if not isinstance(s, str):
            s = str(s)
        i = self.str_index.get(s)
        if i is None:
            i = len(self.str_bytes)
            self.str_index[s] = i
            self.str_bytes.append(_enc(s))
        return i

    def payload(self, b):
        off = self.blob_len
        self.blobs.append(b)
        self.blob_len += len(b)
        return off

    def const(self, c):
        k = c.kind
        kid = KIND_ID[k]
        v = c.value
        row = [kid, 0, 0, 0, 0.0, 0.0]
        if k == "bool":
            row[1] = 1 if v else 0
        elif k == "int":
            v = int(v)
            row[1] = (v > 0) - (v < 0)
            mag = abs(v)
            nb = max(1, (mag.bit_length() + 31) // 32)
            arr = np.frombuffer(mag.to_bytes(nb * 4, "little"), dtype="<u4")
            row[2] = nb
            row[3] = self.nlimbs
            self.limbs.append(arr)
            self.nlimbs += nb
        elif k == "float":
            row[4] = float(v)
        elif k == "complex":
            row[4] = float(v.real)
            row[5] = float(v.imag)
        elif k in ("str", "bytes"):
            b = _enc(v) if k == "str" else bytes(v)
            row[2] = len(b)
            row[3] = ("P", self.payload(b))
        elif k in ("tuple", "frozenset"):
            ids = [self.const(x) for x in v]
            row[2] = len(ids)
            row[3] = len(self.refs)
            self.refs.extend(ids)
        elif k == "code":
            row[3] = self.code(v)
        idx = len(self.consts)
        self.consts.append(row)
        return idx

    def strlist(self, seq):
        ids = [self.sid(s) for s in seq]
        off = len(self.refs)
        self.refs.extend(ids)
        return off, len(ids)

    def code(self, co):
        key = id(co)
        if key in self.obj_index:
            return self.obj_index[key]
        idx = len(self.objs)
        self.obj_index[key] = idx
        row = {}
        self.objs.append(row)
        self.codes.append(bytes(co.code))
        self.excs.append(bytes(co.exceptiontable or b""))
        self.lnts.append(bytes(co.linetable or b""))
        for f in ("argcount", "posonlyargcount", "kwonlyargcount", "nlocals", "stacksize", "firstlineno"):
            row[f] = _clamp(int(getattr(co, f)))
        row["flags"] = _flags62(int(co.flags))
        row["minor"] = int(co.version.minor)
        ids = [self.const(c) for c in co.consts]
        row["consts_off"], row["n_consts"] = len(self.refs), len(ids)
        self.refs.extend(ids)
        for f in ("names", "varnames", "freevars", "cellvars"):
            row[f + "_off"], row["n_" + f] = self.strlist(getattr(co, f))
        row["name"] = self.sid(co.name)
        row["filename"] = self.sid(co.filename)
        row["qualname"] = self.sid(co.qualname or co.name)
        return idx


# Python ints of any size fit the device's int64 fields this way (.pyc inputs are
# 32-bit anyway): counts and sizes saturate at +-2**62, so sums of two and
# stacksize + 6 cannot overflow and every comparison the reference makes
# (validation, depth guard, parameter slicing) keeps its verdict; flags keep their
# low 62 bits (the CO_* tests) and their sign.  Only validation messages that
# print a count of magnitude >= 2**62 differ.
_LIM = 1 << 62


def _clamp(v):
    return _LIM if v > _LIM else -_LIM if v < -_LIM else v


def _flags62(v):
    low = v & (_LIM - 1)
    return low if v >= 0 else low - _LIM


def _align(x, a):
    return (x + a - 1) // a * a


def pack(roots) -> Arena:
    """Pack root code objects (each with its nested code constants) with the
    native packer (csrc/packer.cpp, byte-identical to `pack_py`)."""
    from . import _packer

    blob, offsets, counts, max_code_len, total_units = _packer.pack(list(roots))
    return Arena(np.frombuffer(blob, dtype=np.uint8), offsets, counts, max_code_len, total_units)


def pack_py(roots) -> Arena:
    """Pack root code objects (each with its nested code constants): the Python
    restatement the native packer is checked against (tests/test_packer.py)."""
    p = _Packer()
    root_ids = [p.code(r) for r in roots]
    n_obj = len(p.objs)
    # byte pool: code segments (16-aligned), exception tables, line tables, strings, payloads
    pos = 0
    code_off = []
    for b in p.codes:
        code_off.append(pos)
        pos = _align(pos + len(b), 16)
    code_end = pos
    exc_off = []
    for b in p.excs:
        exc_off.append(pos)
        pos += len(b)
    lnt_off = []
    for b in p.lnts:
        lnt_off.append(pos)
        pos += len(b)
    str_off = []
    for b in p.str_bytes:
        str_off.append(pos)
        pos += len(b)
    payload_base = pos
    pos += p.blob_len
    n_bytes = pos

    counts = {"objs": n_obj, "consts": len(p.consts), "strs": len(p.str_bytes), "refs": len(p.refs),
              "limbs": p.nlimbs, "bytes": n_bytes, "roots": len(root_ids)}
    sizes = {"objs": OBJ_DTYPE.itemsize, "consts": CONST_DTYPE.itemsize, "strs": STR_DTYPE.itemsize,
             "refs": 4, "limbs": 4, "bytes": 1, "roots": 4}
    offsets = {}
    total = 0
    for s in SECTIONS:
        offsets[s] = total
        total = _align(total + counts[s] * sizes[s], ALIGN)
    blob = np.zeros(max(total, ALIGN), dtype=np.uint8)
    arena = Arena(blob, offsets, counts, max((len(b) for b in p.codes), default=0), (code_end + 1) // 2)

    objs = arena.section("objs")
    for i, row in enumerate(p.objs):
        for k, v in row.items():
            objs[k][i] = v
        objs["code_off"][i] = code_off[i]
        objs["code_len"][i] = len(p.codes[i])
        objs["exc_off"][i] = exc_off[i]
        objs["exc_len"][i] = len(p.excs[i])
        objs["lnt_off"][i] = lnt_off[i]
        objs["lnt_len"][i] = len(p.lnts[i])
    consts = arena.section("consts")
    for i, (kid, ival, n, off, re, im) in enumerate(p.consts):
        if isinstance(off, tuple):
            off = payload_base + off[1]
        consts[i] = (kid, ival, n, 0, off, re, im)
    strs = arena.section("strs")
    for i, b in enumerate(p.str_bytes):
        strs[i] = (str_off[i], len(b), 0)
    if p.refs:
        arena.section("refs")[:] = np.asarray(p.refs, dtype="<u4")
    if p.limbs:
        arena.section("limbs")[:] = np.concatenate(p.limbs)
    by = arena.section("bytes")
    for i, b in enumerate(p.codes):
        by[code_off[i]:code_off[i] + len(b)] = np.frombuffer(b, dtype=np.uint8)
    for offs, lst in ((exc_off, p.excs), (lnt_off, p.lnts), (str_off, p.str_bytes)):
        for o, b in zip(offs, lst):
            if b:
                by[o:o + len(b)] = np.frombuffer(b, dtype=np.uint8)
    o = payload_base
    for b in p.blobs:
        if b:
            by[o:o + len(b)] = np.frombuffer(b, dtype=np.uint8)
        o += len(b)
    arena.section("roots")[:] = np.asarray(root_ids, dtype="<i4")
    return arena


def unpack(arena: Arena, code_cls=CodeObject, const_cls=Const, version_cls=VersionTag, objects=None):
    """Rebuild the root CodeObject trees of an arena (inverse of `pack`).

    Used to feed arena-native synthetic corpora to CPU checkers; the classes are
    parameters so the same arena can be rebuilt as any CodeObject flavour.
    `objects` (object indices) selects other objects than the roots."""
    objs = arena.section("objs")
    consts = arena.section("consts")
    strs = arena.section("strs")
    refs = arena.section("refs")
    limbs = arena.section("limbs")
    by = arena.section("bytes")
    sblob = by.tobytes()
    cache_s = {}
    built = {}

    def s(i):
        v = cache_s.get(i)
        if v is None:
            r = strs[i]
            v = sblob[int(r["off"]):int(r["off"]) + int(r["len"])].decode("utf-8", "surrogatepass")
            cache_s[i] = v
        return v

    def const(i):
        r = consts[i]
        kind = KIND_NAME[int(r["kind"])]
        if kind in ("none", "ellipsis"):
            return const_cls(kind)
        if kind == "bool":
            return const_cls(kind, bool(r["ival"]))
        if kind == "int":
            off, n = int(r["off"]), int(r["n"])
            mag = int.from_bytes(limbs[off:off + n].tobytes(), "little")
            return const_cls(kind, mag * int(r["ival"]) if mag else 0)
        if kind == "float":
            return const_cls(kind, float(r["re"]))
        if kind == "complex":
            return const_cls(kind, complex(float(r["re"]), float(r["im"])))
        if kind in ("str", "bytes"):
            raw = sblob[int(r["off"]):int(r["off"]) + int(r["n"])]
            return const_cls(kind, raw.decode("utf-8", "surrogatepass") if kind == "str" else raw)
        if kind in ("tuple", "frozenset"):
            off, n = int(r["off"]), int(r["n"])
            return const_cls(kind, tuple(const(int(j)) for j in refs[off:off + n]))
        return const_cls("code", obj(int(r["off"])))

    def strtuple(off, n):
        return tuple(s(int(j)) for j in refs[off:off + n])

    def obj(i):
        if i in built:
            return built[i]
        r = objs[i]
        co, cl = int(r["code_off"]), int(r["code_len"])
        eo, el = int(r["exc_off"]), int(r["exc_len"])
        lo, ll = int(r["lnt_off"]), int(r["lnt_len"])
        c = code_cls(
            version_cls(3, int(r["minor"])), int(r["argcount"]), int(r["posonlyargcount"]),
            int(r["kwonlyargcount"]), int(r["nlocals"]), int(r["stacksize"]), int(r["flags"]),
            sblob[co:co + cl],
            tuple(const(int(j)) for j in refs[int(r["consts_off"]):int(r["consts_off"]) + int(r["n_consts"])]),
            strtuple(int(r["names_off"]), int(r["n_names"])),
            strtuple(int(r["varnames_off"]), int(r["n_varnames"])),
            strtuple(int(r["freevars_off"]), int(r["n_freevars"])),
            strtuple(int(r["cellvars_off"]), int(r["n_cellvars"])),
            s(int(r["name"])), s(int(r["filename"])), int(r["firstlineno"]),
            sblob[lo:lo + ll], sblob[eo:eo + el], s(int(r["qualname"])),
        )
        built[i] = c
        return c

    which = arena.section("roots") if objects is None else objects
    return [obj(int(i)) for i in which]


def tile(arena: Arena, reps: int) -> Arena:
    """Replicate every object `reps` times.  Each copy gets its own co_code
    bytes (so the decoder reads reps x the bytecode) and its own object
    records and roots; constant, string and name pools are shared read-only.
    Used to build benchmark-scale corpora from a pool of distinct objects."""
    objs = arena.section("objs")
    by = arena.section("bytes")
    roots = arena.section("roots")
    code_end = int(max((int(o) + int(l) for o, l in zip(objs["code_off"], objs["code_len"])), default=0))
    code_end = _align(code_end, 16)
    rest_shift = (reps - 1) * code_end
    n_obj = len(objs)
    counts = dict(arena.counts)
    counts["objs"] = n_obj * reps
    counts["roots"] = len(roots) * reps
    counts["bytes"] = int(arena.counts["bytes"]) + rest_shift
    sizes = {"objs": OBJ_DTYPE.itemsize, "consts": CONST_DTYPE.itemsize, "strs": STR_DTYPE.itemsize,
             "refs": 4, "limbs": 4, "bytes": 1, "roots": 4}
    offsets = {}
    total = 0
    for s in SECTIONS:
        offsets[s] = total
        total = _align(total + counts[s] * sizes[s], ALIGN)
    blob = np.zeros(total, dtype=np.uint8)
    out = Arena(blob, offsets, counts, arena.max_code_len, (code_end * reps + 1) // 2)
    o2 = out.section("objs").reshape(reps, n_obj)
    o2[:] = objs[None, :]
    o2["code_off"] += (np.arange(reps, dtype=np.uint64) * np.uint64(code_end))[:, None]
    o2["exc_off"] += np.uint64(rest_shift)
    o2["lnt_off"] += np.uint64(rest_shift)
    c2 = out.section("consts")
    c2[:] = arena.section("consts")
    pay = (c2["kind"] == KIND_ID["str"]) | (c2["kind"] == KIND_ID["bytes"])
    c2["off"][pay] += np.uint64(rest_shift)
    s2 = out.section("strs")
    s2[:] = arena.section("strs")
    s2["off"] += np.uint64(rest_shift)
    out.section("refs")[:] = arena.section("refs")
    out.section("limbs")[:] = arena.section("limbs")
    b2 = out.section("bytes")
    b2[:code_end * reps].reshape(reps, code_end)[:] = by[:code_end][None, :]
    b2[code_end * reps:] = by[code_end:]
    r2 = out.section("roots").reshape(reps, len(roots))
    r2[:] = roots[None, :] + (np.arange(reps, dtype=np.int32) * n_obj)[:, None]
    return out


def with_roots(arena: Arena, objects) -> Arena:
    """Same objects and pools, roots = the given object indices (a new roots
    section; roots is the last section, so the blob only grows at its end)."""
    roots = np.asarray(objects, dtype="<i4")
    blob = arena.blob.copy()
    off = arena.offsets["roots"]
    need = off + roots.nbytes
    if need > len(blob):
        blob = np.concatenate([blob, np.zeros(need - len(blob), np.uint8)])
    blob[off:off + roots.nbytes] = roots.view(np.uint8)
    counts = dict(arena.counts)
    counts["roots"] = len(roots)
    return Arena(blob, dict(arena.offsets), counts, arena.max_code_len, arena.total_code_units)


def from_blob(blob, header):
    """Arena from a raw blob + the header dict written by the synthetic generator."""
    offsets = {s: int(header["off_" + s]) for s in SECTIONS}
    counts = {s: int(header["n_" + s]) for s in SECTIONS}
    return Arena(blob, offsets, counts, header["max_code_len"], header["total_code_units"])
