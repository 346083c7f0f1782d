"""Writer for CPython .pyc images (PEP 552 header + marshal stream) of 3.8-3.11
code objects, used to build loader corpora: no 3.8-3.11 interpreter exists in
this image, so `.pyc` inputs are synthesised from CodeObject trees.

The stream follows what CPython's marshal (version 4) emits and what the
reference reader accepts (/root/reference/pkg/src/unpyre/pyc.py:57-352):
identifiers as interned short-ASCII strings with FLAG_REF and later uses as
'r' back-references, code objects flagged FLAG_REF, small tuples as ')',
int32 ints as 'i' and larger ones as 15-bit-digit 'l', binary floats 'g' and
complex 'y'.  Options vary the encodings (long-form tuples, 'a'/'u' strings,
no refs) so every reader branch gets exercised.
"""
from __future__ import annotations

import struct

MAGIC = {8: 3413, 9: 3425, 10: 3439, 11: 3495}
FLAG_REF = 0x80


class _W:
    def __init__(self, minor, refs=True, long_tuples=False, unicode_all=False, share_bytes=False):
        self.minor = minor
        self.share_bytes = share_bytes  # equal bytes objects written once, then as 'r' back-references
        self.bytes_refs = {}
        self.out = bytearray()
        self.use_refs = refs
        self.long_tuples = long_tuples
        self.unicode_all = unicode_all
        self.str_refs = {}
        self.nrefs = 0

    def b(self, x):
        self.out += x

    def i32(self, v):
        self.out += struct.pack("<i", v)

    def _new_ref(self):
        i = self.nrefs
        self.nrefs += 1
        return i

    def string(self, s, ident=False):
        key = ("s", s)
        if self.use_refs and ident and key in self.str_refs:
            self.b(b"r")
            self.i32(self.str_refs[key])
            return
        flag = FLAG_REF if (self.use_refs and ident) else 0
        if flag:
            self.str_refs[key] = self._new_ref()
        try:
            raw = s.encode("ascii")
            ascii_ok = not self.unicode_all
        except UnicodeEncodeError:
            ascii_ok = False
        if ascii_ok:
            if len(raw) < 256:
                self.b(bytes([(ord("Z") if ident else ord("z")) | flag, len(raw)]))
            else:
                self.b(bytes([(ord("A") if ident else ord("a")) | flag]))
                self.i32(len(raw))
            self.b(raw)
        else:
            raw = s.encode("utf-8", "surrogatepass")
            self.b(bytes([(ord("t") if ident else ord("u")) | flag]))
            self.i32(len(raw))
            self.b(raw)

    def const(self, c):
        k, v = c.kind, c.value
        if k == "none":
            self.b(b"N")
        elif k == "ellipsis":
            self.b(b".")
        elif k == "bool":
            self.b(b"T" if v else b"F")
        elif k == "int":
            v = int(v)
            if -(1 << 31) <= v < (1 << 31):
                self.b(b"i")
                self.i32(v)
            else:
                mag = abs(v)
                digits = []
                while mag:
                    digits.append(mag & 0x7FFF)
                    mag >>= 15
                self.b(b"l")
                self.i32(-len(digits) if v < 0 else len(digits))
                for d in digits:
                    self.out += struct.pack("<H", d)
        elif k == "float":
            self.b(b"g")
            self.out += struct.pack("<d", v)
        elif k == "complex":
            self.b(b"y")
            self.out += struct.pack("<dd", v.real, v.imag)
        elif k == "str":
            self.string(v, ident=v.isidentifier())
        elif k == "bytes":
            self.b(b"s")
            self.i32(len(v))
            self.b(bytes(v))
        elif k in ("tuple", "frozenset"):
            self.tuple_(v, frozen=k == "frozenset")
        elif k == "code":
            self.code(v)
        else:
            raise ValueError(k)

    def tuple_(self, items, frozen=False, strs=False):
        if frozen:
            self.b(b">")
            self.i32(len(items))
        elif len(items) < 256 and not self.long_tuples:
            self.b(bytes([ord(")"), len(items)]))
        else:
            self.b(b"(")
            self.i32(len(items))
        for x in items:
            if strs:
                self.string(x, ident=True)
            else:
                self.const(x)

    def bytes_(self, b):
        b = bytes(b)
        if self.share_bytes:
            if b in self.bytes_refs:
                self.b(b"r")
                self.i32(self.bytes_refs[b])
                return
            self.bytes_refs[b] = self._new_ref()
            self.b(bytes([ord("s") | FLAG_REF]))
        else:
            self.b(b"s")
        self.i32(len(b))
        self.b(b)

    def code(self, co):
        flag = FLAG_REF if self.use_refs else 0
        if flag:
            self._new_ref()
        self.b(bytes([ord("c") | flag]))
        self.i32(co.argcount)
        self.i32(co.posonlyargcount)
        self.i32(co.kwonlyargcount)
        if self.minor <= 10:
            self.i32(co.nlocals)
        self.i32(co.stacksize)
        self.i32(co.flags)
        self.bytes_(co.code)
        self.tuple_(tuple(co.consts))
        self.tuple_(tuple(co.names), strs=True)
        if self.minor <= 10:
            self.tuple_(tuple(co.varnames), strs=True)
            self.tuple_(tuple(co.freevars), strs=True)
            self.tuple_(tuple(co.cellvars), strs=True)
            self.string(co.filename)
            self.string(co.name, ident=True)
            self.i32(co.firstlineno)
            self.bytes_(co.linetable or b"")
        else:
            names, kinds = [], []
            for v in co.varnames:
                names.append(v)
                kinds.append(0x20 | (0x40 if v in co.cellvars else 0))
            for c in co.cellvars:
                if c not in co.varnames:
                    names.append(c)
                    kinds.append(0x40)
            for f in co.freevars:
                names.append(f)
                kinds.append(0x80)
            self.tuple_(tuple(names), strs=True)
            self.bytes_(bytes(kinds))
            self.string(co.filename)
            self.string(co.name, ident=True)
            self.string(co.qualname or co.name, ident=True)
            self.i32(co.firstlineno)
            self.bytes_(co.linetable or b"")
            self.bytes_(co.exceptiontable or b"")


def dumps(code, minor=None, **opts) -> bytes:
    """Marshal stream of `code` (no pyc header)."""
    minor = code.version.minor if minor is None else minor
    w = _W(minor, **opts)
    w.code(code)
    return bytes(w.out)


def dump_pyc(code, minor=None, **opts) -> bytes:
    """PEP 552 .pyc image: magic, bitfield 0, 8 bytes of mtime/size, marshal."""
    minor = code.version.minor if minor is None else minor
    head = struct.pack("<H", MAGIC[minor]) + b"\r\n" + struct.pack("<I", 0) + struct.pack("<II", 0x5F5E100, 0)
    return head + dumps(code, minor, **opts)
