"""Host-side input records: the reference's CodeObject / Const / VersionTag /
EmitStyle surface, re-stated so callers construct inputs exactly as they do for
the reference (same field names, order, defaults and equality rules).

Reference: /root/reference/pkg/src/unpyre/code_model.py:27-180 (VersionTag,
Const, CodeObject) and emitter.py:46-50 (EmitStyle).  Any object exposing the
same attributes (including the reference's own instances) is accepted by the
arena packer; these classes exist so the product has no dependency on the
reference package.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

from . import errors

SUPPORTED_VERSIONS = ((3, 8), (3, 9), (3, 10), (3, 11))
CO_VARARGS = 0x0004
CO_VARKEYWORDS = 0x0008
CO_GENERATOR = 0x0020
CO_ASYNC_GENERATOR = 0x0200


@dataclass(frozen=True, order=True)
class VersionTag:
    major: int
    minor: int

    def __post_init__(self):
        if (self.major, self.minor) not in SUPPORTED_VERSIONS:
            raise errors.UnsupportedVersion(self.major, self.minor)

    def __str__(self):
        return f"{self.major}.{self.minor}"

    @property
    def pair(self):
        return (self.major, self.minor)


CONST_KINDS = ("none", "bool", "int", "float", "complex", "str", "bytes",
               "tuple", "frozenset", "code", "ellipsis")


class Const:
    """One constant-tree node; kind-tagged, float equality on the bit pattern
    (code_model.py:46-98)."""

    __slots__ = ("kind", "value")

    def __init__(self, kind, value=None):
        if kind not in CONST_KINDS:
            raise ValueError(f"bad const kind {kind!r}")
        self.kind = kind
        self.value = value

    def _key(self):
        k = self.kind
        if k == "float":
            return (k, struct.pack("<d", self.value))
        if k == "complex":
            return (k, struct.pack("<dd", self.value.real, self.value.imag))
        if k == "tuple":
            return (k, tuple(c._key() for c in self.value))
        if k == "frozenset":
            return (k, frozenset(c._key() for c in self.value))
        if k == "code":
            return (k, self.value._key())
        return (k, self.value)

    def __eq__(self, other):
        return isinstance(other, Const) and self._key() == other._key()

    def __hash__(self):
        return hash(self._key())

    def __repr__(self):
        if self.kind in ("none", "ellipsis"):
            return f"Const({self.kind})"
        return f"Const({self.kind}, {self.value!r})"

    @classmethod
    def none(cls):
        return cls("none")


@dataclass(frozen=True)
class CodeObject:
    version: VersionTag
    argcount: int
    posonlyargcount: int
    kwonlyargcount: int
    nlocals: int
    stacksize: int
    flags: int
    code: bytes
    consts: tuple
    names: tuple
    varnames: tuple
    freevars: tuple
    cellvars: tuple
    name: str
    filename: str
    firstlineno: int
    linetable: bytes = b""
    exceptiontable: bytes = b""
    qualname: str = ""

    def __post_init__(self):
        if not self.qualname:
            object.__setattr__(self, "qualname", self.name)

    def _key(self):
        return (self.version.pair, self.argcount, self.posonlyargcount, self.kwonlyargcount,
                self.nlocals, self.stacksize, self.flags, self.code,
                tuple(c._key() for c in self.consts), self.names, self.varnames,
                self.freevars, self.cellvars, self.name, self.firstlineno)

    def code_consts(self):
        return [c.value for c in self.consts if c.kind == "code"]


@dataclass
class EmitStyle:
    indent: str = "    "
    header: bool = False
    tool: str = "unpyre"


def flatten_nested_codes(c):
    """Depth-first (path, code) list in consts order (code_model.py:256-278)."""
    out = []

    def rec(code, path):
        out.append((path, code))
        for child in _code_consts(code.consts):
            rec(child, f"{path}.{child.name}")

    rec(c, c.name)
    return out


def _code_consts(consts):
    for k in consts:
        if k.kind == "code":
            yield k.value
        elif k.kind in ("tuple", "frozenset"):
            yield from _code_consts(k.value)
