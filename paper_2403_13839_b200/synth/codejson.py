"""Lossless JSON form of a CodeObject tree (test fixtures only).

Inputs that cannot be regenerated on the GPU box (the C2 corpus is compiled
from the reference's source files, which exist only in the build container)
are committed in this form: every CodeObject field, the constant tree with
floats / complex parts as float.hex (bit-exact, incl. -0.0 and nan payload
sign), bytes as hex and strings as JSON text (lone surrogates survive
json's \\uXXXX escapes).
"""
from __future__ import annotations

from ..model import CodeObject, Const, VersionTag

_FIELDS = ("argcount", "posonlyargcount", "kwonlyargcount", "nlocals", "stacksize", "flags")
_STRS = ("names", "varnames", "freevars", "cellvars")


def _c2j(c):
    k, v = c.kind, c.value
    if k in ("none", "ellipsis"):
        return [k]
    if k in ("bool", "int", "str"):
        return [k, v]
    if k == "float":
        return [k, v.hex()]
    if k == "complex":
        return [k, v.real.hex(), v.imag.hex()]
    if k == "bytes":
        return [k, v.hex()]
    if k in ("tuple", "frozenset"):
        return [k, [_c2j(x) for x in v]]
    if k == "code":
        return [k, to_json(v)]
    raise ValueError(k)


def _j2c(j):
    k = j[0]
    if k in ("none", "ellipsis"):
        return Const(k)
    if k in ("bool", "int", "str"):
        return Const(k, j[1])
    if k == "float":
        return Const(k, float.fromhex(j[1]))
    if k == "complex":
        return Const(k, complex(float.fromhex(j[1]), float.fromhex(j[2])))
    if k == "bytes":
        return Const(k, bytes.fromhex(j[1]))
    if k in ("tuple", "frozenset"):
        return Const(k, tuple(_j2c(x) for x in j[1]))
    if k == "code":
        return Const(k, from_json(j[1]))
    raise ValueError(k)


def to_json(co):
    d = {"minor": co.version.minor}
    for f in _FIELDS:
        d[f] = getattr(co, f)
    d["code"] = bytes(co.code).hex()
    d["consts"] = [_c2j(c) for c in co.consts]
    for f in _STRS:
        d[f] = list(getattr(co, f))
    d.update(name=co.name, filename=co.filename, firstlineno=co.firstlineno, qualname=co.qualname,
             linetable=bytes(co.linetable).hex(), exceptiontable=bytes(co.exceptiontable).hex())
    return d


def from_json(d):
    return CodeObject(
        VersionTag(3, d["minor"]), *[d[f] for f in _FIELDS], bytes.fromhex(d["code"]),
        tuple(_j2c(c) for c in d["consts"]), *[tuple(d[f]) for f in _STRS], d["name"], d["filename"],
        d["firstlineno"], bytes.fromhex(d["linetable"]), bytes.fromhex(d["exceptiontable"]), d["qualname"])
