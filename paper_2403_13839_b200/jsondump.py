"""The portable JSON code-object dump format (second loader).

`load_json_dump(text, version_override=None) -> [CodeObject]` restates the
reference's reader (/root/reference/pkg/src/unpyre/pyc.py:357-508): the same
schema checks in the same order, the same SchemaError messages and JSON-path
locations (errors.py:37-40).  It is host code that only builds the input
records; the records go to the device through the arena packer like any
other CodeObject.  `dumps(code)` writes the format (used for test corpora and
the CLI's verify fixtures).
"""
from __future__ import annotations

import base64
import json

from . import errors
from .model import CodeObject, Const, VersionTag

# Field schema of one code object, in the order the reference validates it
# (pyc.py:357-375, 420-437): (key, JSON type, type name in the message).
_SCHEMA = tuple((k, t, t.__name__) for k, t in (
    ("argcount", int), ("posonlyargcount", int), ("kwonlyargcount", int), ("nlocals", int),
    ("stacksize", int), ("flags", int), ("code", str), ("consts", list), ("names", list),
    ("varnames", list), ("freevars", list), ("cellvars", list), ("name", str), ("filename", str),
    ("firstlineno", int), ("linetable", str), ("exceptiontable", str)))
_STR_LISTS = ("names", "varnames", "freevars", "cellvars")
_INT_FIELDS = ("argcount", "posonlyargcount", "kwonlyargcount", "nlocals", "stacksize", "flags")


class _Reader:
    """Converts one parsed dump tree into CodeObject/Const records, failing with
    the reference's SchemaError (message, JSON path) at the first violation."""

    def __init__(self, version):
        self.version = version
        # constant tag -> builder(node, path); a builder may raise KeyError (the
        # missing key) or ValueError/TypeError (a malformed value): `const`
        # turns those into the reference's two generic messages (pyc.py:503-506)
        self.tags = {
            "none": lambda n, p: Const("none"),
            "ellipsis": lambda n, p: Const("ellipsis"),
            "bool": lambda n, p: Const("bool", self._typed(n, p, "v", bool, "expected bool")),
            "int": lambda n, p: Const("int", int(n["v"])),
            "float": lambda n, p: Const("float", float.fromhex(n["v"])),
            "complex": lambda n, p: Const("complex", complex(float.fromhex(n["re"]), float.fromhex(n["im"]))),
            "str": lambda n, p: Const("str", self._typed(n, p, "v", str, "expected string")),
            "bytes": lambda n, p: Const("bytes", self.b64(n, p, "v")),
            "tuple": lambda n, p: Const("tuple", self.seq(n["v"], p + ".v")),
            "frozenset": lambda n, p: Const("frozenset", self.seq(n["v"], p + ".v")),
            "code": lambda n, p: Const("code", self.code(n["v"], p + ".v")),
        }

    @staticmethod
    def _typed(node, path, key, typ, msg):
        v = node[key]
        if not isinstance(v, typ):
            raise errors.SchemaError(msg, f"{path}.{key}")
        return v

    @staticmethod
    def b64(node, path, key):
        v = node[key]
        where = f"{path}.{key}"
        if not isinstance(v, str):
            raise errors.SchemaError("expected base64 string", where)
        try:
            return base64.b64decode(v, validate=True)
        except Exception:  # noqa: BLE001 -- binascii.Error / ValueError, as the reference
            raise errors.SchemaError("invalid base64", where) from None

    def seq(self, items, path):
        return tuple(self.const(c, f"{path}[{i}]") for i, c in enumerate(items))

    def const(self, node, path):
        if not (isinstance(node, dict) and "t" in node):
            raise errors.SchemaError("constant must be an object with a 't' tag", path)
        tag = node["t"]
        build = self.tags.get(tag) if isinstance(tag, str) else None
        if build is None:
            raise errors.SchemaError(f"unknown constant tag {tag!r}", f"{path}.t")
        try:
            return build(node, path)
        except KeyError as exc:
            raise errors.SchemaError("missing field", f"{path}.{exc.args[0]}") from None
        except (ValueError, TypeError):
            raise errors.SchemaError(f"bad value for constant of type {tag!r}", path) from None

    def code(self, node, path):
        if not isinstance(node, dict):
            raise errors.SchemaError("code object must be a JSON object", path)
        for key, typ, tname in _SCHEMA:
            if key not in node:
                raise errors.SchemaError("missing field", f"{path}.{key}")
            v = node[key]
            if isinstance(v, bool) or not isinstance(v, typ):
                raise errors.SchemaError(f"expected {tname}", f"{path}.{key}")
        for key in _STR_LISTS:
            if any(not isinstance(x, str) for x in node[key]):
                raise errors.SchemaError("expected list of strings", f"{path}.{key}")
        consts = self.seq(node["consts"], path + ".consts")
        ints = [node[k] for k in _INT_FIELDS]
        code = self.b64(node, path, "code")
        lists = [tuple(node[k]) for k in _STR_LISTS]
        return CodeObject(self.version, *ints, code, consts, *lists, node["name"], node["filename"],
                          node["firstlineno"], self.b64(node, path, "linetable"),
                          self.b64(node, path, "exceptiontable"), node.get("qualname", ""))


def _version_of(doc, override):
    if override is not None:
        return override
    ver = doc.get("python_version")
    if not (isinstance(ver, list) and len(ver) == 2 and all(isinstance(x, int) for x in ver)):
        raise errors.SchemaError("python_version must be [major, minor]", "$.python_version")
    try:
        return VersionTag(*ver)
    except errors.UnsupportedVersion as exc:
        raise errors.SchemaError(str(exc), "$.python_version") from None


def load_json_dump(text: str, version_override=None) -> list:
    """One root code object, returned as a one-element list (pyc.py:378-407)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise errors.SchemaError(f"not valid JSON: {exc.msg}", "$") from None
    if not isinstance(doc, dict):
        raise errors.SchemaError("top level must be an object", "$")
    if doc.get("format_version") != 1:
        raise errors.SchemaError("format_version must be 1", "$.format_version")
    version = _version_of(doc, version_override)
    if "root" not in doc:
        raise errors.SchemaError("missing field", "$.root")
    return [_Reader(version).code(doc["root"], "$.root")]


# ------------------------------------------------------------------ writer

def _wconst(c):
    k, v = c.kind, c.value
    if k in ("none", "ellipsis"):
        return {"t": k}
    if k in ("bool", "str"):
        return {"t": k, "v": v}
    if k == "int":
        return {"t": k, "v": v}
    if k == "float":
        return {"t": k, "v": v.hex()}
    if k == "complex":
        return {"t": k, "re": v.real.hex(), "im": v.imag.hex()}
    if k == "bytes":
        return {"t": k, "v": base64.b64encode(v).decode()}
    if k in ("tuple", "frozenset"):
        return {"t": k, "v": [_wconst(x) for x in v]}
    return {"t": "code", "v": _wcode(v)}


def _wcode(co):
    b = lambda x: base64.b64encode(bytes(x)).decode()  # noqa: E731
    return {
        "argcount": co.argcount, "posonlyargcount": co.posonlyargcount, "kwonlyargcount": co.kwonlyargcount,
        "nlocals": co.nlocals, "stacksize": co.stacksize, "flags": co.flags, "code": b(co.code),
        "consts": [_wconst(c) for c in co.consts], "names": list(co.names), "varnames": list(co.varnames),
        "freevars": list(co.freevars), "cellvars": list(co.cellvars), "name": co.name, "filename": co.filename,
        "firstlineno": co.firstlineno, "linetable": b(co.linetable), "exceptiontable": b(co.exceptiontable),
        "qualname": co.qualname,
    }


def dumps(code, indent=None) -> str:
    return json.dumps({"format_version": 1, "python_version": [code.version.major, code.version.minor],
                       "root": _wcode(code)}, indent=indent)
