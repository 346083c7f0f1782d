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

from .errors import SchemaError, UnsupportedVersion
from .model import CodeObject, Const, VersionTag

_CODE_FIELDS = {  # pyc.py:357-375, checked in this order
    "argcount": int, "posonlyargcount": int, "kwonlyargcount": int, "nlocals": int, "stacksize": int,
    "flags": int, "code": str, "consts": list, "names": list, "varnames": list, "freevars": list,
    "cellvars": list, "name": str, "filename": str, "firstlineno": int, "linetable": str,
    "exceptiontable": str,
}


def load_json_dump(text: str, version_override=None) -> list:
    """pyc.py:378-407: one root code object, returned as a one-element list."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise SchemaError(f"not valid JSON: {exc.msg}", "$") from None
    if not isinstance(doc, dict):
        raise SchemaError("top level must be an object", "$")
    if doc.get("format_version") != 1:
        raise SchemaError("format_version must be 1", "$.format_version")
    ver = doc.get("python_version")
    if version_override is not None:
        version = version_override
    else:
        if not isinstance(ver, list) or len(ver) != 2 or not all(isinstance(x, int) for x in ver):
            raise SchemaError("python_version must be [major, minor]", "$.python_version")
        try:
            version = VersionTag(*ver)
        except UnsupportedVersion as exc:
            raise SchemaError(str(exc), "$.python_version") from None
    if "root" not in doc:
        raise SchemaError("missing field", "$.root")
    return [_code(doc["root"], "$.root", version)]


def _b64(obj, path, key):
    raw = obj[key]
    if not isinstance(raw, str):
        raise SchemaError("expected base64 string", f"{path}.{key}")
    try:
        return base64.b64decode(raw, validate=True)
    except Exception:  # noqa: BLE001 - binascii.Error and friends, as the reference
        raise SchemaError("invalid base64", f"{path}.{key}") from None


def _code(obj, path, version):
    """pyc.py:420-458."""
    if not isinstance(obj, dict):
        raise SchemaError("code object must be a JSON object", path)
    for key, typ in _CODE_FIELDS.items():
        if key not in obj:
            raise SchemaError("missing field", f"{path}.{key}")
        if not isinstance(obj[key], typ) or isinstance(obj[key], bool):
            raise SchemaError(f"expected {typ.__name__}", f"{path}.{key}")
    for key in ("names", "varnames", "freevars", "cellvars"):
        if not all(isinstance(x, str) for x in obj[key]):
            raise SchemaError("expected list of strings", f"{path}.{key}")
    consts = tuple(_const(c, f"{path}.consts[{i}]", version) for i, c in enumerate(obj["consts"]))
    return CodeObject(
        version, obj["argcount"], obj["posonlyargcount"], obj["kwonlyargcount"], obj["nlocals"],
        obj["stacksize"], obj["flags"], _b64(obj, path, "code"), consts, tuple(obj["names"]),
        tuple(obj["varnames"]), tuple(obj["freevars"]), tuple(obj["cellvars"]), obj["name"], obj["filename"],
        obj["firstlineno"], _b64(obj, path, "linetable"), _b64(obj, path, "exceptiontable"),
        obj.get("qualname", ""))


def _const(obj, path, version):
    """pyc.py:461-508."""
    if not isinstance(obj, dict) or "t" not in obj:
        raise SchemaError("constant must be an object with a 't' tag", path)
    t = obj["t"]
    try:
        if t == "none":
            return Const("none")
        if t == "ellipsis":
            return Const("ellipsis")
        if t == "bool":
            if not isinstance(obj["v"], bool):
                raise SchemaError("expected bool", f"{path}.v")
            return Const("bool", obj["v"])
        if t == "int":
            return Const("int", int(obj["v"]))
        if t == "float":
            return Const("float", float.fromhex(obj["v"]))
        if t == "complex":
            return Const("complex", complex(float.fromhex(obj["re"]), float.fromhex(obj["im"])))
        if t == "str":
            if not isinstance(obj["v"], str):
                raise SchemaError("expected string", f"{path}.v")
            return Const("str", obj["v"])
        if t == "bytes":
            return Const("bytes", _b64(obj, path, "v"))
        if t in ("tuple", "frozenset"):
            return Const(t, tuple(_const(c, f"{path}.v[{i}]", version) for i, c in enumerate(obj["v"])))
        if t == "code":
            return Const("code", _code(obj["v"], f"{path}.v", version))
    except KeyError as exc:
        raise SchemaError("missing field", f"{path}.{exc.args[0]}") from None
    except (ValueError, TypeError):
        raise SchemaError(f"bad value for constant of type {t!r}", path) from None
    raise SchemaError(f"unknown constant tag {t!r}", f"{path}.t")


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
