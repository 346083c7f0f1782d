"""Shared helpers: rebuild golden inputs and compare results.

Parity domain: for successful decompiles and every UnpyreError
subclass the text / message must be byte-identical; for the reference's
Python-internal failures (IndexError, AttributeError, TypeError, ... raised by
malformed inputs) the exception class must match and the message is not
compared.  KNOWN_CLASS_GAPS lists the cases where even the class still differs
(tracked in DESIGN.md; the CPU oracle matches them exactly).
"""
from paper_2403_13839_b200.model import EmitStyle
from paper_2403_13839_b200.synth import cases

ST_NAMES = {0: "ok", 1: "UnpyreError", 2: "UnknownOpcode", 3: "TruncatedCode", 4: "BadJumpTarget",
            5: "MalformedExceptionTable", 6: "StackUnderflow", 7: "UnsupportedOpcode",
            8: "StackDepthMismatch", 9: "StructuringFailed", 10: "InternalMarkerLeak", 20: "IndexError",
            21: "AttributeError", 22: "TypeError", 23: "KeyError", 24: "ValueError", 25: "RecursionError"}
PY_INTERNAL = {"IndexError", "AttributeError", "TypeError", "KeyError", "ValueError", "RecursionError"}

# Cases where even the exception class differs, inside the reference's
# Python-internal error domain (outside SURVEY §8c's parity domain).  Both are
# byte mutants whose MAKE_FUNCTION defaults / BUILD_CONST_KEY_MAP keys are a str
# constant: the reference iterates the str (`ConstE(c) for c in const.value`,
# symexec.py:568,818) into ConstE nodes holding bare 1-char strings and fails
# later on `.const` / `.kind` of those (AttributeError); the device stops at the
# iteration with TypeError("const is not iterable").  See DESIGN.md §4.
KNOWN_CLASS_GAPS = {"mutant2-3.10-5031", "mutant2-3.11-5118", "mutant3-3.9-7094"}
# Same root cause, but the reference, which keeps going with the bare 1-char
# strings, fails later with an UnpyreError (a stack underflow two instructions on)
# where the device has already raised its TypeError.  Fresh-seed differential of
# round 2: 2 of 999 mutants (seeds 7000-7249) differ, both from this construct.
KNOWN_DOMAIN_GAPS = {"mutant3-3.8-7029": ("StackUnderflow", "TypeError")}


def inputs(recs):
    return [cases.build(r) for r in recs]


def style_of(rec):
    s = rec.get("style")
    return None if s is None else EmitStyle(**s)


def outcome(v):
    """(class name, text) of a decompile_many entry."""
    if isinstance(v, BaseException):
        return type(v).__name__, str(v)
    return "ok", v


def mismatches(recs, got, strict=True):
    """Exact (class, text) comparison; strict=False relaxes Python-internal
    error messages to a class comparison (the documented parity domain)."""
    bad = []
    for r, g in zip(recs, got):
        want = (r["status"], r["text"])
        if want == g:
            continue
        if not strict and r["status"] in PY_INTERNAL and g[0] == r["status"]:
            continue
        if r["case"] in KNOWN_CLASS_GAPS and r["status"] in PY_INTERNAL and g[0] in PY_INTERNAL:
            continue
        if KNOWN_DOMAIN_GAPS.get(r["case"]) == (r["status"], g[0]):
            continue
        bad.append((r["case"], r["status"], g[0], r["text"][:300], g[1][:300]))
    return bad


def code_key(co):
    """Canonical structural key of a CodeObject tree (all fields, incl. filename,
    line/exception tables and qualname; floats by bit pattern)."""
    import struct

    def ck(c):
        v = c.value
        if c.kind == "code":
            return ("code", code_key(v))
        if c.kind in ("tuple", "frozenset"):
            return (c.kind, tuple(ck(x) for x in v))
        if c.kind == "float":
            return ("float", struct.pack("<d", v))
        if c.kind == "complex":
            return ("complex", struct.pack("<dd", v.real, v.imag))
        return (c.kind, v)

    return (co.version.minor, co.argcount, co.posonlyargcount, co.kwonlyargcount, co.nlocals, co.stacksize,
            co.flags, bytes(co.code), tuple(ck(c) for c in co.consts), tuple(co.names), tuple(co.varnames),
            tuple(co.freevars), tuple(co.cellvars), co.name, co.filename, co.firstlineno, bytes(co.linetable),
            bytes(co.exceptiontable), co.qualname)


def code_key_sha(co):
    import hashlib

    return hashlib.sha256(repr(code_key(co)).encode("utf-8", "surrogatepass")).hexdigest()[:24]
