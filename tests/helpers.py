"""Shared helpers: rebuild golden inputs and compare results by class + text."""
from paper_2403_13839_b200.model import EmitStyle
from paper_2403_13839_b200.synth import cases

ST_NAMES = {0: "ok", 1: "UnpyreError", 2: "UnknownOpcode", 3: "TruncatedCode", 4: "BadJumpTarget",
            5: "MalformedExceptionTable", 6: "StackUnderflow", 7: "UnsupportedOpcode",
            8: "StackDepthMismatch", 9: "StructuringFailed", 10: "InternalMarkerLeak", 20: "IndexError",
            21: "AttributeError", 22: "TypeError", 23: "KeyError", 24: "ValueError", 25: "RecursionError"}


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


def mismatches(recs, got):
    bad = []
    for r, g in zip(recs, got):
        if (r["status"], r["text"]) != g:
            bad.append((r["case"], r["status"], g[0], r["text"][:300], g[1][:300]))
    return bad
