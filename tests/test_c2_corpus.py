"""CPU tier for the C2 corpus (BASELINE configs[1]): the fixture's input trees
are pinned (input_sha), survive the JSON / .pyc round trips, and the 3.10
code generator that produced them lays out the CPython 3.10 shapes the
reference pattern-matches."""
import os

import pytest

from conftest import ROOT, golden_cases
from helpers import code_key_sha, inputs

LIB = os.path.join(ROOT, "paper_2403_13839_b200", "libupy_cuda.so")


def _recs():
    return [r for r in golden_cases(["c2"]) if not r.get("style")]


def test_c2_fixture_inputs_pinned():
    import hashlib

    from paper_2403_13839_b200.synth import codejson

    recs = _recs()
    assert len(recs) == 440 and all(r["status"] == "ok" for r in recs)
    assert sorted({r["minor"] for r in recs}) == [8, 9, 10, 11]
    for r, co in zip(recs, inputs(recs)):
        assert codejson.to_json(co) == r["tree"]
        h = hashlib.sha256()
        stack = [co]
        while stack:
            c = stack.pop()
            h.update(bytes([c.version.minor]))
            h.update(c.code)
            h.update(repr([(k.kind, k.value if k.kind != "code" else None) for k in c.consts]).encode())
            h.update(repr((c.names, c.varnames, c.freevars, c.cellvars, c.name, c.argcount, c.flags)).encode())
            h.update(c.exceptiontable)
            stack.extend(k.value for k in c.consts if k.kind == "code")
        assert h.hexdigest()[:16] == r["input_sha"], r["case"]


@pytest.mark.skipif(not os.path.exists(LIB), reason="CUDA library not built")
def test_c2_pyc_images_load_natively():
    from paper_2403_13839_b200 import arena, loader
    from paper_2403_13839_b200.synth import marshal

    trees = inputs(_recs())
    ar, per_file = loader.load_pyc_batch([marshal.dump_pyc(co) for co in trees])
    roots = arena.unpack(ar)
    assert [code_key_sha(roots[i]) for i in per_file] == [code_key_sha(co) for co in trees]


def _ops(src):
    from paper_2403_13839_b200._optables import TABLES
    from paper_2403_13839_b200.synth import pycodegen

    mod = pycodegen.compile_source(src)
    fn = next(c.value for c in mod.consts if c.kind == "code")
    code = fn.code
    return [(TABLES[10][code[i]][0], code[i + 1]) for i in range(0, len(code), 2)], fn


def test_codegen_rotated_while_loop():
    # CPython 3.10: the test is compiled at the top and again at the bottom
    # (compiler_while), POP_JUMP_IF_TRUE back to the body; jump args in units
    ops, _ = _ops("def f(n):\n    total = 0\n    while n > 0:\n        total += n\n        n -= 1\n"
                  "    return total\n")
    assert ops == [("LOAD_CONST", 1), ("STORE_FAST", 1), ("LOAD_FAST", 0), ("LOAD_CONST", 1), ("COMPARE_OP", 4),
                   ("POP_JUMP_IF_FALSE", 18), ("LOAD_FAST", 1), ("LOAD_FAST", 0), ("INPLACE_ADD", 0),
                   ("STORE_FAST", 1), ("LOAD_FAST", 0), ("LOAD_CONST", 2), ("INPLACE_SUBTRACT", 0),
                   ("STORE_FAST", 0), ("LOAD_FAST", 0), ("LOAD_CONST", 1), ("COMPARE_OP", 4),
                   ("POP_JUMP_IF_TRUE", 6), ("LOAD_FAST", 1), ("RETURN_VALUE", 0)]


def test_codegen_duplicates_unnumbered_exit():
    # duplicate_exits_without_lineno: the implicit `return None` reached by a
    # jump and by fall-through is copied for the jump
    ops, _ = _ops("def f(x):\n    if x:\n        g()\n")
    assert ops == [("LOAD_FAST", 0), ("POP_JUMP_IF_FALSE", 7), ("LOAD_GLOBAL", 0), ("CALL_FUNCTION", 0),
                   ("POP_TOP", 0), ("LOAD_CONST", 0), ("RETURN_VALUE", 0), ("LOAD_CONST", 0), ("RETURN_VALUE", 0)]


def test_codegen_and_or_jump_threading():
    # optimize_basic_block: JUMP_IF_FALSE_OR_POP onto JUMP_IF_TRUE_OR_POP becomes
    # POP_JUMP_IF_FALSE past it
    ops, _ = _ops("def f(a, b, c):\n    x = a and b or c\n    return x\n")
    assert ops[:5] == [("LOAD_FAST", 0), ("POP_JUMP_IF_FALSE", 4), ("LOAD_FAST", 1), ("JUMP_IF_TRUE_OR_POP", 5),
                       ("LOAD_FAST", 2)]


def test_codegen_closures_and_class_cell():
    from paper_2403_13839_b200.synth import pycodegen

    mod = pycodegen.compile_source("def f(base):\n    def add(n):\n        return base + n\n    return add\n"
                                   "class C(B):\n    def m(self):\n        return super().m()\n")
    f, cls = [c.value for c in mod.consts if c.kind == "code"]
    assert f.cellvars == ("base",) and f.flags & 0x40 == 0
    add = next(c.value for c in f.consts if c.kind == "code")
    assert add.freevars == ("base",) and add.flags & 0x10
    assert cls.cellvars == ("__class__",)
    m = next(c.value for c in cls.consts if c.kind == "code")
    assert m.freevars == ("__class__",)


def test_codegen311_try_except_layout_and_exception_table():
    # CPython 3.11: handler entered with PUSH_EXC_INFO / CHECK_EXC_MATCH, the
    # `as` name cleaned up in an artificial block, `COPY 3; POP_EXCEPT;
    # RERAISE 1` cleanup, zero-cost exception table with depth / lasti
    from paper_2403_13839_b200._optables import TABLES
    from paper_2403_13839_b200.synth import pycodegen311

    mod = pycodegen311.compile_source("def f(d, k):\n    try:\n        return d[k]\n    except KeyError as exc:\n"
                                      "        return 'missing:' + repr(exc.args[0])\n")
    fn = mod.consts[0].value
    code = fn.code
    ops = []
    i = 0
    while i < len(code):
        name, _, _, caches = TABLES[11][code[i]]
        ops.append((name, code[i + 1]))
        i += 2 * (1 + caches)
    assert ops[:5] == [("RESUME", 0), ("NOP", 0), ("LOAD_FAST", 0), ("LOAD_FAST", 1), ("BINARY_SUBSCR", 0)]
    assert ("POP_JUMP_FORWARD_IF_FALSE", 39) in ops and ops[-3:] == [("COPY", 3), ("POP_EXCEPT", 0), ("RERAISE", 1)]
    assert ("LOAD_GLOBAL", 3) in ops  # NULL + repr
    # entries (start, size, target, depth<<1|lasti) in code units, varint encoded
    assert fn.exceptiontable == bytes([0x82, 7, 10, 0, 0x8a, 10, 59, 3, 0x94, 28, 54, 3, 0xb0, 1, 59, 3, 0xb6, 5, 59, 3])


def test_codegen39_leading_test_while_loop():
    # CPython 3.9: test at the top, JUMP_ABSOLUTE back to it, byte-offset jump args
    from paper_2403_13839_b200._optables import TABLES
    from paper_2403_13839_b200.synth import pycodegen39

    mod = pycodegen39.compile_source("def f(n):\n    total = 0\n    while n > 0:\n        total += n\n"
                                     "        n -= 1\n    return total\n")
    code = next(c.value for c in mod.consts if c.kind == "code").code
    ops = [(TABLES[9][code[i]][0], code[i + 1]) for i in range(0, len(code), 2)]
    assert ops == [("LOAD_CONST", 1), ("STORE_FAST", 1), ("LOAD_FAST", 0), ("LOAD_CONST", 1), ("COMPARE_OP", 4),
                   ("POP_JUMP_IF_FALSE", 30), ("LOAD_FAST", 1), ("LOAD_FAST", 0), ("INPLACE_ADD", 0),
                   ("STORE_FAST", 1), ("LOAD_FAST", 0), ("LOAD_CONST", 2), ("INPLACE_SUBTRACT", 0),
                   ("STORE_FAST", 0), ("JUMP_ABSOLUTE", 4), ("LOAD_FAST", 1), ("RETURN_VALUE", 0)]


def test_codegen38_finally_and_exception_match():
    # CPython 3.8: BEGIN_FINALLY / END_FINALLY / CALL_FINALLY finally machinery,
    # COMPARE_OP 10 (exception match), BUILD_LIST_UNPACK for starred displays
    from paper_2403_13839_b200._optables import TABLES
    from paper_2403_13839_b200.synth import pycodegen38

    mod = pycodegen38.compile_source("def f(a, xs):\n    try:\n        return g(a)\n    except KeyError:\n"
                                     "        pass\n    finally:\n        h()\n    return [*xs, 1]\n")
    code = next(c.value for c in mod.consts if c.kind == "code").code
    names = [TABLES[8][code[i]][0] for i in range(0, len(code), 2)]
    for op in ("SETUP_FINALLY", "CALL_FINALLY", "BEGIN_FINALLY", "END_FINALLY", "POP_EXCEPT",
               "BUILD_LIST_UNPACK"):
        assert op in names, op
    assert ("COMPARE_OP", 10) in [(TABLES[8][code[i]][0], code[i + 1]) for i in range(0, len(code), 2)]
