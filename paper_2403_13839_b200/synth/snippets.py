"""Hand-assembled code objects covering the SPEC known-answer examples
(/root/reference/SPEC.md `examples:` lines) and targeted constructs.  Each
builder takes the minor version and returns a CodeObject.
"""
from __future__ import annotations

from ..model import CodeObject, Const, VersionTag
from .asm import Asm, L

NB = {"+": 0, "&": 1, "//": 2, "<<": 3, "@": 4, "*": 5, "%": 6, "|": 7, "**": 8, ">>": 9, "-": 10,
      "/": 11, "^": 12}
B310 = {"+": "BINARY_ADD", "-": "BINARY_SUBTRACT", "*": "BINARY_MULTIPLY", "/": "BINARY_TRUE_DIVIDE",
        "//": "BINARY_FLOOR_DIVIDE", "%": "BINARY_MODULO", "**": "BINARY_POWER", "<<": "BINARY_LSHIFT",
        ">>": "BINARY_RSHIFT", "&": "BINARY_AND", "|": "BINARY_OR", "^": "BINARY_XOR",
        "@": "BINARY_MATRIX_MULTIPLY"}
SNIPPETS = {}


def snippet(minors=(8, 9, 10, 11)):
    def deco(fn):
        fn.minors = minors
        SNIPPETS[fn.__name__] = fn
        return fn
    return deco


def _start(m, *vars_):
    a = Asm(m)
    a.const(None)
    for v in vars_:
        a.var(v)
    if m >= 11:
        a("RESUME", 0)
    return a


def binop(a, op):
    if a.minor >= 11:
        a("BINARY_OP", NB[op])
    else:
        a(B310[op])


def jf(a, lab):
    a("POP_JUMP_FORWARD_IF_FALSE" if a.minor >= 11 else "POP_JUMP_IF_FALSE", lab)


def jt(a, lab):
    a("POP_JUMP_FORWARD_IF_TRUE" if a.minor >= 11 else "POP_JUMP_IF_TRUE", lab)


def ret_none(a):
    a("LOAD_CONST", 0)
    a("RETURN_VALUE")


@snippet()
def ret_const(m):  # SPEC.md:188  64 01 53 00 -> return 1
    a = _start(m)
    a("LOAD_CONST", a.const(1))
    a("RETURN_VALUE")
    return a.build("f")


@snippet()
def precedence(m):
    a = _start(m, "a", "b", "c")
    for ops, order in ((("+", "*"), "ab+c*"), (("+", "+"), "ab+c+"), (("**", "**"), "abc**")):
        if order == "abc**":
            for v in "abc":
                a("LOAD_FAST", a.var(v))
            binop(a, "**")
            binop(a, "**")
        else:
            a("LOAD_FAST", 0); a("LOAD_FAST", 1); binop(a, ops[0]); a("LOAD_FAST", 2); binop(a, ops[1])
        a("STORE_FAST", a.var("x" + str(len(a.varnames))))
    a("LOAD_FAST", 0); a("UNARY_NEGATIVE"); a("LOAD_FAST", 1); binop(a, "**"); a("STORE_FAST", a.var("y"))
    a("LOAD_FAST", 0); a("LOAD_FAST", 1); a("UNARY_NEGATIVE"); binop(a, "-"); a("STORE_FAST", a.var("z"))
    a("LOAD_FAST", 0); a("LOAD_FAST", 1); a("LOAD_FAST", 2); binop(a, "-"); binop(a, "-"); a("RETURN_VALUE")
    return a.build("prec", argcount=3)


@snippet()
def constants(m):  # SPEC.md:465-467 and constant rendering corners
    a = _start(m, "x")
    vals = [10 ** 30, -0.0, 0.1, 1e16, 1e-05, 123.456, float("inf"), float("-inf"), float("nan"), 2.5j,
            complex(1.5, -2.0), complex(0.0, -2.0), complex(-0.0, 1.0), "it's", 'say "hi"', "both ' \"",
            "tab\tnl\n\x00\x7fé​\U0001F600", b"\x00'\xff", (1,), (), (1, "a", None),
            frozenset([1]), True, False, Ellipsis, -7, 2 ** 64 + 1, -(2 ** 100), 5e-324, 1.7976931348623157e308,
            0.30000000000000004, 100.0, 1e22, 123456789012345680.0]
    for v in vals:
        a("LOAD_CONST", a.const(v))
        a("STORE_FAST", 0)
    a("LOAD_CONST", a.const(7)); a("LOAD_ATTR", a.name("real")); a("RETURN_VALUE")
    return a.build("consts")


@snippet()
def ternary(m):  # SPEC.md:391  x = 1 if c else 2
    a = _start(m, "c", "x")
    e, j = L("else"), L("join")
    a("LOAD_FAST", 0); jf(a, e); a("LOAD_CONST", a.const(1)); a("JUMP_FORWARD", j)
    a.label(e); a("LOAD_CONST", a.const(2)); a.label(j); a("STORE_FAST", 1)
    a("LOAD_FAST", 1); a("RETURN_VALUE")
    return a.build("tern", argcount=1)


@snippet()
def underflow(m):  # SPEC.md:326  RETURN_VALUE on an empty stack
    a = _start(m)
    a("RETURN_VALUE")
    return a.build("f")


@snippet()
def odd_code(m):
    co = ret_const(m)
    return CodeObject(co.version, 0, 0, 0, 0, 1, 0x43, co.code + b"\x00", co.consts, (), (), (), (), "f", "<s>", 1)


@snippet(minors=(8, 9, 10))
def exctable_old(m):  # SPEC.md:63  exception table on <3.11
    co = ret_const(m)
    return CodeObject(co.version, 0, 0, 0, 0, 1, 0x43, co.code, co.consts, (), (), (), (), "f", "<s>", 1,
                      b"", b"\x80\x00\x00\x00")


@snippet()
def unknown_opcode(m):
    co = ret_const(m)
    return CodeObject(co.version, 0, 0, 0, 0, 1, 0x43, co.code[:2] + b"\xfe\x00" + co.code[2:], co.consts,
                      (), (), (), (), "f", "<s>", 1)


@snippet()
def bad_jump(m):  # SPEC.md:199  jump into the middle of an EXTENDED_ARG pair
    a = _start(m, "x")
    a("LOAD_FAST", 0)
    a("POP_JUMP_FORWARD_IF_FALSE" if m >= 11 else "POP_JUMP_IF_FALSE", 0)
    a("LOAD_CONST", 0)
    a("RETURN_VALUE")
    co = a.build("f", argcount=1)
    code = bytearray(co.code)
    # retarget the conditional jump into the middle of its own unit pair
    for i in range(0, len(code), 2):
        if code[i] in (114, 115):
            code[i + 1] = 3 if m == 10 else 7
    return CodeObject(co.version, 1, 0, 0, 1, 4, 0x43, bytes(code), co.consts, (), ("x",), (), (), "f", "<s>", 1)


@snippet()
def chained_compare(m):  # a < b < c  (DUP/ROT + JUMP_IF_FALSE_OR_POP)
    a = _start(m, "a", "b", "c")
    cl, end = L("cleanup"), L("end")
    a("LOAD_FAST", 0); a("LOAD_FAST", 1)
    if m >= 11:
        a("SWAP", 2); a("COPY", 2)
    else:
        a("DUP_TOP"); a("ROT_THREE")
    a("COMPARE_OP", 0)
    a("JUMP_IF_FALSE_OR_POP", cl)
    a("LOAD_FAST", 2); a("COMPARE_OP", 0); a("RETURN_VALUE")
    a.label(cl)
    if m >= 11:
        a("SWAP", 2)
    else:
        a("ROT_TWO")
    a("POP_TOP"); a("RETURN_VALUE")
    return a.build("chain", argcount=3)


@snippet()
def boolops(m):  # x = a and b or c ; return not (a == b)
    a = _start(m, "a", "b", "c", "x")
    l1, l2 = L("l1"), L("l2")
    a("LOAD_FAST", 0); a("JUMP_IF_FALSE_OR_POP", l1); a("LOAD_FAST", 1); a.label(l1)
    a("JUMP_IF_TRUE_OR_POP", l2); a("LOAD_FAST", 2); a.label(l2); a("STORE_FAST", 3)
    a("LOAD_FAST", 0); a("LOAD_FAST", 1); a("COMPARE_OP", 2); a("UNARY_NOT"); a("RETURN_VALUE")
    return a.build("bools", argcount=3)


@snippet()
def assert_stmt(m):
    a = _start(m, "x")
    ok = L("ok")
    a("LOAD_FAST", 0); jt(a, ok)
    if m >= 9:
        a("LOAD_ASSERTION_ERROR")
    else:
        a("LOAD_GLOBAL", a.name("AssertionError") << (1 if m >= 11 else 0))
    a("LOAD_CONST", a.const("bad x"))
    if m >= 11:
        a("PRECALL", 0); a("CALL", 0)
    else:
        a("CALL_FUNCTION", 1)
    a("RAISE_VARARGS", 1)
    a.label(ok); ret_none(a)
    return a.build("chk", argcount=1)


@snippet()
def unpack_swap(m):  # a, b = b, a ; x, (y, *z) = w
    a = _start(m, "a", "b", "w", "x", "y", "z")
    a("LOAD_FAST", 1); a("LOAD_FAST", 0)
    if m >= 11:
        a("SWAP", 2)
    else:
        a("ROT_TWO")
    a("STORE_FAST", 0); a("STORE_FAST", 1)
    a("LOAD_FAST", 2); a("UNPACK_SEQUENCE", 2); a("STORE_FAST", 3); a("UNPACK_EX", 1)
    a("STORE_FAST", 4); a("STORE_FAST", 5)
    ret_none(a)
    return a.build("swap", argcount=3)


@snippet()
def displays_calls(m):  # f(*a, k=1, **b); {'x': 1, **c}; [1, *d]; s[1:2, ::3]
    a = _start(m, "a", "b", "c", "d", "s")
    if m >= 11:
        a("LOAD_GLOBAL", (a.name("f") << 1) | 1)
    else:
        a("LOAD_GLOBAL", a.name("f"))
    a("LOAD_FAST", 0)
    if m >= 9:
        a("LOAD_CONST", a.const("k")); a("LOAD_CONST", a.const(1)); a("BUILD_MAP", 1)
        a("LOAD_FAST", 1); a("DICT_MERGE", 1)
    else:
        a("LOAD_CONST", a.const("k")); a("LOAD_CONST", a.const(1)); a("BUILD_MAP", 1)
        a("LOAD_FAST", 1); a("BUILD_MAP_UNPACK_WITH_CALL", 2)
    a("CALL_FUNCTION_EX", 1); a("POP_TOP")
    a("LOAD_CONST", a.const("x")); a("LOAD_CONST", a.const(1)); a("BUILD_MAP", 1)
    if m >= 9:
        a("LOAD_FAST", 2); a("DICT_UPDATE", 1)
    else:
        a("LOAD_FAST", 2); a("BUILD_MAP_UNPACK", 2)
    a("STORE_FAST", 1)
    if m >= 9:
        a("LOAD_CONST", a.const(1)); a("BUILD_LIST", 1); a("LOAD_FAST", 3); a("LIST_EXTEND", 1)
    else:
        a("LOAD_CONST", a.const(1)); a("BUILD_LIST", 1); a("LOAD_FAST", 3); a("BUILD_LIST_UNPACK", 2)
    a("STORE_FAST", 3)
    a("LOAD_FAST", 4); a("LOAD_CONST", a.const(1)); a("LOAD_CONST", a.const(2)); a("BUILD_SLICE", 2)
    a("LOAD_CONST", 0); a("LOAD_CONST", 0); a("LOAD_CONST", a.const(3)); a("BUILD_SLICE", 3)
    a("BUILD_TUPLE", 2); a("BINARY_SUBSCR"); a("RETURN_VALUE")
    return a.build("disp", argcount=5)


@snippet()
def fstring(m):  # f"{a!r:>{w}} and {b}{{x}}"
    a = _start(m, "a", "b", "w")
    a("LOAD_FAST", 0); a("LOAD_CONST", a.const(">")); a("LOAD_FAST", 2); a("FORMAT_VALUE", 0)
    a("BUILD_STRING", 2); a("FORMAT_VALUE", 2 | 4)
    a("LOAD_CONST", a.const(" and ")); a("LOAD_FAST", 1); a("FORMAT_VALUE", 0)
    a("LOAD_CONST", a.const("{x}'\"")); a("BUILD_STRING", 4); a("RETURN_VALUE")
    return a.build("fs", argcount=3)


@snippet(minors=(8, 9, 10))
def try_except_legacy(m):
    a = _start(m, "x")
    h, rr, end = L("h"), L("rr"), L("end")
    a("SETUP_FINALLY", h)
    a("LOAD_GLOBAL", a.name("g")); a("CALL_FUNCTION", 0); a("STORE_FAST", 0)
    a("POP_BLOCK"); a("JUMP_FORWARD", end)
    a.label(h); a("DUP_TOP"); a("LOAD_GLOBAL", a.name("ValueError"))
    if m >= 9:
        a("JUMP_IF_NOT_EXC_MATCH", rr)
    else:
        a("COMPARE_OP", 10); a("POP_JUMP_IF_FALSE", rr)
    a("POP_TOP"); a("POP_TOP"); a("POP_TOP")
    a("LOAD_CONST", a.const(0)); a("STORE_FAST", 0); a("POP_EXCEPT"); a("JUMP_FORWARD", end)
    a.label(rr)
    if m >= 9:
        a("RERAISE", 0) if m >= 10 else a("RERAISE")
    else:
        a("END_FINALLY")
    a.label(end); a("LOAD_FAST", 0); a("RETURN_VALUE")
    return a.build("tryx")


@snippet(minors=(10,))
def with_stmt(m):  # with open(p) as f: g(f)
    a = _start(m, "p", "f")
    h, end = L("h"), L("end")
    a("LOAD_GLOBAL", a.name("open")); a("LOAD_FAST", 0); a("CALL_FUNCTION", 1)
    a("SETUP_WITH", h); a("STORE_FAST", 1)
    a("LOAD_GLOBAL", a.name("g")); a("LOAD_FAST", 1); a("CALL_FUNCTION", 1); a("POP_TOP")
    a("POP_BLOCK"); a("LOAD_CONST", 0); a("DUP_TOP"); a("DUP_TOP"); a("CALL_FUNCTION", 3); a("POP_TOP")
    a("JUMP_FORWARD", end)
    a.label(h); a("WITH_EXCEPT_START"); a("POP_JUMP_IF_TRUE", L("sup")); a("RERAISE", 1)
    a.label("sup"); a("POP_TOP"); a("POP_TOP"); a("POP_TOP"); a("POP_EXCEPT"); a("POP_TOP")
    a.label(end); ret_none(a)
    return a.build("w", argcount=1)


@snippet(minors=(10,))
def nested_defs(m):  # module with def + lambda + listcomp + class
    comp = Asm(m)
    comp.var(".0"); comp.var("x")
    top, end = L("top"), L("end")
    comp("BUILD_LIST", 0); comp("LOAD_FAST", 0); comp.label(top); comp("FOR_ITER", end)
    comp("STORE_FAST", 1); comp("LOAD_FAST", 1); comp("LOAD_FAST", 1); comp("BINARY_MULTIPLY")
    comp("LIST_APPEND", 2); comp("JUMP_ABSOLUTE", top); comp.label(end); comp("RETURN_VALUE")
    comp_co = comp.build("<listcomp>", argcount=1, flags=0x13, qualname="f.<locals>.<listcomp>")
    lam = Asm(m)
    lam.var("p")
    lam("LOAD_FAST", 0); lam("LOAD_CONST", lam.const(1)); lam("BINARY_SUBSCR"); lam("RETURN_VALUE")
    lam_co = lam.build("<lambda>", argcount=1, flags=0x13)
    f = Asm(m)
    f.const("doc of f")
    f.var("xs"); f.var("k")
    f("LOAD_CONST", f.const(comp_co)); f("LOAD_CONST", f.const("f.<locals>.<listcomp>"))
    f("MAKE_FUNCTION", 0); f("LOAD_FAST", 0); f("GET_ITER"); f("CALL_FUNCTION", 1); f("STORE_FAST", 1)
    f("LOAD_GLOBAL", f.name("sorted")); f("LOAD_FAST", 1)
    f("LOAD_CONST", f.const(lam_co)); f("LOAD_CONST", f.const("f.<locals>.<lambda>")); f("MAKE_FUNCTION", 0)
    f("LOAD_CONST", f.const(("key",))); f("CALL_FUNCTION_KW", 2); f("RETURN_VALUE")
    f_co = f.build("f", argcount=1)
    mod = Asm(m)
    mod.const("module doc")
    mod("LOAD_CONST", 0); mod("STORE_NAME", mod.name("__doc__"))
    mod("LOAD_CONST", mod.const(0)); mod("LOAD_CONST", mod.const(None)); mod("IMPORT_NAME", mod.name("os"))
    mod("STORE_NAME", mod.name("os"))
    mod("LOAD_CONST", mod.const(f_co)); mod("LOAD_CONST", mod.const("f")); mod("MAKE_FUNCTION", 0)
    mod("STORE_NAME", mod.name("f")); mod("LOAD_CONST", mod.const(None)); mod("RETURN_VALUE")
    return mod.build("<module>", flags=0x40)
