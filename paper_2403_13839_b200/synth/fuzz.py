"""Random structured programs for parity fuzzing (3.8-3.11).

`program(seed, minor)` assembles a function whose body is a random tree of
statements and expressions laid out the way CPython's compiler lays them out
for that version (rotated loops on 3.10+, legacy SETUP_FINALLY regions on
<=3.10, exception tables on 3.11, PRECALL/CALL/KW_NAMES on 3.11, ...), with
nested code objects (lambda, list/set/dict comprehensions, generator
expressions).  `mode="mutant"` flips a few bytes of such a program so the
decoder / simulator error paths (and the device code's robustness on
malformed input) are exercised too.
"""
from __future__ import annotations

from .asm import Asm, L
from .corpus import Rng, splitmix64

CONSTS = [0, 1, 2, -1, 7, 255, 256, 10 ** 20, -(2 ** 70), 0.5, -0.0, 1e-07, 1e16, 3.14159, float("inf"),
          1j, complex(2, -3), "s", "it's", 'q"d', "a\nb\t\\", "üñï", "​", b"", b"\x01'\"", None, True,
          False, (1, 2), ("x",), (), frozenset(), frozenset([2]), Ellipsis]
LOCALS = ["a", "b", "c", "d", "e", "f", "g", "h"]
GLOBALS = ["print", "len", "obj", "mod", "fn", "data", "Exc"]
ATTRS = ["x", "y", "real", "items", "append", "value", "keys"]
BINOPS = ["+", "-", "*", "/", "//", "%", "**", "<<", ">>", "&", "|", "^", "@"]
NB = {"+": 0, "&": 1, "//": 2, "<<": 3, "@": 4, "*": 5, "%": 6, "|": 7, "**": 8, ">>": 9, "-": 10, "/": 11,
      "^": 12}
B310 = {"+": "ADD", "-": "SUBTRACT", "*": "MULTIPLY", "/": "TRUE_DIVIDE", "//": "FLOOR_DIVIDE", "%": "MODULO",
        "**": "POWER", "<<": "LSHIFT", ">>": "RSHIFT", "&": "AND", "|": "OR", "^": "XOR", "@": "MATRIX_MULTIPLY"}


class Fuzz:
    def __init__(self, seed, minor, name="f", depth_limit=4, size=40, comp_kind=None):
        self.r = Rng(splitmix64(0xF022 ^ (seed * 1000003 + minor)))
        self.m = minor
        self.a = Asm(minor)
        self.a.const(None)
        self.name = name
        self.depth_limit = depth_limit
        self.budget = size
        self.loops = []      # stack of (continue_label, break_label, in_try)
        self.seed = seed
        self.nested = 0
        for v in LOCALS[:2 + self.r.below(len(LOCALS) - 2)]:
            self.a.var(v)
        if minor >= 11:
            self.a("RESUME", 0)

    # ------------------------------------------------------------ helpers
    def op(self, name, arg=None):
        self.a(name, arg)

    def chance(self, p):
        return self.r.below(1000) < p * 1000

    def jf(self, lab):
        self.op("POP_JUMP_FORWARD_IF_FALSE" if self.m >= 11 else "POP_JUMP_IF_FALSE", lab)

    def jt(self, lab):
        self.op("POP_JUMP_FORWARD_IF_TRUE" if self.m >= 11 else "POP_JUMP_IF_TRUE", lab)

    def jback(self, lab):
        self.op("JUMP_BACKWARD" if self.m >= 11 else "JUMP_ABSOLUTE", lab)

    def local(self):
        return self.r.below(len(self.a.varnames))

    def load_global(self, name, null=False):
        i = self.a.name(name)
        if self.m >= 11:
            self.op("LOAD_GLOBAL", (i << 1) | (1 if null else 0))
        else:
            self.op("LOAD_GLOBAL", i)

    def binop(self, sym, inplace=False):
        if self.m >= 11:
            self.op("BINARY_OP", NB[sym] + (13 if inplace else 0))
        else:
            self.op(("INPLACE_" if inplace else "BINARY_") + B310[sym])

    def dup(self):
        self.op("COPY", 1) if self.m >= 11 else self.op("DUP_TOP")

    def rot2(self):
        self.op("SWAP", 2) if self.m >= 11 else self.op("ROT_TWO")

    def call(self, nargs, kwnames=(), method=False):
        """Stack: [callable-prefix] args... -> call.  Caller pushed the callable."""
        if self.m >= 11:
            if kwnames:
                self.op("KW_NAMES", self.a.const(tuple(kwnames)))
            self.op("PRECALL", nargs)
            self.op("CALL", nargs)
        elif method:
            self.op("CALL_METHOD", nargs)
        elif kwnames:
            self.op("LOAD_CONST", self.a.const(tuple(kwnames)))
            self.op("CALL_FUNCTION_KW", nargs)
        else:
            self.op("CALL_FUNCTION", nargs)

    # ------------------------------------------------------------ expressions
    def expr(self, d=0):
        r = self.r
        if d >= 3 or self.chance(0.3):
            k = r.below(10)
            if k < 5:
                self.op("LOAD_FAST", self.local())
            elif k < 8:
                self.op("LOAD_CONST", self.a.const(r.choice(CONSTS)))
            else:
                self.load_global(r.choice(GLOBALS))
            return
        k = r.below(17)
        if k == 0:
            self.expr(d + 1)
            self.expr(d + 1)
            self.binop(r.choice(BINOPS))
        elif k == 1:
            self.expr(d + 1)
            self.op(r.choice(["UNARY_NEGATIVE", "UNARY_POSITIVE", "UNARY_INVERT", "UNARY_NOT"]))
        elif k == 2:
            self.expr(d + 1)
            self.expr(d + 1)
            c = r.below(10)
            if c < 6:
                self.op("COMPARE_OP", c)
            elif self.m == 8:
                self.op("COMPARE_OP", c)
            else:
                self.op("IS_OP" if c >= 8 else "CONTAINS_OP", r.below(2))
        elif k == 3:
            self.expr(d + 1)
            self.op("LOAD_ATTR", self.a.name(r.choice(ATTRS)))
        elif k == 4:
            self.expr(d + 1)
            self.expr(d + 1)
            self.op("BINARY_SUBSCR")
        elif k == 5:  # slice subscript
            self.expr(d + 1)
            n = 2 + r.below(2)
            for _ in range(n):
                if self.chance(0.3):
                    self.op("LOAD_CONST", 0)
                else:
                    self.expr(d + 2)
            self.op("BUILD_SLICE", n)
            self.op("BINARY_SUBSCR")
        elif k in (6, 7):  # call of a global / of an expression
            name = r.choice(GLOBALS)
            self.load_global(name, null=True)
            n = r.below(4)
            for _ in range(n):
                self.expr(d + 1)
            kw = ()
            if n and self.chance(0.3):
                kw = tuple(r.choice(["key", "default", "sep"]) + str(i) for i in range(1 + r.below(n)))
            self.call(n, kw)
        elif k == 8:  # method call
            self.expr(d + 1)
            self.op("LOAD_METHOD", self.a.name(r.choice(ATTRS)))
            n = r.below(3)
            for _ in range(n):
                self.expr(d + 1)
            self.call(n, method=True)
        elif k == 9:  # displays
            n = r.below(4)
            for _ in range(n):
                self.expr(d + 1)
            self.op(r.choice(["BUILD_TUPLE", "BUILD_LIST", "BUILD_SET"]), n)
        elif k == 10:  # dict
            n = r.below(3)
            if n and self.chance(0.5):
                for _ in range(n):
                    self.expr(d + 1)
                self.op("LOAD_CONST", self.a.const(tuple(f"k{i}" for i in range(n))))
                self.op("BUILD_CONST_KEY_MAP", n)
            else:
                for _ in range(n):
                    self.expr(d + 1)
                    self.expr(d + 1)
                self.op("BUILD_MAP", n)
        elif k == 11:  # ternary
            e, j = self.a.fresh("te"), self.a.fresh("tj")
            self.expr(d + 1)
            self.jf(e)
            self.expr(d + 1)
            self.op("JUMP_FORWARD", j)
            self.a.label(e)
            self.expr(d + 1)
            self.a.label(j)
        elif k == 12:  # and / or
            j = self.a.fresh("bj")
            self.expr(d + 1)
            self.op(r.choice(["JUMP_IF_FALSE_OR_POP", "JUMP_IF_TRUE_OR_POP"]), j)
            self.expr(d + 1)
            self.a.label(j)
        elif k == 13:  # f-string
            n = 1 + r.below(3)
            for _ in range(n):
                if self.chance(0.4):
                    self.op("LOAD_CONST", self.a.const(r.choice(["x=", " {b} ", "'", '"', "é"])))
                else:
                    self.expr(d + 1)
                    flags = r.below(4)
                    if self.chance(0.2):
                        self.op("LOAD_CONST", self.a.const(r.choice([">10", ".3f", "x"])))
                        flags |= 4
                    self.op("FORMAT_VALUE", flags)
            self.op("BUILD_STRING", n)
        elif k == 14 and self.nested < 2:
            self.lambda_expr(d)
        elif k == 15 and self.nested < 2:
            self.comprehension(d)
        else:
            self.op("LOAD_FAST", self.local())

    def nested_code(self, name, build):
        sub = Fuzz(self.seed * 31 + self.nested + 7, self.m, name)
        sub.nested = self.nested + 1
        sub.a = Asm(self.m)
        return sub

    def lambda_expr(self, d):
        sub = Fuzz(self.seed * 131 + len(self.a.items), self.m, "<lambda>")
        sub.nested = self.nested + 1
        sub.a = Asm(self.m)
        for v in ("p", "q")[:1 + self.r.below(2)]:
            sub.a.var(v)
        if self.m >= 11:
            sub.a("RESUME", 0)
        sub.expr(1)
        sub.op("RETURN_VALUE")
        co = sub.a.build("<lambda>", argcount=len(sub.a.varnames), flags=0x13,
                         qualname=f"{self.name}.<locals>.<lambda>")
        ndef = self.r.below(2) if len(sub.a.varnames) else 0
        if ndef:
            self.op("LOAD_CONST", self.a.const((1,)))
        self.op("LOAD_CONST", self.a.const(co))
        if self.m <= 10:
            self.op("LOAD_CONST", self.a.const(f"{self.name}.<locals>.<lambda>"))
        self.op("MAKE_FUNCTION", 1 if ndef else 0)

    def comprehension(self, d):
        kind = self.r.choice(["<listcomp>", "<setcomp>", "<dictcomp>", "<genexpr>"])
        sub = Fuzz(self.seed * 137 + len(self.a.items), self.m, kind)
        sub.nested = self.nested + 1
        sub.a = Asm(self.m)
        sub.a.var(".0")
        sub.a.var("x")
        a = sub.a
        gen = kind == "<genexpr>"
        if self.m >= 11:
            if gen:
                a("RETURN_GENERATOR")
                a("POP_TOP")
            a("RESUME", 0)
        if not gen:
            a({"<listcomp>": "BUILD_LIST", "<setcomp>": "BUILD_SET", "<dictcomp>": "BUILD_MAP"}[kind], 0)
        elif self.m == 10:
            a("GEN_START", 0)
        top, end = L("ct"), L("ce")
        a("LOAD_FAST", 0)
        a.label(top)
        a("FOR_ITER", end)
        a("STORE_FAST", 1)
        if sub.chance(0.5):
            sub.expr(2)
            sub.jf(top) if sub.m < 11 else a("POP_JUMP_BACKWARD_IF_FALSE", top)
        if kind == "<dictcomp>":
            sub.expr(2)
            sub.expr(2)
            a("MAP_ADD", 2)
        else:
            sub.expr(2)
            if gen:
                a("YIELD_VALUE")
                if self.m >= 11:
                    a("RESUME", 1)
                a("POP_TOP")
            else:
                a("LIST_APPEND" if kind == "<listcomp>" else "SET_ADD", 2)
        sub.jback(top)
        a.label(end)
        if gen:
            a("LOAD_CONST", a.const(None))
        a("RETURN_VALUE")
        co = a.build(kind, argcount=1, flags=0x33 if gen else 0x13, qualname=f"{self.name}.<locals>.{kind}")
        self.op("LOAD_CONST", self.a.const(co))
        if self.m <= 10:
            self.op("LOAD_CONST", self.a.const(f"{self.name}.<locals>.{kind}"))
        self.op("MAKE_FUNCTION", 0)
        self.expr(d + 1)
        self.op("GET_ITER")
        self.call(1) if self.m <= 10 else (self.op("PRECALL", 0), self.op("CALL", 0))

    # ------------------------------------------------------------ statements
    def block(self, depth, n):
        for _ in range(n):
            if self.budget <= 0:
                break
            self.stmt(depth)

    def stmt(self, depth):
        r = self.r
        self.budget -= 1
        k = r.below(24) if depth < self.depth_limit else r.below(8)
        if k <= 2:  # assignment to a local
            self.expr()
            self.op("STORE_FAST", self.local())
        elif k == 3:  # attribute / subscript store
            self.expr()
            self.expr(2)
            if self.chance(0.5):
                self.op("STORE_ATTR", self.a.name(r.choice(ATTRS)))
            else:
                self.expr(2)
                self.op("STORE_SUBSCR")
        elif k == 4:  # augmented assignment
            t = self.local()
            self.op("LOAD_FAST", t)
            self.expr(1)
            self.binop(r.choice(BINOPS), inplace=True)
            self.op("STORE_FAST", t)
        elif k == 5:  # expression statement
            self.expr()
            self.op("POP_TOP")
        elif k == 6:  # chained assignment / swap / unpack
            c = r.below(3)
            if c == 0:
                self.expr()
                self.dup()
                self.op("STORE_FAST", self.local())
                self.op("STORE_FAST", self.local())
            elif c == 1:
                x, y = self.local(), self.local()
                self.op("LOAD_FAST", y)
                self.op("LOAD_FAST", x)
                self.rot2()
                self.op("STORE_FAST", x)
                self.op("STORE_FAST", y)
            else:
                self.expr()
                n = 2 + r.below(2)
                self.op("UNPACK_SEQUENCE", n)
                for _ in range(n):
                    self.op("STORE_FAST", self.local())
        elif k == 7:  # global store / del / import
            c = r.below(3)
            if c == 0:
                self.expr()
                self.op("STORE_GLOBAL", self.a.name(r.choice(GLOBALS)))
            elif c == 1:
                self.op("DELETE_FAST", self.local())
            else:
                self.op("LOAD_CONST", self.a.const(0))
                if self.chance(0.5):
                    self.op("LOAD_CONST", self.a.const(None))
                    self.op("IMPORT_NAME", self.a.name(r.choice(["os", "os.path", "json"])))
                    self.op("STORE_FAST", self.local())
                else:
                    names = tuple(r.choice(["join", "dumps", "sep"]) for _ in range(1 + r.below(2)))
                    self.op("LOAD_CONST", self.a.const(names))
                    self.op("IMPORT_NAME", self.a.name(r.choice(["os", "json"])))
                    for nm in names:
                        self.op("IMPORT_FROM", self.a.name(nm))
                        self.op("STORE_FAST", self.local())
                    self.op("POP_TOP")
        elif k in (8, 9):  # if / if-else / elif
            els, end = self.a.fresh("e"), self.a.fresh("x")
            self.expr(1)
            self.jf(els)
            self.block(depth + 1, 1 + r.below(3))
            if self.chance(0.5):
                self.op("JUMP_FORWARD", end)
                self.a.label(els)
                self.block(depth + 1, 1 + r.below(3))
                self.a.label(end)
            else:
                self.a.label(els)
        elif k in (10, 11):  # while
            self.while_loop(depth)
        elif k in (12, 13):  # for
            self.for_loop(depth)
        elif k == 14 and self.loops and not self.loops[-1][2]:  # break / continue
            cont, brk, _ = self.loops[-1]
            if self.chance(0.5):
                self.op("JUMP_FORWARD" if self.m >= 11 else "JUMP_ABSOLUTE", brk)
            elif self.m >= 11:
                placed = any(x == cont for x in self.a.items if isinstance(x, str))
                self.op("JUMP_BACKWARD" if placed else "JUMP_FORWARD", cont)
            else:
                self.op("JUMP_ABSOLUTE", cont)
            self.a.label(self.a.fresh("dead"))
        elif k == 15:  # assert
            ok = self.a.fresh("ok")
            self.expr(1)
            self.jt(ok)
            if self.m >= 9:
                self.op("LOAD_ASSERTION_ERROR")
            else:
                self.load_global("AssertionError")
            if self.chance(0.5):
                self.op("LOAD_CONST", self.a.const("message"))
                self.call(0) if self.m >= 11 else self.op("CALL_FUNCTION", 1)
            self.op("RAISE_VARARGS", 1)
            self.a.label(ok)
        elif k in (16, 17) and not self.loops:
            self.try_stmt(depth)
        elif k == 18 and self.m in (9, 10) and not self.loops:
            self.with_stmt(depth)
        elif k == 19:  # return inside a branch
            e = self.a.fresh("r")
            self.expr(1)
            self.jf(e)
            self.expr(1)
            self.op("RETURN_VALUE")
            self.a.label(e)
        else:
            self.expr()
            self.op("STORE_FAST", self.local())

    def while_loop(self, depth):
        a = self.a
        top, end, test = a.fresh("wt"), a.fresh("we"), a.fresh("wc")
        if self.m <= 9:
            a.label(top)
            self.expr(1)
            self.jf(end)
            self.loops.append((top, end, False))
            self.block(depth + 1, 1 + self.r.below(3))
            self.loops.pop()
            self.op("JUMP_ABSOLUTE", top)
            a.label(end)
            return
        self.expr(1)
        self.jf(end)
        a.label(top)
        self.loops.append((test, end, False))
        self.block(depth + 1, 1 + self.r.below(3))
        self.loops.pop()
        a.label(test)
        self.expr(1)
        if self.m >= 11:
            self.op("POP_JUMP_BACKWARD_IF_TRUE", top)
        else:
            self.op("POP_JUMP_IF_TRUE", top)
        a.label(end)

    def for_loop(self, depth):
        a = self.a
        top, end = a.fresh("ft"), a.fresh("fe")
        self.expr(1)
        self.op("GET_ITER")
        a.label(top)
        self.op("FOR_ITER", end)
        self.op("STORE_FAST", self.local())
        self.loops.append((top, end, False))
        self.block(depth + 1, 1 + self.r.below(3))
        self.loops.pop()
        self.jback(top)
        a.label(end)
        if self.chance(0.2):  # for-else body
            self.block(depth + 1, 1)

    def try_stmt(self, depth):
        if self.m >= 11:
            return self.try311(depth)
        a = self.a
        h, rr, end = a.fresh("h"), a.fresh("rr"), a.fresh("te")
        finally_ = self.chance(0.3)
        if finally_ and self.m >= 9:
            fin = a.fresh("fin")
            self.op("SETUP_FINALLY", fin)
            self.block(depth + 1, 1 + self.r.below(2))
            self.op("POP_BLOCK")
            # straight-line finally body, emitted twice (normal + exceptional path)
            mark = len(a.items)
            for _ in range(1 + self.r.below(2)):
                self.expr(3)
                self.op("STORE_FAST", self.local())
            copy = a.items[mark:]
            self.op("JUMP_FORWARD", end)
            a.label(fin)
            a.items.extend(copy)
            self.op("RERAISE", 0) if self.m >= 10 else self.op("RERAISE")
            a.label(end)
            return
        self.op("SETUP_FINALLY", h)
        self.block(depth + 1, 1 + self.r.below(3))
        self.op("POP_BLOCK")
        self.op("JUMP_FORWARD", end)
        a.label(h)
        if self.chance(0.3):  # bare except
            self.op("POP_TOP")
            self.op("POP_TOP")
            self.op("POP_TOP")
            self.block(depth + 1, 1)
            self.op("POP_EXCEPT")
            self.op("JUMP_FORWARD", end)
            if self.m == 8:
                self.op("END_FINALLY")
        else:
            self.op("DUP_TOP")
            self.load_global(self.r.choice(["ValueError", "KeyError", "Exc"]))
            if self.m >= 9:
                self.op("JUMP_IF_NOT_EXC_MATCH", rr)
            else:
                self.op("COMPARE_OP", 10)
                self.op("POP_JUMP_IF_FALSE", rr)
            self.op("POP_TOP")
            if self.chance(0.3):
                self.op("STORE_FAST", self.local())
            else:
                self.op("POP_TOP")
            self.op("POP_TOP")
            self.block(depth + 1, 1 + self.r.below(2))
            self.op("POP_EXCEPT")
            self.op("JUMP_FORWARD", end)
            a.label(rr)
            if self.m >= 10:
                self.op("RERAISE", 0)
            elif self.m == 9:
                self.op("RERAISE")
            else:
                self.op("END_FINALLY")
        a.label(end)

    def try311(self, depth):
        a = self.a
        s, e, h, cl, end, rr = (a.fresh("t") for _ in range(6))
        self.op("NOP")
        a.label(s)
        self.budget -= 3
        for _ in range(1 + self.r.below(3)):
            self.expr(1)
            self.op("STORE_FAST", self.local())
        a.label(e)
        self.op("JUMP_FORWARD", end)
        a.label(h)
        self.op("PUSH_EXC_INFO")
        self.load_global(self.r.choice(["ValueError", "KeyError"]))
        self.op("CHECK_EXC_MATCH")
        self.op("POP_JUMP_FORWARD_IF_FALSE", rr)
        self.op("POP_TOP")
        for _ in range(1 + self.r.below(2)):
            self.expr(1)
            self.op("STORE_FAST", self.local())
        self.op("POP_EXCEPT")
        self.op("JUMP_FORWARD", end)
        a.label(rr)
        self.op("RERAISE", 0)
        a.label(cl)
        self.op("COPY", 3)
        self.op("POP_EXCEPT")
        self.op("RERAISE", 1)
        a.label(end)
        a.exc.append((s, e, h, 0, False))
        a.exc.append((h, cl, cl, 1, True))

    def with_stmt(self, depth):
        a = self.a
        h, end, sup = a.fresh("wh"), a.fresh("wx"), a.fresh("ws")
        self.expr(1)
        self.op("SETUP_WITH", h)
        if self.chance(0.6):
            self.op("STORE_FAST", self.local())
        else:
            self.op("POP_TOP")
        self.block(depth + 1, 1 + self.r.below(2))
        self.op("POP_BLOCK")
        self.op("LOAD_CONST", 0)
        self.op("DUP_TOP")
        self.op("DUP_TOP")
        self.op("CALL_FUNCTION", 3)
        self.op("POP_TOP")
        self.op("JUMP_FORWARD", end)
        a.label(h)
        self.op("WITH_EXCEPT_START")
        self.op("POP_JUMP_IF_TRUE", sup)
        self.op("RERAISE", 1) if self.m >= 10 else self.op("RERAISE")
        a.label(sup)
        for _ in range(3):
            self.op("POP_TOP")
        self.op("POP_EXCEPT")
        self.op("POP_TOP")
        a.label(end)

    def finish(self, argcount):
        if self.chance(0.7):
            self.op("LOAD_CONST", 0)
        else:
            self.expr(1)
        self.op("RETURN_VALUE")
        return self.a.build(self.name, argcount=min(argcount, len(self.a.varnames)), stacksize=64)


def program(seed, minor=10, size=30, mode="valid"):
    fz = Fuzz(seed, minor, size=size)
    fz.block(0, size)
    co = fz.finish(fz.r.below(3))
    if mode == "mutant":
        co = mutate(co, Rng(splitmix64(0xBAD ^ seed)))
    return co


def mutate(co, r):
    from ..model import CodeObject

    code = bytearray(co.code)
    for _ in range(1 + r.below(3)):
        i = r.below(len(code))
        code[i] = r.below(256) if r.below(2) else (code[i] ^ (1 << r.below(8)))
    if r.below(10) == 0 and len(code) > 4:
        code = code[:len(code) - 2 * (1 + r.below(2))]
    return CodeObject(co.version, co.argcount, co.posonlyargcount, co.kwonlyargcount, co.nlocals,
                      co.stacksize, co.flags, bytes(code), co.consts, co.names, co.varnames, co.freevars,
                      co.cellvars, co.name, co.filename, co.firstlineno, co.linetable, co.exceptiontable,
                      co.qualname)
