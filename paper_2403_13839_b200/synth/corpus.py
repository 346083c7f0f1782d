"""Synthetic corpora named by BASELINE.json's configs.

  C1  fig1(minor)           the paper's Figure-1 function, its Dynamo-transformed
                            code and the two resume functions
  C3  c3(seed, minor)       ~200-unit straight-line objects: 33 statements drawn from
                            {x = a + b * K, x = g(a, b.attr), x = a.m(b)[c], a.attr = b - c}
  C4  c4(seed, minor, n)    long functions (~n units) of nested if / if-else / for /
                            rotated while / try-except NameError, EXTENDED_ARG jumps

Seeds are splitmix64-derived so a (config, index) pair always yields the same
object; the benchmark tiles a pool of distinct objects (see bench.py).
"""
from __future__ import annotations

from .asm import Asm, L

MASK64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class Rng:
    def __init__(self, seed):
        self.s = seed & MASK64

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        return splitmix64(self.s)

    def below(self, n):
        return self.next() % n

    def choice(self, seq):
        return seq[self.below(len(seq))]


# ----------------------------------------------------------------- C1

def _toy_body(a, minor, lv):
    """x = a / (torch.abs(a) + 1); if b.sum() < 0: b = b * -1; return x * b"""
    c1, c0, cm1 = a.const(1), a.const(0), a.const(-1)
    if minor >= 11:
        a("LOAD_FAST", lv["a"]); a("LOAD_GLOBAL", a.name("torch") << 1); a("LOAD_METHOD", a.name("abs"))
        a("LOAD_FAST", lv["a"]); a("PRECALL", 1); a("CALL", 1); a("LOAD_CONST", c1); a("BINARY_OP", 0)
        a("BINARY_OP", 11); a("STORE_FAST", lv["x"])
        a("LOAD_FAST", lv["b"]); a("LOAD_METHOD", a.name("sum")); a("PRECALL", 0); a("CALL", 0)
        a("LOAD_CONST", c0); a("COMPARE_OP", 0); a("POP_JUMP_FORWARD_IF_FALSE", L("skip"))
        a("LOAD_FAST", lv["b"]); a("LOAD_CONST", cm1); a("BINARY_OP", 5); a("STORE_FAST", lv["b"])
        a.label("skip"); a("LOAD_FAST", lv["x"]); a("LOAD_FAST", lv["b"]); a("BINARY_OP", 5); a("RETURN_VALUE")
        return
    a("LOAD_FAST", lv["a"]); a("LOAD_GLOBAL", a.name("torch")); a("LOAD_METHOD", a.name("abs"))
    a("LOAD_FAST", lv["a"]); a("CALL_METHOD", 1); a("LOAD_CONST", c1); a("BINARY_ADD")
    a("BINARY_TRUE_DIVIDE"); a("STORE_FAST", lv["x"])
    a("LOAD_FAST", lv["b"]); a("LOAD_METHOD", a.name("sum")); a("CALL_METHOD", 0)
    a("LOAD_CONST", c0); a("COMPARE_OP", 0); a("POP_JUMP_IF_FALSE", L("skip"))
    a("LOAD_FAST", lv["b"]); a("LOAD_CONST", cm1); a("BINARY_MULTIPLY"); a("STORE_FAST", lv["b"])
    a.label("skip"); a("LOAD_FAST", lv["x"]); a("LOAD_FAST", lv["b"]); a("BINARY_MULTIPLY"); a("RETURN_VALUE")


def fig1(minor=10):
    """The four Figure-1 code objects (toy, transformed, two resume functions)."""
    out = []
    a = Asm(minor)
    a.const(None)
    lv = {n: a.var(n) for n in ("a", "b", "x")}
    if minor >= 11:
        a("RESUME", 0)
    _toy_body(a, minor, lv)
    out.append(a.build("toy_example", argcount=2))

    t = Asm(minor)
    t.const(None)
    for n in ("a", "b", "x", "__temp_1"):
        t.var(n)
    c0, c1 = t.const(0), t.const(1)
    if minor >= 11:
        t("RESUME", 0)
        t("LOAD_GLOBAL", (t.name("__compiled_fn_0") << 1) | 1)
        t("LOAD_FAST", 0); t("LOAD_FAST", 1); t("PRECALL", 2); t("CALL", 2)
    else:
        t("LOAD_GLOBAL", t.name("__compiled_fn_0")); t("LOAD_FAST", 0); t("LOAD_FAST", 1)
        t("CALL_FUNCTION", 2)
    t("STORE_FAST", 3)
    t("LOAD_FAST", 3); t("LOAD_CONST", c0); t("BINARY_SUBSCR"); t("STORE_FAST", 2)
    t("LOAD_FAST", 3); t("LOAD_CONST", c1); t("BINARY_SUBSCR")
    t("POP_JUMP_FORWARD_IF_FALSE" if minor >= 11 else "POP_JUMP_IF_FALSE", L("other"))
    for target, lab in (("__resume_at_30_1", None), ("__resume_at_38_2", "other")):
        if lab:
            t.label(lab)
        if minor >= 11:
            t("LOAD_GLOBAL", (t.name(target) << 1) | 1); t("LOAD_FAST", 1); t("LOAD_FAST", 2)
            t("PRECALL", 2); t("CALL", 2)
        else:
            t("LOAD_GLOBAL", t.name(target)); t("LOAD_FAST", 1); t("LOAD_FAST", 2); t("CALL_FUNCTION", 2)
        t("RETURN_VALUE")
    out.append(t.build("__transformed_code_0_for_toy_example", argcount=2))

    for rname, resume_at in (("__resume_at_30_1", "body"), ("__resume_at_38_2", "skip")):
        r = Asm(minor)
        r.const(None)
        rv = {n: r.var(n) for n in ("b", "x", "a")}
        if minor >= 11:
            r("RESUME", 0)
            r("JUMP_FORWARD", L(resume_at))
        else:
            r("JUMP_ABSOLUTE", L(resume_at))
        # the original body copy; the resume label marks the continuation point
        c1_, c0_, cm1 = r.const(1), r.const(0), r.const(-1)
        r("LOAD_FAST", rv["a"]); r("LOAD_GLOBAL", r.name("torch") << (1 if minor >= 11 else 0))
        r("LOAD_METHOD", r.name("abs")); r("LOAD_FAST", rv["a"])
        if minor >= 11:
            r("PRECALL", 1); r("CALL", 1); r("LOAD_CONST", c1_); r("BINARY_OP", 0); r("BINARY_OP", 11)
        else:
            r("CALL_METHOD", 1); r("LOAD_CONST", c1_); r("BINARY_ADD"); r("BINARY_TRUE_DIVIDE")
        r("STORE_FAST", rv["x"])
        r("LOAD_FAST", rv["b"]); r("LOAD_METHOD", r.name("sum"))
        if minor >= 11:
            r("PRECALL", 0); r("CALL", 0)
        else:
            r("CALL_METHOD", 0)
        r("LOAD_CONST", c0_); r("COMPARE_OP", 0)
        r("POP_JUMP_FORWARD_IF_FALSE" if minor >= 11 else "POP_JUMP_IF_FALSE", L("skip"))
        r.label("body")
        r("LOAD_FAST", rv["b"]); r("LOAD_CONST", cm1)
        r("BINARY_OP", 5) if minor >= 11 else r("BINARY_MULTIPLY")
        r("STORE_FAST", rv["b"])
        r.label("skip")
        r("LOAD_FAST", rv["x"]); r("LOAD_FAST", rv["b"])
        r("BINARY_OP", 5) if minor >= 11 else r("BINARY_MULTIPLY")
        r("RETURN_VALUE")
        out.append(r.build(rname, argcount=2))
    return out


# ----------------------------------------------------------------- C3 / C4 statements

_LOCALS = ("a", "b", "c", "d", "e", "f")
_NAMES = ("g", "h", "attr", "m", "n", "k")


class _Gen:
    def __init__(self, minor, rng):
        self.a = Asm(minor)
        self.minor = minor
        self.r = rng
        self.a.const(None)
        for n in _LOCALS:
            self.a.var(n)
        for n in _NAMES:
            self.a.name(n)
        if minor >= 11:
            self.a("RESUME", 0)

    def lv(self):
        return self.r.below(len(_LOCALS))

    def nm(self):
        return self.r.below(len(_NAMES))

    def binop(self, v310, nb):
        if self.minor >= 11:
            self.a("BINARY_OP", nb)
        else:
            self.a(v310)

    def simple(self):
        a, r = self.a, self.r
        t = r.below(4)
        if t == 0:  # x = a + b * K
            a("LOAD_FAST", self.lv()); a("LOAD_FAST", self.lv()); a("LOAD_CONST", a.const(1 + r.below(3)))
            self.binop("BINARY_MULTIPLY", 5); self.binop("BINARY_ADD", 0); a("STORE_FAST", self.lv())
        elif t == 1:  # x = g(a, b.attr)
            if self.minor >= 11:
                a("LOAD_GLOBAL", (self.nm() << 1) | 1)
            else:
                a("LOAD_GLOBAL", self.nm())
            a("LOAD_FAST", self.lv()); a("LOAD_FAST", self.lv()); a("LOAD_ATTR", self.nm())
            if self.minor >= 11:
                a("PRECALL", 2); a("CALL", 2)
            else:
                a("CALL_FUNCTION", 2)
            a("STORE_FAST", self.lv())
        elif t == 2:  # x = a.m(b)[c]
            a("LOAD_FAST", self.lv()); a("LOAD_METHOD", self.nm()); a("LOAD_FAST", self.lv())
            if self.minor >= 11:
                a("PRECALL", 1); a("CALL", 1)
            else:
                a("CALL_METHOD", 1)
            a("LOAD_FAST", self.lv()); a("BINARY_SUBSCR"); a("STORE_FAST", self.lv())
        else:  # a.attr = b - c
            a("LOAD_FAST", self.lv()); a("LOAD_FAST", self.lv()); self.binop("BINARY_SUBTRACT", 10)
            a("LOAD_FAST", self.lv()); a("STORE_ATTR", self.nm())

    def cond(self):
        a = self.a
        a("LOAD_FAST", self.lv()); a("LOAD_FAST", self.lv()); a("COMPARE_OP", self.r.below(6))

    def jf(self, label):  # pop-jump-if-false forward
        self.a("POP_JUMP_FORWARD_IF_FALSE" if self.minor >= 11 else "POP_JUMP_IF_FALSE", label)

    def finish(self):
        self.a("LOAD_CONST", 0); self.a("RETURN_VALUE")

    def units(self):
        return len(self.a.items)


def c3(seed, minor=10, n_stmts=33):
    g = _Gen(minor, Rng(splitmix64(0xC3 ^ seed)))
    for _ in range(n_stmts):
        g.simple()
    g.finish()
    return g.a.build(f"c3_{seed}", argcount=2)


def c4(seed, minor=10, target_units=10000, max_depth=8):
    """Long nested-control-flow function of roughly target_units instructions."""
    g = _Gen(minor, Rng(splitmix64(0xC4 ^ seed)))

    def full():
        return g.units() >= target_units

    def block(depth, n):
        for _ in range(n):
            if full():
                break
            stmt(depth)

    def stmt(depth):
        a, r = g.a, g.r
        kind = r.below(10) if depth < max_depth else 0
        if kind <= 3:
            g.simple()
        elif kind == 4:  # if
            end = a.fresh()
            g.cond(); g.jf(end); block(depth + 1, 1 + r.below(4)); a.label(end)
        elif kind == 5:  # if / else
            els, end = a.fresh(), a.fresh()
            g.cond(); g.jf(els); block(depth + 1, 1 + r.below(4)); a("JUMP_FORWARD", end)
            a.label(els); block(depth + 1, 1 + r.below(4)); a.label(end)
        elif kind == 6:  # for
            top, end = a.fresh(), a.fresh()
            a("LOAD_FAST", g.lv()); a("GET_ITER"); a.label(top); a("FOR_ITER", end)
            a("STORE_FAST", g.lv()); block(depth + 1, 1 + r.below(4))
            a("JUMP_BACKWARD" if g.minor >= 11 else "JUMP_ABSOLUTE", top); a.label(end)
        elif kind == 7:  # rotated while
            top, end = a.fresh(), a.fresh()
            g.cond(); g.jf(end); a.label(top); block(depth + 1, 1 + r.below(4)); g.cond()
            if g.minor >= 11:
                a("POP_JUMP_BACKWARD_IF_TRUE", top)
            else:
                a("POP_JUMP_IF_TRUE", top)
            a.label(end)
        else:  # try / except NameError
            if g.minor >= 11:
                _try311(g, depth, block)
            else:
                h, rr, end = a.fresh(), a.fresh(), a.fresh()
                a("SETUP_FINALLY", h); block(depth + 1, 1 + r.below(4)); a("POP_BLOCK")
                a("JUMP_FORWARD", end)
                a.label(h); a("DUP_TOP"); a("LOAD_GLOBAL", a.name("NameError"))
                a("JUMP_IF_NOT_EXC_MATCH", rr); a("POP_TOP"); a("POP_TOP"); a("POP_TOP")
                block(depth + 1, 1 + r.below(3)); a("POP_EXCEPT"); a("JUMP_FORWARD", end)
                a.label(rr); a("RERAISE", 0); a.label(end)

    while not full():
        stmt(0)
    g.finish()
    return g.a.build(f"c4_{seed}", argcount=2, stacksize=32)


def _try311(g, depth, block):
    """3.11 try/except NameError with a varint exception table."""
    a, r = g.a, g.r
    s, e, h, cl, end, rr = (a.fresh() for _ in range(6))
    a("NOP")
    # straight-line body and handler: nested control flow inside a 3.11
    # protected range needs CPython's range splitting, which this generator skips
    a.label(s)
    for _ in range(1 + r.below(4)):
        g.simple()
    a.label(e)
    a("JUMP_FORWARD", end)
    a.label(h); a("PUSH_EXC_INFO"); a("LOAD_GLOBAL", a.name("NameError") << 1); a("CHECK_EXC_MATCH")
    a("POP_JUMP_FORWARD_IF_FALSE", rr); a("POP_TOP")
    for _ in range(1 + r.below(3)):
        g.simple()
    a("POP_EXCEPT"); a("JUMP_FORWARD", end)
    a.label(rr); a("RERAISE", 0)
    a.label(cl); a("COPY", 3); a("POP_EXCEPT"); a("RERAISE", 1)
    a.label(end)
    depth_stack = 0
    a.exc.append((s, e, h, depth_stack, False))
    a.exc.append((h, cl, cl, depth_stack + 1, True))


def shared_bytes(minor=10):
    """A module whose second function's co_code equals a bytes constant and the
    line table of the first (`def f(): return <bytes>` / `def g(): return None`),
    so a marshal writer that shares equal bytes objects emits g's co_code as an
    'r' back-reference to f's objects (the loader must not move that payload)."""
    def fn(name, value):
        a = Asm(minor)
        a.const(None)
        if minor >= 11:
            a("RESUME", 0)
        a("LOAD_CONST", a.const(value, "bytes") if value is not None else 0)
        a("RETURN_VALUE")
        return a.build(name)

    import dataclasses

    g = fn("g", None)
    f = fn("f", bytes(g.code))
    # f's line table (the last bytes object written for f) equals g's code too
    f = dataclasses.replace(f, linetable=bytes(g.code))
    m = Asm(minor)
    if minor >= 11:
        m("RESUME", 0)
    for co in (f, g):
        m("LOAD_CONST", m.const(co, "code"))
        if minor <= 10:
            m("LOAD_CONST", m.const(co.name))
        m("MAKE_FUNCTION", 0)
        m("STORE_NAME", m.name(co.name))
    m("LOAD_CONST", m.const(None))
    m("RETURN_VALUE")
    return m.build("<module>", flags=0x40)
