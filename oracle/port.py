"""TEST INFRASTRUCTURE ONLY -- oracle entry point: decompile_source on the CPU.

Restates, from /root/reference/pkg/src/unpyre:
  code_model.py:198-253   validation               -> check()
  recover.py:25-357       nested-code recovery     -> Recover, scope_decls()
  pipeline.py:90-160      body pipeline / wrapper  -> body(), decompile_source()
  emitter.py:19-551       source rendering         -> Writer
"""
from __future__ import annotations

import math

from paper_2403_13839_b200.errors import InternalMarkerLeak, UnpyreError

from . import lift, shape
from . import nodes as n

COMP_KIND = {"<listcomp>": "list", "<setcomp>": "set", "<dictcomp>": "dict", "<genexpr>": "gen"}


def params_of(co, defaults=(), kwdefaults=()):
    """params_from_code (ir.py:432-450)."""
    names = co.varnames
    k = co.argcount
    p = n.Params(list(names[:k]), co.posonlyargcount, None, list(names[k:k + co.kwonlyargcount]), None,
                 list(defaults), dict(kwdefaults))
    i = k + co.kwonlyargcount
    if co.flags & 0x4:
        p.vararg = names[i]
        i += 1
    if co.flags & 0x8:
        p.kwarg = names[i]
    return p


def _doc_const(co):
    return co.consts[0] if co.consts and co.consts[0].kind == "str" else None


# ------------------------------------------------------------------ recovery

class Recover:
    """DefRecovery (recover.py:81-227) with map_expr/_map_pair/_stmt_exprs."""

    def __init__(self, co):
        self.co = co
        self.hoisted = []
        self.lambdas = 0

    def mx(self, e):
        if not n.is_expr(e):
            return e
        r = self.pre(e)
        if r is not None:
            return r
        for name, _ in e.kind_fields:
            v = getattr(e, name)
            if n.is_expr(v):
                setattr(e, name, self.mx(v))
            elif isinstance(v, list):
                setattr(e, name, [self.mx(x) if n.is_expr(x) else self.pair(x) for x in v])
        return self.post(e)

    def pair(self, x):
        if isinstance(x, tuple) and len(x) == 2 and n.is_expr(x[1]):
            return (x[0], self.mx(x[1]))
        if isinstance(x, n.CompFor):
            x.target = self.mx(x.target)
            x.iter = self.mx(x.iter)
            x.ifs = [self.mx(i) for i in x.ifs]
        return x

    def pre(self, e):
        if isinstance(e, n.Call) and isinstance(e.func, n.FuncExpr):
            kind = COMP_KIND.get(e.func.code.name)
            if kind and len(e.args) == 1 and not e.keywords:
                arg = self.mx(e.args[0])
                comp = self.comprehension(kind, e.func.code, arg)
                if comp is not None:
                    return comp
        if isinstance(e, n.FuncExpr) and e.code.name == "<lambda>":
            lam = self.lam(e)
            if lam is not None:
                return lam
        return None

    def post(self, e):
        if isinstance(e, n.FuncExpr):
            name = e.code.name
            if name == "<lambda>":
                name = f"__lambda_{self.lambdas}"
                self.lambdas += 1
            self.hoisted.append(self.funcdef(name, e))
            return n.Name(name, "fast")
        return e

    def funcdef(self, name, fe):
        ps = params_of(fe.code, [self.mx(d) for d in fe.defaults], [(k, self.mx(d)) for k, d in fe.kwdefaults])
        b = body(fe.code)
        doc = _doc_const(fe.code)
        if doc is not None:
            b = [n.ExprStmt(n.ConstE(doc))] + b
        return n.FuncDef(name, ps, b or [n.Pass()])

    def classdef(self, name, call):
        args = call.args
        if len(args) < 2 or not isinstance(args[0], n.FuncExpr):
            return None
        code = args[0].code
        bases = [self.mx(x) for x in args[2:]]
        kws = [(k, self.mx(v)) for k, v in call.keywords]
        b = _class_body(body(code))
        return n.ClassDef(name, bases, kws, b or [n.Pass()])

    def lam(self, fe):
        b = body(fe.code)
        if len(b) == 1 and isinstance(b[0], n.Return):
            return n.Lambda(params_of(fe.code, fe.defaults, fe.kwdefaults), b[0].value)
        return None

    def comprehension(self, kind, code, it):
        m = _comp_shape(body(code))
        if m is None:
            return None
        acc, gens = m
        gens[0].iter = it
        if kind == "dict":
            if not isinstance(acc, n.CompAccum) or acc.kind != "map":
                return None
            return n.CompExpr("dict", None, acc.key, acc.value, gens)
        if isinstance(acc, n.CompAccum):
            return n.CompExpr(kind, acc.value, None, None, gens)
        return n.CompExpr(kind, acc, None, None, gens)

    def as_def(self, target, value):
        decos = []
        inner = value
        while isinstance(inner, n.Call) and len(inner.args) == 1 and not inner.keywords \
                and not isinstance(inner.func, n.BuildClass):
            decos.append(inner.func)
            inner = inner.args[0]
        if isinstance(inner, n.Call) and isinstance(inner.func, n.BuildClass):
            made = self.classdef(target.id, inner)
            if made is None:
                return None
            made.decorators = [self.mx(d) for d in decos]
            return made
        if isinstance(inner, n.FuncExpr) and inner.code.name == target.id:
            made = self.funcdef(target.id, inner)
            made.decorators = [self.mx(d) for d in decos]
            return made
        return None

    def stmt(self, s):
        if isinstance(s, n.Assign) and len(s.targets) == 1 and isinstance(s.targets[0], n.Name):
            made = self.as_def(s.targets[0], s.value)
            if made is not None:
                return [made]
        for f in shape.BLOCK_FIELDS:
            sub = getattr(s, f, None)
            if isinstance(sub, list) and sub and n.is_stmt(sub[0]):
                setattr(s, f, self.block(sub))
        if isinstance(s, n.Try):
            for h in s.handlers:
                h.body = self.block(h.body)
        if isinstance(s, n.With):
            s.body = self.block(s.body)
        for name, _ in s.kind_fields:
            v = getattr(s, name)
            if n.is_expr(v):
                setattr(s, name, self.mx(v))
            elif isinstance(v, list) and v and all(n.is_expr(x) for x in v):
                setattr(s, name, [self.mx(x) for x in v])
            elif isinstance(v, list):
                for x in v:
                    if isinstance(x, n.WithItem):
                        x.context = self.mx(x.context)
                        if x.target is not None:
                            x.target = self.mx(x.target)
                    elif isinstance(x, tuple) and len(x) == 2 and n.is_expr(x[1]):
                        v[v.index(x)] = (x[0], self.mx(x[1]))
        return [s]

    def block(self, stmts):
        res = []
        for s in stmts:
            rep = self.stmt(s)
            res.extend(self.hoisted)
            self.hoisted = []
            res.extend(rep)
        return res


def _comp_shape(b):
    """_match_comp_body (recover.py:230-279)."""
    seq = list(b)
    if seq and isinstance(seq[-1], n.Return):
        seq = seq[:-1]
    if len(seq) != 1 or not isinstance(seq[0], n.For):
        return None
    node = seq[0]
    gens = []
    while True:
        if node.orelse:
            return None
        g = n.CompFor(node.target, node.iter, [])
        gens.append(g)
        inner = node.body
        while True:
            if (len(inner) >= 2 and isinstance(inner[0], n.If) and len(inner[0].then) == 1
                    and isinstance(inner[0].then[0], n.Continue) and not inner[0].orelse):
                g.ifs.append(lift.negate(inner[0].cond))
                inner = inner[1:]
                continue
            if (len(inner) == 1 and isinstance(inner[0], n.If) and not inner[0].orelse
                    and not (len(inner[0].then) == 1 and isinstance(inner[0].then[0], n.Continue))):
                g.ifs.append(inner[0].cond)
                inner = inner[0].then
                continue
            break
        if len(inner) == 1 and isinstance(inner[0], n.For):
            node = inner[0]
            continue
        if len(inner) == 1 and isinstance(inner[0], n.CompAccum):
            return inner[0], gens
        if len(inner) == 1 and isinstance(inner[0], n.ExprStmt) and isinstance(inner[0].value, n.Yield):
            return inner[0].value.value, gens
        return None


def _class_body(b):
    """_clean_class_body (recover.py:282-301)."""
    res = []
    for s in b:
        if isinstance(s, n.Assign) and len(s.targets) == 1 and isinstance(s.targets[0], n.Name):
            t = s.targets[0].id
            if (t == "__module__" and isinstance(s.value, n.Name)) or \
                    (t == "__qualname__" and isinstance(s.value, n.ConstE)) or t == "__classcell__":
                continue
            if t == "__doc__" and isinstance(s.value, n.ConstE):
                res.append(n.ExprStmt(s.value))
                continue
        if isinstance(s, n.Return):
            continue
        res.append(s)
    return res


def _children(s):
    if isinstance(s, n.If):
        return [s.then, s.orelse]
    if isinstance(s, (n.While, n.For)):
        return [s.body, s.orelse]
    if isinstance(s, n.Try):
        return [s.body, *[h.body for h in s.handlers], s.orelse, s.final]
    if isinstance(s, n.With):
        return [s.body]
    return []


def scope_decls(b, co):
    """add_scope_decls (recover.py:304-357)."""
    gl, nl = [], []
    free = set(co.freevars)

    def note(t):
        if isinstance(t, n.Name):
            if t.scope == "global" and t.id not in gl:
                gl.append(t.id)
            if t.scope == "deref" and t.id in free and t.id not in nl:
                nl.append(t.id)
        elif isinstance(t, (n.TupleE, n.ListE)):
            for e in t.elts:
                note(e)
        elif isinstance(t, n.Starred):
            note(t.value)

    def scan(stmts):
        for s in stmts:
            if isinstance(s, (n.FuncDef, n.ClassDef)):
                continue
            if isinstance(s, (n.Assign, n.Delete)):
                for t in s.targets:
                    note(t)
            elif isinstance(s, n.AugAssign):
                note(s.target)
            elif isinstance(s, n.For):
                note(s.target)
            for sub in _children(s):
                scan(sub)

    scan(b)
    decls = ([n.Global(gl)] if gl else []) + ([n.Nonlocal(nl)] if nl else [])
    if not decls:
        return b
    at = 1 if b and isinstance(b[0], n.ExprStmt) and isinstance(b[0].value, n.ConstE) else 0
    return b[:at] + decls + b[at:]


def _ret_none(s):
    return isinstance(s, n.Return) and isinstance(s.value, n.ConstE) and s.value.const.kind == "none"


def body(co):
    """decompile_body (pipeline.py:90-110)."""
    instrs, rows, g, loops = lift.analyze(co)
    stmts = shape.Shaper(co, instrs, g, loops, rows).top()
    stmts = shape.canon(stmts)
    stmts = Recover(co).block(stmts)
    stmts = scope_decls(stmts, co)
    if co.flags & (0x20 | 0x200):
        while stmts and _ret_none(stmts[-1]):
            stmts.pop()
    elif stmts and _ret_none(stmts[-1]):
        stmts.pop()
    return stmts


# ------------------------------------------------------------------ validation

def check(co):
    """validate_code_object (code_model.py:198-253): list of violations."""
    out = []

    def one(c, path, seen):
        where = f"{path or c.name}: " if path else ""
        if id(c) in seen:
            out.append(f"{where}code constant cycle detected")
            return
        seen = seen | {id(c)}
        if len(c.code) % 2:
            out.append(f"{where}code length not word-aligned")
        if not c.code:
            out.append(f"{where}empty code")
        if c.stacksize < 0:
            out.append(f"{where}negative stacksize")
        if c.flags < 0:
            out.append(f"{where}negative flags")
        if c.exceptiontable and c.version.minor < 11:
            out.append(f"{where}exception table requires >=3.11")
        if c.version.minor <= 10:
            if not (c.argcount + c.kwonlyargcount <= c.nlocals <= len(c.varnames)):
                out.append(f"{where}argcount {c.argcount}+kwonly {c.kwonlyargcount} vs nlocals {c.nlocals} "
                           f"vs varnames {len(c.varnames)} inconsistent")
        else:
            if c.nlocals != len(c.varnames):
                out.append(f"{where}nlocals {c.nlocals} != len(varnames) {len(c.varnames)}")
            if c.argcount + c.kwonlyargcount > c.nlocals:
                out.append(f"{where}more arguments than local slots")
        if c.posonlyargcount > c.argcount:
            out.append(f"{where}posonlyargcount exceeds argcount")
        consts(c, c.consts, where, seen, 0)

    def consts(owner, cs, where, seen, depth):
        if depth > 128:
            out.append(f"{where}constant tree too deep")
            return
        for k in cs:
            if k.kind == "code":
                ch = k.value
                if ch.version != owner.version:
                    out.append(f"{where}nested code {ch.name!r} has version {ch.version}, parent has {owner.version}")
                one(ch, f"{where}{ch.name}", seen)
            elif k.kind in ("tuple", "frozenset"):
                consts(owner, k.value, where, seen, depth + 1)

    one(co, "", set())
    return out


# ------------------------------------------------------------------ emitter

PREC = dict(LAMBDA=1, TERNARY=2, OR=3, AND=4, NOT=5, COMPARE=6, BITOR=7, BITXOR=8, BITAND=9, SHIFT=10, ARITH=11,
            TERM=12, UNARY=13, POWER=14, AWAIT=15, ATOM=16)
P = type("P", (), PREC)
BINPREC = {"|": P.BITOR, "^": P.BITXOR, "&": P.BITAND, "<<": P.SHIFT, ">>": P.SHIFT, "+": P.ARITH, "-": P.ARITH,
           "*": P.TERM, "/": P.TERM, "//": P.TERM, "%": P.TERM, "@": P.TERM, "**": P.POWER}


def float_text(v):
    if math.isnan(v):
        return "float('nan')"
    if math.isinf(v):
        return "float('inf')" if v > 0 else "float('-inf')"
    if v == 0.0 and math.copysign(1.0, v) < 0:
        return "-0.0"
    return repr(v)


def imag_text(im):
    if math.isinf(im):
        return "complex(0.0, %s)" % float_text(im)
    return repr(im) + "j"


def const_text(c):
    """render_constant (emitter.py:53-109)."""
    k = c.kind
    if k == "none":
        return "None"
    if k == "bool":
        return "True" if c.value else "False"
    if k == "ellipsis":
        return "..."
    if k in ("int", "str", "bytes"):
        return repr(c.value)
    if k == "float":
        return float_text(c.value)
    if k == "complex":
        re, im = c.value.real, c.value.imag
        if re == 0.0 and math.copysign(1.0, re) > 0 and not math.isnan(im):
            return imag_text(im)
        if math.isnan(re) or math.isinf(re) or math.isnan(im) or math.isinf(im):
            return f"complex({float_text(re)}, {float_text(im)})"
        if math.copysign(1.0, im) >= 0:
            return f"({float_text(re)} + {imag_text(im)})"
        return f"({float_text(re)} - {imag_text(-im)})"
    if k == "tuple":
        if not c.value:
            return "()"
        inner = ", ".join(const_text(x) for x in c.value)
        return f"({inner},)" if len(c.value) == 1 else f"({inner})"
    if k == "frozenset":
        if not c.value:
            return "frozenset()"
        return "frozenset({%s})" % ", ".join(const_text(x) for x in c.value)
    raise InternalMarkerLeak(f"constant kind {k} cannot be rendered inline")


class Writer:
    """Emitter (emitter.py:112-532)."""

    def __init__(self, indent="    "):
        self.indent = indent
        self.lines = []
        self.depth = 0

    def put(self, text):
        self.lines.append(self.indent * self.depth + text)

    def suite(self, stmts):
        self.depth += 1
        if not stmts:
            self.put("pass")
        for s in stmts:
            self.stmt(s)
        self.depth -= 1

    def stmt(self, s):
        if isinstance(s, n.MARKERS) or type(s).__name__ in ("CompAccum", "_WhileShape"):
            raise InternalMarkerLeak(f"marker survived structuring: {s!r}")
        fn = STMT.get(type(s).__name__)
        if fn is None:
            raise InternalMarkerLeak(f"no emitter for {type(s).__name__}")
        fn(self, s)

    def if_chain(self, s, kw):
        self.put(f"{kw} {self.ex(s.cond)}:")
        self.suite(s.then)
        if not s.orelse:
            return
        if len(s.orelse) == 1 and isinstance(s.orelse[0], n.If):
            self.if_chain(s.orelse[0], "elif")
            return
        self.put("else:")
        self.suite(s.orelse)

    def params(self, p):
        parts = []
        nd = len(p.defaults)
        for i, a in enumerate(p.args):
            di = i - (len(p.args) - nd)
            parts.append(f"{a}={self.ex(p.defaults[di])}" if di >= 0 else a)
            if p.posonly and i + 1 == p.posonly:
                parts.append("/")
        if p.vararg:
            parts.append("*" + p.vararg)
        elif p.kwonly:
            parts.append("*")
        for k in p.kwonly:
            parts.append(f"{k}={self.ex(p.kwdefaults[k])}" if k in p.kwdefaults else k)
        if p.kwarg:
            parts.append("**" + p.kwarg)
        return ", ".join(parts)

    def tgt(self, t, nested=False):
        if isinstance(t, (n.TupleE, n.ListE)) and t.elts:
            inner = ", ".join(self.tgt(e, True) for e in t.elts)
            if isinstance(t, n.ListE):
                return f"[{inner}]"
            if len(t.elts) == 1:
                inner += ","
            return f"({inner})" if nested else inner
        if isinstance(t, n.Starred):
            return "*" + self.tgt(t.value, nested)
        return self.ex(t)

    def ex(self, e, parent=0, right=False):
        fn = EXPR.get(type(e).__name__)
        if fn is None:
            raise InternalMarkerLeak(f"no emitter for expression {type(e).__name__}: {e!r}")
        text, prec = fn(self, e)
        if prec < parent or (prec == parent and right and prec != P.ATOM):
            return f"({text})"
        return text

    def arg(self, a):
        if isinstance(a, n.Starred):
            return "*" + self.ex(a.value, P.LAMBDA)
        return self.ex(a, P.LAMBDA)

    def index(self, i):
        if isinstance(i, n.SliceE):
            return self.slice(i)
        if isinstance(i, n.TupleE) and i.elts and any(isinstance(x, n.SliceE) for x in i.elts):
            return ", ".join(self.slice(x) if isinstance(x, n.SliceE) else self.ex(x) for x in i.elts)
        return self.ex(i)

    def slice(self, s):
        lo = self.ex(s.lower, P.TERNARY) if s.lower is not None else ""
        hi = self.ex(s.upper, P.TERNARY) if s.upper is not None else ""
        t = f"{lo}:{hi}"
        if s.step is not None:
            t += f":{self.ex(s.step, P.TERNARY)}"
        return t

    def fpart(self, fv):
        inner = self.ex(fv.value, P.TERNARY)
        if inner.startswith("{"):
            inner = " " + inner
        t = "{" + inner
        if fv.conversion:
            t += "!" + fv.conversion
        if fv.format_spec is not None:
            t += ":" + self.fspec(fv.format_spec)
        return t + "}"

    def fspec(self, spec):
        if isinstance(spec, n.ConstE):
            return str(spec.const.value)
        if isinstance(spec, n.FString):
            return "".join(p if isinstance(p, str) else self.fpart(p) for p in spec.parts)
        return "{" + self.ex(spec, P.TERNARY) + "}"


def _s_assign(w, s):
    w.put(" = ".join(w.tgt(t) for t in s.targets) + f" = {w.ex(s.value)}")


def _s_return(w, s):
    if isinstance(s.value, n.ConstE) and s.value.const.kind == "none":
        w.put("return None")
    else:
        w.put(f"return {w.ex(s.value)}")


def _s_raise(w, s):
    if s.exc is None:
        w.put("raise")
    elif s.cause is not None:
        w.put(f"raise {w.ex(s.exc)} from {w.ex(s.cause)}")
    else:
        w.put(f"raise {w.ex(s.exc)}")


def _s_loop(kw):
    def f(w, s):
        if kw == "while":
            w.put(f"while {w.ex(s.cond)}:")
        else:
            w.put(f"for {w.tgt(s.target)} in {w.ex(s.iter)}:")
        w.suite(s.body)
        if s.orelse:
            w.put("else:")
            w.suite(s.orelse)
    return f


def _s_try(w, s):
    w.put("try:")
    w.suite(s.body)
    for h in s.handlers:
        if h.type is None:
            w.put("except:")
        elif h.name:
            w.put(f"except {w.ex(h.type)} as {h.name}:")
        else:
            w.put(f"except {w.ex(h.type)}:")
        w.suite(h.body)
    if s.orelse:
        w.put("else:")
        w.suite(s.orelse)
    if s.final:
        w.put("finally:")
        w.suite(s.final)


def _s_with(w, s):
    items = []
    for it in s.items:
        part = w.ex(it.context)
        if it.target is not None:
            part += f" as {w.tgt(it.target, True)}"
        items.append(part)
    w.put("with " + ", ".join(items) + ":")
    w.suite(s.body)


def _s_funcdef(w, s):
    for d in s.decorators:
        w.put("@" + w.ex(d))
    w.put(f"def {s.name}({w.params(s.params)}):")
    w.suite(s.body)


def _s_classdef(w, s):
    for d in s.decorators:
        w.put("@" + w.ex(d))
    head = f"class {s.name}"
    args = [w.ex(b) for b in s.bases] + [f"{k}={w.ex(v)}" for k, v in s.keywords]
    if args:
        head += "(" + ", ".join(args) + ")"
    w.put(head + ":")
    w.suite(s.body)


STMT = {
    "Assign": _s_assign,
    "AugAssign": lambda w, s: w.put(f"{w.tgt(s.target)} {s.op}= {w.ex(s.value)}"),
    "ExprStmt": lambda w, s: w.put(w.ex(s.value)),
    "Return": _s_return, "Raise": _s_raise,
    "Delete": lambda w, s: w.put("del " + ", ".join(w.tgt(t) for t in s.targets)),
    "Pass": lambda w, s: w.put("pass"), "Break": lambda w, s: w.put("break"),
    "Continue": lambda w, s: w.put("continue"),
    "Global": lambda w, s: w.put("global " + ", ".join(s.names)),
    "Nonlocal": lambda w, s: w.put("nonlocal " + ", ".join(s.names)),
    "Assert": lambda w, s: w.put(f"assert {w.ex(s.test)}, {w.ex(s.msg)}" if s.msg is not None
                                 else f"assert {w.ex(s.test)}"),
    "Import": lambda w, s: w.put(f"import {s.module} as {s.asname}" if s.asname else f"import {s.module}"),
    "ImportFrom": lambda w, s: w.put(f"from {'.' * s.level + s.module} import "
                                     + ", ".join(f"{a} as {b}" if b else a for a, b in s.names)),
    "ImportStar": lambda w, s: w.put(f"from {'.' * s.level + s.module} import *"),
    "If": lambda w, s: w.if_chain(s, "if"),
    "While": _s_loop("while"), "For": _s_loop("for"), "Try": _s_try, "With": _s_with,
    "FuncDef": _s_funcdef, "ClassDef": _s_classdef,
}


def _e_const(w, e):
    t = const_text(e.const)
    return t, (P.UNARY if t.startswith("-") or e.const.kind == "complex" else P.ATOM)


def _e_binop(w, e):
    p = BINPREC[e.op]
    if e.op == "**":
        return f"{w.ex(e.left, p, True)} ** {w.ex(e.right, p)}", p
    return f"{w.ex(e.left, p)} {e.op} {w.ex(e.right, p, True)}", p


def _e_unary(w, e):
    if e.op == "not":
        return f"not {w.ex(e.operand, P.NOT)}", P.NOT
    return f"{e.op}{w.ex(e.operand, P.UNARY)}", P.UNARY


def _e_compare(w, e):
    parts = [w.ex(e.left, P.COMPARE, True)]
    for op, x in zip(e.ops, e.comparators):
        parts.append(op)
        parts.append(w.ex(x, P.COMPARE, True))
    return " ".join(parts), P.COMPARE


def _e_boolop(w, e):
    p = P.OR if e.op == "or" else P.AND
    return f" {e.op} ".join(w.ex(v, p, i > 0) for i, v in enumerate(e.values)), p


def _e_call(w, e):
    fn = w.ex(e.func, P.ATOM)
    args = [w.arg(a) for a in e.args]
    for k, v in e.keywords:
        args.append("**" + w.ex(v, P.LAMBDA) if k is None else f"{k}={w.ex(v, P.LAMBDA)}")
    return f"{fn}({', '.join(args)})", P.ATOM


def _e_attr(w, e):
    base = w.ex(e.value, P.ATOM)
    if isinstance(e.value, n.ConstE) and e.value.const.kind == "int":
        base = f"({base})"
    return f"{base}.{e.name}", P.ATOM


def _e_tuple(w, e):
    if not e.elts:
        return "()", P.ATOM
    inner = ", ".join(w.arg(x) for x in e.elts)
    return (f"({inner},)" if len(e.elts) == 1 else f"({inner})"), P.ATOM


def _e_set(w, e):
    if not e.elts:
        return "set()", P.ATOM
    return "{" + ", ".join(w.arg(x) for x in e.elts) + "}", P.ATOM


def _e_dict(w, e):
    parts = []
    for k, v in zip(e.keys, e.values):
        parts.append("**" + w.ex(v, P.LAMBDA) if k is None else f"{w.ex(k, P.LAMBDA)}: {w.ex(v, P.LAMBDA)}")
    return "{" + ", ".join(parts) + "}", P.ATOM


def _e_yield(w, e):
    if e.value is None or (isinstance(e.value, n.ConstE) and e.value.const.kind == "none"):
        return "(yield)", P.ATOM
    return f"(yield {w.ex(e.value, P.LAMBDA)})", P.ATOM


def _e_comp(w, e):
    gens = []
    for g in e.generators:
        part = f"for {w.tgt(g.target)} in {w.ex(g.iter, P.TERNARY)}"
        for c in g.ifs:
            part += f" if {w.ex(c, P.TERNARY)}"
        gens.append(part)
    spine = " ".join(gens)
    if e.kind == "dict":
        return "{" + f"{w.ex(e.key, P.TERNARY)}: {w.ex(e.value, P.TERNARY)} {spine}" + "}", P.ATOM
    elt = w.ex(e.elt, P.TERNARY)
    if e.kind == "list":
        return f"[{elt} {spine}]", P.ATOM
    if e.kind == "set":
        return "{" + f"{elt} {spine}" + "}", P.ATOM
    return f"({elt} {spine})", P.ATOM


def _e_fstring(w, e):
    bits = [p.replace("{", "{{").replace("}", "}}") if isinstance(p, str) else w.fpart(p) for p in e.parts]
    text = "".join(bits)
    q = "'" if "'" not in text else '"'
    if "'" in text and '"' in text:
        text = text.replace("'", "\\'")
        q = "'"
    return f"f{q}{text}{q}", P.ATOM


def _e_lambda(w, e):
    ps = w.params(e.params)
    head = f"lambda {ps}: " if ps else "lambda: "
    return head + w.ex(e.body, P.LAMBDA), P.LAMBDA


EXPR = {
    "ConstE": _e_const, "Name": lambda w, e: (e.id, P.ATOM), "StackTemp": lambda w, e: (f"__stack_{e.index}", P.ATOM),
    "BinOp": _e_binop, "UnaryOp": _e_unary, "Compare": _e_compare, "BoolOp": _e_boolop,
    "Ternary": lambda w, e: (f"{w.ex(e.then, P.TERNARY, True)} if {w.ex(e.cond, P.TERNARY, True)} else "
                             f"{w.ex(e.orelse, P.TERNARY)}", P.TERNARY),
    "Lambda": _e_lambda,
    "NamedExpr": lambda w, e: (f"{e.target.id} := {w.ex(e.value, P.LAMBDA)}", P.LAMBDA),
    "Call": _e_call, "Attr": _e_attr,
    "Subscript": lambda w, e: (f"{w.ex(e.value, P.ATOM)}[{w.index(e.index)}]", P.ATOM),
    "TupleE": _e_tuple, "ListE": lambda w, e: ("[" + ", ".join(w.arg(x) for x in e.elts) + "]", P.ATOM),
    "SetE": _e_set, "DictE": _e_dict, "Starred": lambda w, e: ("*" + w.ex(e.value, P.LAMBDA), P.LAMBDA),
    "Yield": _e_yield, "YieldFrom": lambda w, e: (f"(yield from {w.ex(e.value, P.LAMBDA)})", P.ATOM),
    "CompExpr": _e_comp, "FString": _e_fstring,
}


# ------------------------------------------------------------------ entry

def decompile_source(co, style=None):
    """decompile_source (pipeline.py:143-160) + emit_module (emitter.py:535-547)."""
    problems = check(co)
    if problems:
        raise UnpyreError("validation failed: " + "; ".join(problems))
    b = body(co)
    if co.name == "<module>":
        if b and isinstance(b[0], n.Assign) and len(b[0].targets) == 1 and isinstance(b[0].targets[0], n.Name) \
                and b[0].targets[0].id == "__doc__" and isinstance(b[0].value, n.ConstE):
            b[0] = n.ExprStmt(b[0].value)
        tree = b or [n.Pass()]
    else:
        doc = _doc_const(co)
        if doc is not None:
            b = [n.ExprStmt(n.ConstE(doc))] + b
        tree = [n.FuncDef(co.name, params_of(co), b or [n.Pass()])]
    w = Writer("    " if style is None else style.indent)
    if style is not None and style.header:
        w.put(f"# decompiled by {style.tool} from {co.qualname or co.name} (python {co.version})")
    if not tree:
        w.put("pass")
    for s in tree:
        w.stmt(s)
    return "\n".join(w.lines) + "\n"


def outcome(co, style=None):
    """("ok", text) or (exception class name, message)."""
    try:
        return "ok", decompile_source(co, style)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e)
