"""Python source -> CPython 3.10 code objects (test-corpus generator, not product).

SURVEY.md §8(c)/(d) C2: the reference's syntax corpus (`pkg/corpus/*.py`) is
source text, and no 3.8-3.11 interpreter exists in this image, so the C2
parity corpus needs an in-repo compiler.  This module restates CPython 3.10's
code generator for the statement/expression subset the corpus uses:

* scope analysis (Python/symtable.c: LOCAL / GLOBAL_EXPLICIT / GLOBAL_IMPLICIT /
  FREE / CELL, the implicit `__class__` cell for zero-argument super());
* the AST constant folder (Python/ast_opt.c: unary/binary folding on
  constants, constant tuples, list/set literals in `in` and `for` become
  tuple/frozenset constants, `not (a in b)` -> `a not in b`);
* code generation (Python/compile.c: compiler_jump_if, rotated while loops,
  try/except/finally with SETUP_FINALLY + POP_BLOCK, SETUP_WITH, frame-block
  unwinding for return/break/continue, comprehensions as nested functions,
  LOAD_METHOD/CALL_METHOD, CALL_FUNCTION_KW/EX, BUILD_CONST_KEY_MAP, ...);
* the CFG optimiser (optimize_basic_block, clean_basic_block,
  extend_block / exit-block copying, mark_reachable,
  eliminate_empty_basic_blocks, redundant-jump removal,
  duplicate_exits_without_lineno), with line numbers tracked so the same NOPs
  survive;
* stack-depth computation and the assembler (synth/asm.py handles
  EXTENDED_ARG sizing and the 3.10 jump encoding).

Parity does not depend on this being bit-identical to CPython: every C2 input
is decompiled by the reference itself to make the golden text
(tests/golden/make_c2_golden.py).  Fidelity only decides how much of the
reference's pattern matching the corpus exercises.
"""
from __future__ import annotations

import ast
import math

from .asm import Label, assemble
from ..model import CodeObject, Const, VersionTag

CO_OPTIMIZED, CO_NEWLOCALS, CO_VARARGS, CO_VARKEYWORDS = 1, 2, 4, 8
CO_NESTED, CO_GENERATOR, CO_NOFREE = 0x10, 0x20, 0x40
STACK_USE_GUIDELINE = 30
MAX_COPY_SIZE = 4

LOCAL, GLOBAL_EXPLICIT, GLOBAL_IMPLICIT, FREE, CELL = 1, 2, 3, 4, 5

BINOP = {ast.Add: "ADD", ast.Sub: "SUBTRACT", ast.Mult: "MULTIPLY", ast.Div: "TRUE_DIVIDE",
         ast.FloorDiv: "FLOOR_DIVIDE", ast.Mod: "MODULO", ast.Pow: "POWER", ast.LShift: "LSHIFT",
         ast.RShift: "RSHIFT", ast.BitAnd: "AND", ast.BitOr: "OR", ast.BitXor: "XOR",
         ast.MatMult: "MATRIX_MULTIPLY"}
UNOP = {ast.UAdd: "UNARY_POSITIVE", ast.USub: "UNARY_NEGATIVE", ast.Not: "UNARY_NOT",
        ast.Invert: "UNARY_INVERT"}
CMPOP = {ast.Lt: 0, ast.LtE: 1, ast.Eq: 2, ast.NotEq: 3, ast.Gt: 4, ast.GtE: 5}

JUMPS = {"JUMP_ABSOLUTE", "JUMP_FORWARD", "POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE",
         "JUMP_IF_FALSE_OR_POP", "JUMP_IF_TRUE_OR_POP", "JUMP_IF_NOT_EXC_MATCH", "FOR_ITER",
         "SETUP_FINALLY", "SETUP_WITH",
         # 3.11 pseudo / new jumps (pycodegen311.py), direction fixed by normalize_jumps
         "JUMP", "JUMP_NO_INTERRUPT", "POP_JUMP_IF_NONE", "POP_JUMP_IF_NOT_NONE", "SETUP_CLEANUP", "SEND"}
UNCOND = {"JUMP_ABSOLUTE", "JUMP_FORWARD", "JUMP", "JUMP_NO_INTERRUPT"}
SETUPS = {"SETUP_FINALLY", "SETUP_WITH", "SETUP_CLEANUP"}
EXITS = {"RETURN_VALUE", "RAISE_VARARGS", "RERAISE"}


class CompileError(Exception):
    pass


# ---------------------------------------------------------------- constant folding (ast_opt.c)

_SAFE_MULT, _SAFE_POW, _SAFE_LSHIFT = 128, 128, 128


def _is_const(n):
    return isinstance(n, ast.Constant)


def _fold_binop(op, a, b):
    """safe_multiply / safe_power / safe_lshift limits of ast_opt.c."""
    if isinstance(op, ast.Pow) and isinstance(a, int) and isinstance(b, int) and b >= 0:
        if a and b > 0 and a.bit_length() * b > _SAFE_POW:
            return None
    if isinstance(op, ast.LShift) and isinstance(a, int) and isinstance(b, int):
        if b < 0 or b > _SAFE_LSHIFT or a.bit_length() > _SAFE_LSHIFT - b:
            return None
    if isinstance(op, ast.Mult):
        if isinstance(a, int) and isinstance(b, int) and a and b and a.bit_length() + b.bit_length() > _SAFE_MULT:
            return None
        if isinstance(a, (str, bytes, tuple)) or isinstance(b, (str, bytes, tuple)):
            return None
    if isinstance(op, ast.Mod) and isinstance(a, (str, bytes)):
        return None
    fn = {ast.Add: lambda x, y: x + y, ast.Sub: lambda x, y: x - y, ast.Mult: lambda x, y: x * y,
          ast.Div: lambda x, y: x / y, ast.FloorDiv: lambda x, y: x // y, ast.Mod: lambda x, y: x % y,
          ast.Pow: lambda x, y: x ** y, ast.LShift: lambda x, y: x << y, ast.RShift: lambda x, y: x >> y,
          ast.BitAnd: lambda x, y: x & y, ast.BitOr: lambda x, y: x | y, ast.BitXor: lambda x, y: x ^ y}.get(type(op))
    if fn is None:
        return None
    try:
        v = fn(a, b)
    except Exception:  # noqa: BLE001 - folding never raises (ast_opt.c clears the error)
        return None
    if isinstance(v, (str, bytes)) and len(v) > 4096:
        return None
    return (v,)


class _Folder(ast.NodeTransformer):
    def visit_UnaryOp(self, n):
        self.generic_visit(n)
        o = n.operand
        if isinstance(n.op, ast.Not) and isinstance(o, ast.Compare) and len(o.ops) == 1:
            inv = {ast.Is: ast.IsNot, ast.IsNot: ast.Is, ast.In: ast.NotIn, ast.NotIn: ast.In}.get(type(o.ops[0]))
            if inv is not None:
                return ast.copy_location(ast.Compare(o.left, [inv()], o.comparators), n)
        if _is_const(o):
            try:
                v = {ast.UAdd: lambda x: +x, ast.USub: lambda x: -x, ast.Invert: lambda x: ~x,
                     ast.Not: lambda x: not x}[type(n.op)](o.value)
            except Exception:  # noqa: BLE001
                return n
            return ast.copy_location(ast.Constant(v), n)
        return n

    def visit_BinOp(self, n):
        self.generic_visit(n)
        if _is_const(n.left) and _is_const(n.right):
            r = _fold_binop(n.op, n.left.value, n.right.value)
            if r is not None:
                return ast.copy_location(ast.Constant(r[0]), n)
        return n

    def visit_Tuple(self, n):
        self.generic_visit(n)
        if isinstance(n.ctx, ast.Load) and all(_is_const(e) for e in n.elts):
            return ast.copy_location(ast.Constant(tuple(e.value for e in n.elts)), n)
        return n

    @staticmethod
    def _fold_iter(it):
        if isinstance(it, ast.List) and not any(isinstance(e, ast.Starred) for e in it.elts):
            t = ast.copy_location(ast.Tuple(it.elts, ast.Load()), it)
            return _Folder.visit_Tuple(_Folder(), t)
        if isinstance(it, ast.Set) and all(_is_const(e) for e in it.elts):
            return ast.copy_location(ast.Constant(frozenset(e.value for e in it.elts)), it)
        return it

    def visit_Compare(self, n):
        self.generic_visit(n)
        if isinstance(n.ops[-1], (ast.In, ast.NotIn)):
            n.comparators[-1] = self._fold_iter(n.comparators[-1])
        return n

    def visit_For(self, n):
        self.generic_visit(n)
        n.iter = self._fold_iter(n.iter)
        return n

    def visit_comprehension(self, n):
        self.generic_visit(n)
        n.iter = self._fold_iter(n.iter)
        return n

    def visit_Name(self, n):
        if n.id == "__debug__" and isinstance(n.ctx, ast.Load):
            return ast.copy_location(ast.Constant(True), n)
        return n


# ---------------------------------------------------------------- symbol tables (symtable.c)

class Scope:
    def __init__(self, kind, name, node, parent):
        self.kind = kind            # "module" | "class" | "function"
        self.name = name
        self.node = node
        self.parent = parent
        self.params = []
        self.assigned = set()
        self.used = set()
        self.globals = set()
        self.nonlocals = set()
        self.children = []
        self.generator = False
        self.varargs = self.varkw = False
        self.comprehension = False
        self.lambda_ = False
        self.scope = {}
        self.cells = set()
        self.free = set()
        self.needs_class_closure = False
        self.nested = bool(parent and (parent.nested or parent.kind == "function"))

    def all_names(self):
        return set(self.params) | self.assigned | self.used | self.globals | self.nonlocals

    def lookup(self, name):
        return self.scope.get(name, GLOBAL_IMPLICIT)


class _ScopeBuilder(ast.NodeVisitor):
    def __init__(self):
        self.by_node = {}
        self.cur = None

    def _enter(self, kind, name, node):
        s = Scope(kind, name, node, self.cur)
        if self.cur is not None:
            self.cur.children.append(s)
        self.by_node[id(node)] = s
        self.cur = s
        return s

    def _leave(self, s):
        self.cur = s.parent

    def visit_Module(self, n):
        s = self._enter("module", "<module>", n)
        for st in n.body:
            self.visit(st)
        self._leave(s)

    def _args(self, a):
        s = self.cur
        for x in a.posonlyargs + a.args + a.kwonlyargs:
            s.params.append(x.arg)
        if a.vararg:
            s.params.append(a.vararg.arg)
            s.varargs = True
        if a.kwarg:
            s.params.append(a.kwarg.arg)
            s.varkw = True

    def visit_FunctionDef(self, n):
        self.cur.assigned.add(n.name)
        for d in n.args.defaults:
            self.visit(d)
        for d in n.args.kw_defaults:
            if d is not None:
                self.visit(d)
        for d in n.decorator_list:
            self.visit(d)
        s = self._enter("function", n.name, n)
        self._args(n.args)
        for st in n.body:
            self.visit(st)
        self._leave(s)

    visit_AsyncFunctionDef = visit_FunctionDef

    def visit_Lambda(self, n):
        for d in n.args.defaults:
            self.visit(d)
        for d in n.args.kw_defaults:
            if d is not None:
                self.visit(d)
        s = self._enter("function", "<lambda>", n)
        s.lambda_ = True
        self._args(n.args)
        self.visit(n.body)
        self._leave(s)

    def visit_ClassDef(self, n):
        self.cur.assigned.add(n.name)
        for b in n.bases:
            self.visit(b)
        for k in n.keywords:
            self.visit(k.value)
        for d in n.decorator_list:
            self.visit(d)
        s = self._enter("class", n.name, n)
        for st in n.body:
            self.visit(st)
        self._leave(s)

    def _comp(self, n, name, elts):
        gens = n.generators
        self.visit(gens[0].iter)
        s = self._enter("function", name, n)
        s.comprehension = True
        s.params.append(".0")
        for i, g in enumerate(gens):
            if i:
                self.visit(g.iter)
            self.visit(g.target)
            for c in g.ifs:
                self.visit(c)
        for e in elts:
            self.visit(e)
        if name == "<genexpr>":
            s.generator = True
        self._leave(s)

    def visit_ListComp(self, n):
        self._comp(n, "<listcomp>", [n.elt])

    def visit_SetComp(self, n):
        self._comp(n, "<setcomp>", [n.elt])

    def visit_GeneratorExp(self, n):
        self._comp(n, "<genexpr>", [n.elt])

    def visit_DictComp(self, n):
        self._comp(n, "<dictcomp>", [n.key, n.value])

    def visit_Name(self, n):
        if isinstance(n.ctx, ast.Load):
            self.cur.used.add(n.id)
            if n.id == "super" and self.cur.kind == "function":
                self.cur.used.add("__class__")
        else:
            self.cur.assigned.add(n.id)

    def visit_NamedExpr(self, n):
        self.visit(n.value)
        s = self.cur
        while s.comprehension:
            s = s.parent
        s.assigned.add(n.target.id)
        if s is not self.cur:
            self.cur.used.add(n.target.id)

    def visit_Global(self, n):
        self.cur.globals.update(n.names)

    def visit_Nonlocal(self, n):
        self.cur.nonlocals.update(n.names)

    def visit_Import(self, n):
        for a in n.names:
            self.cur.assigned.add(a.asname or a.name.split(".")[0])

    def visit_ImportFrom(self, n):
        for a in n.names:
            if a.name != "*":
                self.cur.assigned.add(a.asname or a.name)

    def visit_ExceptHandler(self, n):
        if n.type is not None:
            self.visit(n.type)
        if n.name:
            self.cur.assigned.add(n.name)
        for st in n.body:
            self.visit(st)

    def visit_Yield(self, n):
        self.cur.generator = True
        self.generic_visit(n)

    visit_YieldFrom = visit_Yield


def _analyze(s, bound):
    """analyze_block: resolve every name of `s`; returns the names `s` needs
    from enclosing scopes (its free set)."""
    local = set(s.params) | s.assigned
    for name in s.all_names():
        if name in s.globals:
            s.scope[name] = GLOBAL_EXPLICIT
        elif name in s.nonlocals:
            s.scope[name] = FREE
        elif name in local:
            s.scope[name] = LOCAL
        elif s.kind != "module" and name in bound:
            s.scope[name] = FREE
        else:
            s.scope[name] = GLOBAL_IMPLICIT
    if s.kind == "function":
        child_bound = (bound | local) - s.globals
    elif s.kind == "class":
        child_bound = (bound - s.globals) | {"__class__"}
    else:
        child_bound = set()
    child_free = set()
    for c in s.children:
        child_free |= _analyze(c, child_bound)
    for name in child_free:
        if s.kind == "function" and s.scope.get(name) == LOCAL:
            s.scope[name] = CELL
        elif s.kind == "class" and name == "__class__":
            s.needs_class_closure = True
        elif s.kind != "module":
            if s.scope.get(name) in (None, GLOBAL_IMPLICIT):
                s.scope[name] = FREE
    s.free = {n for n, k in s.scope.items() if k == FREE}
    s.cells = {n for n, k in s.scope.items() if k == CELL}
    if s.kind == "class":
        s.free.discard("__class__")
        s.scope.pop("__class__", None)
    return set(s.free)


# ---------------------------------------------------------------- CFG

class Block:
    __slots__ = ("instrs", "next", "idx", "exit", "nofall", "preds", "label", "depth",
                 "visited", "exc", "lasti")  # the last three: 3.11 exception labelling

    def __init__(self, idx):
        self.instrs = []     # [opname, arg, target Block | None, lineno]
        self.next = None
        self.idx = idx
        self.exit = False
        self.nofall = False
        self.preds = 0
        self.label = None
        self.depth = -1
        self.visited = False
        self.exc = None
        self.lasti = False


def _is_jump(ins):
    return ins[0] in JUMPS


class FBlock:
    __slots__ = ("kind", "block", "exit", "datum")

    def __init__(self, kind, block, exit_, datum):
        self.kind, self.block, self.exit, self.datum = kind, block, exit_, datum


class Unit:
    """One code object being compiled (compiler_unit)."""

    def __init__(self, scope, name, qualname, firstlineno, kind, minor=10):
        self.minor = minor
        self.scope = scope
        self.name = name
        self.qualname = qualname
        self.firstlineno = firstlineno
        self.kind = kind     # module | class | function | lambda | comprehension
        self.consts = []
        self.const_idx = {}
        self.names = []
        self.varnames = list(scope.params)
        self.cellvars = sorted(scope.cells)
        if scope.needs_class_closure:
            self.cellvars = ["__class__"]
        self.freevars = sorted(scope.free)
        self.blocks = []       # creation order
        self.fblocks = []
        self.lineno = firstlineno
        self.entry = self.new_block()
        self.cur = self.entry
        self.order = [self.entry]
        self.argcount = self.posonly = self.kwonly = 0

    def new_block(self):
        b = Block(len(getattr(self, "blocks", [])))
        self.blocks.append(b)
        return b

    def use(self, b):
        self.cur.next = b
        self.cur = b
        self.order.append(b)

    def next_block(self):
        self.use(self.new_block())

    # pools
    def const(self, v):
        c = v if isinstance(v, Const) else _const(v)
        key = (c._key(), id(c.value) if c.kind == "code" else 0)
        i = self.const_idx.get(key)
        if i is None:
            i = self.const_idx[key] = len(self.consts)
            self.consts.append(c)
        return i

    def name_idx(self, s):
        if s not in self.names:
            self.names.append(s)
        return self.names.index(s)

    def var_idx(self, s):
        if s not in self.varnames:
            self.varnames.append(s)
        return self.varnames.index(s)

    def deref_idx(self, s):
        if s in self.cellvars:
            return self.cellvars.index(s)
        return len(self.cellvars) + self.freevars.index(s)

    def emit(self, op, arg=None, target=None, lineno=None):
        b = self.cur
        if b.instrs and (b.instrs[-1][0] in JUMPS or b.instrs[-1][0] in EXITS):
            self.next_block()
            b = self.cur
        b.instrs.append([op, arg, target, self.lineno if lineno is None else lineno])


def _const(v):
    if v is None:
        return Const("none")
    if v is Ellipsis:
        return Const("ellipsis")
    if isinstance(v, bool):
        return Const("bool", v)
    if isinstance(v, int):
        return Const("int", v)
    if isinstance(v, float):
        return Const("float", v)
    if isinstance(v, complex):
        return Const("complex", v)
    if isinstance(v, str):
        return Const("str", v)
    if isinstance(v, bytes):
        return Const("bytes", v)
    if isinstance(v, tuple):
        return Const("tuple", tuple(_const(x) for x in v))
    if isinstance(v, frozenset):
        return Const("frozenset", tuple(_const(x) for x in v))
    if isinstance(v, CodeObject):
        return Const("code", v)
    raise CompileError(f"unsupported constant {type(v).__name__}")


def _truthy(c):
    k, v = c.kind, c.value
    if k == "none":
        return False
    if k == "ellipsis" or k == "code":
        return True
    if k in ("tuple", "frozenset"):
        return len(v) > 0
    return bool(v)


# ---------------------------------------------------------------- the compiler

class Compiler:
    MINORS = (10,)

    def __init__(self, source, filename="<corpus>", minor=10):
        if minor not in self.MINORS:
            raise CompileError(f"{type(self).__name__} targets CPython 3.{self.MINORS[0]} bytecode")
        self.minor = minor
        self.filename = filename
        tree = ast.parse(source, filename)
        tree = ast.fix_missing_locations(_Folder().visit(tree))
        sb = _ScopeBuilder()
        sb.visit(tree)
        self.scopes = sb.by_node
        _analyze(self.scopes[id(tree)], set())
        self.tree = tree
        self.u = None
        self.stack = []

    # ------------------------------------------------------------ units
    def _new_unit(self, scope, name, qual, firstlineno, kind):
        return Unit(scope, name, qual, firstlineno, kind)

    def compile_module(self):
        s = self.scopes[id(self.tree)]
        self.u = self._new_unit(s, "<module>", "<module>", 1, "module")
        body = self.tree.body
        if body:
            self.u.lineno = body[0].lineno
        self._body(body)
        return self._assemble(add_none=True)

    def _enter(self, node, name, kind, firstlineno):
        scope = self.scopes[id(node)]
        parent = self.u
        qual = name
        if parent is not None and parent.kind != "module":
            force_global = False
            if kind in ("function", "class") and parent.scope.lookup(name) == GLOBAL_EXPLICIT:
                force_global = True
            if not force_global:
                if parent.kind in ("function", "lambda"):
                    qual = f"{parent.qualname}.<locals>.{name}"
                else:
                    qual = f"{parent.qualname}.{name}"
        self.stack.append(self.u)
        self.u = self._new_unit(scope, name, qual, firstlineno, kind)
        return self.u

    def _exit(self):
        self.u = self.stack.pop()

    def _flags(self):
        u = self.u
        s = u.scope
        flags = 0
        if u.kind in ("function", "lambda", "comprehension"):
            flags |= CO_OPTIMIZED | CO_NEWLOCALS
            if s.nested:
                flags |= CO_NESTED
            if s.generator:
                flags |= CO_GENERATOR
            if s.varargs:
                flags |= CO_VARARGS
            if s.varkw:
                flags |= CO_VARKEYWORDS
        if not u.cellvars and not u.freevars:
            flags |= CO_NOFREE
        return flags

    def _assemble(self, add_none):
        u = self.u
        last = u.cur
        if not any(i[0] == "RETURN_VALUE" for i in last.instrs):
            saved = u.lineno
            u.lineno = -1
            if add_none:
                u.emit("LOAD_CONST", u.const(None))
            u.emit("RETURN_VALUE")
            u.lineno = saved
        flags = self._flags()
        if flags & CO_GENERATOR:
            u.entry.instrs.insert(0, ["GEN_START", 0, None, -1])
        _optimize(u)
        stacksize = _stackdepth(u)
        items = []
        lab = {}
        for b in _chain(u.entry):
            lab[id(b)] = Label(f"B{b.idx}")
        for b in _chain(u.entry):
            items.append(lab[id(b)])
            for op, arg, tgt, _ln in b.instrs:
                if tgt is not None:
                    items.append((op, lab[id(tgt)]))
                else:
                    items.append((op, arg))
        code = assemble(items, self.minor)
        return CodeObject(
            VersionTag(3, self.minor), u.argcount, u.posonly, u.kwonly, len(u.varnames), stacksize, flags,
            code, tuple(u.consts), tuple(u.names), tuple(u.varnames), tuple(u.freevars),
            tuple(u.cellvars), u.name, self.filename, u.firstlineno, b"", b"",
            # co_qualname exists from 3.11 on; a 3.10 code object's qualname is its name
            u.qualname if self.minor >= 11 else "")

    # ------------------------------------------------------------ helpers
    def emit(self, op, arg=None, target=None):
        self.u.emit(op, arg, target)

    def load_const(self, v):
        self.emit("LOAD_CONST", self.u.const(v))

    def nameop(self, name, ctx):
        u = self.u
        sc = u.scope.lookup(name)
        if name == "__class__" and u.kind == "class" and u.scope.needs_class_closure:
            sc = CELL
        if u.kind == "class" and name in u.freevars and sc == GLOBAL_IMPLICIT:
            sc = FREE
        fn = u.kind in ("function", "lambda", "comprehension")
        op_kind = "NAME"
        if sc in (FREE, CELL):
            op_kind = "DEREF"
        elif sc == LOCAL and fn:
            op_kind = "FAST"
        elif sc == GLOBAL_IMPLICIT and fn:
            op_kind = "GLOBAL"
        elif sc == GLOBAL_EXPLICIT:
            op_kind = "GLOBAL"
        verb = {"load": "LOAD", "store": "STORE", "del": "DELETE"}[ctx]
        if op_kind == "DEREF":
            op = f"{verb}_DEREF"
            if ctx == "load" and u.kind == "class":
                op = "LOAD_CLASSDEREF"
            self.emit(op, u.deref_idx(name))
        elif op_kind == "FAST":
            self.emit(f"{verb}_FAST", u.var_idx(name))
        else:
            self.emit(f"{verb}_{op_kind}", u.name_idx(name))

    def _push_fb(self, kind, block, exit_=None, datum=None):
        self.u.fblocks.append(FBlock(kind, block, exit_, datum))

    def _pop_fb(self):
        self.u.fblocks.pop()

    def _set_loc(self, node):
        self.u.lineno = node.lineno

    # ------------------------------------------------------------ statements
    def _body(self, stmts):
        """compiler_body: docstring of modules / classes -> __doc__."""
        i = 0
        if stmts and _docstring(stmts) is not None:
            self._set_loc(stmts[0])
            self.expr(stmts[0].value)
            self.nameop("__doc__", "store")
            i = 1
        for st in stmts[i:]:
            self.stmt(st)

    def stmt(self, s):
        self._set_loc(s)
        m = getattr(self, "s_" + type(s).__name__, None)
        if m is None:
            raise CompileError(f"unsupported statement {type(s).__name__}")
        m(s)

    def stmts(self, seq):
        for s in seq:
            self.stmt(s)

    def s_Expr(self, s):
        if isinstance(s.value, ast.Constant):
            self.emit("NOP")
            return
        self.expr(s.value)
        self.emit("POP_TOP")

    def s_Pass(self, s):
        self.emit("NOP")

    def s_Assign(self, s):
        self.expr(s.value)
        n = len(s.targets)
        for i, t in enumerate(s.targets):
            if i < n - 1:
                self.emit("DUP_TOP")
            self.store(t)

    def s_AugAssign(self, s):
        e = s.target
        old = self.u.lineno
        self._set_loc(e)
        if isinstance(e, ast.Attribute):
            self.expr(e.value)
            self.emit("DUP_TOP")
            self.u.lineno = e.end_lineno
            self.emit("LOAD_ATTR", self.u.name_idx(e.attr))
        elif isinstance(e, ast.Subscript):
            self.expr(e.value)
            self.expr(e.slice)
            self.emit("DUP_TOP_TWO")
            self.emit("BINARY_SUBSCR")
        else:
            self.nameop(e.id, "load")
        self.u.lineno = old
        self.expr(s.value)
        self.emit("INPLACE_" + BINOP[type(s.op)])
        self._set_loc(e)
        if isinstance(e, ast.Attribute):
            self.u.lineno = e.end_lineno
            self.emit("ROT_TWO")
            self.emit("STORE_ATTR", self.u.name_idx(e.attr))
        elif isinstance(e, ast.Subscript):
            self.emit("ROT_THREE")
            self.emit("STORE_SUBSCR")
        else:
            self.nameop(e.id, "store")

    def s_Delete(self, s):
        for t in s.targets:
            self.delete(t)

    def delete(self, t):
        if isinstance(t, ast.Name):
            self.nameop(t.id, "del")
        elif isinstance(t, ast.Attribute):
            self.expr(t.value)
            self.emit("DELETE_ATTR", self.u.name_idx(t.attr))
        elif isinstance(t, ast.Subscript):
            self.expr(t.value)
            self.expr(t.slice)
            self.emit("DELETE_SUBSCR")
        elif isinstance(t, (ast.Tuple, ast.List)):
            for e in t.elts:
                self.delete(e)
        else:
            raise CompileError("bad delete target")

    def s_Return(self, s):
        v = s.value
        preserve = v is not None and not isinstance(v, ast.Constant)
        if preserve:
            self.expr(v)
        elif v is not None:
            self._set_loc(v)
            self.emit("NOP")
        if v is None or v.lineno != s.lineno:
            self._set_loc(s)
            self.emit("NOP")
        self.unwind_stack(preserve, None)
        if v is None:
            self.load_const(None)
        elif not preserve:
            self.load_const(v.value)
        self.emit("RETURN_VALUE")
        self.u.next_block()

    def s_Raise(self, s):
        n = 0
        if s.exc is not None:
            self.expr(s.exc)
            n = 1
            if s.cause is not None:
                self.expr(s.cause)
                n = 2
        self.emit("RAISE_VARARGS", n)
        self.u.next_block()

    def s_Assert(self, s):
        end = self.u.new_block()
        self.jump_if(s.test, end, True)
        self.emit("LOAD_ASSERTION_ERROR")
        if s.msg is not None:
            self.expr(s.msg)
            self.emit("CALL_FUNCTION", 1)
        self.emit("RAISE_VARARGS", 1)
        self.u.use(end)

    def s_Global(self, s):
        pass

    s_Nonlocal = s_Global

    def s_Break(self, s):
        self.emit("NOP")
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise CompileError("'break' outside loop")
        self.unwind(loop, False)
        self.emit("JUMP_ABSOLUTE", target=loop.exit)
        self.u.next_block()

    def s_Continue(self, s):
        self.emit("NOP")
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise CompileError("'continue' not properly in loop")
        self.emit("JUMP_ABSOLUTE", target=loop.block)
        self.u.next_block()

    def s_If(self, s):
        u = self.u
        end = u.new_block()
        nxt = u.new_block() if s.orelse else end
        self.jump_if(s.test, nxt, False)
        self.stmts(s.body)
        if s.orelse:
            self.emit_noline("JUMP_FORWARD", end)
            u.use(nxt)
            self.stmts(s.orelse)
        u.use(end)

    def s_While(self, s):
        u = self.u
        loop, body, anchor, end = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        u.use(loop)
        self._push_fb("WHILE_LOOP", loop, end)
        self.jump_if(s.test, anchor, False)
        u.use(body)
        self.stmts(s.body)
        self._set_loc(s)
        self.jump_if(s.test, body, True)
        self._pop_fb()
        u.use(anchor)
        if s.orelse:
            self.stmts(s.orelse)
        u.use(end)

    def s_For(self, s):
        u = self.u
        start, body, cleanup, end = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        self._push_fb("FOR_LOOP", start, end)
        self.expr(s.iter)
        self.emit("GET_ITER")
        u.use(start)
        self.emit("FOR_ITER", target=cleanup)
        u.use(body)
        self.store(s.target)
        self.stmts(s.body)
        self.emit_noline("JUMP_ABSOLUTE", start)
        u.use(cleanup)
        self._pop_fb()
        self.stmts(s.orelse)
        u.use(end)

    def emit_noline(self, op, target=None, arg=None):
        saved = self.u.lineno
        self.u.lineno = -1
        self.emit(op, arg, target)
        self.u.lineno = saved

    def s_Try(self, s):
        if s.finalbody:
            self.try_finally(s)
        else:
            self.try_except(s)

    def try_finally(self, s):
        u = self.u
        body, end, exit_ = u.new_block(), u.new_block(), u.new_block()
        self.emit("SETUP_FINALLY", target=end)
        u.use(body)
        self._push_fb("FINALLY_TRY", body, end, s.finalbody)
        if s.handlers:
            self.try_except(s)
        else:
            self.stmts(s.body)
        self.emit_noline("POP_BLOCK")
        self._pop_fb()
        self.stmts(s.finalbody)
        self.emit_noline("JUMP_FORWARD", exit_)
        u.use(end)
        self._push_fb("FINALLY_END", end)
        self.stmts(s.finalbody)
        self._pop_fb()
        self.emit("RERAISE", 0)
        u.use(exit_)

    def try_except(self, s):
        u = self.u
        body, except_, orelse, end = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        self.emit("SETUP_FINALLY", target=except_)
        u.use(body)
        self._push_fb("TRY_EXCEPT", body)
        self.stmts(s.body)
        self._pop_fb()
        self.emit_noline("POP_BLOCK")
        self.emit_noline("JUMP_FORWARD", orelse)
        n = len(s.handlers)
        u.use(except_)
        self._push_fb("EXCEPTION_HANDLER", None)
        for i, h in enumerate(s.handlers):
            self._set_loc(h)
            if h.type is None and i < n - 1:
                raise CompileError("default 'except:' must be last")
            except_ = u.new_block()
            if h.type is not None:
                self.emit("DUP_TOP")
                self.expr(h.type)
                self.emit("JUMP_IF_NOT_EXC_MATCH", target=except_)
                u.next_block()
            self.emit("POP_TOP")
            if h.name:
                cleanup_end, cleanup_body = u.new_block(), u.new_block()
                self.nameop(h.name, "store")
                self.emit("POP_TOP")
                self.emit("SETUP_FINALLY", target=cleanup_end)
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, None, h.name)
                self.stmts(h.body)
                self._pop_fb()
                u.lineno = -1
                self.emit("POP_BLOCK")
                self.emit("POP_EXCEPT")
                self.load_const(None)
                self.nameop(h.name, "store")
                self.nameop(h.name, "del")
                self.emit("JUMP_FORWARD", target=end)
                u.use(cleanup_end)
                u.lineno = -1
                self.load_const(None)
                self.nameop(h.name, "store")
                self.nameop(h.name, "del")
                self.emit("RERAISE", 1)
            else:
                cleanup_body = u.new_block()
                self.emit("POP_TOP")
                self.emit("POP_TOP")
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, None, None)
                self.stmts(h.body)
                self._pop_fb()
                u.lineno = -1
                self.emit("POP_EXCEPT")
                self.emit("JUMP_FORWARD", target=end)
            u.use(except_)
        self._pop_fb()
        u.lineno = -1
        self.emit("RERAISE", 0)
        u.use(orelse)
        self.stmts(s.orelse)
        u.use(end)

    def s_With(self, s, pos=0):
        u = self.u
        item = s.items[pos]
        block, final, exit_ = u.new_block(), u.new_block(), u.new_block()
        self.expr(item.context_expr)
        self.emit("SETUP_WITH", target=final)
        u.use(block)
        self._push_fb("WITH", block, final, s)
        if item.optional_vars is not None:
            self.store(item.optional_vars)
        else:
            self.emit("POP_TOP")
        if pos + 1 == len(s.items):
            self.stmts(s.body)
        else:
            self.s_With(s, pos + 1)
        u.lineno = -1
        self.emit("POP_BLOCK")
        self._pop_fb()
        self._set_loc(s)
        self.call_exit_with_nones()
        self.emit("POP_TOP")
        self.emit("JUMP_FORWARD", target=exit_)
        u.use(final)
        self.emit("WITH_EXCEPT_START")
        ex = u.new_block()
        self.emit("POP_JUMP_IF_TRUE", target=ex)
        u.next_block()
        self.emit("RERAISE", 1)
        u.use(ex)
        for op in ("POP_TOP", "POP_TOP", "POP_TOP", "POP_EXCEPT", "POP_TOP"):
            self.emit(op)
        u.use(exit_)

    def call_exit_with_nones(self):
        self.load_const(None)
        self.emit("DUP_TOP")
        self.emit("DUP_TOP")
        self.emit("CALL_FUNCTION", 3)

    # frame-block unwinding (compiler_unwind_fblock / _stack)
    def unwind(self, fb, preserve):
        u = self.u
        k = fb.kind
        if k in ("WHILE_LOOP", "EXCEPTION_HANDLER"):
            return
        if k == "FOR_LOOP":
            if preserve:
                self.emit("ROT_TWO")
            self.emit("POP_TOP")
        elif k == "TRY_EXCEPT":
            self.emit("POP_BLOCK")
        elif k == "FINALLY_TRY":
            self.emit("POP_BLOCK")
            if preserve:
                self._push_fb("POP_VALUE", None)
            self.stmts(fb.datum)
            if preserve:
                self._pop_fb()
            u.lineno = -1
        elif k == "FINALLY_END":
            if preserve:
                self.emit("ROT_FOUR")
            self.emit("POP_TOP")
            self.emit("POP_TOP")
            self.emit("POP_TOP")
            if preserve:
                self.emit("ROT_FOUR")
            self.emit("POP_EXCEPT")
        elif k == "WITH":
            self._set_loc(fb.datum)
            self.emit("POP_BLOCK")
            if preserve:
                self.emit("ROT_TWO")
            self.call_exit_with_nones()
            self.emit("POP_TOP")
            u.lineno = -1
        elif k == "HANDLER_CLEANUP":
            if fb.datum:
                self.emit("POP_BLOCK")
            if preserve:
                self.emit("ROT_FOUR")
            self.emit("POP_EXCEPT")
            if fb.datum:
                self.load_const(None)
                self.nameop(fb.datum, "store")
                self.nameop(fb.datum, "del")
        elif k == "POP_VALUE":
            if preserve:
                self.emit("ROT_TWO")
            self.emit("POP_TOP")

    def unwind_stack(self, preserve, loop):
        u = self.u
        if not u.fblocks:
            return None
        top = u.fblocks[-1]
        if loop is not None and top.kind in ("WHILE_LOOP", "FOR_LOOP"):
            return top
        u.fblocks.pop()
        self.unwind(top, preserve)
        r = self.unwind_stack(preserve, loop)
        u.fblocks.append(top)
        return r

    def s_Import(self, s):
        for a in s.names:
            self.load_const(0)
            self.load_const(None)
            self.emit("IMPORT_NAME", self.u.name_idx(a.name))
            if a.asname:
                parts = a.name.split(".")
                if len(parts) > 1:
                    for j, attr in enumerate(parts[1:]):
                        self.emit("IMPORT_FROM", self.u.name_idx(attr))
                        if j + 2 < len(parts):
                            self.emit("ROT_TWO")
                            self.emit("POP_TOP")
                    self.nameop(a.asname, "store")
                    self.emit("POP_TOP")
                else:
                    self.nameop(a.asname, "store")
            else:
                self.nameop(a.name.split(".")[0], "store")

    def s_ImportFrom(self, s):
        self.load_const(s.level)
        self.load_const(tuple(a.name for a in s.names))
        self.emit("IMPORT_NAME", self.u.name_idx(s.module or ""))
        for a in s.names:
            if a.name == "*":
                self.emit("IMPORT_STAR")
                return
            self.emit("IMPORT_FROM", self.u.name_idx(a.name))
            self.nameop(a.asname or a.name, "store")
        self.emit("POP_TOP")

    def s_FunctionDef(self, s):
        for d in s.decorator_list:
            self.expr(d)
        firstlineno = s.decorator_list[0].lineno if s.decorator_list else s.lineno
        flags = self.default_args(s.args)
        doc = _docstring(s.body)
        self._enter(s, s.name, "function", firstlineno)
        u = self.u
        u.const(doc if doc is not None else None)
        self._params(s.args)
        for st in s.body[1 if doc is not None else 0:]:
            self.stmt(st)
        co = self._assemble(add_none=True)
        qual = u.qualname
        self._exit()
        self._set_loc(s)
        self.make_closure(co, flags, qual)
        for _ in s.decorator_list:
            self.emit("CALL_FUNCTION", 1)
        self.nameop(s.name, "store")

    def _params(self, a):
        u = self.u
        u.argcount = len(a.posonlyargs) + len(a.args)
        u.posonly = len(a.posonlyargs)
        u.kwonly = len(a.kwonlyargs)

    def default_args(self, a):
        flags = 0
        if a.defaults:
            for d in a.defaults:
                self.expr(d)
            self.emit("BUILD_TUPLE", len(a.defaults))
            flags |= 1
        keys = []
        for arg, d in zip(a.kwonlyargs, a.kw_defaults):
            if d is not None:
                keys.append(arg.arg)
                self.expr(d)
        if keys:
            self.load_const(tuple(keys))
            self.emit("BUILD_CONST_KEY_MAP", len(keys))
            flags |= 2
        return flags

    def make_closure(self, co, flags, qualname):
        if co.freevars:
            for name in co.freevars:
                self.emit("LOAD_CLOSURE", self.u.deref_idx(name))
            flags |= 8
            self.emit("BUILD_TUPLE", len(co.freevars))
        self.load_const(co)
        self.load_const(qualname)
        self.emit("MAKE_FUNCTION", flags)

    def s_ClassDef(self, s):
        for d in s.decorator_list:
            self.expr(d)
        firstlineno = s.decorator_list[0].lineno if s.decorator_list else s.lineno
        self._enter(s, s.name, "class", firstlineno)
        u = self.u
        u.lineno = s.lineno
        self.nameop("__name__", "load")
        self.nameop("__module__", "store")
        self.load_const(u.qualname)
        self.nameop("__qualname__", "store")
        self._body(s.body)
        u.lineno = -1
        if u.scope.needs_class_closure:
            self.emit("LOAD_CLOSURE", 0)
            self.emit("DUP_TOP")
            self.nameop("__classcell__", "store")
        else:
            self.load_const(None)
        self.emit("RETURN_VALUE")
        co = self._assemble(add_none=True)
        self._exit()
        self._set_loc(s)
        self.emit("LOAD_BUILD_CLASS")
        self.make_closure(co, 0, co.name)
        self.load_const(s.name)
        self.call_helper(2, s.bases, s.keywords)
        for _ in s.decorator_list:
            self.emit("CALL_FUNCTION", 1)
        self.nameop(s.name, "store")

    # ------------------------------------------------------------ stores
    def store(self, t):
        if isinstance(t, ast.Name):
            self.nameop(t.id, "store")
        elif isinstance(t, ast.Attribute):
            old = self.u.lineno
            self._set_loc(t)
            self.expr(t.value)
            self.emit("STORE_ATTR", self.u.name_idx(t.attr))
            self.u.lineno = old
        elif isinstance(t, ast.Subscript):
            old = self.u.lineno
            self._set_loc(t)
            self.expr(t.value)
            self.expr(t.slice)
            self.emit("STORE_SUBSCR")
            self.u.lineno = old
        elif isinstance(t, (ast.Tuple, ast.List)):
            n = len(t.elts)
            star = [i for i, e in enumerate(t.elts) if isinstance(e, ast.Starred)]
            if star:
                i = star[0]
                self.emit("UNPACK_EX", i + ((n - i - 1) << 8))
            else:
                self.emit("UNPACK_SEQUENCE", n)
            for e in t.elts:
                self.store(e.value if isinstance(e, ast.Starred) else e)
        else:
            raise CompileError(f"bad store target {type(t).__name__}")

    # ------------------------------------------------------------ expressions
    def expr(self, e):
        u = self.u
        old = u.lineno
        u.lineno = e.lineno
        m = getattr(self, "e_" + type(e).__name__, None)
        if m is None:
            raise CompileError(f"unsupported expression {type(e).__name__}")
        m(e)
        u.lineno = old

    def e_Constant(self, e):
        self.load_const(e.value)

    def e_Name(self, e):
        self.nameop(e.id, "load")

    def e_BinOp(self, e):
        self.expr(e.left)
        self.expr(e.right)
        self.emit("BINARY_" + BINOP[type(e.op)])

    def e_UnaryOp(self, e):
        self.expr(e.operand)
        self.emit(UNOP[type(e.op)])

    def e_BoolOp(self, e):
        end = self.u.new_block()
        op = "JUMP_IF_FALSE_OR_POP" if isinstance(e.op, ast.And) else "JUMP_IF_TRUE_OR_POP"
        for v in e.values[:-1]:
            self.expr(v)
            self.emit(op, target=end)
            self.u.next_block()
        self.expr(e.values[-1])
        self.u.use(end)

    def compare_op(self, op):
        if isinstance(op, (ast.Is, ast.IsNot)):
            self.emit("IS_OP", int(isinstance(op, ast.IsNot)))
        elif isinstance(op, (ast.In, ast.NotIn)):
            self.emit("CONTAINS_OP", int(isinstance(op, ast.NotIn)))
        else:
            self.emit("COMPARE_OP", CMPOP[type(op)])

    def e_Compare(self, e):
        u = self.u
        self.expr(e.left)
        n = len(e.ops) - 1
        if n == 0:
            self.expr(e.comparators[0])
            self.compare_op(e.ops[0])
            return
        cleanup = u.new_block()
        for i in range(n):
            self.expr(e.comparators[i])
            self.emit("DUP_TOP")
            self.emit("ROT_THREE")
            self.compare_op(e.ops[i])
            self.emit("JUMP_IF_FALSE_OR_POP", target=cleanup)
            u.next_block()
        self.expr(e.comparators[n])
        self.compare_op(e.ops[n])
        end = u.new_block()
        self.emit_noline("JUMP_FORWARD", end)
        u.use(cleanup)
        self.emit("ROT_TWO")
        self.emit("POP_TOP")
        u.use(end)

    def jump_if(self, e, nxt, cond):
        """compiler_jump_if."""
        u = self.u
        old = u.lineno
        u.lineno = e.lineno
        try:
            if isinstance(e, ast.UnaryOp) and isinstance(e.op, ast.Not):
                return self.jump_if(e.operand, nxt, not cond)
            if isinstance(e, ast.BoolOp):
                cond2 = isinstance(e.op, ast.Or)
                nxt2 = nxt
                if cond2 != cond:
                    nxt2 = u.new_block()
                for v in e.values[:-1]:
                    self.jump_if(v, nxt2, cond2)
                self.jump_if(e.values[-1], nxt, cond)
                if nxt2 is not nxt:
                    u.use(nxt2)
                return
            if isinstance(e, ast.IfExp):
                end, nxt2 = u.new_block(), u.new_block()
                self.jump_if(e.test, nxt2, False)
                self.jump_if(e.body, nxt, cond)
                self.emit_noline("JUMP_FORWARD", end)
                u.use(nxt2)
                self.jump_if(e.orelse, nxt, cond)
                u.use(end)
                return
            if isinstance(e, ast.Compare) and len(e.ops) > 1:
                n = len(e.ops) - 1
                cleanup = u.new_block()
                self.expr(e.left)
                for i in range(n):
                    self.expr(e.comparators[i])
                    self.emit("DUP_TOP")
                    self.emit("ROT_THREE")
                    self.compare_op(e.ops[i])
                    self.emit("POP_JUMP_IF_FALSE", target=cleanup)
                    u.next_block()
                self.expr(e.comparators[n])
                self.compare_op(e.ops[n])
                self.emit("POP_JUMP_IF_TRUE" if cond else "POP_JUMP_IF_FALSE", target=nxt)
                end = u.new_block()
                self.emit_noline("JUMP_FORWARD", end)
                u.use(cleanup)
                self.emit("POP_TOP")
                if not cond:
                    self.emit_noline("JUMP_FORWARD", nxt)
                u.use(end)
                return
            self.expr(e)
            self.emit("POP_JUMP_IF_TRUE" if cond else "POP_JUMP_IF_FALSE", target=nxt)
            u.next_block()
        finally:
            u.lineno = old

    def e_IfExp(self, e):
        u = self.u
        end, nxt = u.new_block(), u.new_block()
        self.jump_if(e.test, nxt, False)
        self.expr(e.body)
        self.emit_noline("JUMP_FORWARD", end)
        u.use(nxt)
        self.expr(e.orelse)
        u.use(end)

    def e_NamedExpr(self, e):
        self.expr(e.value)
        self.emit("DUP_TOP")
        self.store(e.target)

    def e_Attribute(self, e):
        self.expr(e.value)
        old = self.u.lineno
        self.u.lineno = e.end_lineno
        self.emit("LOAD_ATTR", self.u.name_idx(e.attr))
        self.u.lineno = old

    def e_Subscript(self, e):
        self.expr(e.value)
        self.expr(e.slice)
        self.emit("BINARY_SUBSCR")

    def e_Slice(self, e):
        n = 2
        if e.lower is not None:
            self.expr(e.lower)
        else:
            self.load_const(None)
        if e.upper is not None:
            self.expr(e.upper)
        else:
            self.load_const(None)
        if e.step is not None:
            self.expr(e.step)
            n = 3
        self.emit("BUILD_SLICE", n)

    def starunpack(self, elts, pushed, build, add, extend, tuple_):
        n = len(elts)
        if n > 2 and all(isinstance(x, ast.Constant) for x in elts):
            folded = tuple(x.value for x in elts)
            if tuple_:
                self.load_const(folded)
            else:
                if add == "SET_ADD":
                    folded = frozenset(folded)
                self.emit(build, pushed)
                self.load_const(folded)
                self.emit(extend, 1)
            return
        big = n + pushed > STACK_USE_GUIDELINE
        seen_star = any(isinstance(x, ast.Starred) for x in elts)
        if not seen_star and not big:
            for x in elts:
                self.expr(x)
            self.emit("BUILD_TUPLE" if tuple_ else build, n + pushed)
            return
        built = False
        if big:
            self.emit(build, pushed)
            built = True
        for i, x in enumerate(elts):
            if isinstance(x, ast.Starred):
                if not built:
                    self.emit(build, i + pushed)
                    built = True
                self.expr(x.value)
                self.emit(extend, 1)
            else:
                self.expr(x)
                if built:
                    self.emit(add, 1)
        if tuple_:
            self.emit("LIST_TO_TUPLE")

    def e_Tuple(self, e):
        self.starunpack(e.elts, 0, "BUILD_LIST", "LIST_APPEND", "LIST_EXTEND", True)

    def e_List(self, e):
        self.starunpack(e.elts, 0, "BUILD_LIST", "LIST_APPEND", "LIST_EXTEND", False)

    def e_Set(self, e):
        self.starunpack(e.elts, 0, "BUILD_SET", "SET_ADD", "SET_UPDATE", False)

    def subdict(self, e, begin, end):
        n = end - begin
        big = n * 2 > STACK_USE_GUIDELINE
        keys = e.keys[begin:end]
        if n > 1 and not big and all(isinstance(k, ast.Constant) for k in keys):
            for v in e.values[begin:end]:
                self.expr(v)
            self.load_const(tuple(k.value for k in keys))
            self.emit("BUILD_CONST_KEY_MAP", n)
            return
        if big:
            self.emit("BUILD_MAP", 0)
        for k, v in zip(keys, e.values[begin:end]):
            self.expr(k)
            self.expr(v)
            if big:
                self.emit("MAP_ADD", 1)
        if not big:
            self.emit("BUILD_MAP", n)

    def e_Dict(self, e):
        n = len(e.values)
        have = False
        elements = 0
        for i in range(n):
            if e.keys[i] is None:
                if elements:
                    self.subdict(e, i - elements, i)
                    if have:
                        self.emit("DICT_UPDATE", 1)
                    have = True
                    elements = 0
                if not have:
                    self.emit("BUILD_MAP", 0)
                    have = True
                self.expr(e.values[i])
                self.emit("DICT_UPDATE", 1)
            else:
                if elements * 2 > STACK_USE_GUIDELINE:
                    self.subdict(e, i - elements, i + 1)
                    if have:
                        self.emit("DICT_UPDATE", 1)
                    have = True
                    elements = 0
                else:
                    elements += 1
        if elements:
            self.subdict(e, n - elements, n)
            if have:
                self.emit("DICT_UPDATE", 1)
            have = True
        if not have:
            self.emit("BUILD_MAP", 0)

    def e_Call(self, e):
        f = e.func
        if (isinstance(f, ast.Attribute) and not e.keywords and len(e.args) < STACK_USE_GUIDELINE
                and not any(isinstance(a, ast.Starred) for a in e.args)):
            self.expr(f.value)
            old = self.u.lineno
            self.u.lineno = f.end_lineno
            self.emit("LOAD_METHOD", self.u.name_idx(f.attr))
            for a in e.args:
                self.expr(a)
            self.u.lineno = f.end_lineno
            self.emit("CALL_METHOD", len(e.args))
            self.u.lineno = old
            return
        self.expr(f)
        self.call_helper(0, e.args, e.keywords)

    def call_helper(self, n, args, keywords):
        if not any(isinstance(a, ast.Starred) for a in args) and not any(k.arg is None for k in keywords):
            for a in args:
                self.expr(a)
            if keywords:
                for k in keywords:
                    self.expr(k.value)
                self.load_const(tuple(k.arg for k in keywords))
                self.emit("CALL_FUNCTION_KW", n + len(args) + len(keywords))
            else:
                self.emit("CALL_FUNCTION", n + len(args))
            return
        if n == 0 and len(args) == 1 and isinstance(args[0], ast.Starred):
            self.expr(args[0].value)
        else:
            self.starunpack(args, n, "BUILD_LIST", "LIST_APPEND", "LIST_EXTEND", True)
        if keywords:
            have = False
            nseen = 0
            for i, k in enumerate(keywords):
                if k.arg is None:
                    if nseen:
                        self.subkwargs(keywords[i - nseen:i])
                        if have:
                            self.emit("DICT_MERGE", 1)
                        have = True
                        nseen = 0
                    if not have:
                        self.emit("BUILD_MAP", 0)
                        have = True
                    self.expr(k.value)
                    self.emit("DICT_MERGE", 1)
                else:
                    nseen += 1
            if nseen:
                self.subkwargs(keywords[len(keywords) - nseen:])
                if have:
                    self.emit("DICT_MERGE", 1)
        self.emit("CALL_FUNCTION_EX", int(bool(keywords)))

    def subkwargs(self, kws):
        n = len(kws)
        big = n * 2 > STACK_USE_GUIDELINE
        if n > 1 and not big:
            for k in kws:
                self.expr(k.value)
            self.load_const(tuple(k.arg for k in kws))
            self.emit("BUILD_CONST_KEY_MAP", n)
            return
        if big:
            self.emit_noline("BUILD_MAP", arg=0)
        for k in kws:
            self.load_const(k.arg)
            self.expr(k.value)
            if big:
                self.emit_noline("MAP_ADD", arg=1)
        if not big:
            self.emit("BUILD_MAP", n)

    def e_Lambda(self, e):
        flags = self.default_args(e.args)
        self._enter(e, "<lambda>", "lambda", e.lineno)
        u = self.u
        u.const(None)
        self._params(e.args)
        self.expr(e.body)
        if u.scope.generator:
            self.emit("POP_TOP")
            self.load_const(None)
        self.emit("RETURN_VALUE")
        co = self._assemble(add_none=False)
        qual = u.qualname
        self._exit()
        self.make_closure(co, flags, qual)

    def _comprehension(self, e, name, kind, elt, val=None):
        gens = e.generators
        self._enter(e, name, "comprehension", e.lineno)
        u = self.u
        u.argcount = 1
        if kind != "genexp":
            self.emit({"list": "BUILD_LIST", "set": "BUILD_SET", "dict": "BUILD_MAP"}[kind], 0)
        self._comp_gen(gens, 0, 0, elt, val, kind)
        if kind != "genexp":
            self.emit("RETURN_VALUE")
        co = self._assemble(add_none=True)
        qual = u.qualname
        self._exit()
        self.make_closure(co, 0, qual)
        self.expr(gens[0].iter)
        self.emit("GET_ITER")
        self.emit("CALL_FUNCTION", 1)

    def _comp_gen(self, gens, idx, depth, elt, val, kind):
        u = self.u
        start, if_cleanup, anchor = u.new_block(), u.new_block(), u.new_block()
        g = gens[idx]
        if idx == 0:
            self.emit("LOAD_FAST", 0)
        else:
            it = g.iter
            elts = it.elts if isinstance(it, (ast.List, ast.Tuple)) else None
            if elts is not None and len(elts) == 1 and not isinstance(elts[0], ast.Starred):
                self.expr(elts[0])
                start = None
            elif isinstance(it, ast.Constant) and isinstance(it.value, tuple) and len(it.value) == 1:
                self.load_const(it.value[0])
                start = None
            if start is not None:
                self.expr(it)
                self.emit("GET_ITER")
        if start is not None:
            depth += 1
            u.use(start)
            self.emit("FOR_ITER", target=anchor)
            u.next_block()
        self.store(g.target)
        for c in g.ifs:
            self.jump_if(c, if_cleanup, False)
            u.next_block()
        idx += 1
        if idx < len(gens):
            self._comp_gen(gens, idx, depth, elt, val, kind)
        else:
            if kind == "genexp":
                self.expr(elt)
                self.emit("YIELD_VALUE")
                self.emit("POP_TOP")
            elif kind == "list":
                self.expr(elt)
                self.emit("LIST_APPEND", depth + 1)
            elif kind == "set":
                self.expr(elt)
                self.emit("SET_ADD", depth + 1)
            else:
                self.expr(elt)
                self.expr(val)
                self.emit("MAP_ADD", depth + 1)
        u.use(if_cleanup)
        if start is not None:
            self.emit("JUMP_ABSOLUTE", target=start)
            u.use(anchor)

    def e_ListComp(self, e):
        self._comprehension(e, "<listcomp>", "list", e.elt)

    def e_SetComp(self, e):
        self._comprehension(e, "<setcomp>", "set", e.elt)

    def e_GeneratorExp(self, e):
        self._comprehension(e, "<genexpr>", "genexp", e.elt)

    def e_DictComp(self, e):
        self._comprehension(e, "<dictcomp>", "dict", e.key, e.value)

    def e_Yield(self, e):
        if e.value is not None:
            self.expr(e.value)
        else:
            self.load_const(None)
        self.emit("YIELD_VALUE")

    def e_YieldFrom(self, e):
        self.expr(e.value)
        self.emit("GET_YIELD_FROM_ITER")
        self.load_const(None)
        self.emit("YIELD_FROM")

    def e_JoinedStr(self, e):
        for v in e.values:
            self.expr(v)
        if len(e.values) != 1:
            self.emit("BUILD_STRING", len(e.values))

    def e_FormattedValue(self, e):
        self.expr(e.value)
        oparg = {-1: 0, 115: 1, 114: 2, 97: 3}[e.conversion]
        if e.format_spec is not None:
            self.expr(e.format_spec)
            oparg |= 4
        self.emit("FORMAT_VALUE", oparg)

    def e_Starred(self, e):
        raise CompileError("can't use starred expression here")


def _docstring(body):
    if body and isinstance(body[0], ast.Expr) and isinstance(body[0].value, ast.Constant) \
            and isinstance(body[0].value.value, str):
        return body[0].value.value
    return None


# ---------------------------------------------------------------- CFG optimiser (compile.c 3.10)

def _chain(entry):
    b = entry
    while b is not None:
        yield b
        b = b.next


def _first_nonempty(b):
    while b is not None and not b.instrs:
        b = b.next
    return b


def _normalize(u):
    for b in _chain(u.entry):
        b.exit = b.nofall = False
        for i, ins in enumerate(b.instrs):
            op = ins[0]
            if op in EXITS:
                b.exit = b.nofall = True
            elif op in JUMPS:
                if op in UNCOND:
                    b.nofall = True
                if i != len(b.instrs) - 1:
                    raise CompileError("malformed control flow graph")
                ins[2] = _first_nonempty(ins[2])


def _clean(b, prev_lineno):
    """clean_basic_block: drop NOPs whose line number is redundant."""
    out = []
    ins = b.instrs
    for src in range(len(ins)):
        cur = ins[src]
        lineno = cur[3]
        if cur[0] == "NOP":
            if lineno < 0:
                continue
            if prev_lineno == lineno:
                continue
            if src < len(ins) - 1:
                nl = ins[src + 1][3]
                if nl < 0 or nl == lineno:
                    ins[src + 1][3] = lineno
                    continue
            else:
                nxt = _first_nonempty(b.next)
                if nxt is not None and lineno == nxt.instrs[0][3]:
                    continue
        out.append(cur)
        prev_lineno = lineno
    b.instrs = out


def _optimize_block(u, b):
    i = 0
    while i < len(b.instrs):
        ins = b.instrs[i]
        op = ins[0]
        nxt = b.instrs[i + 1] if i + 1 < len(b.instrs) else None
        nextop = nxt[0] if nxt else None
        tgt = None
        if op in JUMPS:
            ins[2] = _first_nonempty(ins[2])
            tgt = ins[2].instrs[0]
        redo = False
        if op == "LOAD_CONST" and nextop in ("POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE"):
            is_true = _truthy(u.consts[ins[1]])
            ins[0] = "NOP"
            if is_true == (nextop == "POP_JUMP_IF_TRUE"):
                nxt[0] = "JUMP_ABSOLUTE"
                b.nofall = True
            else:
                nxt[0] = "NOP"
                nxt[2] = None
        elif op == "LOAD_CONST" and nextop in ("JUMP_IF_FALSE_OR_POP", "JUMP_IF_TRUE_OR_POP"):
            is_true = _truthy(u.consts[ins[1]])
            if is_true == (nextop == "JUMP_IF_TRUE_OR_POP"):
                nxt[0] = "JUMP_ABSOLUTE"
                b.nofall = True
            else:
                ins[0] = "NOP"
                nxt[0] = "NOP"
                nxt[2] = None
        elif op == "BUILD_TUPLE":
            n = ins[1]
            if nextop == "UNPACK_SEQUENCE" and nxt[1] == n:
                if n == 1:
                    ins[0] = "NOP"
                    nxt[0] = "NOP"
                elif n == 2:
                    ins[0] = "ROT_TWO"
                    nxt[0] = "NOP"
                elif n == 3:
                    ins[0] = "ROT_THREE"
                    nxt[0] = "ROT_TWO"
            elif i >= n and all(b.instrs[j][0] == "LOAD_CONST" for j in range(i - n, i)):
                vals = tuple(u.consts[b.instrs[j][1]] for j in range(i - n, i))
                for j in range(i - n, i):
                    b.instrs[j][0] = "NOP"
                ins[0] = "LOAD_CONST"
                ins[1] = u.const(Const("tuple", vals))
        elif op == "JUMP_IF_FALSE_OR_POP" or op == "JUMP_IF_TRUE_OR_POP":
            same = "POP_JUMP_IF_FALSE" if op == "JUMP_IF_FALSE_OR_POP" else "POP_JUMP_IF_TRUE"
            other = "JUMP_IF_TRUE_OR_POP" if op == "JUMP_IF_FALSE_OR_POP" else "JUMP_IF_FALSE_OR_POP"
            t = tgt[0]
            if t == same:
                if ins[3] == tgt[3]:
                    ins[0], ins[1], ins[2] = tgt[0], tgt[1], tgt[2]
                    redo = True
            elif t in ("JUMP_ABSOLUTE", "JUMP_FORWARD", op):
                if ins[3] == tgt[3] and ins[2] is not tgt[2]:
                    ins[2] = tgt[2]
                    redo = True
            elif t == other:
                if ins[3] == tgt[3]:
                    ins[0] = same
                    ins[2] = ins[2].next
                    redo = True
        elif op in ("POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE"):
            if tgt[0] in UNCOND and ins[3] == tgt[3] and ins[2] is not tgt[2]:
                ins[2] = tgt[2]
                redo = True
        elif op in UNCOND:
            if tgt[0] in UNCOND:
                if ins[2] is not tgt[2]:
                    newop = "JUMP_FORWARD" if (op == "JUMP_FORWARD" and tgt[0] == "JUMP_FORWARD") else "JUMP_ABSOLUTE"
                    ins[0] = "NOP"
                    ins[2] = None
                    b.instrs.append([newop, None, tgt[2], tgt[3]])
        elif op == "FOR_ITER":
            if tgt[0] == "JUMP_FORWARD":
                ins[2] = tgt[2]
        if not redo:
            i += 1


def _extend_block(b):
    if not b.instrs:
        return
    last = b.instrs[-1]
    if last[0] not in UNCOND:
        return
    t = last[2]
    if t.exit and len(t.instrs) <= MAX_COPY_SIZE:
        last[0] = "NOP"
        last[2] = None
        b.instrs.extend([list(x) for x in t.instrs])
        b.exit = True


def _mark_reachable(u):
    for b in u.blocks:
        b.preds = 0
    u.entry.preds = 1
    stack = [u.entry]
    while stack:
        b = stack.pop()
        if b.next is not None and not b.nofall:
            if b.next.preds == 0:
                stack.append(b.next)
            b.next.preds += 1
        for ins in b.instrs:
            if ins[0] in JUMPS and ins[2] is not None:
                t = ins[2]
                if t.preds == 0:
                    stack.append(t)
                t.preds += 1


def _eliminate_empty(u):
    for b in _chain(u.entry):
        n = b.next
        if n is not None:
            while not n.instrs and n.next is not None:
                n = n.next
            b.next = n
    for b in _chain(u.entry):
        if b.instrs and b.instrs[-1][0] in JUMPS:
            b.instrs[-1][2] = _first_nonempty(b.instrs[-1][2])


def _optimize(u, optimize_block=None):
    optimize_block = optimize_block or _optimize_block
    _normalize(u)
    for b in _chain(u.entry):
        optimize_block(u, b)
        _clean(b, -1)
    for b in sorted(u.blocks, key=lambda x: -x.idx):
        _extend_block(b)
    _mark_reachable(u)
    for b in _chain(u.entry):
        if b.preds == 0:
            b.instrs = []
            b.nofall = False
    pred = None
    for b in _chain(u.entry):
        prev = pred.instrs[-1][3] if (pred is not None and pred.instrs) else -1
        _clean(b, prev)
        pred = None if b.nofall else b
    _eliminate_empty(u)
    changed = False
    for b in _chain(u.entry):
        if b.instrs and b.instrs[-1][0] in UNCOND and b.instrs[-1][2] is b.next:
            b.nofall = False
            b.instrs[-1][0] = "NOP"
            b.instrs[-1][2] = None
            _clean(b, -1)
            changed = True
    if changed:
        _eliminate_empty(u)
    # duplicate_exits_without_lineno
    _normalize(u)
    _mark_reachable(u)
    live = [b for b in _chain(u.entry)]
    for b in sorted(live, key=lambda x: -x.idx):
        if b.instrs and b.instrs[-1][0] in JUMPS and b.instrs[-1][0] not in SETUPS:
            t = b.instrs[-1][2]
            if t.exit and t.instrs[0][3] < 0 and t.preds > 1:
                nb = u.new_block()
                nb.instrs = [list(x) for x in t.instrs]
                nb.instrs[0][3] = b.instrs[-1][3]
                nb.exit = True
                nb.nofall = True
                b.instrs[-1][2] = nb
                t.preds -= 1
                nb.preds = 1
                nb.next = t.next
                t.next = nb
    for b in _chain(u.entry):
        while b.next is not None and not b.next.instrs:
            b.next = b.next.next
    if u.minor >= 11:
        return  # jump directions are chosen by normalize_jumps (pycodegen311.py)
    # relative jumps must point forward
    pos = {}
    k = 0
    for b in _chain(u.entry):
        pos[id(b)] = k
        k += 1
    for b in _chain(u.entry):
        if b.instrs and b.instrs[-1][0] == "JUMP_FORWARD" and pos[id(b.instrs[-1][2])] <= pos[id(b)]:
            b.instrs[-1][0] = "JUMP_ABSOLUTE"


# ---------------------------------------------------------------- stack depth

def _effect(op, arg, jump):
    fixed = {
        "NOP": 0, "POP_TOP": -1, "ROT_TWO": 0, "ROT_THREE": 0, "ROT_FOUR": 0, "DUP_TOP": 1, "DUP_TOP_TWO": 2,
        "UNARY_POSITIVE": 0, "UNARY_NEGATIVE": 0, "UNARY_NOT": 0, "UNARY_INVERT": 0, "GET_ITER": 0,
        "BINARY_SUBSCR": -1, "STORE_SUBSCR": -3, "DELETE_SUBSCR": -2, "LOAD_BUILD_CLASS": 1,
        "RETURN_VALUE": -1, "IMPORT_STAR": -1, "YIELD_VALUE": 0, "YIELD_FROM": -1, "POP_BLOCK": 0,
        "POP_EXCEPT": -3, "STORE_NAME": -1, "DELETE_NAME": 0, "STORE_ATTR": -2, "DELETE_ATTR": -1,
        "STORE_GLOBAL": -1, "DELETE_GLOBAL": 0, "LOAD_CONST": 1, "LOAD_NAME": 1, "LOAD_ATTR": 0,
        "COMPARE_OP": -1, "IS_OP": -1, "CONTAINS_OP": -1, "JUMP_IF_NOT_EXC_MATCH": -2, "IMPORT_NAME": -1,
        "IMPORT_FROM": 1, "JUMP_FORWARD": 0, "JUMP_ABSOLUTE": 0, "POP_JUMP_IF_FALSE": -1,
        "POP_JUMP_IF_TRUE": -1, "LOAD_GLOBAL": 1, "RERAISE": -3, "WITH_EXCEPT_START": 1, "LOAD_FAST": 1,
        "STORE_FAST": -1, "DELETE_FAST": 0, "LOAD_CLOSURE": 1, "LOAD_DEREF": 1, "LOAD_CLASSDEREF": 1,
        "STORE_DEREF": -1, "DELETE_DEREF": 0, "LOAD_METHOD": 1, "LIST_APPEND": -1, "SET_ADD": -1,
        "MAP_ADD": -2, "LIST_EXTEND": -1, "SET_UPDATE": -1, "DICT_UPDATE": -1, "DICT_MERGE": -1,
        "LIST_TO_TUPLE": 0, "GET_YIELD_FROM_ITER": 0, "LOAD_ASSERTION_ERROR": 1, "GEN_START": -1,
        "PRINT_EXPR": -1,
    }
    if op in fixed:
        return fixed[op]
    if op.startswith("BINARY_") or op.startswith("INPLACE_"):
        return -1
    if op == "UNPACK_SEQUENCE":
        return arg - 1
    if op == "UNPACK_EX":
        return (arg & 0xFF) + (arg >> 8)
    if op == "FOR_ITER":
        return -1 if jump else 1
    if op in ("BUILD_TUPLE", "BUILD_LIST", "BUILD_SET", "BUILD_STRING",
              # 3.8 (pycodegen38.py)
              "BUILD_TUPLE_UNPACK", "BUILD_LIST_UNPACK", "BUILD_SET_UNPACK", "BUILD_MAP_UNPACK",
              "BUILD_TUPLE_UNPACK_WITH_CALL", "BUILD_MAP_UNPACK_WITH_CALL"):
        return 1 - arg
    # 3.8 finally machinery (Python/compile.c 3.8 stack_effect)
    if op == "BEGIN_FINALLY":
        return 6
    if op in ("END_FINALLY", "POP_FINALLY"):
        return -6 if op == "END_FINALLY" else 0
    if op == "CALL_FINALLY":
        return 1 if jump else 0
    if op == "WITH_CLEANUP_START":
        return 2
    if op == "WITH_CLEANUP_FINISH":
        return -3
    if op == "BUILD_MAP":
        return 1 - 2 * arg
    if op == "BUILD_CONST_KEY_MAP":
        return -arg
    if op in ("JUMP_IF_TRUE_OR_POP", "JUMP_IF_FALSE_OR_POP"):
        return 0 if jump else -1
    if op == "SETUP_FINALLY":
        return 6 if jump else 0
    if op == "SETUP_WITH":
        return 6 if jump else 1
    if op == "RAISE_VARARGS":
        return -arg
    if op == "CALL_FUNCTION":
        return -arg
    if op == "CALL_METHOD":
        return -arg - 1
    if op == "CALL_FUNCTION_KW":
        return -arg - 1
    if op == "CALL_FUNCTION_EX":
        return -1 - (arg & 1)
    if op == "MAKE_FUNCTION":
        return -1 - bin(arg & 0xF).count("1")
    if op == "BUILD_SLICE":
        return -1 if arg == 2 else -2
    if op == "FORMAT_VALUE":
        return -1 if arg & 4 else 0
    raise CompileError(f"no stack effect for {op}")


def _stackdepth(u):
    blocks = list(_chain(u.entry))
    for b in blocks:
        b.depth = -1
    maxd = 0
    stack = []
    u.entry.depth = 0
    stack.append(u.entry)
    while stack:
        b = stack.pop()
        d = b.depth
        fall = True
        for op, arg, tgt, _ln in b.instrs:
            if tgt is not None:
                nd = d + _effect(op, arg, True)
                maxd = max(maxd, nd)
                if tgt.depth < nd:
                    tgt.depth = nd
                    stack.append(tgt)
            d += _effect(op, arg, False)
            maxd = max(maxd, d)
            if op in UNCOND or op in EXITS:
                fall = False
                break
        if fall and b.next is not None and b.next.depth < d:
            b.next.depth = d
            stack.append(b.next)
    return maxd


def compile_source(source, filename="<corpus>", minor=10):
    """Compile module source text to a 3.10 CodeObject tree."""
    return Compiler(source, filename, minor).compile_module()
