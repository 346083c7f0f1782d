"""Python source -> CPython 3.11 code objects (test-corpus generator, not product).

The 3.11 counterpart of pycodegen.py (C2 corpus per version).
It reuses the 3.10 scope analysis, constant folder and statement walk, and
restates what CPython 3.11's compile.c changed:

* every scope starts with RESUME 0, preceded by COPY_FREE_VARS / MAKE_CELL /
  RETURN_GENERATOR + POP_TOP (insert_prefix_instructions); cell and free
  variables are addressed by their localsplus slot (fix_cell_offsets);
* calls are PUSH_NULL + callable + args + [KW_NAMES] + PRECALL n + CALL n
  (PUSH_NULL folds into LOAD_GLOBAL's low bit), methods LOAD_METHOD ... CALL
  (now also with keywords, except on names imported at module level),
  decorators / assert messages / comprehension calls use PRECALL 0 + CALL 0;
  MAKE_FUNCTION no longer takes a qualname (co_qualname);
* BINARY_OP n for binary and in-place operators, COPY / SWAP for the old
  DUP_TOP / ROT_* shapes (apply_static_swaps reorders STORE_FAST / POP_TOP
  runs instead of swapping);
* zero-cost exceptions: SETUP_FINALLY / SETUP_CLEANUP / SETUP_WITH / POP_BLOCK
  pseudo instructions during optimisation, handlers entered with
  PUSH_EXC_INFO and CHECK_EXC_MATCH, `COPY 3; POP_EXCEPT; RERAISE 1` cleanup
  blocks, then label_exception_targets -> exception table (depth from the
  handler's entry stack depth, lasti for cleanup / with handlers);
* yields as YIELD_VALUE + RESUME 1, `yield from` as SEND / YIELD_VALUE /
  RESUME 2 / JUMP_BACKWARD_NO_INTERRUPT;
* jump threading only across equal line numbers, `x is None` tests as
  POP_JUMP_IF_(NOT_)NONE, and normalize_jumps choosing the FORWARD / BACKWARD
  opcode of every jump from the final block order.
"""
from __future__ import annotations

import ast

from . import pycodegen as P
from .asm import Label, assemble, encode_exception_table
from ..model import CodeObject, VersionTag

NB = {ast.Add: 0, ast.BitAnd: 1, ast.FloorDiv: 2, ast.LShift: 3, ast.MatMult: 4, ast.Mult: 5, ast.Mod: 6,
      ast.BitOr: 7, ast.Pow: 8, ast.RShift: 9, ast.Sub: 10, ast.Div: 11, ast.BitXor: 12}
NB_INPLACE = 13


class Unit311(P.Unit):
    def deref_idx(self, s):
        return ("deref", s)   # resolved to a localsplus slot at assembly (fix_cell_offsets)

    def localsplus(self):
        extra = [c for c in self.cellvars if c not in self.varnames]
        return list(self.varnames) + extra + list(self.freevars)


class Compiler311(P.Compiler):
    MINORS = (11,)

    def __init__(self, source, filename="<corpus>", minor=11):
        super().__init__(source, filename, minor)
        mod = self.scopes[id(self.tree)]
        # is_import_originated: names bound by an import at module level
        self.module_imports = set()
        for st in self.tree.body:
            if isinstance(st, (ast.Import, ast.ImportFrom)):
                for a in st.names:
                    if a.name != "*":
                        self.module_imports.add(a.asname or a.name.split(".")[0])
        self._mod_scope = mod

    def _new_unit(self, scope, name, qual, firstlineno, kind):
        u = Unit311(scope, name, qual, firstlineno, kind, minor=11)
        saved = u.lineno
        u.lineno = -1 if kind == "module" else firstlineno
        u.emit("RESUME", 0)
        u.lineno = saved
        return u

    # ------------------------------------------------------------ names
    def nameop(self, name, ctx):
        u = self.u
        sc = u.scope.lookup(name)
        if name == "__class__" and u.kind == "class" and u.scope.needs_class_closure:
            sc = P.CELL
        if u.kind == "class" and name in u.freevars and sc == P.GLOBAL_IMPLICIT:
            sc = P.FREE
        fn = u.kind in ("function", "lambda", "comprehension")
        verb = {"load": "LOAD", "store": "STORE", "del": "DELETE"}[ctx]
        if sc in (P.FREE, P.CELL):
            op = "LOAD_CLASSDEREF" if (ctx == "load" and u.kind == "class") else f"{verb}_DEREF"
            self.emit(op, ("deref", name))
        elif sc == P.LOCAL and fn:
            self.emit(f"{verb}_FAST", u.var_idx(name))
        elif (sc == P.GLOBAL_IMPLICIT and fn) or sc == P.GLOBAL_EXPLICIT:
            idx = u.name_idx(name)
            self.emit(f"{verb}_GLOBAL", idx << 1 if ctx == "load" else idx)
        else:
            self.emit(f"{verb}_NAME", u.name_idx(name))

    # ------------------------------------------------------------ statements
    def s_Assign(self, s):
        self.expr(s.value)
        n = len(s.targets)
        for i, t in enumerate(s.targets):
            if i < n - 1:
                self.emit("COPY", 1)
            self.store(t)

    def s_AugAssign(self, s):
        e = s.target
        old = self.u.lineno
        self._set_loc(e)
        if isinstance(e, ast.Attribute):
            self.expr(e.value)
            self.emit("COPY", 1)
            self.u.lineno = e.end_lineno
            self.emit("LOAD_ATTR", self.u.name_idx(e.attr))
        elif isinstance(e, ast.Subscript):
            self.expr(e.value)
            self.expr(e.slice)
            self.emit("COPY", 2)
            self.emit("COPY", 2)
            self.emit("BINARY_SUBSCR")
        else:
            self.nameop(e.id, "load")
        self.u.lineno = old
        self.expr(s.value)
        self.emit("BINARY_OP", NB[type(s.op)] + NB_INPLACE)
        self._set_loc(e)
        if isinstance(e, ast.Attribute):
            self.u.lineno = e.end_lineno
            self.emit("SWAP", 2)
            self.emit("STORE_ATTR", self.u.name_idx(e.attr))
        elif isinstance(e, ast.Subscript):
            self.emit("SWAP", 3)
            self.emit("SWAP", 2)
            self.emit("STORE_SUBSCR")
        else:
            self.nameop(e.id, "store")

    def s_Assert(self, s):
        end = self.u.new_block()
        self.jump_if(s.test, end, True)
        self.emit("LOAD_ASSERTION_ERROR")
        if s.msg is not None:
            self.expr(s.msg)
            self.emit("PRECALL", 0)
            self.emit("CALL", 0)
        self.emit("RAISE_VARARGS", 1)
        self.u.use(end)

    def s_Break(self, s):
        self.emit("NOP")
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise P.CompileError("'break' outside loop")
        self.unwind(loop, False)
        self.emit("JUMP", target=loop.exit)
        self.u.next_block()

    def s_Continue(self, s):
        self.emit("NOP")
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise P.CompileError("'continue' not properly in loop")
        self.emit("JUMP", target=loop.block)
        self.u.next_block()

    def s_If(self, s):
        u = self.u
        end = u.new_block()
        nxt = u.new_block() if s.orelse else end
        self.jump_if(s.test, nxt, False)
        self.stmts(s.body)
        if s.orelse:
            self.emit_noline("JUMP", end)
            u.use(nxt)
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
        self.emit_noline("JUMP", start)
        u.use(cleanup)
        self._pop_fb()
        self.stmts(s.orelse)
        u.use(end)

    def _pop_except_and_reraise(self):
        self.emit("COPY", 3)
        self.emit("POP_EXCEPT")
        self.emit("RERAISE", 1)

    def try_finally(self, s):
        u = self.u
        body, end, exit_, cleanup = u.new_block(), u.new_block(), u.new_block(), u.new_block()
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
        self.emit_noline("JUMP", exit_)
        u.use(end)
        u.lineno = -1
        self.emit("SETUP_CLEANUP", target=cleanup)
        self.emit("PUSH_EXC_INFO")
        self._push_fb("FINALLY_END", end)
        self.stmts(s.finalbody)
        self._pop_fb()
        self.emit("RERAISE", 0)
        u.use(cleanup)
        self._pop_except_and_reraise()
        u.use(exit_)

    def try_except(self, s):
        u = self.u
        body, except_, end, cleanup = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        self.emit("SETUP_FINALLY", target=except_)
        u.use(body)
        self._push_fb("TRY_EXCEPT", body)
        self.stmts(s.body)
        self._pop_fb()
        self.emit_noline("POP_BLOCK")
        if s.orelse:
            self.stmts(s.orelse)
        self.emit_noline("JUMP", end)
        n = len(s.handlers)
        u.use(except_)
        u.lineno = -1
        self.emit("SETUP_CLEANUP", target=cleanup)
        self.emit("PUSH_EXC_INFO")
        self._push_fb("EXCEPTION_HANDLER", None)
        for i, h in enumerate(s.handlers):
            self._set_loc(h)
            if h.type is None and i < n - 1:
                raise P.CompileError("default 'except:' must be last")
            except_ = u.new_block()
            if h.type is not None:
                self.expr(h.type)
                self.emit("CHECK_EXC_MATCH")
                self.emit("POP_JUMP_IF_FALSE", target=except_)
            if h.name:
                cleanup_end, cleanup_body = u.new_block(), u.new_block()
                self.nameop(h.name, "store")
                self.emit("SETUP_CLEANUP", target=cleanup_end)
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, None, h.name)
                self.stmts(h.body)
                self._pop_fb()
                u.lineno = -1
                self.emit("POP_BLOCK")
                self.emit("POP_BLOCK")
                self.emit("POP_EXCEPT")
                self.load_const(None)
                self.nameop(h.name, "store")
                self.nameop(h.name, "del")
                self.emit("JUMP", target=end)
                u.use(cleanup_end)
                u.lineno = -1
                self.load_const(None)
                self.nameop(h.name, "store")
                self.nameop(h.name, "del")
                self.emit("RERAISE", 1)
            else:
                cleanup_body = u.new_block()
                self.emit("POP_TOP")
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, None, None)
                self.stmts(h.body)
                self._pop_fb()
                u.lineno = -1
                self.emit("POP_BLOCK")
                self.emit("POP_EXCEPT")
                self.emit("JUMP", target=end)
            u.use(except_)
        u.lineno = -1
        self._pop_fb()
        self.emit("RERAISE", 0)
        u.use(cleanup)
        self._pop_except_and_reraise()
        u.use(end)

    def s_With(self, s, pos=0):
        u = self.u
        item = s.items[pos]
        block, final, exit_, cleanup = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        self.expr(item.context_expr)
        self.emit("BEFORE_WITH")
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
        self.emit("JUMP", target=exit_)
        u.use(final)
        self.emit("SETUP_CLEANUP", target=cleanup)
        self.emit("PUSH_EXC_INFO")
        self.emit("WITH_EXCEPT_START")
        # compiler_with_except_finish
        u.lineno = -1
        ex = u.new_block()
        self.emit("POP_JUMP_IF_TRUE", target=ex)
        self.emit("RERAISE", 2)
        u.use(cleanup)
        self._pop_except_and_reraise()
        u.use(ex)
        for op in ("POP_TOP", "POP_BLOCK", "POP_EXCEPT", "POP_TOP", "POP_TOP"):
            self.emit(op)
        u.use(exit_)

    def call_exit_with_nones(self):
        self.load_const(None)
        self.load_const(None)
        self.load_const(None)
        self.emit("PRECALL", 2)
        self.emit("CALL", 2)

    def unwind(self, fb, preserve):
        u = self.u
        k = fb.kind
        if k in ("WHILE_LOOP", "EXCEPTION_HANDLER"):
            return
        if k == "FOR_LOOP":
            if preserve:
                self.emit("SWAP", 2)
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
                self.emit("SWAP", 2)
            self.emit("POP_TOP")
            if preserve:
                self.emit("SWAP", 2)
            self.emit("POP_BLOCK")
            self.emit("POP_EXCEPT")
        elif k == "WITH":
            self._set_loc(fb.datum)
            self.emit("POP_BLOCK")
            if preserve:
                self.emit("SWAP", 2)
            self.call_exit_with_nones()
            self.emit("POP_TOP")
            u.lineno = -1
        elif k == "HANDLER_CLEANUP":
            if fb.datum:
                self.emit("POP_BLOCK")
            if preserve:
                self.emit("SWAP", 2)
            self.emit("POP_BLOCK")
            self.emit("POP_EXCEPT")
            if fb.datum:
                self.load_const(None)
                self.nameop(fb.datum, "store")
                self.nameop(fb.datum, "del")
        elif k == "POP_VALUE":
            if preserve:
                self.emit("SWAP", 2)
            self.emit("POP_TOP")

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
                            self.emit("SWAP", 2)
                            self.emit("POP_TOP")
                    self.nameop(a.asname, "store")
                    self.emit("POP_TOP")
                else:
                    self.nameop(a.asname, "store")
            else:
                self.nameop(a.name.split(".")[0], "store")

    def s_FunctionDef(self, s):
        for d in s.decorator_list:
            self.expr(d)
        firstlineno = s.decorator_list[0].lineno if s.decorator_list else s.lineno
        flags = self.default_args(s.args)
        doc = P._docstring(s.body)
        self._enter(s, s.name, "function", firstlineno)
        u = self.u
        u.const(doc if doc is not None else None)
        self._params(s.args)
        for st in s.body[1 if doc is not None else 0:]:
            self.stmt(st)
        co = self._assemble(add_none=True)
        self._exit()
        self._set_loc(s)
        self.make_closure(co, flags, None)
        for _ in s.decorator_list:
            self.emit("PRECALL", 0)
            self.emit("CALL", 0)
        self.nameop(s.name, "store")

    def make_closure(self, co, flags, qualname):
        if co.freevars:
            for name in co.freevars:
                self.emit("LOAD_CLOSURE", ("deref", name))
            flags |= 8
            self.emit("BUILD_TUPLE", len(co.freevars))
        self.load_const(co)
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
            self.emit("LOAD_CLOSURE", ("deref", "__class__"))
            self.emit("COPY", 1)
            self.nameop("__classcell__", "store")
        else:
            self.load_const(None)
        self.emit("RETURN_VALUE")
        co = self._assemble(add_none=True)
        self._exit()
        self._set_loc(s)
        self.emit("PUSH_NULL")
        self.emit("LOAD_BUILD_CLASS")
        self.make_closure(co, 0, None)
        self.load_const(s.name)
        self.call_helper(2, s.bases, s.keywords)
        for _ in s.decorator_list:
            self.emit("PRECALL", 0)
            self.emit("CALL", 0)
        self.nameop(s.name, "store")

    # ------------------------------------------------------------ expressions
    def e_BinOp(self, e):
        self.expr(e.left)
        self.expr(e.right)
        self.emit("BINARY_OP", NB[type(e.op)])

    def e_NamedExpr(self, e):
        self.expr(e.value)
        self.emit("COPY", 1)
        self.store(e.target)

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
            self.emit("SWAP", 2)
            self.emit("COPY", 2)
            self.compare_op(e.ops[i])
            self.emit("JUMP_IF_FALSE_OR_POP", target=cleanup)
            u.next_block()
        self.expr(e.comparators[n])
        self.compare_op(e.ops[n])
        end = u.new_block()
        self.emit_noline("JUMP", end)
        u.use(cleanup)
        self.emit("SWAP", 2)
        self.emit("POP_TOP")
        u.use(end)

    def jump_if(self, e, nxt, cond):
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
                self.emit_noline("JUMP", end)
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
                    self.emit("SWAP", 2)
                    self.emit("COPY", 2)
                    self.compare_op(e.ops[i])
                    self.emit("POP_JUMP_IF_FALSE", target=cleanup)
                    u.next_block()
                self.expr(e.comparators[n])
                self.compare_op(e.ops[n])
                self.emit("POP_JUMP_IF_TRUE" if cond else "POP_JUMP_IF_FALSE", target=nxt)
                end = u.new_block()
                self.emit_noline("JUMP", end)
                u.use(cleanup)
                self.emit("POP_TOP")
                if not cond:
                    self.emit_noline("JUMP", nxt)
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
        self.emit_noline("JUMP", end)
        u.use(nxt)
        self.expr(e.orelse)
        u.use(end)

    def e_Call(self, e):
        f = e.func
        if (isinstance(f, ast.Attribute) and
                not (isinstance(f.value, ast.Name) and f.value.id in self.module_imports) and
                len(e.args) + len(e.keywords) + (1 if e.keywords else 0) < P.STACK_USE_GUIDELINE and
                not any(isinstance(a, ast.Starred) for a in e.args) and
                not any(k.arg is None for k in e.keywords)):
            self.expr(f.value)
            old = self.u.lineno
            self.u.lineno = f.end_lineno
            self.emit("LOAD_METHOD", self.u.name_idx(f.attr))
            for a in e.args:
                self.expr(a)
            if e.keywords:
                for k in e.keywords:
                    self.expr(k.value)
                self.emit("KW_NAMES", self.u.const(tuple(k.arg for k in e.keywords)))
            self.u.lineno = f.end_lineno
            n = len(e.args) + len(e.keywords)
            self.emit("PRECALL", n)
            self.emit("CALL", n)
            self.u.lineno = old
            return
        old = self.u.lineno
        self.u.lineno = f.lineno
        self.emit("PUSH_NULL")
        self.u.lineno = old
        self.expr(f)
        self.call_helper(0, e.args, e.keywords)

    def call_helper(self, n, args, keywords):
        simple = (len(args) + 2 * len(keywords) <= P.STACK_USE_GUIDELINE and
                  not any(isinstance(a, ast.Starred) for a in args) and not any(k.arg is None for k in keywords))
        if simple:
            for a in args:
                self.expr(a)
            if keywords:
                for k in keywords:
                    self.expr(k.value)
                self.emit("KW_NAMES", self.u.const(tuple(k.arg for k in keywords)))
            self.emit("PRECALL", n + len(args) + len(keywords))
            self.emit("CALL", n + len(args) + len(keywords))
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
        self._exit()
        self.make_closure(co, flags, None)

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
        self._exit()
        self.make_closure(co, 0, None)
        self.expr(gens[0].iter)
        self.emit("GET_ITER")
        self.emit("PRECALL", 0)
        self.emit("CALL", 0)

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
                self.emit("RESUME", 1)
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
            self.emit("JUMP", target=start)
            u.use(anchor)

    def e_Yield(self, e):
        if e.value is not None:
            self.expr(e.value)
        else:
            self.load_const(None)
        self.emit("YIELD_VALUE")
        self.emit("RESUME", 1)

    def e_YieldFrom(self, e):
        u = self.u
        self.expr(e.value)
        self.emit("GET_YIELD_FROM_ITER")
        self.load_const(None)
        start, resume, exit_ = u.new_block(), u.new_block(), u.new_block()
        u.use(start)
        self.emit("SEND", target=exit_)
        u.use(resume)
        self.emit("YIELD_VALUE")
        self.emit("RESUME", 2)
        self.emit("JUMP_NO_INTERRUPT", target=start)
        u.use(exit_)

    # ------------------------------------------------------------ assembly
    def _flags(self):
        f = super()._flags()
        return f & ~P.CO_NOFREE   # CO_NOFREE is gone in 3.11

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
        # insert_prefix_instructions
        prefix = []
        if u.freevars:
            prefix.append(["COPY_FREE_VARS", len(u.freevars), None, -1])
        for c in u.cellvars:
            prefix.append(["MAKE_CELL", ("deref", c), None, -1])
        if flags & P.CO_GENERATOR:
            prefix += [["RETURN_GENERATOR", 0, None, u.firstlineno], ["POP_TOP", 0, None, u.firstlineno]]
        u.entry.instrs[0:0] = prefix
        P._optimize(u, _optimize_block311)
        stacksize = _stackdepth311(u)
        _label_exception_targets(u)
        for b in P._chain(u.entry):
            for ins in b.instrs:
                if ins[0] in P.SETUPS or ins[0] == "POP_BLOCK":
                    ins[0], ins[1], ins[2] = "NOP", None, None
        for b in P._chain(u.entry):
            P._clean(b, -1)
        _normalize_jumps(u)
        # fix_cell_offsets: ("deref", name) -> localsplus slot
        lp = u.localsplus()
        for b in P._chain(u.entry):
            for ins in b.instrs:
                if isinstance(ins[1], tuple) and ins[1] and ins[1][0] == "deref":
                    ins[1] = lp.index(ins[1][1])
        items = []
        lab = {}
        k = 0
        order = []
        for b in P._chain(u.entry):
            lab[id(b)] = Label(f"B{b.idx}")
        for b in P._chain(u.entry):
            items.append(lab[id(b)])
            for ins in b.instrs:
                il = Label(f"I{k}")
                items.append(il)
                order.append((il, ins))
                k += 1
                op, arg, tgt, _ln = ins[:4]
                items.append((op, lab[id(tgt)]) if tgt is not None else (op, 0 if arg is None else arg))
        items.append(Label("END"))
        code, labels = assemble(items, self.minor, return_labels=True)
        # assemble_exception_table: runs of instructions with the same handler
        entries = []
        handler, start = None, 0
        for il, ins in order:
            h = ins[4] if len(ins) > 4 else None
            if h is not handler:
                if handler is not None:
                    entries.append((start, labels[il], handler))
                start, handler = labels[il], h
        if handler is not None:
            entries.append((start, labels[Label("END")], handler))
        table = []
        for s0, e0, h in entries:
            depth = h.depth - 1 - (1 if getattr(h, "lasti", False) else 0)
            table.append((s0, e0, labels[lab[id(h)]], depth, bool(getattr(h, "lasti", False))))
        exctable = encode_exception_table(table)
        return CodeObject(
            VersionTag(3, self.minor), u.argcount, u.posonly, u.kwonly, len(u.varnames), stacksize, flags,
            code, tuple(u.consts), tuple(u.names), tuple(u.varnames), tuple(u.freevars),
            tuple(u.cellvars), u.name, self.filename, u.firstlineno, b"", exctable, u.qualname)


# ---------------------------------------------------------------- 3.11 optimiser pieces

def _jump_thread(ins, tgt, opcode):
    if ins[3] == tgt[3] and ins[2] is not tgt[2]:
        ins[2] = tgt[2]
        ins[0] = opcode
        return True
    return False


def _next_swappable(instrs, i, lineno):
    while True:
        i += 1
        if i >= len(instrs):
            return -1
        ins = instrs[i]
        if lineno >= 0 and ins[3] != lineno:
            return -1
        if ins[0] == "NOP":
            continue
        if ins[0] in ("STORE_FAST", "POP_TOP"):
            return i
        return -1


def _apply_static_swaps(instrs, i):
    while i >= 0:
        sw = instrs[i]
        if sw[0] != "SWAP":
            if sw[0] in ("NOP", "STORE_FAST", "POP_TOP"):
                i -= 1
                continue
            return
        j = _next_swappable(instrs, i, -1)
        if j < 0:
            return
        k = j
        lineno = instrs[j][3]
        for _ in range(sw[1] - 1):
            k = _next_swappable(instrs, k, lineno)
            if k < 0:
                return
        sw[0], sw[1] = "NOP", None
        instrs[j], instrs[k] = instrs[k], instrs[j]
        i -= 1


def _optimize_block311(u, b):
    i = 0
    while i < len(b.instrs):
        ins = b.instrs[i]
        op = ins[0]
        nxt = b.instrs[i + 1] if i + 1 < len(b.instrs) else None
        nextop = nxt[0] if nxt else None
        tgt = None
        if op in P.JUMPS:
            ins[2] = P._first_nonempty(ins[2])
            tgt = ins[2].instrs[0]
        redo = False
        if op == "PUSH_NULL" and nextop == "LOAD_GLOBAL" and (nxt[1] & 1) == 0:
            ins[0], ins[1] = "NOP", None
            nxt[1] |= 1
        elif op == "LOAD_CONST" and nextop in ("POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE"):
            is_true = P._truthy(u.consts[ins[1]])
            ins[0] = "NOP"
            if is_true == (nextop == "POP_JUMP_IF_TRUE"):
                nxt[0] = "JUMP"
                b.nofall = True
            else:
                nxt[0], nxt[2] = "NOP", None
        elif op == "LOAD_CONST" and nextop == "IS_OP" and u.consts[ins[1]].kind == "none":
            jop = b.instrs[i + 2][0] if i + 2 < len(b.instrs) else None
            if jop in ("POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE"):
                inv = nxt[1]
                ins[0] = "NOP"
                nxt[0], nxt[1] = "NOP", None
                jump_if_not_none = bool(inv) ^ (jop == "POP_JUMP_IF_FALSE")
                b.instrs[i + 2][0] = "POP_JUMP_IF_NOT_NONE" if jump_if_not_none else "POP_JUMP_IF_NONE"
        elif op == "BUILD_TUPLE":
            n = ins[1]
            if nextop == "UNPACK_SEQUENCE" and nxt[1] == n:
                if n == 1:
                    ins[0] = "NOP"
                    nxt[0] = "NOP"
                elif n in (2, 3):
                    ins[0], ins[1] = "NOP", None
                    nxt[0], nxt[1] = "SWAP", n
                    i += 1
                    continue
            elif i >= n and all(b.instrs[j][0] == "LOAD_CONST" for j in range(i - n, i)):
                vals = tuple(u.consts[b.instrs[j][1]] for j in range(i - n, i))
                for j in range(i - n, i):
                    b.instrs[j][0] = "NOP"
                ins[0] = "LOAD_CONST"
                ins[1] = u.const(P.Const("tuple", vals))
        elif op == "SWAP":
            if ins[1] == 1:
                ins[0], ins[1] = "NOP", None
            else:
                _apply_static_swaps(b.instrs, i)
        elif op in ("JUMP_IF_FALSE_OR_POP", "JUMP_IF_TRUE_OR_POP"):
            same = "POP_JUMP_IF_FALSE" if op == "JUMP_IF_FALSE_OR_POP" else "POP_JUMP_IF_TRUE"
            other = "JUMP_IF_TRUE_OR_POP" if op == "JUMP_IF_FALSE_OR_POP" else "JUMP_IF_FALSE_OR_POP"
            t = tgt[0]
            if t == same:
                redo = _jump_thread(ins, tgt, same)
            elif t in ("JUMP", op):
                redo = _jump_thread(ins, tgt, op)
            elif t == other:
                if ins[3] == tgt[3]:
                    ins[0] = same
                    ins[2] = ins[2].next
                    redo = True
        elif op in ("POP_JUMP_IF_FALSE", "POP_JUMP_IF_TRUE", "POP_JUMP_IF_NONE", "POP_JUMP_IF_NOT_NONE"):
            if tgt[0] == "JUMP":
                redo = _jump_thread(ins, tgt, op)
        elif op == "JUMP":
            if tgt[0] == "JUMP":
                redo = _jump_thread(ins, tgt, "JUMP")
        if not redo:
            i += 1


_FIXED = {
    "NOP": 0, "POP_TOP": -1, "PUSH_NULL": 1, "UNARY_POSITIVE": 0, "UNARY_NEGATIVE": 0, "UNARY_NOT": 0,
    "UNARY_INVERT": 0, "GET_ITER": 0, "BINARY_SUBSCR": -1, "STORE_SUBSCR": -3, "DELETE_SUBSCR": -2,
    "LOAD_BUILD_CLASS": 1, "RETURN_VALUE": -1, "IMPORT_STAR": -1, "YIELD_VALUE": 0, "POP_EXCEPT": -1,
    "PUSH_EXC_INFO": 1, "CHECK_EXC_MATCH": 0, "STORE_NAME": -1, "DELETE_NAME": 0, "STORE_ATTR": -2,
    "DELETE_ATTR": -1, "STORE_GLOBAL": -1, "DELETE_GLOBAL": 0, "LOAD_CONST": 1, "LOAD_NAME": 1, "LOAD_ATTR": 0,
    "COMPARE_OP": -1, "IS_OP": -1, "CONTAINS_OP": -1, "IMPORT_NAME": -1, "IMPORT_FROM": 1, "JUMP": 0,
    "JUMP_NO_INTERRUPT": 0, "POP_JUMP_IF_FALSE": -1, "POP_JUMP_IF_TRUE": -1, "POP_JUMP_IF_NONE": -1,
    "POP_JUMP_IF_NOT_NONE": -1, "RERAISE": -1, "WITH_EXCEPT_START": 1, "BEFORE_WITH": 1, "LOAD_FAST": 1,
    "STORE_FAST": -1, "DELETE_FAST": 0, "LOAD_CLOSURE": 1, "LOAD_DEREF": 1, "LOAD_CLASSDEREF": 1,
    "STORE_DEREF": -1, "DELETE_DEREF": 0, "LOAD_METHOD": 1, "LIST_APPEND": -1, "SET_ADD": -1, "MAP_ADD": -2,
    "LIST_EXTEND": -1, "SET_UPDATE": -1, "DICT_UPDATE": -1, "DICT_MERGE": -1, "LIST_TO_TUPLE": 0,
    "GET_YIELD_FROM_ITER": 0, "LOAD_ASSERTION_ERROR": 1, "RESUME": 0, "RETURN_GENERATOR": 0, "MAKE_CELL": 0,
    "COPY_FREE_VARS": 0, "KW_NAMES": 0, "BINARY_OP": -1, "COPY": 1, "SWAP": 0, "POP_BLOCK": 0, "CALL": -1,
    "PRINT_EXPR": -1,
}


def _effect311(op, arg, jump):
    if op in _FIXED:
        return _FIXED[op]
    if op == "LOAD_GLOBAL":
        return 1 + (arg & 1)
    if op == "PRECALL":
        return -arg
    if op == "UNPACK_SEQUENCE":
        return arg - 1
    if op == "UNPACK_EX":
        return (arg & 0xFF) + (arg >> 8)
    if op == "FOR_ITER":
        return -1 if jump else 1
    if op == "SEND":
        return -1 if jump else 0
    if op in ("BUILD_TUPLE", "BUILD_LIST", "BUILD_SET", "BUILD_STRING"):
        return 1 - arg
    if op == "BUILD_MAP":
        return 1 - 2 * arg
    if op == "BUILD_CONST_KEY_MAP":
        return -arg
    if op in ("JUMP_IF_TRUE_OR_POP", "JUMP_IF_FALSE_OR_POP"):
        return 0 if jump else -1
    if op in ("SETUP_FINALLY", "SETUP_WITH"):
        return 1 if jump else 0
    if op == "SETUP_CLEANUP":
        return 2 if jump else 0
    if op == "RAISE_VARARGS":
        return -arg
    if op == "CALL_FUNCTION_EX":
        return -2 - (arg & 1)
    if op == "MAKE_FUNCTION":
        return -bin(arg & 0xF).count("1")
    if op == "BUILD_SLICE":
        return -1 if arg == 2 else -2
    if op == "FORMAT_VALUE":
        return -1 if arg & 4 else 0
    raise P.CompileError(f"no 3.11 stack effect for {op}")


def _stackdepth311(u):
    """stackdepth(): max depth, and each block's entry depth (b_startdepth),
    which the exception table's depth field is derived from."""
    for b in P._chain(u.entry):
        b.depth = -1
    for b in u.blocks:
        b.depth = -1
    maxd = 0
    u.entry.depth = 0
    stack = [u.entry]
    while stack:
        b = stack.pop()
        d = b.depth
        fall = True
        for ins in b.instrs:
            op, arg, tgt = ins[0], ins[1], ins[2]
            if tgt is not None:
                nd = d + _effect311(op, arg, True)
                maxd = max(maxd, nd)
                if tgt.depth < nd:
                    tgt.depth = nd
                    stack.append(tgt)
            d += _effect311(op, arg, False)
            maxd = max(maxd, d)
            if op in P.UNCOND or op in P.EXITS:
                fall = False
                break
        if fall and b.next is not None and b.next.depth < d:
            b.next.depth = d
            stack.append(b.next)
    return maxd


def _label_exception_targets(u):
    """label_exception_targets: every instruction gets the innermost active
    handler block (ins[4]); SETUP_CLEANUP / SETUP_WITH handlers keep lasti."""
    for b in u.blocks:
        b.visited = False
        b.exc = None
    entry = u.entry
    entry.exc = []
    entry.visited = True
    todo = [entry]
    while todo:
        b = todo.pop()
        stack = b.exc
        b.exc = None
        handler = stack[-1] if stack else None
        for ins in b.instrs:
            while len(ins) < 5:
                ins.append(None)
            op = ins[0]
            if op in P.SETUPS:
                t = ins[2]
                if not t.visited:
                    t.exc = list(stack)
                    t.visited = True
                    todo.append(t)
                if op in ("SETUP_WITH", "SETUP_CLEANUP"):
                    t.lasti = True
                stack.append(t)
                handler = t
            elif op == "POP_BLOCK":
                stack.pop()
                handler = stack[-1] if stack else None
            elif op in P.JUMPS:
                ins[4] = handler
                t = ins[2]
                if not t.visited:
                    t.exc = list(stack) if not b.nofall else stack
                    t.visited = True
                    todo.append(t)
            else:
                ins[4] = handler
        if not b.nofall and b.next is not None and not b.next.visited:
            b.next.exc = stack
            b.next.visited = True
            todo.append(b.next)


def _normalize_jumps(u):
    seen = set()
    for b in P._chain(u.entry):
        seen.add(id(b))
        if not b.instrs:
            continue
        last = b.instrs[-1]
        if last[0] not in P.JUMPS:
            continue
        fwd = id(last[2]) not in seen
        op = last[0]
        if op == "JUMP":
            last[0] = "JUMP_FORWARD" if fwd else "JUMP_BACKWARD"
        elif op == "JUMP_NO_INTERRUPT":
            last[0] = "JUMP_FORWARD" if fwd else "JUMP_BACKWARD_NO_INTERRUPT"
        elif op.startswith("POP_JUMP_IF_"):
            last[0] = ("POP_JUMP_FORWARD_IF_" if fwd else "POP_JUMP_BACKWARD_IF_") + op[len("POP_JUMP_IF_"):]


def compile_source(source, filename="<corpus>"):
    """Compile module source text to a 3.11 CodeObject tree."""
    return Compiler311(source, filename, 11).compile_module()
