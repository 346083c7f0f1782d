"""Python source -> CPython 3.8 code objects (test-corpus generator, not product).

The 3.8 counterpart of pycodegen.py / pycodegen39.py (C2 corpus per version,
SURVEY.md §8(d)).  On top of the 3.9 layout (peephole era, leading-test loops)
CPython 3.8's compile.c differs in:

* finally machinery: SETUP_FINALLY + POP_BLOCK + BEGIN_FINALLY before the
  finally body, END_FINALLY after it; `return` / `break` / `continue` out of a
  try-finally call the finally body with CALL_FINALLY, leave a finally body
  with POP_FINALLY; `except E as n` is a nested try/finally whose cleanup
  ends in END_FINALLY + POP_EXCEPT; with-statements end in
  WITH_CLEANUP_START / WITH_CLEANUP_FINISH / END_FINALLY;
* exception matching is COMPARE_OP 10 (`exception match`) + POP_JUMP_IF_FALSE,
  `is` / `in` are COMPARE_OP 8/9 and 6/7 (no IS_OP / CONTAINS_OP), asserts load
  the global AssertionError;
* starred displays and calls build with BUILD_{LIST,TUPLE,SET}_UNPACK /
  BUILD_TUPLE_UNPACK_WITH_CALL, dict merges with BUILD_MAP_UNPACK(_WITH_CALL)
  (no LIST_EXTEND / DICT_MERGE, no constant-list folding).
"""
from __future__ import annotations

import ast

from . import pycodegen as P
from .pycodegen39 import Compiler39

CMP38 = {ast.Lt: 0, ast.LtE: 1, ast.Eq: 2, ast.NotEq: 3, ast.Gt: 4, ast.GtE: 5, ast.In: 6, ast.NotIn: 7,
         ast.Is: 8, ast.IsNot: 9}


class Compiler38(Compiler39):
    MINORS = (8,)

    def __init__(self, source, filename="<corpus>", minor=8):
        P.Compiler.__init__(self, source, filename, minor)

    def _new_unit(self, scope, name, qual, firstlineno, kind):
        return P.Unit(scope, name, qual, firstlineno, kind, minor=8)

    def emit(self, op, arg=None, target=None):
        self.u.emit(op, arg, target)

    def compare_op(self, op):
        self.emit("COMPARE_OP", CMP38[type(op)])

    # ------------------------------------------------------------ frame blocks
    def unwind(self, fb, preserve):
        k = fb.kind
        if k in ("WHILE_LOOP", "EXCEPTION_HANDLER"):
            return
        if k == "FINALLY_END":
            fb.exit = None
            self.emit("POP_FINALLY", int(preserve))
            if preserve:
                self.emit("ROT_TWO")
            self.emit("POP_TOP")
        elif k == "FOR_LOOP":
            if preserve:
                self.emit("ROT_TWO")
            self.emit("POP_TOP")
        elif k == "TRY_EXCEPT":
            self.emit("POP_BLOCK")
        elif k == "FINALLY_TRY":
            self.emit("POP_BLOCK")
            self.emit("CALL_FINALLY", target=fb.exit)
        elif k == "WITH":
            self.emit("POP_BLOCK")
            if preserve:
                self.emit("ROT_TWO")
            self.emit("BEGIN_FINALLY")
            self.emit("WITH_CLEANUP_START")
            self.emit("WITH_CLEANUP_FINISH")
            self.emit("POP_FINALLY", 0)
        elif k == "HANDLER_CLEANUP":
            if preserve:
                self.emit("ROT_FOUR")
            if fb.exit is not None:
                self.emit("POP_BLOCK")
                self.emit("POP_EXCEPT")
                self.emit("CALL_FINALLY", target=fb.exit)
            else:
                self.emit("POP_EXCEPT")

    def s_Return(self, s):
        v = s.value
        preserve = v is not None and not isinstance(v, ast.Constant)
        if preserve:
            self.expr(v)
        for fb in reversed(list(self.u.fblocks)):
            self.unwind(fb, preserve)
        if v is None:
            self.load_const(None)
        elif not preserve:
            self.load_const(v.value)
        self.emit("RETURN_VALUE")

    def s_Break(self, s):
        for fb in reversed(list(self.u.fblocks)):
            self.unwind(fb, False)
            if fb.kind in ("WHILE_LOOP", "FOR_LOOP"):
                self.emit("JUMP_ABSOLUTE", target=fb.exit)
                return
        raise P.CompileError("'break' outside loop")

    def s_Continue(self, s):
        for fb in reversed(list(self.u.fblocks)):
            if fb.kind in ("WHILE_LOOP", "FOR_LOOP"):
                self.emit("JUMP_ABSOLUTE", target=fb.block)
                return
            self.unwind(fb, False)
        raise P.CompileError("'continue' not properly in loop")

    # ------------------------------------------------------------ try / with
    def try_finally(self, s):
        u = self.u
        body, end = u.new_block(), u.new_block()
        self.emit("SETUP_FINALLY", target=end)
        u.use(body)
        self._push_fb("FINALLY_TRY", body, end)
        if s.handlers:
            self.try_except(s)
        else:
            self.stmts(s.body)
        self.emit("POP_BLOCK")
        self.emit("BEGIN_FINALLY")
        self._pop_fb()
        u.use(end)
        self._push_fb("FINALLY_END", end)
        self.stmts(s.finalbody)
        self.emit("END_FINALLY")
        self._pop_fb()

    def try_except(self, s):
        u = self.u
        body, except_, orelse, end = u.new_block(), u.new_block(), u.new_block(), u.new_block()
        self.emit("SETUP_FINALLY", target=except_)
        u.use(body)
        self._push_fb("TRY_EXCEPT", body)
        self.stmts(s.body)
        self.emit("POP_BLOCK")
        self._pop_fb()
        self.emit("JUMP_FORWARD", target=orelse)
        n = len(s.handlers)
        u.use(except_)
        for i, h in enumerate(s.handlers):
            if h.type is None and i < n - 1:
                raise P.CompileError("default 'except:' must be last")
            except_ = u.new_block()
            if h.type is not None:
                self.emit("DUP_TOP")
                self.expr(h.type)
                self.emit("COMPARE_OP", 10)
                self.emit("POP_JUMP_IF_FALSE", target=except_)
            self.emit("POP_TOP")
            if h.name:
                cleanup_end, cleanup_body = u.new_block(), u.new_block()
                self.nameop(h.name, "store")
                self.emit("POP_TOP")
                self.emit("SETUP_FINALLY", target=cleanup_end)
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, cleanup_end)
                self.stmts(h.body)
                self.emit("POP_BLOCK")
                self.emit("BEGIN_FINALLY")
                self._pop_fb()
                u.use(cleanup_end)
                self._push_fb("FINALLY_END", cleanup_end)
                self.load_const(None)
                self.nameop(h.name, "store")
                self.nameop(h.name, "del")
                self.emit("END_FINALLY")
                self.emit("POP_EXCEPT")
                self._pop_fb()
            else:
                cleanup_body = u.new_block()
                self.emit("POP_TOP")
                self.emit("POP_TOP")
                u.use(cleanup_body)
                self._push_fb("HANDLER_CLEANUP", cleanup_body, None)
                self.stmts(h.body)
                self._pop_fb()
                self.emit("POP_EXCEPT")
            self.emit("JUMP_FORWARD", target=end)
            u.use(except_)
        self.emit("END_FINALLY")
        u.use(orelse)
        self.stmts(s.orelse)
        u.use(end)

    def s_With(self, s, pos=0):
        u = self.u
        item = s.items[pos]
        block, final = u.new_block(), u.new_block()
        self.expr(item.context_expr)
        self.emit("SETUP_WITH", target=final)
        u.use(block)
        self._push_fb("WITH", block, final)
        if item.optional_vars is not None:
            self.store(item.optional_vars)
        else:
            self.emit("POP_TOP")
        if pos + 1 == len(s.items):
            self.stmts(s.body)
        else:
            self.s_With(s, pos + 1)
        self.emit("POP_BLOCK")
        self.emit("BEGIN_FINALLY")
        self._pop_fb()
        u.use(final)
        self._push_fb("FINALLY_END", final)
        self.emit("WITH_CLEANUP_START")
        self.emit("WITH_CLEANUP_FINISH")
        self.emit("END_FINALLY")
        self._pop_fb()

    def s_Assert(self, s):
        end = self.u.new_block()
        self.jump_if(s.test, end, True)
        self.emit("LOAD_GLOBAL", self.u.name_idx("AssertionError"))
        if s.msg is not None:
            self.expr(s.msg)
            self.emit("CALL_FUNCTION", 1)
        self.emit("RAISE_VARARGS", 1)
        self.u.use(end)

    # ------------------------------------------------------------ displays / calls
    def _unpack_helper38(self, elts, single, inner, outer):
        nsub = nseen = 0
        for x in elts:
            if isinstance(x, ast.Starred):
                if nseen:
                    self.emit(inner, nseen)
                    nseen = 0
                    nsub += 1
                self.expr(x.value)
                nsub += 1
            else:
                self.expr(x)
                nseen += 1
        if nsub:
            if nseen:
                self.emit(inner, nseen)
                nsub += 1
            self.emit(outer, nsub)
        else:
            self.emit(single, nseen)

    def e_Tuple(self, e):
        self._unpack_helper38(e.elts, "BUILD_TUPLE", "BUILD_TUPLE", "BUILD_TUPLE_UNPACK")

    def e_List(self, e):
        self._unpack_helper38(e.elts, "BUILD_LIST", "BUILD_TUPLE", "BUILD_LIST_UNPACK")

    def e_Set(self, e):
        self._unpack_helper38(e.elts, "BUILD_SET", "BUILD_SET", "BUILD_SET_UNPACK")

    def subdict(self, e, begin, end):
        n = end - begin
        keys = e.keys[begin:end]
        if n > 1 and all(isinstance(k, ast.Constant) for k in keys):
            for v in e.values[begin:end]:
                self.expr(v)
            self.load_const(tuple(k.value for k in keys))
            self.emit("BUILD_CONST_KEY_MAP", n)
            return
        for k, v in zip(keys, e.values[begin:end]):
            self.expr(k)
            self.expr(v)
        self.emit("BUILD_MAP", n)

    def e_Dict(self, e):
        n = len(e.values)
        containers = elements = 0
        is_unpacking = False
        for i in range(n):
            is_unpacking = e.keys[i] is None
            if elements == 0xFFFF or (elements and is_unpacking):
                self.subdict(e, i - elements, i)
                containers += 1
                elements = 0
            if is_unpacking:
                self.expr(e.values[i])
                containers += 1
            else:
                elements += 1
        if elements or containers == 0:
            self.subdict(e, n - elements, n)
            containers += 1
        if containers > 1 or is_unpacking:
            self.emit("BUILD_MAP_UNPACK", containers)

    def e_Call(self, e):
        f = e.func
        if (isinstance(f, ast.Attribute) and not e.keywords and
                not any(isinstance(a, ast.Starred) for a in e.args)):
            self.expr(f.value)
            self.emit("LOAD_METHOD", self.u.name_idx(f.attr))
            for a in e.args:
                self.expr(a)
            self.emit("CALL_METHOD", len(e.args))
            return
        self.expr(f)
        self.call_helper(0, e.args, e.keywords)

    def subkwargs(self, kws):
        n = len(kws)
        if n > 1:
            for k in kws:
                self.expr(k.value)
            self.load_const(tuple(k.arg for k in kws))
            self.emit("BUILD_CONST_KEY_MAP", n)
            return
        for k in kws:
            self.load_const(k.arg)
            self.expr(k.value)
        self.emit("BUILD_MAP", n)

    def call_helper(self, n, args, keywords):
        must_dict = any(k.arg is None for k in keywords)
        nsubargs = nsubkw = 0
        nseen = n
        for a in args:
            if isinstance(a, ast.Starred):
                if nseen:
                    self.emit("BUILD_TUPLE", nseen)
                    nseen = 0
                    nsubargs += 1
                self.expr(a.value)
                nsubargs += 1
            else:
                self.expr(a)
                nseen += 1
        if nsubargs or must_dict:
            if nseen:
                self.emit("BUILD_TUPLE", nseen)
                nsubargs += 1
            if nsubargs > 1:
                self.emit("BUILD_TUPLE_UNPACK_WITH_CALL", nsubargs)
            elif nsubargs == 0:
                self.emit("BUILD_TUPLE", 0)
            nseen = 0
            for i, k in enumerate(keywords):
                if k.arg is None:
                    if nseen:
                        self.subkwargs(keywords[i - nseen:i])
                        nsubkw += 1
                        nseen = 0
                    self.expr(k.value)
                    nsubkw += 1
                else:
                    nseen += 1
            if nseen:
                self.subkwargs(keywords[len(keywords) - nseen:])
                nsubkw += 1
            if nsubkw > 1:
                self.emit("BUILD_MAP_UNPACK_WITH_CALL", nsubkw)
            self.emit("CALL_FUNCTION_EX", int(nsubkw > 0))
            return
        if keywords:
            for k in keywords:
                self.expr(k.value)
            self.load_const(tuple(k.arg for k in keywords))
            self.emit("CALL_FUNCTION_KW", nseen + len(keywords))
        else:
            self.emit("CALL_FUNCTION", nseen)


def compile_source(source, filename="<corpus>"):
    """Compile module source text to a 3.8 CodeObject tree."""
    return Compiler38(source, filename, 8).compile_module()
