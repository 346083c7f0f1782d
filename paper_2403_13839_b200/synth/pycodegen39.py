"""Python source -> CPython 3.9 code objects (test-corpus generator, not product).

The 3.9 counterpart of pycodegen.py (C2 corpus per version).
CPython 3.9 compiles the same statement shapes as 3.10 with these differences,
restated here:

* `while` is not rotated: the test is compiled once at the top and the body
  ends with JUMP_ABSOLUTE back to it (compiler_while); a constant-true test
  emits no test at all;
* no GEN_START, RERAISE takes no argument, jump arguments are byte offsets
  (handled by the assembler), no line-number NOPs;
* no CFG optimiser: the peephole optimiser (Python/peephole.c) folds
  LOAD_CONST + conditional jumps, BUILD_TUPLE + UNPACK_SEQUENCE and constant
  tuples, threads jumps to unconditional jumps (no line-number guard),
  drops code after RETURN / RAISE / unconditional jumps up to the next jump
  target and removes NOPs; exit blocks are never copied, so a function's
  implicit `return None` is shared by fall-through and jumps and unreachable
  trailing returns that are still jump targets survive.
"""
from __future__ import annotations

import ast

from . import pycodegen as P


class Compiler39(P.Compiler):
    MINORS = (9,)

    def __init__(self, source, filename="<corpus>", minor=9):
        super().__init__(source, filename, minor)

    def _new_unit(self, scope, name, qual, firstlineno, kind):
        return P.Unit(scope, name, qual, firstlineno, kind, minor=9)

    def s_Return(self, s):
        v = s.value
        preserve = v is not None and not isinstance(v, ast.Constant)
        if preserve:
            self.expr(v)
        self.unwind_stack(preserve, None)
        if v is None:
            self.load_const(None)
        elif not preserve:
            self.load_const(v.value)
        self.emit("RETURN_VALUE")

    def s_Break(self, s):
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise P.CompileError("'break' outside loop")
        self.unwind(loop, False)
        self.emit("JUMP_ABSOLUTE", target=loop.exit)

    def s_Continue(self, s):
        loop = self.unwind_stack(False, "loop")
        if loop is None:
            raise P.CompileError("'continue' not properly in loop")
        self.emit("JUMP_ABSOLUTE", target=loop.block)

    def s_While(self, s):
        u = self.u
        t = s.test
        constant = bool(t.value) if isinstance(t, ast.Constant) else None
        if constant is False:
            if s.orelse:
                self.stmts(s.orelse)
            return
        loop, end = u.new_block(), u.new_block()
        anchor = u.new_block() if constant is None else None
        u.use(loop)
        self._push_fb("WHILE_LOOP", loop, end)
        if constant is None:
            self.jump_if(t, anchor, False)
        self.stmts(s.body)
        self.emit("JUMP_ABSOLUTE", target=loop)
        if constant is None:
            u.use(anchor)
        self._pop_fb()
        if s.orelse:
            self.stmts(s.orelse)
        u.use(end)

    def emit(self, op, arg=None, target=None):
        if op == "RERAISE":
            arg = None   # 3.9 RERAISE has no argument
        self.u.emit(op, arg, target)

    def _assemble(self, add_none):
        u = self.u
        last = u.cur
        if not any(i[0] == "RETURN_VALUE" for i in last.instrs):
            if add_none:
                u.emit("LOAD_CONST", u.const(None))
            u.emit("RETURN_VALUE")
        flags = self._flags()
        _peephole39(u)
        stacksize = P._stackdepth(u)
        items = []
        lab = {id(b): P.Label(f"B{b.idx}") for b in P._chain(u.entry)}
        for b in P._chain(u.entry):
            items.append(lab[id(b)])
            for op, arg, tgt, _ln in b.instrs:
                items.append((op, lab[id(tgt)]) if tgt is not None else (op, arg))
        code = P.assemble(items, self.minor)
        return P.CodeObject(
            P.VersionTag(3, self.minor), u.argcount, u.posonly, u.kwonly, len(u.varnames), stacksize, flags,
            code, tuple(u.consts), tuple(u.names), tuple(u.varnames), tuple(u.freevars),
            tuple(u.cellvars), u.name, self.filename, u.firstlineno, b"", b"", "")


def _peephole39(u):
    # peephole.c has no line-number guards: make every jump-threading check pass
    for b in u.blocks:
        for ins in b.instrs:
            ins[3] = 0
    P._normalize(u)
    for b in P._chain(u.entry):
        P._optimize_block(u, b)
    # unreachable code is dropped only up to the next jump target (dead jumps count)
    targeted = set()
    for b in P._chain(u.entry):
        for ins in b.instrs:
            if ins[0] in P.JUMPS and ins[0] != "NOP" and ins[2] is not None:
                targeted.add(id(ins[2]))
    P._mark_reachable(u)
    for b in P._chain(u.entry):
        if b.preds == 0 and id(b) not in targeted:
            b.instrs = []
    for b in P._chain(u.entry):
        b.instrs = [ins for ins in b.instrs if ins[0] != "NOP"]
    P._eliminate_empty(u)
    for b in P._chain(u.entry):
        while b.next is not None and not b.next.instrs:
            b.next = b.next.next
    pos = {}
    for k, b in enumerate(P._chain(u.entry)):
        pos[id(b)] = k
    for b in P._chain(u.entry):
        if b.instrs and b.instrs[-1][0] == "JUMP_FORWARD" and pos[id(b.instrs[-1][2])] <= pos[id(b)]:
            b.instrs[-1][0] = "JUMP_ABSOLUTE"


def compile_source(source, filename="<corpus>"):
    """Compile module source text to a 3.9 CodeObject tree."""
    return Compiler39(source, filename, 9).compile_module()
