"""Oracle: decoding, control-flow facts and block simulation.

Restates disasm.py:71-214, pipeline.py:17-87, cfg.py:61-313,
structurer.py:62-173 and symexec.py:128-1051 of /root/reference/pkg/src/unpyre.
Instructions are small mutable records; the CFG is kept as parallel lists.
"""
from __future__ import annotations

from paper_2403_13839_b200._optables import CMP_OP, TABLES
from paper_2403_13839_b200.errors import (BadJumpTarget, MalformedExceptionTable, StackDepthMismatch,
                                          StackUnderflow, StructuringFailed, TruncatedCode, UnknownOpcode,
                                          UnsupportedOpcode)
from paper_2403_13839_b200.model import Const

from . import nodes as n

JUMPS = ("jump_rel", "jump_abs", "jump_back")
SETUPS = ("SETUP_FINALLY", "SETUP_WITH", "SETUP_ASYNC_WITH")


class Ins:
    __slots__ = ("offset", "op_offset", "opname", "opcode", "arg", "argval", "nprefix", "cache", "kind")

    def __init__(self, offset, op_offset, opname, opcode, arg, nprefix, cache, kind):
        self.offset = offset
        self.op_offset = op_offset
        self.opname = opname
        self.opcode = opcode
        self.arg = arg
        self.argval = None
        self.nprefix = nprefix
        self.cache = cache
        self.kind = kind

    @property
    def end(self):
        return self.offset + 2 * (1 + self.nprefix + self.cache)

    @property
    def jumps(self):
        return self.kind in JUMPS


def localsplus(co):
    extra = tuple(c for c in co.cellvars if c not in co.varnames)
    return co.varnames + extra + co.freevars


def decode(co):
    """decode_instructions (disasm.py:71-122) + argvals (:125-145) + targets (:148-172)."""
    table = TABLES[co.version.minor]
    code = co.code
    if not code:
        raise TruncatedCode("empty code object")
    if len(code) % 2:
        raise TruncatedCode("odd code length")
    out = []
    pos = 0
    acc = 0
    npre = 0
    start = 0
    while pos < len(code):
        op = code[pos]
        info = table.get(op)
        if info is None:
            raise UnknownOpcode(op, pos)
        name, has_arg, kind, cache = info
        if op == 144:
            acc = (acc | code[pos + 1]) << 8
            npre += 1
            pos += 2
            if pos >= len(code):
                raise TruncatedCode(f"code ends inside EXTENDED_ARG run at {pos}")
            continue
        ins = Ins(start, pos, name, op, (code[pos + 1] | acc) if has_arg else None, npre, cache, kind)
        pos += 2
        if cache:
            if pos + 2 * cache > len(code):
                raise TruncatedCode(f"code ends inside inline cache of {name} at {pos}")
            pos += 2 * cache
        out.append(ins)
        acc = 0
        npre = 0
        start = pos
    if not out:
        raise TruncatedCode("code holds no instruction")
    minor = co.version.minor
    cmp_op = CMP_OP[minor]
    for ins in out:
        a = ins.arg
        if a is None:
            continue
        k = ins.kind
        if k == "const":
            ins.argval = co.consts[a] if a < len(co.consts) else None
        elif k == "name":
            i = a >> 1 if (minor >= 11 and ins.opname == "LOAD_GLOBAL") else a
            ins.argval = co.names[i] if i < len(co.names) else None
        elif k == "local":
            tab = co.varnames if minor <= 10 else localsplus(co)
            ins.argval = tab[a] if a < len(tab) else None
        elif k == "free":
            tab = localsplus(co) if minor >= 11 else co.cellvars + co.freevars
            ins.argval = tab[a] if a < len(tab) else None
        elif k == "compare":
            ins.argval = cmp_op[a] if a < len(cmp_op) else None
    starts = {i.offset for i in out}
    for ins in out:
        if not ins.jumps:
            continue
        if ins.kind == "jump_abs":
            t = ins.arg * 2 if minor == 10 else ins.arg
        elif ins.kind == "jump_back":
            t = ins.op_offset + 2 - 2 * ins.arg
        else:
            t = ins.op_offset + 2 + (ins.arg * 2 if minor >= 10 else ins.arg)
        if t not in starts:
            raise BadJumpTarget(ins.offset, t)
        ins.argval = t
    return out


def exception_table(co):
    """decode_exception_table (disasm.py:175-214): list of (start, end, target, depth, lasti)."""
    data = co.exceptiontable
    at = [0]

    def num(first):
        p = at[0]
        if p >= len(data):
            raise MalformedExceptionTable(f"truncated varint at byte {p}")
        b = data[p]
        if first and not b & 0x80:
            raise MalformedExceptionTable(f"missing entry marker at byte {p}")
        p += 1
        v = b & 0x3F
        while b & 0x40:
            if p >= len(data):
                raise MalformedExceptionTable(f"truncated varint at byte {p}")
            b = data[p]
            if b & 0x80:
                raise MalformedExceptionTable(f"entry marker inside varint at byte {p}")
            p += 1
            v = (v << 6) | (b & 0x3F)
        at[0] = p
        return v

    rows = []
    while at[0] < len(data):
        s = num(True) * 2
        ln = num(False) * 2
        t = num(False) * 2
        dl = num(False)
        if ln <= 0:
            raise MalformedExceptionTable(f"empty range in entry at byte {at[0]}")
        rows.append((s, s + ln, t, dl >> 1, bool(dl & 1)))
    return rows


def collapse_send(instrs):
    """rewrite_yield_from (pipeline.py:57-87)."""
    res = []
    i = 0
    while i < len(instrs):
        x = instrs[i]
        if x.opname == "SEND":
            names = [y.opname for y in instrs[i + 1:i + 4]]
            k = 3 if names[:2] == ["YIELD_VALUE", "JUMP_BACKWARD_NO_INTERRUPT"] else (
                4 if names == ["YIELD_VALUE", "RESUME", "JUMP_BACKWARD_NO_INTERRUPT"] else 0)
            if k and instrs[i + k - 1].argval == x.offset:
                units = (instrs[i + k - 1].end - x.offset) // 2 - 1
                res.append(Ins(x.offset, x.offset, "YIELD_FROM_311", -1, None, 0, units, "none"))
                i += k
                continue
        res.append(x)
        i += 1
    return res


def find_index(instrs, off):
    """_index_of (structurer.py:163-173) by bisection."""
    lo, hi = 0, len(instrs)
    while lo < hi:
        mid = (lo + hi) // 2
        if instrs[mid].offset < off:
            lo = mid + 1
        else:
            hi = mid
    if lo == len(instrs) or instrs[lo].offset != off:
        raise StructuringFailed(off, "offset is not an instruction boundary")
    return lo


class Region:
    __slots__ = ("start", "end", "handler", "kind", "setup")

    def __init__(self, start, end, handler, kind, setup=-1):
        self.start, self.end, self.handler, self.kind, self.setup = start, end, handler, kind, setup


def regions(co, instrs, table_rows):
    """match_try_regions (structurer.py:62-151)."""
    if co.version.minor <= 10:
        found = []
        for x in instrs:
            if x.opname not in ("SETUP_FINALLY", "SETUP_WITH"):
                continue
            if x.opname == "SETUP_WITH":
                kind = "with"
            else:
                j = find_index(instrs, x.argval)
                first = instrs[j]
                if first.opname == "DUP_TOP" or (
                        first.opname == "POP_TOP" and j + 2 < len(instrs)
                        and instrs[j + 1].opname == "POP_TOP" and instrs[j + 2].opname == "POP_TOP"):
                    kind = "except"
                else:
                    kind = "finally"
            found.append(Region(x.end, x.argval, x.argval, kind, x.offset))
        return found
    at = {x.offset: x for x in instrs}
    by_handler = {}
    for (s, e, t, _d, _l) in table_rows:
        tgt = at.get(t)
        if tgt is None or tgt.opname != "PUSH_EXC_INFO":
            continue
        j = find_index(instrs, t)
        kind = "finally"
        nxt = j + 1
        if nxt < len(instrs) and instrs[nxt].opname == "WITH_EXCEPT_START":
            kind = "with"
        else:
            k = nxt
            while k < len(instrs) and k < nxt + 24:
                nm = instrs[k].opname
                if nm == "CHECK_EXC_MATCH" or (nm == "POP_TOP" and k == nxt):
                    kind = "except"
                    break
                if nm in ("LOAD_GLOBAL", "LOAD_NAME", "LOAD_FAST", "LOAD_CONST", "LOAD_ATTR", "BUILD_TUPLE",
                          "EXTENDED_ARG"):
                    k += 1
                    continue
                break
            if kind != "except":
                seq = [y.opname for y in instrs[j + 1:j + 4]][:3]
                if seq in (["LOAD_CONST", "STORE_FAST", "DELETE_FAST"], ["LOAD_CONST", "STORE_NAME", "DELETE_NAME"]):
                    kind = "as_cleanup"
        r = by_handler.get(t)
        if r is None:
            by_handler[t] = Region(s, e, t, kind)
        else:
            r.start = min(r.start, s)
            r.end = max(r.end, e)
    return list(by_handler.values())


# ------------------------------------------------------------------ CFG

class Graph:
    """Basic blocks as parallel lists indexed by block id (cfg.py:72-141)."""

    def __init__(self):
        self.start = []
        self.stop = []
        self.body = []       # list of Ins lists
        self.succ = []       # list of [(dst, kind)]
        self.pred = []
        self.at = {}         # start offset -> id (alive only after pruning)
        self.entry = 0
        self.alive = []


ENDS = ("RETURN_VALUE", "RAISE_VARARGS", "RERAISE", "END_FINALLY")
CONDS = ("JUMP_IF_FALSE_OR_POP", "JUMP_IF_TRUE_OR_POP", "JUMP_IF_NOT_EXC_MATCH", "CALL_FINALLY")


def blocks(instrs, rows):
    g = Graph()
    last = instrs[-1].end
    lead = {instrs[0].offset}
    for x in instrs:
        if x.jumps:
            lead.add(x.argval)
    for x in instrs:
        if (x.opname in ENDS or (x.jumps and x.opname not in SETUPS)) and x.end < last:
            lead.add(x.end)
    for (s, e, t, _d, _l) in rows:
        lead.add(t)
        lead.add(s)
        if e < last:
            lead.add(e)
    order = sorted(lead)
    k = 0
    for i, s in enumerate(order):
        e = order[i + 1] if i + 1 < len(order) else last
        while k < len(instrs) and instrs[k].offset < s:
            k += 1
        j = k
        while j < len(instrs) and instrs[j].offset < e:
            j += 1
        g.start.append(s)
        g.stop.append(e)
        g.body.append(instrs[k:j] if e > s else [])
        g.succ.append([])
        g.pred.append([])
        g.alive.append(True)
        g.at[s] = i

    def edge(src, off, kind):
        dst = g.at[off]
        g.succ[src].append((dst, kind))
        g.pred[dst].append(src)

    for b in range(len(order)):
        if not g.body[b]:
            continue
        x = g.body[b][-1]
        falls = True
        if x.opname in ("RETURN_VALUE", "RAISE_VARARGS", "RERAISE"):
            falls = False
        elif x.opname == "FOR_ITER":
            edge(b, x.argval, "jump_taken")
            edge(b, x.end, "jump_not_taken")
            falls = False
        elif x.jumps and x.opname not in SETUPS:
            edge(b, x.argval, "jump_taken")
            if x.opname.startswith("POP_JUMP") or x.opname in CONDS:
                edge(b, x.end, "jump_not_taken")
            falls = False
        if falls and g.stop[b] < last:
            edge(b, g.stop[b], "fallthrough")
    for (s, e, t, _d, _l) in rows:
        h = g.at[t]
        for b in range(len(order)):
            if g.start[b] < e and g.stop[b] > s and (h, "exception") not in g.succ[b] and b != h:
                g.succ[b].append((h, "exception"))
                g.pred[h].append(b)
    g.entry = g.at[instrs[0].offset]
    return g


def reach(g, root, with_exc=False):
    seen = set()
    todo = [root]
    while todo:
        b = todo.pop()
        if b in seen:
            continue
        seen.add(b)
        for d, k in g.succ[b]:
            if (with_exc or k != "exception") and d not in seen:
                todo.append(d)
    return seen


def prune(g):
    keep = reach(g, g.entry, True)
    for b in range(len(g.start)):
        if b not in keep:
            g.alive[b] = False
            continue
        g.succ[b] = [(d, k) for d, k in g.succ[b] if d in keep]
        g.pred[b] = [p for p in g.pred[b] if p in keep]
    g.at = {off: b for off, b in g.at.items() if b in keep}


def _normal_edge(g, p, b):
    return any(d == b and k != "exception" for d, k in g.succ[p])


def idoms(g, root, universe):
    """compute_dominators (cfg.py:160-220) with an explicit-stack DFS."""
    post = []
    seen = {root}
    stack = [(root, iter(g.succ[root]))]
    while stack:
        b, it = stack[-1]
        for d, k in it:
            if k != "exception" and d in universe and d not in seen:
                seen.add(d)
                stack.append((d, iter(g.succ[d])))
                break
        else:
            post.append(b)
            stack.pop()
    rpo = post[::-1]
    pos = {b: i for i, b in enumerate(rpo)}
    dom = {root: root}
    changed = True
    while changed:
        changed = False
        for b in rpo:
            if b == root:
                continue
            ps = [p for p in g.pred[b] if p in dom and p in universe and _normal_edge(g, p, b)]
            if not ps:
                continue
            cur = ps[0]
            for p in ps[1:]:
                x, y = cur, p
                while x != y:
                    while pos[x] > pos[y]:
                        x = dom[x]
                    while pos[y] > pos[x]:
                        y = dom[y]
                cur = x
            if dom.get(b) != cur:
                dom[b] = cur
                changed = True
    return dom


def dominates(dom, a, b):
    while True:
        if a == b:
            return True
        up = dom.get(b)
        if up is None or up == b:
            return a == b
        b = up


class LoopInfo:
    __slots__ = ("header", "body", "tails")

    def __init__(self, header, body, tails):
        self.header, self.body, self.tails = header, body, tails


def loops_of(g, dom, universe):
    """analyze_loops (cfg.py:241-313): (reducible, {header: LoopInfo})."""
    roots = [b for b in sorted(universe) if all(p not in universe for p in g.pred[b])]
    root = roots[0] if roots else (g.entry if g.entry in universe else min(universe))
    retreat = []
    seen = {root}
    active = {root}
    stack = [(root, iter(g.succ[root]))]
    while stack:
        u, it = stack[-1]
        for v, k in it:
            if k == "exception" or v not in universe:
                continue
            if v not in seen:
                seen.add(v)
                active.add(v)
                stack.append((v, iter(g.succ[v])))
                break
            if v in active:
                retreat.append((u, v))
        else:
            active.discard(u)
            stack.pop()
    ok = True
    tails = {}
    for u, v in retreat:
        if dominates(dom, v, u):
            tails.setdefault(v, []).append(u)
        else:
            ok = False
    out = {}
    for h, ts in tails.items():
        body = {h}
        todo = list(ts)
        while todo:
            x = todo.pop()
            if x in body:
                continue
            body.add(x)
            for p in g.pred[x]:
                if p in universe and _normal_edge(g, p, x):
                    todo.append(p)
        out[h] = LoopInfo(h, body, list(ts))
    return ok, out


def analyze(co):
    """pipeline.py:17-54: instructions, table rows, graph and loop map."""
    instrs = decode(co)
    if co.version.minor >= 11:
        instrs = collapse_send(instrs)
        offs = {x.offset for x in instrs}
        rows = [r for r in exception_table(co) if r[2] in offs]
    else:
        rows = [(r.start, r.end, r.handler, 0, False) for r in regions(co, instrs, ())]
    g = blocks(instrs, rows)
    prune(g)
    dom = idoms(g, g.entry, reach(g, g.entry))
    ok, loops = loops_of(g, dom, set(dom))
    if not ok:
        raise StructuringFailed(g.entry, "irreducible control flow")
    covered = set(dom)
    for (_s, _e, t, _d, _l) in rows:
        root = g.at.get(t)
        if root is None or root in covered:
            continue
        uni = reach(g, root) - covered
        if not uni:
            continue
        sub = idoms(g, root, uni | {root})
        ok, sl = loops_of(g, sub, set(sub))
        if not ok:
            raise StructuringFailed(root, "irreducible control flow in handler")
        for h, lp in sl.items():
            loops.setdefault(h, lp)
        covered |= set(sub)
    return instrs, rows, g, loops


# ------------------------------------------------------------------ simulation

NB_OPS = ["+", "&", "//", "<<", "@", "*", "%", "|", "**", ">>", "-", "/", "^"]
BIN = {"ADD": "+", "SUBTRACT": "-", "MULTIPLY": "*", "TRUE_DIVIDE": "/", "FLOOR_DIVIDE": "//", "MODULO": "%",
       "POWER": "**", "LSHIFT": "<<", "RSHIFT": ">>", "AND": "&", "OR": "|", "XOR": "^", "MATRIX_MULTIPLY": "@"}
UNARY = {"UNARY_NEGATIVE": "-", "UNARY_POSITIVE": "+", "UNARY_INVERT": "~"}
ASYNC = {"GET_AITER", "GET_ANEXT", "BEFORE_ASYNC_WITH", "SETUP_ASYNC_WITH", "END_ASYNC_FOR", "GET_AWAITABLE",
         "ASYNC_GEN_WRAP", "SEND"}
NOOPS = {"NOP", "RESUME", "PRECALL", "MAKE_CELL", "COPY_FREE_VARS", "GEN_START", "SETUP_ANNOTATIONS",
         "POP_BLOCK", "GET_ITER", "GET_YIELD_FROM_ITER", "CALL_FINALLY"}
COND = {  # name -> (jump_when, none_test, pops)
    "POP_JUMP_IF_FALSE": (False, None, True), "POP_JUMP_IF_TRUE": (True, None, True),
    "POP_JUMP_FORWARD_IF_FALSE": (False, None, True), "POP_JUMP_FORWARD_IF_TRUE": (True, None, True),
    "POP_JUMP_BACKWARD_IF_FALSE": (False, None, True), "POP_JUMP_BACKWARD_IF_TRUE": (True, None, True),
    "POP_JUMP_FORWARD_IF_NONE": (True, True, True), "POP_JUMP_FORWARD_IF_NOT_NONE": (True, False, True),
    "POP_JUMP_BACKWARD_IF_NONE": (True, True, True), "POP_JUMP_BACKWARD_IF_NOT_NONE": (True, False, True),
    "JUMP_IF_FALSE_OR_POP": (False, None, False), "JUMP_IF_TRUE_OR_POP": (True, None, False),
}
PLAIN_JUMPS = ("JUMP_FORWARD", "JUMP_ABSOLUTE", "JUMP_BACKWARD", "JUMP_BACKWARD_NO_INTERRUPT")
SCALAR_STORE = {"STORE_FAST": "fast", "STORE_NAME": "name", "STORE_GLOBAL": "global", "STORE_DEREF": "deref"}
FLIP = {"==": "!=", "!=": "==", "<": ">=", ">=": "<", ">": "<=", "<=": ">", "in": "not in", "not in": "in",
        "is": "is not", "is not": "is"}


def negate(e):
    """symexec.py:1002-1012."""
    if isinstance(e, n.Compare) and len(e.ops) == 1 and e.ops[0] in FLIP:
        return n.Compare(e.left, [FLIP[e.ops[0]]], e.comparators)
    if isinstance(e, n.UnaryOp) and e.op == "not":
        return e.operand
    return n.UnaryOp("not", e)


def effectful(e):
    return not isinstance(e, (n.ConstE, n.FuncExpr, n.Lambda, n.NullSlot, n.MethodSelf))


def splice(v, as_set=False):
    """_spread (symexec.py:991-999)."""
    if isinstance(v, (n.TupleE, n.ListE)) or (as_set and isinstance(v, n.SetE)):
        return list(v.elts)
    if isinstance(v, n.ConstE) and v.const.kind in ("tuple", "frozenset"):
        return [n.ConstE(c) for c in v.const.value]
    return [n.Starred(v)]


def _root_attr(e):
    while isinstance(e, n.Attr):
        e = e.value
    return e


def _nullify(e):
    return None if isinstance(e, n.ConstE) and e.const.kind == "none" else e


class Outcome:
    """BlockResult (symexec.py:103-112)."""
    __slots__ = ("stmts", "fall", "jump", "term")

    def __init__(self, stmts, fall, jump, term):
        self.stmts, self.fall, self.jump, self.term = stmts, fall, jump, term


class Machine:
    """Per-code-object simulator (symexec.py:128-944)."""

    def __init__(self, co):
        self.co = co
        self.minor = co.version.minor
        self.kw = None
        self.comp = co.name in ("<listcomp>", "<setcomp>", "<dictcomp>")

    # -- stack helpers
    def pop(self, st, x):
        if not st:
            raise StackUnderflow(x.offset, x.opname)
        return st.pop()

    def take(self, st, x):
        v = self.pop(st, x)
        pend = getattr(v, "_pending_targets", None)
        if pend:
            last = pend.pop()
            del v._pending_targets
            w = n.NamedExpr(last, v)
            for t in reversed(pend):
                w = n.NamedExpr(t, w)
            return w
        return v

    def many(self, st, x, k):
        if len(st) < k:
            raise StackUnderflow(x.offset, x.opname)
        vals = st[len(st) - k:]
        del st[len(st) - k:]
        return vals

    @staticmethod
    def fold(v):
        pend = getattr(v, "_pending_targets", None)
        if pend:
            del v._pending_targets
            for t in reversed(pend):
                v = n.NamedExpr(t, v)
        return v

    def run(self, body, entry, block_id):
        st = list(entry)
        out = []
        i = 0
        while i < len(body):
            x = body[i]
            nm = x.opname
            if nm in ASYNC:
                raise UnsupportedOpcode(nm, x.offset)
            if nm in NOOPS:
                i += 1
                continue
            if nm == "RETURN_VALUE":
                out.append(n.Return(self.pop(st, x)))
                return Outcome(out, None, None, x)
            if nm == "RAISE_VARARGS":
                exc = cause = None
                if x.arg >= 2:
                    cause = self.pop(st, x)
                if x.arg >= 1:
                    exc = self.pop(st, x)
                out.append(n.Raise(exc, cause))
                return Outcome(out, None, None, x)
            if nm == "RERAISE":
                return Outcome(out, None, None, x)
            if nm in PLAIN_JUMPS:
                out.append(n.JumpMarker(x.argval))
                return Outcome(out, None, list(st), x)
            if nm in COND:
                when, none_test, pops = COND[nm]
                if pops:
                    c = self.pop(st, x)
                    if none_test is not None:
                        c = n.Compare(c, ["is" if none_test else "is not"], [n.ConstE(Const("none"))])
                    out.append(n.CondJumpMarker(c, when, x.argval))
                    return Outcome(out, list(st), list(st), x)
                c = st[-1] if st else self.pop(st, x)
                out.append(n.CondJumpMarker(c, when, x.argval, False))
                return Outcome(out, st[:-1], list(st), x)
            if nm == "JUMP_IF_NOT_EXC_MATCH":
                ty = self.pop(st, x)
                ex = self.pop(st, x)
                out.append(n.CondJumpMarker(n.Compare(ex, ["exception match"], [ty]), False, x.argval))
                return Outcome(out, list(st), list(st), x)
            if nm == "FOR_ITER":
                return Outcome(out, st + [n.ForItem(st[-1] if st else None)], st[:-1] if st else [], x)
            if nm == "END_FINALLY":
                if st and isinstance(st[-1], n.FinallySentinel):
                    st.pop()
                return Outcome(out, list(st), None, x)
            fn = OPS.get(nm)
            if fn is None:
                if nm.startswith("BINARY_") and nm[7:] in BIN:
                    fn = _binop(BIN[nm[7:]], False)
                elif nm.startswith("INPLACE_") and nm[8:] in BIN:
                    fn = _binop(BIN[nm[8:]], True)
                else:
                    raise UnsupportedOpcode(nm, x.offset)
            used = fn(self, x, st, out, body, i)
            i += 1 + (used or 0)
            if len(st) > self.co.stacksize + 6:
                raise StackDepthMismatch(block_id, len(st))
        return Outcome(out, list(st), None, None)

    # -- stores
    def store(self, x, st, out, body, i, target):
        """_store (symexec.py:295-399)."""
        v = self.pop(st, x)
        if isinstance(v, n.UnpackSlot):
            v.group.targets[v.index] = target
            self.finish_group(v.group, out)
            return 0
        if isinstance(v, n.ImportExpr) and v.fromlist is None:
            root = v.module.split(".")[0]
            if type(target) is n.Name and target.id == root:
                out.append(n.Import(v.module))
            else:
                out.append(n.Import(v.module, target.id if isinstance(target, n.Name) else None))
            return 0
        if isinstance(v, n.ImportFromExpr) and isinstance(v.source, n.ImportExpr):
            imp = v.source
            if imp.fromlist is None:
                out.append(n.Import(imp.module, target.id if isinstance(target, n.Name) else None))
                return 0
            alias = target.id if isinstance(target, n.Name) and target.id != v.name else None
            if out and isinstance(out[-1], n.ImportFrom) and getattr(out[-1], "_source", None) is imp:
                out[-1].names.append((v.name, alias))
            else:
                s = n.ImportFrom(imp.module, [(v.name, alias)], imp.level)
                s._source = imp
                out.append(s)
            return 0
        if isinstance(v, n.Attr) and isinstance(_root_attr(v), n.ImportExpr):
            out.append(n.Import(_root_attr(v).module, target.id if isinstance(target, n.Name) else None))
            return 0
        if any(e is v for e in st):
            pend = getattr(v, "_pending_targets", None)
            if pend is None:
                v._pending_targets = pend = []
            pend.append(target)
            return 0
        targets = [target]
        pend = getattr(v, "_pending_targets", None)
        if pend:
            targets = pend + [target]
            del v._pending_targets
        if len(targets) == 1 and isinstance(v, n.BinOp) and v.inplace and v.left == target:
            out.append(n.AugAssign(target, v.op, v.right))
            return 0
        blockers = (n.UnpackSlot, n.NullSlot, n.MethodSelf)
        rest = body[i + 1:]
        if (len(targets) == 1 and x.opname in SCALAR_STORE and rest and rest[0].opname in SCALAR_STORE and st
                and not isinstance(st[-1], blockers) and not hasattr(st[-1], "_pending_targets")
                and not any(e is st[-1] for e in st[:-1])):
            pairs = [(target, v)]
            k = 0
            while k < len(rest) and rest[k].opname in SCALAR_STORE and st and not isinstance(st[-1], blockers):
                y = rest[k]
                pairs.append((n.Name(y.argval, SCALAR_STORE[y.opname]), self.pop(st, y)))
                k += 1
            if self.minor >= 11:
                pairs.reverse()
            out.append(n.Assign([n.TupleE([t for t, _ in pairs])], n.TupleE([u for _, u in pairs])))
            return k
        out.append(n.Assign(targets, v))
        return 0

    def finish_group(self, g, out):
        if any(t is None for t in g.targets):
            return
        elts = list(g.targets)
        if g.star_index >= 0:
            elts[g.star_index] = n.Starred(elts[g.star_index])
        tup = n.TupleE(elts)
        if g.parent is None:
            out.append(n.Assign([tup], g.source))
        else:
            pg, idx = g.parent
            pg.targets[idx] = tup
            self.finish_group(pg, out)

    def unpack(self, st, src, total, star):
        g = n.UnpackGroup(src, total, star, [None] * total,
                          (src.group, src.index) if isinstance(src, n.UnpackSlot) else None)
        for idx in range(total - 1, -1, -1):
            st.append(n.UnpackSlot(src, total, idx, -1, 0, g))


def _binop(sym, inplace):
    def f(m, x, st, out, body, i):
        r = m.take(st, x)
        l = m.take(st, x)
        st.append(n.BinOp(sym, l, r, inplace))
    return f


def _push(fn):
    def f(m, x, st, out, body, i):
        st.extend(fn(m, x))
    return f


def _store_name(scope):
    def f(m, x, st, out, body, i):
        return m.store(x, st, out, body, i, n.Name(x.argval, scope))
    return f


def _del_name(scope):
    def f(m, x, st, out, body, i):
        out.append(n.Delete([n.Name(x.argval, scope)]))
    return f


def _op_store_attr(m, x, st, out, body, i):
    obj = m.pop(st, x)
    return m.store(x, st, out, body, i, n.Attr(obj, x.argval))


def _op_store_subscr(m, x, st, out, body, i):
    idx = m.pop(st, x)
    obj = m.pop(st, x)
    return m.store(x, st, out, body, i, n.Subscript(obj, idx))


def _op_unpack_seq(m, x, st, out, body, i):
    m.unpack(st, m.pop(st, x), x.arg, -1)


def _op_unpack_ex(m, x, st, out, body, i):
    src = m.pop(st, x)
    lo, hi = x.arg & 0xFF, x.arg >> 8
    m.unpack(st, src, lo + 1 + hi, lo)


def _op_del_attr(m, x, st, out, body, i):
    out.append(n.Delete([n.Attr(m.pop(st, x), x.argval)]))


def _op_del_subscr(m, x, st, out, body, i):
    idx = m.pop(st, x)
    obj = m.pop(st, x)
    out.append(n.Delete([n.Subscript(obj, idx)]))


def _op_binary_op(m, x, st, out, body, i):
    inplace = x.arg >= 13
    _binop(NB_OPS[x.arg - 13 if inplace else x.arg], inplace)(m, x, st, out, body, i)


def _op_subscr(m, x, st, out, body, i):
    idx = m.take(st, x)
    obj = m.take(st, x)
    st.append(n.Subscript(obj, idx))


def _cmp(label):
    def f(m, x, st, out, body, i):
        r = m.take(st, x)
        l = m.take(st, x)
        st.append(n.Compare(l, [label(x)], [r]))
    return f


def _op_pop_top(m, x, st, out, body, i):
    v = m.pop(st, x)
    if isinstance(v, (n.ImportExpr, n.NullSlot, n.MethodSelf, n.ExcValue, n.FinallySentinel, n.WithEnter)):
        return
    if getattr(v, "_loop_iter", False):
        return
    if isinstance(v, n.Call) and isinstance(v.func, n.WithExit):
        return
    pend = getattr(v, "_pending_targets", None)
    if pend:
        del v._pending_targets
        out.append(n.Assign(pend, v))
        return
    if effectful(v):
        out.append(n.ExprStmt(v))


def _op_rot2(m, x, st, out, body, i):
    st[-1], st[-2] = st[-2], st[-1]


def _op_rot3(m, x, st, out, body, i):
    st[-1], st[-2], st[-3] = st[-2], st[-3], st[-1]


def _op_rot4(m, x, st, out, body, i):
    st[-1], st[-2], st[-3], st[-4] = st[-2], st[-3], st[-4], st[-1]


def _op_rotn(m, x, st, out, body, i):
    top = st[-1]
    del st[-1]
    st.insert(len(st) - (x.arg - 1), top)


def _op_swap(m, x, st, out, body, i):
    st[-1], st[-x.arg] = st[-x.arg], st[-1]


def _op_copy(m, x, st, out, body, i):
    st.append(st[-x.arg])


def _op_dup(m, x, st, out, body, i):
    st.append(st[-1])


def _op_dup2(m, x, st, out, body, i):
    st.extend(st[-2:])


def _op_not(m, x, st, out, body, i):
    st.append(negate(m.take(st, x)))


def _unary(sym):
    def f(m, x, st, out, body, i):
        st.append(n.UnaryOp(sym, m.take(st, x)))
    return f


def _build(cls):
    def f(m, x, st, out, body, i):
        st.append(cls([m.fold(v) for v in m.many(st, x, x.arg)]))
    return f


def _op_build_map(m, x, st, out, body, i):
    kv = m.many(st, x, 2 * x.arg)
    ks = [m.fold(v) for v in kv[0::2]]
    vs = [m.fold(v) for v in kv[1::2]]
    st.append(n.DictE(ks, vs))


def _op_const_key_map(m, x, st, out, body, i):
    kc = m.pop(st, x)
    vs = [m.fold(v) for v in m.many(st, x, x.arg)]
    st.append(n.DictE([n.ConstE(k) for k in kc.const.value], vs))


def _op_build_slice(m, x, st, out, body, i):
    parts = m.many(st, x, x.arg)
    lo, hi = parts[0], parts[1]
    step = parts[2] if x.arg == 3 else None
    st.append(n.SliceE(_nullify(lo), _nullify(hi), _nullify(step) if step is not None else None))


def _op_build_string(m, x, st, out, body, i):
    parts = []
    for v in m.many(st, x, x.arg):
        if isinstance(v, n.ConstE) and v.const.kind == "str":
            parts.append(v.const.value)
        elif isinstance(v, n.FString):
            parts.extend(v.parts)
        else:
            parts.append(v)
    st.append(n.FString(parts))


def _op_format_value(m, x, st, out, body, i):
    spec = m.pop(st, x) if x.arg & 4 else None
    val = m.take(st, x)
    st.append(n.FString([n.FormattedValue(val, ("", "s", "r", "a")[x.arg & 3], spec)]))


def _accum(kind, cls, label):
    def f(m, x, st, out, body, i):
        v = m.take(st, x)
        if m.comp:
            out.append(n.CompAccum(kind, v, None, x.arg))
            return
        t = st[-x.arg]
        if not isinstance(t, cls):
            raise UnsupportedOpcode(label, x.offset)
        t.elts.append(v)
    return f


def _op_map_add(m, x, st, out, body, i):
    v = m.take(st, x)
    k = m.take(st, x)
    if m.comp:
        out.append(n.CompAccum("map", v, k, x.arg))
        return
    t = st[-x.arg]
    if not isinstance(t, n.DictE):
        raise UnsupportedOpcode("MAP_ADD outside display", x.offset)
    t.keys.append(k)
    t.values.append(v)


def _extend(cls, as_set, label):
    def f(m, x, st, out, body, i):
        it = m.take(st, x)
        t = st[-x.arg]
        if not isinstance(t, cls):
            raise UnsupportedOpcode(label, x.offset)
        t.elts.extend(splice(it, as_set))
    return f


def _op_dict_update(m, x, st, out, body, i):
    other = m.take(st, x)
    t = st[-x.arg]
    if not isinstance(t, n.DictE):
        raise UnsupportedOpcode("DICT_UPDATE outside display", x.offset)
    if isinstance(other, n.DictE) and len(other.keys) <= 8 and all(k is not None for k in other.keys):
        t.keys.extend(other.keys)
        t.values.extend(other.values)
    else:
        t.keys.append(None)
        t.values.append(other)


def _op_list_to_tuple(m, x, st, out, body, i):
    v = m.pop(st, x)
    st.append(n.TupleE(v.elts) if isinstance(v, n.ListE) else v)


def _unpack_display(cls):
    def f(m, x, st, out, body, i):
        parts = []
        for v in m.many(st, x, x.arg):
            parts.extend(splice(v, cls is n.SetE))
        st.append(cls(parts))
    return f


def _op_map_unpack(m, x, st, out, body, i):
    ks, vs = [], []
    for v in m.many(st, x, x.arg):
        if isinstance(v, n.DictE) and all(k is not None for k in v.keys):
            ks.extend(v.keys)
            vs.extend(v.values)
        else:
            ks.append(None)
            vs.append(v)
    st.append(n.DictE(ks, vs))


def _op_load_attr(m, x, st, out, body, i):
    st.append(n.Attr(m.take(st, x), x.argval))


def _op_load_method(m, x, st, out, body, i):
    obj = m.take(st, x)
    st.append(n.Attr(obj, x.argval))
    st.append(n.MethodSelf())


def _op_kw_names(m, x, st, out, body, i):
    m.kw = tuple(c.value for c in x.argval.value)


def _call_done(m, st, x, args, kwnames=()):
    kws = []
    if kwnames:
        k = len(kwnames)
        kws = list(zip(kwnames, args[-k:]))
        args = args[:-k]
    top = m.pop(st, x)
    if m.minor >= 11:
        under = m.pop(st, x)
        if isinstance(under, n.NullSlot):
            fn = top
        elif isinstance(top, n.MethodSelf):
            fn = under
        else:
            fn = under
            args = [top] + args
    else:
        fn = top
    st.append(n.Call(fn, args, kws))


def _op_call_function(m, x, st, out, body, i):
    _call_done(m, st, x, [m.fold(v) for v in m.many(st, x, x.arg)])


def _op_call_function_kw(m, x, st, out, body, i):
    names = tuple(c.value for c in m.pop(st, x).const.value)
    _call_done(m, st, x, [m.fold(v) for v in m.many(st, x, x.arg)], names)


def _op_call_method(m, x, st, out, body, i):
    args = [m.fold(v) for v in m.many(st, x, x.arg)]
    m.pop(st, x)
    st.append(n.Call(m.pop(st, x), args, []))


def _op_call(m, x, st, out, body, i):
    args = [m.fold(v) for v in m.many(st, x, x.arg)]
    kw = m.kw or ()
    m.kw = None
    _call_done(m, st, x, args, kw)


def _op_call_ex(m, x, st, out, body, i):
    kwargs = m.take(st, x) if x.arg & 1 else None
    pos = m.take(st, x)
    fn = m.pop(st, x)
    if m.minor >= 11 and st and isinstance(st[-1], n.NullSlot):
        st.pop()
    args = list(splice(pos))
    kws = []
    if kwargs is not None:
        if isinstance(kwargs, n.DictE):
            for k, v in zip(kwargs.keys, kwargs.values):
                if k is None:
                    kws.append((None, v))
                elif isinstance(k, n.ConstE) and k.const.kind == "str":
                    kws.append((k.const.value, v))
                else:
                    kws.append((None, n.DictE([k], [v])))
        else:
            kws.append((None, kwargs))
    st.append(n.Call(fn, args, kws))


def _op_make_function(m, x, st, out, body, i):
    flags = x.arg
    if m.minor <= 10:
        m.pop(st, x)
    cc = m.pop(st, x)
    closure, ann, kwd, dflt = (), [], [], []
    if flags & 8:
        closure = tuple(c.id for c in m.pop(st, x).elts)
    if flags & 4:
        a = m.pop(st, x)
        if isinstance(a, n.DictE):
            ann = [(k.const.value, v) for k, v in zip(a.keys, a.values)]
        elif isinstance(a, n.ConstE):
            names = [c.value for c in a.const.value]
            ann = list(zip(names, [None] * len(names)))
    if flags & 2:
        d = m.pop(st, x)
        kwd = [(k.const.value, v) for k, v in zip(d.keys, d.values)]
    if flags & 1:
        d = m.pop(st, x)
        dflt = list(d.elts) if isinstance(d, n.TupleE) else [n.ConstE(c) for c in d.const.value]
    st.append(n.FuncExpr(cc.const.value, dflt, kwd, ann, closure))


def _op_import_name(m, x, st, out, body, i):
    fl = m.pop(st, x)
    lv = m.pop(st, x)
    names = tuple(c.value for c in fl.const.value) if fl.const.kind == "tuple" else None
    st.append(n.ImportExpr(x.argval, names, lv.const.value))


def _op_import_from(m, x, st, out, body, i):
    st.append(n.ImportFromExpr(st[-1], x.argval))


def _op_import_star(m, x, st, out, body, i):
    imp = m.pop(st, x)
    out.append(n.ImportStar(imp.module, imp.level))


def _op_yield(m, x, st, out, body, i):
    st.append(n.Yield(m.take(st, x)))


def _op_yield_from(m, x, st, out, body, i):
    m.pop(st, x)
    st.append(n.YieldFrom(m.pop(st, x)))


def _op_pop_finally(m, x, st, out, body, i):
    keep = m.pop(st, x) if x.arg else None
    if st and isinstance(st[-1], n.FinallySentinel):
        st.pop()
    if keep is not None:
        st.append(keep)


def _op_pop_except(m, x, st, out, body, i):
    for _ in range(1 if m.minor >= 11 else 3):
        if st:
            st.pop()


def _op_push_exc_info(m, x, st, out, body, i):
    e = m.pop(st, x)
    st.append(n.ExcValue(1))
    st.append(e)


def _op_check_exc_match(m, x, st, out, body, i):
    ty = m.take(st, x)
    st.append(n.Compare(st[-1], ["exception match"], [ty]))


def _op_setup_with(m, x, st, out, body, i):
    c = m.take(st, x)
    st.append(n.WithExit(c))
    st.append(n.WithEnter(c))


def _op_with_cleanup_start(m, x, st, out, body, i):
    if len(st) >= 2 and isinstance(st[-1], n.FinallySentinel) and isinstance(st[-2], n.WithExit):
        s = st.pop()
        st.pop()
        st.append(s)
        st.append(n.NullSlot())
        return
    raise UnsupportedOpcode(x.opname, x.offset)


def _op_with_cleanup_finish(m, x, st, out, body, i):
    if st and isinstance(st[-1], n.NullSlot):
        st.pop()
        return
    raise UnsupportedOpcode(x.opname, x.offset)


def _op_unsupported(m, x, st, out, body, i):
    raise UnsupportedOpcode(x.opname, x.offset)


def _op_get_len(m, x, st, out, body, i):
    st.append(n.Call(n.Name("len", "global"), [st[-1]], []))


def _nothing(m, x, st, out, body, i):
    return None


OPS = {
    "LOAD_CONST": _push(lambda m, x: [n.ConstE(x.argval)]),
    "LOAD_FAST": _push(lambda m, x: [n.Name(x.argval, "fast")]),
    "LOAD_GLOBAL": _push(lambda m, x: ([n.NullSlot()] if m.minor >= 11 and x.arg & 1 else [])
                         + [n.Name(x.argval, "global")]),
    "LOAD_NAME": _push(lambda m, x: [n.Name(x.argval, "name")]),
    "LOAD_DEREF": _push(lambda m, x: [n.Name(x.argval, "deref")]),
    "LOAD_CLASSDEREF": _push(lambda m, x: [n.Name(x.argval, "deref")]),
    "LOAD_CLOSURE": _push(lambda m, x: [n.Name(x.argval, "cell")]),
    "LOAD_ASSERTION_ERROR": _push(lambda m, x: [n.Name("AssertionError", "global")]),
    "LOAD_BUILD_CLASS": _push(lambda m, x: [n.BuildClass()]),
    "PUSH_NULL": _push(lambda m, x: [n.NullSlot()]),
    "STORE_FAST": _store_name("fast"), "STORE_NAME": _store_name("name"),
    "STORE_GLOBAL": _store_name("global"), "STORE_DEREF": _store_name("deref"),
    "STORE_ATTR": _op_store_attr, "STORE_SUBSCR": _op_store_subscr,
    "UNPACK_SEQUENCE": _op_unpack_seq, "UNPACK_EX": _op_unpack_ex,
    "DELETE_FAST": _del_name("fast"), "DELETE_NAME": _del_name("name"),
    "DELETE_GLOBAL": _del_name("global"), "DELETE_DEREF": _del_name("deref"),
    "DELETE_ATTR": _op_del_attr, "DELETE_SUBSCR": _op_del_subscr,
    "BINARY_OP": _op_binary_op, "BINARY_SUBSCR": _op_subscr,
    "COMPARE_OP": _cmp(lambda x: x.argval),
    "IS_OP": _cmp(lambda x: "is not" if x.arg else "is"),
    "CONTAINS_OP": _cmp(lambda x: "not in" if x.arg else "in"),
    "POP_TOP": _op_pop_top, "ROT_TWO": _op_rot2, "ROT_THREE": _op_rot3, "ROT_FOUR": _op_rot4,
    "ROT_N": _op_rotn, "SWAP": _op_swap, "COPY": _op_copy, "DUP_TOP": _op_dup, "DUP_TOP_TWO": _op_dup2,
    "UNARY_NOT": _op_not, **{k: _unary(v) for k, v in UNARY.items()},
    "BUILD_TUPLE": _build(n.TupleE), "BUILD_LIST": _build(n.ListE), "BUILD_SET": _build(n.SetE),
    "BUILD_MAP": _op_build_map, "BUILD_CONST_KEY_MAP": _op_const_key_map, "BUILD_SLICE": _op_build_slice,
    "BUILD_STRING": _op_build_string, "FORMAT_VALUE": _op_format_value,
    "LIST_APPEND": _accum("list", n.ListE, "LIST_APPEND outside display"),
    "SET_ADD": _accum("set", n.SetE, "SET_ADD outside display"),
    "MAP_ADD": _op_map_add,
    "LIST_EXTEND": _extend(n.ListE, False, "LIST_EXTEND outside display"),
    "SET_UPDATE": _extend(n.SetE, True, "SET_UPDATE outside display"),
    "DICT_UPDATE": _op_dict_update, "DICT_MERGE": _op_dict_update, "LIST_TO_TUPLE": _op_list_to_tuple,
    "BUILD_TUPLE_UNPACK": _unpack_display(n.TupleE), "BUILD_TUPLE_UNPACK_WITH_CALL": _unpack_display(n.TupleE),
    "BUILD_LIST_UNPACK": _unpack_display(n.ListE), "BUILD_SET_UNPACK": _unpack_display(n.SetE),
    "BUILD_MAP_UNPACK": _op_map_unpack, "BUILD_MAP_UNPACK_WITH_CALL": _op_map_unpack,
    "LOAD_ATTR": _op_load_attr, "LOAD_METHOD": _op_load_method, "KW_NAMES": _op_kw_names,
    "CALL_FUNCTION": _op_call_function, "CALL_FUNCTION_KW": _op_call_function_kw,
    "CALL_METHOD": _op_call_method, "CALL": _op_call, "CALL_FUNCTION_EX": _op_call_ex,
    "MAKE_FUNCTION": _op_make_function, "IMPORT_NAME": _op_import_name, "IMPORT_FROM": _op_import_from,
    "IMPORT_STAR": _op_import_star, "YIELD_VALUE": _op_yield, "YIELD_FROM": _op_yield_from,
    "YIELD_FROM_311": _op_yield_from, "RETURN_GENERATOR": _push(lambda m, x: [n.NullSlot()]),
    "SETUP_FINALLY": _nothing, "BEGIN_FINALLY": _push(lambda m, x: [n.FinallySentinel()]),
    "POP_FINALLY": _op_pop_finally, "POP_EXCEPT": _op_pop_except, "PUSH_EXC_INFO": _op_push_exc_info,
    "CHECK_EXC_MATCH": _op_check_exc_match, "SETUP_WITH": _op_setup_with, "BEFORE_WITH": _op_setup_with,
    "WITH_CLEANUP_START": _op_with_cleanup_start, "WITH_CLEANUP_FINISH": _op_with_cleanup_finish,
    "WITH_EXCEPT_START": _op_unsupported, "GET_LEN": _op_get_len,
}
