"""Oracle: region structuring and tree canonicalisation.

Restates structurer.py:176-1197 of /root/reference/pkg/src/unpyre.  Walk
exits are (kind, target, stack) tuples; contexts are small immutable tuples.
"""
from __future__ import annotations

from paper_2403_13839_b200.errors import StackDepthMismatch, StructuringFailed
from paper_2403_13839_b200.model import Const

from . import lift
from . import nodes as n

FALL, JUMP, ENDED, NEXT, ENDFIN = "fall", "jump", "ended", "next", "end_finally"
FAR = 1 << 60


class Ctx:
    __slots__ = ("cont", "brk", "joins", "range_end")

    def __init__(self, cont=frozenset(), brk=-1, joins=(), range_end=FAR):
        self.cont, self.brk, self.joins, self.range_end = cont, brk, joins, range_end

    def join(self, off):
        return Ctx(self.cont, self.brk, self.joins + (off,), self.range_end)

    def nojoins(self):
        return Ctx(self.cont, self.brk, (), self.range_end)

    def ranged(self, end):
        return Ctx(self.cont, self.brk, self.joins, end)


def bool_join(op, a, b):
    parts = []
    for e in (a, b):
        if isinstance(e, n.BoolOp) and e.op == op:
            parts.extend(e.values)
        else:
            parts.append(e)
    return n.BoolOp(op, parts)


def trim_continue(body):
    """_strip_trailing_continue (structurer.py:992-1002), in place."""
    while body and isinstance(body[-1], n.Continue):
        body.pop()
    if body and isinstance(body[-1], n.Try):
        t = body[-1]
        trim_continue(t.body)
        for h in t.handlers:
            trim_continue(h.body)
        if t.orelse:
            trim_continue(t.orelse)
    return body


BLOCK_FIELDS = ("then", "orelse", "body", "final")


def _cleanup_pair(st, name):
    return (len(st) == 2 and isinstance(st[0], n.Assign) and len(st[0].targets) == 1
            and isinstance(st[0].targets[0], n.Name) and st[0].targets[0].id == name
            and isinstance(st[0].value, n.ConstE) and st[0].value.const.kind == "none"
            and isinstance(st[1], n.Delete) and isinstance(st[1].targets[0], n.Name)
            and st[1].targets[0].id == name)


def drop_as_cleanup(body, name):
    if name is None:
        return body
    if (len(body) == 1 and isinstance(body[0], n.Try) and not body[0].handlers and not body[0].orelse
            and _cleanup_pair(body[0].final, name)):
        return body[0].body
    if len(body) >= 2 and _cleanup_pair(body[-2:], name):
        return body[:-2]
    return body


def drop_final_copies(stmts, final):
    """strip_finally_copies (structurer.py:1089-1112)."""
    if not final:
        return stmts
    k = len(final)
    res = []
    i = 0
    while i < len(stmts):
        if stmts[i:i + k] == final:
            nxt = stmts[i + k] if i + k < len(stmts) else None
            if nxt is None or isinstance(nxt, (n.Return, n.Break, n.Continue)):
                i += k
                continue
        s = stmts[i]
        for f in BLOCK_FIELDS:
            sub = getattr(s, f, None)
            if isinstance(sub, list):
                setattr(s, f, drop_final_copies(sub, final))
        if isinstance(s, n.Try):
            for h in s.handlers:
                h.body = drop_final_copies(h.body, final)
        res.append(s)
        i += 1
    return res


class Shaper:
    """Structurer (structurer.py:176-971)."""

    def __init__(self, co, instrs, g, loops, rows):
        self.co = co
        self.minor = co.version.minor
        self.ins = instrs
        self.g = g
        self.loops = loops
        self.regs = lift.regions(co, instrs, rows)
        self.by_start = {}
        for r in self.regs:
            if r.kind in ("except", "finally", "with"):
                self.by_start.setdefault(r.start, []).append(r)
        for rs in self.by_start.values():
            rs.sort(key=lambda r: -r.end)
        self.m = lift.Machine(co)
        self.temps = 0
        self.active_regs = []
        self.active_loops = set()
        self.end = instrs[-1].end

    def block(self, off):
        b = self.g.at.get(off)
        if b is None:
            raise StructuringFailed(off, "no block starts here")
        return b

    def sim(self, b, stack):
        return self.m.run(self.g.body[b], stack, b)

    def top(self):
        return self.walk([(self.ins[0].offset, self.end)], [], Ctx())[0]

    def walk(self, segs, stack, ctx):
        out = []
        si = 0
        pos = segs[0][0]
        while True:
            if pos >= segs[si][1]:
                si += 1
                if si >= len(segs):
                    return out, (FALL, pos, stack)
                pos = segs[si][0]
                continue
            if pos not in self.g.at:
                return out, (ENDED, -1, None)
            cand = [r for r in self.by_start.get(pos, []) if r not in self.active_regs]
            if cand:
                pos, stack = self.region(cand[0], out, stack, ctx)
                if pos is None:
                    return out, (ENDED, -1, None)
                continue
            b = self.g.at[pos]
            lp = self.loops.get(b)
            if lp is not None and b not in self.active_loops:
                pos, stack = self.loop(lp, b, out, stack, ctx)
                if pos is None:
                    return out, (ENDED, -1, None)
                continue
            res = self.sim(b, stack)
            ex = self.consume(b, res, out, stack, ctx.ranged(segs[si][1]))
            if ex is None:
                pos, stack = self.g.stop[b], res.fall
                continue
            if ex[0] == NEXT:
                pos, stack = ex[1], ex[2]
                continue
            return out, ex

    def consume(self, b, res, out, stack, ctx):
        t = res.term
        if t is None:
            out.extend(res.stmts)
            return None
        nm = t.opname
        if nm in ("RETURN_VALUE", "RAISE_VARARGS", "RERAISE"):
            out.extend(res.stmts)
            return (ENDED, -1, None)
        if nm == "END_FINALLY":
            out.extend(res.stmts)
            return (ENDFIN, self.g.stop[b], res.fall)
        if nm in lift.PLAIN_JUMPS:
            out.extend(res.stmts[:-1])
            return self.jump_to(t.argval, res.jump, out, ctx)
        if nm == "FOR_ITER":
            raise StructuringFailed(b, "FOR_ITER outside a loop header")
        out.extend(res.stmts[:-1])
        return self.conditional(b, res.stmts[-1], res, out, stack, ctx)

    def jump_to(self, target, stack, out, ctx):
        if target in ctx.cont:
            out.append(n.Continue())
            return (ENDED, -1, None)
        if target == ctx.brk:
            out.append(n.Break())
            return (ENDED, -1, None)
        return (JUMP, target, stack)

    # ------------------------------------------------------------ loops
    def exits_max(self, lo, hi):
        best = -1
        for x in self.ins:
            if lo <= x.offset < hi and x.jumps and x.opname not in lift.SETUPS and x.argval >= hi:
                best = max(best, x.argval)
        return best

    def loop(self, lp, h, out, stack, ctx):
        lo = min(self.g.start[b] for b in lp.body)
        hi = max(self.g.stop[b] for b in lp.body)
        self.active_loops.add(h)
        try:
            hr = self.sim(h, stack)
            t = hr.term
            if t is not None and t.opname == "FOR_ITER":
                return self.for_loop(h, hr, out, stack, ctx)
            if (t is not None and not hr.stmts[:-1] and isinstance(hr.stmts[-1], n.CondJumpMarker)
                    and hr.stmts[-1].pops_on_jump and not (lo <= t.argval < hi)):
                mk = hr.stmts[-1]
                cond = mk.cond if not mk.jump_when else lift.negate(mk.cond)
                after = t.argval
                brk = max(self.exits_max(self.g.stop[h], after), after)
                body, _ = self.walk([(self.g.stop[h], after)], hr.jump,
                                    Ctx(frozenset({self.g.start[h]}), brk))
                body = trim_continue(body) or [n.Pass()]
                orelse, after = self.loop_else(after, brk, stack, ctx)
                out.append(n.While(cond, body, orelse))
                return after, stack
            return self.while_true(lp, h, out, stack, ctx, lo, hi)
        finally:
            self.active_loops.discard(h)

    def for_loop(self, h, hr, out, stack, ctx):
        after = hr.term.argval
        it = stack[-1] if stack else None
        if it is None:
            raise StructuringFailed(h, "FOR_ITER with empty stack")
        it._loop_iter = True
        out.extend(hr.stmts)
        brk = max(self.exits_max(self.g.stop[h], after), after)
        body, _ = self.walk([(self.g.stop[h], after)], hr.fall, Ctx(frozenset({self.g.start[h]}), brk))
        if not body:
            raise StructuringFailed(h, "empty for body")
        first = body[0]
        if not (isinstance(first, n.Assign) and len(first.targets) == 1 and isinstance(first.value, n.ForItem)):
            raise StructuringFailed(h, "for loop does not store its item")
        target, body = first.targets[0], body[1:]
        body = trim_continue(body) or [n.Pass()]
        orelse, nxt = self.loop_else(after, brk, stack, ctx)
        out.append(n.For(target, it, body, orelse))
        return nxt, stack[:-1]

    def while_true(self, lp, h, out, stack, ctx, lo, hi):
        after = hi
        brk = max(self.exits_max(lo, hi), hi)
        tail = None
        for u in lp.tails:
            last = self.g.body[u][-1]
            if last.opname.startswith("POP_JUMP") or last.opname in ("JUMP_IF_TRUE_OR_POP", "JUMP_IF_FALSE_OR_POP"):
                tail = u
                break
        hs = self.g.start[h]
        cont = {hs} if tail is None else {hs, self.g.start[tail]}
        bctx = Ctx(frozenset(cont), brk)
        segs = [(hs, hi)]
        if lo < hs:
            segs.append((lo, hs))
        if tail is not None and self.g.start[tail] >= hs:
            segs[0] = (hs, self.g.start[tail])
            if lo < hs:
                raise StructuringFailed(h, "rotated loop with tail re-test")
        body, _ = self.walk(segs, list(stack), bctx)
        tail_cond = None
        if tail is not None:
            tr = self.sim(tail, stack)
            mk = tr.stmts[-1] if tr.stmts else None
            if isinstance(mk, n.CondJumpMarker) and not tr.stmts[:-1] and mk.target == hs:
                tail_cond = mk.cond if mk.jump_when else lift.negate(mk.cond)
            else:
                extra, ex = self.walk([(self.g.start[tail], hi)], list(stack), bctx)
                body.extend(extra)
                if ex[0] == FALL:
                    body.append(n.Break())
        body = trim_continue(body) or [n.Pass()]
        orelse, nxt = self.loop_else(after, brk, stack, ctx)
        out.append(n._WhileShape(n.ConstE(Const("bool", True)), body, orelse, tail_cond))
        return nxt, stack

    def loop_else(self, after, brk, stack, ctx):
        if brk > after:
            orelse, _ = self.walk([(after, brk)], list(stack), ctx.join(brk))
            return orelse, brk
        return [], after

    # ------------------------------------------------------------ conditionals
    def conditional(self, b, mk, res, out, stack, ctx):
        cond, when, target = mk.cond, mk.jump_when, mk.target
        fall, jstate = res.fall, res.jump
        bstart, bend = self.g.start[b], self.g.stop[b]
        if target <= bstart:
            if target in ctx.cont:
                out.append(n.If(cond if when else lift.negate(cond), [n.Continue()], []))
                return (NEXT, bend, fall)
            raise StructuringFailed(b, "unexpected backward conditional jump")
        if not mk.pops_on_jump:
            return self.orpop(b, mk, res, out, ctx)
        p, target, fpos, fall = self.chain(lift.negate(cond) if when else cond, target, bend, fall)
        if target in ctx.cont:
            out.append(n.If(lift.negate(p), [n.Continue()], []))
            return (NEXT, fpos, fall)
        if target == ctx.brk and target not in set(ctx.joins):
            out.append(n.If(lift.negate(p), [n.Break()], []))
            return (NEXT, fpos, fall)
        then, tx = self.walk([(fpos, target)], list(fall), ctx.join(target))
        if tx[0] == FALL and tx[1] > target:
            out.append(n.If(p, then, []))
            return (NEXT, tx[1], tx[2] if tx[2] is not None else jstate)
        if (len(then) == 1 and isinstance(then[0], n.Raise) and tx[0] == ENDED and _asserts(then[0])):
            exc = then[0].exc
            msg = exc.args[0] if isinstance(exc, n.Call) and exc.args else None
            out.append(n.Assert(lift.negate(p), msg))
            return (NEXT, target, jstate)
        if tx[0] == ENDED:
            out.append(n.If(p, then, []))
            return (NEXT, target, jstate)
        if tx[0] == JUMP and tx[1] != target:
            join = tx[1]
            if join <= target or join > ctx.range_end:
                more, _ = self.walk([(join, self.end)], tx[2], ctx)
                then.extend(more)
                out.append(n.If(p, then, []))
                return (NEXT, target, jstate)
            other, ox = self.walk([(target, join)], list(jstate), ctx.join(join))
            ts = tx[2]
            es = ox[2] if ox[0] in (JUMP, FALL) else None
            if (not then and not other and ts is not None and es is not None and len(ts) == len(fall) + 1
                    and len(es) == len(fall) + 1 and ts[:-1] == es[:-1]):
                return (NEXT, join, ts[:-1] + [n.Ternary(p, ts[-1], es[-1])])
            if ts is not None and es is not None:
                if len(ts) != len(es):
                    raise StackDepthMismatch(b, [len(ts), len(es)])
                if ts == es:
                    out.append(n.If(p, then, other))
                    return (NEXT, join, ts)
                merged = self.spill([ts, es], b, [then, other])
                out.append(n.If(p, then, other))
                return (NEXT, join, merged)
            out.append(n.If(p, then, other))
            return (NEXT, join, ts if ts is not None else es)
        ts = tx[2]
        if ts is not None and len(ts) != len(jstate):
            raise StructuringFailed(b, "branch leaves a value on one path")
        if ts is not None and ts != jstate:
            pre = []
            merged = self.spill([ts, jstate], b, [then, pre])
            out.extend(pre)
            out.append(n.If(p, then, []))
            return (NEXT, target, merged)
        out.append(n.If(p, then, []))
        return (NEXT, target, ts if ts is not None else jstate)

    def spill(self, states, b, sinks):
        """merge_stack_states (symexec.py:1027-1051); spill assigns go to sinks."""
        depths = sorted({len(s) for s in states})
        if len(depths) != 1:
            raise StackDepthMismatch(b, depths)
        merged = []
        for slot in range(depths[0]):
            vals = [s[slot] for s in states]
            if all(v == vals[0] for v in vals[1:]):
                merged.append(vals[0])
                continue
            name = f"__stack_{self.temps}"
            self.temps += 1
            for v, sink in zip(vals, sinks):
                sink.append(n.Assign([n.Name(name, "fast")], v))
            merged.append(n.Name(name, "fast"))
        return merged

    def chain(self, p, target, fpos, fall):
        """_collect_chain (structurer.py:619-655)."""
        while True:
            b = self.g.at.get(fpos)
            if b is None:
                break
            if b in self.loops or self.g.start[b] in self.by_start:
                break
            r = self.sim(b, fall)
            mk = r.stmts[-1] if r.stmts else None
            if (r.term is None or not isinstance(mk, n.CondJumpMarker) or r.stmts[:-1] or not mk.pops_on_jump
                    or mk.target <= self.g.start[b]):
                break
            p2 = lift.negate(mk.cond) if mk.jump_when else mk.cond
            if mk.target == target:
                p = bool_join("and", p, p2)
            elif target == self.g.stop[b]:
                p = bool_join("or", lift.negate(p), p2)
                target = mk.target
            else:
                break
            fpos, fall = self.g.stop[b], r.fall
        return p, target, fpos, fall

    def orpop(self, b, mk, res, out, ctx):
        """_structure_orpop (structurer.py:657-719)."""
        op = "or" if mk.jump_when else "and"
        join = mk.target
        kept = res.jump[-1]
        chained = (op == "and" and isinstance(kept, n.Compare) and len(res.jump) >= 2
                   and res.jump[-2] is kept.comparators[-1])
        rhs, rx = self.walk([(self.g.stop[b], join)], list(res.fall), ctx.join(join))
        if chained and not rhs and rx[0] in (JUMP, FALL):
            s2 = rx[2]
            if (s2 is not None and len(s2) == len(res.fall) and isinstance(s2[-1], n.Compare)
                    and s2[-1].left is kept.comparators[-1]):
                fused = n.Compare(kept.left, kept.ops + s2[-1].ops, kept.comparators + s2[-1].comparators)
                if self.fixup(join):
                    return (NEXT, rx[1], s2[:-1] + [fused])
        if (chained and rx[0] == ENDED and len(rhs) == 1 and isinstance(rhs[0], n.Return)
                and isinstance(rhs[0].value, n.Compare) and rhs[0].value.left is kept.comparators[-1]
                and self.fixup(join, True)):
            r = rhs[0].value
            out.append(n.Return(n.Compare(kept.left, kept.ops + r.ops, kept.comparators + r.comparators)))
            return (ENDED, -1, None)
        if rhs or rx[0] == ENDED or rx[2] is None or len(rx[2]) != len(res.jump):
            raise StructuringFailed(b, "unstructured short-circuit value")
        return (NEXT, join, res.jump[:-1] + [bool_join(op, kept, rx[2][-1])])

    def fixup(self, off, returning=False):
        b = self.g.at.get(off)
        if b is None:
            return False
        names = [x.opname for x in self.g.body[b]]
        if returning:
            return names in (["ROT_TWO", "POP_TOP", "RETURN_VALUE"], ["SWAP", "POP_TOP", "RETURN_VALUE"])
        return names in (["ROT_TWO", "POP_TOP"], ["SWAP", "POP_TOP"])

    # ------------------------------------------------------------ regions
    def region(self, r, out, stack, ctx):
        self.active_regs.append(r)
        try:
            if r.kind == "with":
                return self.with_region(r, out, stack, ctx)
            if r.kind == "finally":
                return self.finally_region(r, out, stack, ctx)
            return self.except_region(r, out, stack, ctx)
        finally:
            self.active_regs.remove(r)

    def exc_stack(self, base):
        if self.minor >= 11:
            return list(base) + [n.ExcValue(0)]
        return list(base) + [n.ExcValue(i) for i in range(6)]

    def with_region(self, r, out, stack, ctx):
        ce = None
        for e in reversed(stack):
            if isinstance(e, n.WithExit):
                ce = e.context
                break
        if ce is None:
            raise StructuringFailed(self.g.at.get(r.start, -1), "with region without context on stack")
        target = None
        if out and isinstance(out[-1], n.Assign) and isinstance(out[-1].value, n.WithEnter) \
                and out[-1].value.context is ce:
            target = out.pop().targets[0]
        body, bx = self.walk([(r.start, r.handler)], list(stack), ctx)
        if target is None and body:
            f = body[0]
            if isinstance(f, n.Assign) and isinstance(f.value, n.WithEnter) and f.value.context is ce:
                target = f.targets[0]
                body = body[1:]
        rest = [e for e in stack if not (isinstance(e, (n.WithExit, n.WithEnter)) and e.context is ce)]
        if self.minor == 8 and bx[0] == FALL:
            extra, x2 = self.walk([(r.handler, self.end)], bx[2], ctx.nojoins())
            body.extend(extra)
            bx = (JUMP, x2[1], rest) if x2[0] in (ENDFIN, JUMP, FALL) else (ENDED, -1, None)
        out.append(n.With([n.WithItem(ce, target)], body or [n.Pass()]))
        if bx[0] == JUMP:
            return bx[1], rest
        if bx[0] == FALL and bx[1] < r.handler:
            return bx[1], rest
        return None, rest

    def after_handler(self, r):
        i = lift.find_index(self.ins, r.handler)
        depth = 0
        while i < len(self.ins):
            x = self.ins[i]
            if x.opname in ("RERAISE", "END_FINALLY") and depth == 0:
                return x.end
            if x.opname in ("SETUP_FINALLY", "SETUP_WITH"):
                depth += 1
            if x.opname == "POP_BLOCK" and depth:
                depth -= 1
            i += 1
        return self.end

    def finally_region(self, r, out, stack, ctx):
        if self.minor == 8:
            return self.finally_38(r, out, stack, ctx)
        final, _ = self.walk([(r.handler, self.end)], self.exc_stack([]), ctx.nojoins())
        bctx = ctx.join(r.handler)
        body, bx = self.walk([(r.start, r.end)], list(stack), bctx)
        if bx[0] == ENDED:
            tail, tx = [], bx
        else:
            tail, tx = self.walk([(max(r.end, bx[1]), r.handler)], bx[2], bctx)
        body.extend(tail)
        body = drop_final_copies(body, final)
        out.append(n.Try(body or [n.Pass()], [], [], final or [n.Pass()]))
        if tx[0] == JUMP:
            return tx[1], stack
        if tx[0] == FALL and tx[1] > r.handler:
            return tx[1], stack
        if tx[0] == ENDED:
            return None, stack
        return self.after_handler(r), stack

    def finally_38(self, r, out, stack, ctx):
        final, fx = self.walk([(r.handler, self.end)], list(stack) + [n.FinallySentinel()], ctx.nojoins())
        bctx = ctx.join(r.handler)
        body, bx = self.walk([(r.start, r.end)], list(stack), bctx)
        if bx[0] != ENDED:
            tail, _ = self.walk([(max(r.end, bx[1]), r.handler)], bx[2], bctx)
            body.extend(tail)
        out.append(n.Try(body or [n.Pass()], [], [], final or [n.Pass()]))
        if fx[0] == ENDFIN:
            return fx[1], stack
        i = lift.find_index(self.ins, r.handler)
        while i < len(self.ins) and self.ins[i].opname != "END_FINALLY":
            i += 1
        return (self.ins[i].end if i < len(self.ins) else self.end), stack

    def except_region(self, r, out, stack, ctx):
        bctx = ctx.join(r.handler)
        body, bx = self.walk([(r.start, r.end)], list(stack), bctx)
        bj = -1
        if bx[0] == JUMP and bx[1] >= r.handler:
            bj = bx[1]
        elif bx[0] != ENDED:
            tail, tx = self.walk([(max(r.end, bx[1]), r.handler)], bx[2], bctx)
            body.extend(tail)
            if tx[0] == JUMP:
                bj = tx[1]
            elif tx[0] == FALL and tx[1] > r.handler:
                bj = tx[1]
        handlers, hj = self.handlers(r, ctx)
        orelse = []
        join = max(bj, hj)
        if bj != -1 and hj != -1 and bj < hj:
            orelse, _ = self.walk([(bj, hj)], list(stack), ctx.join(hj))
            join = hj
        out.append(n.Try(body or [n.Pass()], handlers, orelse, []))
        return (None if join == -1 else join), stack

    def handlers(self, r, ctx):
        """_parse_handlers (structurer.py:911-953)."""
        hs, joins = [], []
        h = r.handler
        count = 0
        while h is not None and count < 64:
            count += 1
            b = self.block(h)
            entry = self.exc_stack([])
            res = self.sim(b, entry)
            mk = res.stmts[-1] if res.stmts and isinstance(res.stmts[-1], n.CondJumpMarker) else None
            if mk is not None and isinstance(mk.cond, n.Compare) and mk.cond.ops == ["exception match"]:
                ty, nxt, start, st = mk.cond.comparators[0], mk.target, self.g.stop[b], res.fall
            elif res.term is not None and res.term.opname in ("RERAISE", "END_FINALLY") and not res.stmts:
                break
            else:
                ty, nxt, start, st = None, None, h, entry
            end = nxt if nxt is not None else self.end
            body, ex = self.walk([(start, end)], list(st), ctx.nojoins())
            name = None
            if body and isinstance(body[0], n.Assign) and isinstance(body[0].value, n.ExcValue):
                t = body[0].targets[0]
                if isinstance(t, n.Name):
                    name = t.id
                    body = body[1:]
            body = drop_as_cleanup(body, name)
            j = -1
            if ex[0] == JUMP:
                j = ex[1]
            elif ex[0] == FALL and ex[1] > end:
                j = ex[1]
            hs.append(n.ExceptHandler(ty, name, body or [n.Pass()]))
            if j != -1:
                joins.append(j)
            h = nxt
            if ty is None:
                break
        return hs, (max(joins) if joins else -1)


def _asserts(stmt):
    e = stmt.exc
    return ((isinstance(e, n.Name) and e.id == "AssertionError")
            or (isinstance(e, n.Call) and isinstance(e.func, n.Name) and e.func.id == "AssertionError"))


# ------------------------------------------------------------ tree passes

def canon(stmts):
    """canonicalize_tree (structurer.py:1118-1197)."""
    return [_canon(s) for s in stmts]


def _kids(s):
    for f in BLOCK_FIELDS:
        sub = getattr(s, f, None)
        if isinstance(sub, list):
            setattr(s, f, canon(sub))
    if isinstance(s, n.Try):
        for h in s.handlers:
            h.body = canon(h.body)
    return s


def _guard_merge(cond, shape):
    body = list(shape.body)
    tail = shape.tail_cond
    while True:
        if tail is not None and tail == cond:
            return n.While(cond, body or [n.Pass()], shape.orelse)
        if not body:
            return None
        last = body[-1]
        if isinstance(last, n.If) and not last.orelse and len(last.then) == 1 and isinstance(last.then[0], n.Break):
            piece = lift.negate(last.cond)
            tail = piece if tail is None else bool_join("and", piece, tail)
            body.pop()
            continue
        return None


def _canon(s):
    if isinstance(s, n.If) and len(s.then) == 1 and isinstance(s.then[0], n._WhileShape) and not s.orelse:
        merged = _guard_merge(s.cond, s.then[0])
        if merged is not None:
            return _kids(merged)
    if isinstance(s, n._WhileShape):
        body = s.body
        if s.tail_cond is not None:
            body = body + [n.If(lift.negate(s.tail_cond), [n.Break()], [])]
        return _kids(n.While(s.cond, body, s.orelse))
    s = _kids(s)
    if isinstance(s, n.If):
        if len(s.then) == 1 and isinstance(s.then[0], n.If) and not s.orelse and not s.then[0].orelse:
            inner = s.then[0]
            return n.If(bool_join("and", s.cond, inner.cond), inner.then, [])
        return s
    if isinstance(s, n.With) and len(s.body) == 1 and isinstance(s.body[0], n.With):
        inner = s.body[0]
        return n.With(s.items + inner.items, inner.body)
    return s
