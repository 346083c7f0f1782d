"""Label assembler for CPython 3.8-3.11 wordcode.

Builds CodeObjects directly from (opname, arg|label) items: opcode numbers and
inline-cache counts come from the per-version tables (_optables.py), jump args
are encoded per version by inverting the reference's target formulas
(disasm.py:158-164), EXTENDED_ARG prefixes are sized by fixpoint iteration,
and 3.11 exception tables are varint-encoded per disasm.py:175-214.

No 3.8-3.11 interpreter exists in this image, so every synthetic input of the
parity suite and the benchmark corpus is assembled here.
"""
from __future__ import annotations

from .._optables import BY_NAME, TABLES
from ..model import CodeObject, Const, VersionTag

EXT = 144


class Label(str):
    pass


def L(name):
    return Label(name)


class Asm:
    """Accumulates instructions plus const/name/varname pools for one code object."""

    def __init__(self, minor):
        self.minor = minor
        self.items = []
        self.consts = []
        self._const_keys = {}
        self.names = []
        self.varnames = []
        self.freevars = []
        self.cellvars = []
        self.exc = []  # (start_label, end_label, target_label, depth, lasti)
        self._n = 0

    # pools -------------------------------------------------------------
    def const(self, value, kind=None):
        c = value if isinstance(value, Const) else _to_const(value, kind)
        key = (c._key(), id(c.value) if c.kind == "code" else 0)
        if key not in self._const_keys:
            self._const_keys[key] = len(self.consts)
            self.consts.append(c)
        return self._const_keys[key]

    def name(self, s):
        if s not in self.names:
            self.names.append(s)
        return self.names.index(s)

    def var(self, s):
        if s not in self.varnames:
            self.varnames.append(s)
        return self.varnames.index(s)

    def fresh(self, stem="L"):
        self._n += 1
        return Label(f"{stem}{self._n}")

    # emission -----------------------------------------------------------
    def op(self, opname, arg=None):
        self.items.append((opname, arg))
        return self

    def label(self, lab):
        self.items.append(Label(lab) if not isinstance(lab, Label) else lab)
        return self

    def __call__(self, opname, arg=None):
        return self.op(opname, arg)

    def code_bytes(self):
        return assemble(self.items, self.minor)

    def build(self, name="f", argcount=0, posonly=0, kwonly=0, flags=0x43, stacksize=None,
              filename="<synth>", firstlineno=1, qualname="", nlocals=None):
        code, labels = assemble(self.items, self.minor, return_labels=True)
        exctable = encode_exception_table(
            [(labels[s], labels[e], labels[t], d, lasti) for s, e, t, d, lasti in self.exc]
        ) if self.exc else b""
        return CodeObject(
            VersionTag(3, self.minor), argcount, posonly, kwonly,
            len(self.varnames) if nlocals is None else nlocals,
            stacksize if stacksize is not None else 16, flags, code, tuple(self.consts),
            tuple(self.names), tuple(self.varnames), tuple(self.freevars), tuple(self.cellvars),
            name, filename, firstlineno, b"", exctable, qualname,
        )


def _to_const(v, kind=None):
    if kind is not None:
        return Const(kind, v)
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
        return Const("tuple", tuple(_to_const(x) for x in v))
    if isinstance(v, frozenset):
        return Const("frozenset", tuple(_to_const(x) for x in v))
    if isinstance(v, CodeObject) or hasattr(v, "co_code_like"):
        return Const("code", v)
    if hasattr(v, "version") and hasattr(v, "code"):
        return Const("code", v)
    raise TypeError(f"cannot make a Const from {type(v)}")


def _nprefix(arg):
    n = 0
    arg >>= 8
    while arg:
        n += 1
        arg >>= 8
    return n


def assemble(items, minor, return_labels=False):
    table = TABLES[minor]
    by_name = BY_NAME[minor]
    # sizes: units per item (prefixes + 1 + caches); iterate to a fixpoint
    ops = [it for it in items if not isinstance(it, Label)]
    prefixes = [0] * len(ops)
    for _ in range(16):
        labels = {}
        offsets = []
        pos = 0
        k = 0
        for it in items:
            if isinstance(it, Label):
                labels[it] = pos
                continue
            opname, arg = it
            offsets.append(pos)
            info = table[by_name[opname]]
            pos += 2 * (1 + prefixes[k] + info[3])
            k += 1
        changed = False
        args = []
        for k, (opname, arg) in enumerate(ops):
            info = table[by_name[opname]]
            a = arg
            if isinstance(arg, Label):
                tgt = labels[arg]
                op_off = offsets[k] + 2 * prefixes[k]
                kind = info[2]
                if kind == "jump_abs":
                    a = tgt // 2 if minor == 10 else tgt
                elif kind == "jump_back":
                    a = (op_off + 2 - tgt) // 2
                elif kind == "jump_rel":
                    a = (tgt - op_off - 2) // (2 if minor >= 10 else 1)
                else:
                    raise ValueError(f"label arg on non-jump {opname}")
                if a < 0:
                    raise ValueError(f"negative jump arg for {opname} -> {arg}")
            if a is None:
                a = 0
            args.append(a)
            need = _nprefix(a) if info[1] else 0
            if need > prefixes[k]:
                prefixes[k] = need
                changed = True
        if not changed:
            break
    else:
        raise RuntimeError("EXTENDED_ARG sizing did not converge")
    out = bytearray()
    for k, (opname, _arg) in enumerate(ops):
        code = by_name[opname]
        info = table[code]
        a = args[k]
        for j in range(prefixes[k], 0, -1):
            out += bytes((EXT, (a >> (8 * j)) & 0xFF))
        out += bytes((code, a & 0xFF if info[1] else 0))
        out += b"\x00\x00" * info[3]
    if return_labels:
        return bytes(out), labels
    return bytes(out)


def _varint(v, first):
    chunks = [v & 0x3F]
    v >>= 6
    while v:
        chunks.append(v & 0x3F)
        v >>= 6
    chunks.reverse()
    out = []
    for i, c in enumerate(chunks):
        b = c
        if i + 1 < len(chunks):
            b |= 0x40
        if i == 0 and first:
            b |= 0x80
        out.append(b)
    return out


def encode_exception_table(entries):
    """entries: (start, end, target, depth, lasti) in byte offsets."""
    out = []
    for start, end, target, depth, lasti in entries:
        out += _varint(start // 2, True)
        out += _varint((end - start) // 2, False)
        out += _varint(target // 2, False)
        out += _varint((depth << 1) | int(bool(lasti)), False)
    return bytes(out)
