"""Secondary outputs of the decoder and CFG stages on the GPU path:

* `decode_many(codes)` -- `decode_instructions` (disasm.py:71-172) for a batch: the
  decode kernel writes the 12-byte records (upy_decode_batch, include/upy.h), the
  host wraps them as `Instruction`s and resolves argvals from the caller's objects
  (`_resolve_argvals`, disasm.py:125-145; jump targets, disasm.py:148-172);
* `format_listing(instrs)` -- the text listing (disasm.py:224-236);
* `to_dot_many(codes)` -- `to_dot(analyze(code)[2])` (cfg.py:331-344,
  pipeline.py:17-54): the CFG analysis and the Graphviz text are produced on the
  device (csrc/dot.h, upy_options.output = 1), one thread per code object.

Errors follow the reference: an entry is the exception instance decode /
analyze would raise (same class and message).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import errors
from ._optables import CMP_OP, TABLES

EXTENDED_ARG = 144
_JUMPS = ("jump_rel", "jump_abs", "jump_back")


@dataclass
class Instruction:
    """disasm.py:28-58 (same fields, defaults and repr)."""
    offset: int
    op_offset: int
    opname: str
    opcode: int
    arg: int | None
    argval: object = None
    is_jump_target: bool = False
    n_prefixes: int = 0
    cache_units: int = 0
    kind: str = "none"

    @property
    def size(self):
        return 2 * (1 + self.n_prefixes + self.cache_units)

    @property
    def end_offset(self):
        return self.offset + self.size

    @property
    def is_jump(self):
        return self.kind in _JUMPS

    def __repr__(self):
        bits = f"{self.offset} {self.opname}"
        if self.arg is not None:
            bits += f" {self.arg}"
            if self.argval is not None and self.argval != self.arg:
                bits += f" ({self.argval})"
        return f"<{bits}>"


def _localsplus(co):
    """code_model.py:127-139."""
    extra = tuple(c for c in co.cellvars if c not in co.varnames)
    return tuple(co.varnames) + extra + tuple(co.freevars)


def _deref_names(co):
    """code_model.py:141-145."""
    if co.version.minor >= 11:
        return _localsplus(co)
    return tuple(co.cellvars) + tuple(co.freevars)


def _full_arg(code, rec):
    """The record's arg as the reference's Python int (records saturate at
    2**32-1; wide args are re-folded from the EXTENDED_ARG prefix bytes)."""
    if not int(rec["flags"]) & 2:
        return int(rec["arg"])
    off = int(rec["offset"])
    a = 0
    for p in range(int(rec["n_prefixes"])):
        a = (a | code[off + 2 * p + 1]) << 8
    return a | code[off + 2 * int(rec["n_prefixes"]) + 1]


def instructions(co, recs):
    """Instruction list of one object from its decoded records, argvals resolved
    on the host (disasm.py:125-172)."""
    minor = co.version.minor
    table = TABLES[minor]
    cmp_op = CMP_OP[minor]
    code = co.code
    consts, names = co.consts, co.names
    local_names = co.varnames if minor <= 10 else _localsplus(co)
    free_names = None
    out = []
    for r in recs:
        op = int(r["opcode"])
        opname, _has, kind, _cache = table[op]
        has_arg = bool(int(r["flags"]) & 1)
        arg = _full_arg(code, r) if has_arg else None
        n_pre = int(r["n_prefixes"])
        off = int(r["offset"])
        ins = Instruction(offset=off, op_offset=off + 2 * n_pre, opname=opname, opcode=op, arg=arg,
                          is_jump_target=bool(int(r["flags"]) & 4), n_prefixes=n_pre,
                          cache_units=int(r["cache_units"]), kind=kind)
        if arg is not None:
            if kind == "const":
                ins.argval = consts[arg] if arg < len(consts) else None
            elif kind == "name":
                idx = arg >> 1 if (minor >= 11 and opname == "LOAD_GLOBAL") else arg
                ins.argval = names[idx] if idx < len(names) else None
            elif kind == "local":
                ins.argval = local_names[arg] if arg < len(local_names) else None
            elif kind == "free":
                if free_names is None:
                    free_names = _deref_names(co)
                ins.argval = free_names[arg] if arg < len(free_names) else None
            elif kind == "compare":
                ins.argval = cmp_op[arg] if arg < len(cmp_op) else None
            elif kind in _JUMPS:
                if kind == "jump_abs":
                    ins.argval = arg * 2 if minor == 10 else arg
                elif kind == "jump_back":
                    ins.argval = ins.op_offset + 2 - 2 * arg
                else:
                    ins.argval = ins.op_offset + 2 + (arg * 2 if minor >= 10 else arg)
        out.append(ins)
    return out


def decode_exception(co, status, aux0, aux1):
    """The exception decode_instructions raises for a device decode status
    (aux conventions: csrc/decode.h; messages: disasm.py:76-120, errors.py:45-66)."""
    if status == errors.ST_UNKNOWN_OPCODE:
        return errors.make_exception(status, f"unknown opcode {aux0} at offset {aux1}", (aux0, aux1))
    if status == errors.ST_BAD_JUMP_TARGET:
        return errors.make_exception(status, f"jump at offset {aux0} targets {aux1}, not an instruction boundary",
                                     (aux0, aux1))
    if status == errors.ST_TRUNCATED_CODE:
        if aux0 == 1:
            msg = "empty code object"
        elif aux0 == 2:
            msg = "odd code length"
        elif aux0 == 3:
            msg = f"code ends inside EXTENDED_ARG run at {aux1}"
        elif aux0 == 4:
            op = co.code[aux1 - 2]
            msg = f"code ends inside inline cache of {TABLES[co.version.minor][op][0]} at {aux1}"
        else:
            msg = "code holds no instruction"
        return errors.make_exception(status, msg, (0, 0))
    return errors.DeviceCapacityError(f"decode status {status}")


def decode_many(codes, device=None):
    """decode_instructions for every code object of `codes` (each decoded on its
    own; nested code constants are not expanded): list of Instruction lists or
    exception instances, on the GPU decode kernel."""
    import torch

    from .api import DeviceArena
    from .arena import DECODED_DTYPE, INS_DTYPE, pack

    codes = list(codes)
    if not codes:
        return []
    ar = pack(codes)
    da = DeviceArena(ar, device=device)
    da.upload()
    da.run(mode="decode")
    torch.cuda.synchronize(da.device)
    units = ar.total_code_units + 1
    dec_off = (units * INS_DTYPE.itemsize + 255) & ~255
    ws = da.ws[:dec_off + DECODED_DTYPE.itemsize * ar.n_objs].cpu().numpy()
    ins = ws[:units * INS_DTYPE.itemsize].view(INS_DTYPE)
    dec = ws[dec_off:dec_off + DECODED_DTYPE.itemsize * ar.n_objs].view(DECODED_DTYPE)
    objs = ar.section("objs")
    roots = ar.section("roots")
    out = []
    for co, o in zip(codes, roots):
        d = dec[int(o)]
        st = int(d["status"])
        if st != errors.ST_OK:
            out.append(decode_exception(co, st, int(d["aux0"]), int(d["aux1"])))
            continue
        base = int(objs[int(o)]["code_off"]) >> 1
        out.append(instructions(co, ins[base:base + int(d["n_instrs"])]))
    return out


def decode_instructions(code, device=None):
    """Drop-in for unpyre.disasm.decode_instructions (disasm.py:71)."""
    v = decode_many([code], device)[0]
    if isinstance(v, BaseException):
        raise v
    return v


def format_listing(instrs) -> str:
    """disasm.py:224-236."""
    lines = []
    for ins in instrs:
        mark = ">>" if ins.is_jump_target else "  "
        argpart = "" if ins.arg is None else f" {ins.arg}"
        valpart = ""
        if ins.is_jump:
            valpart = f" (to {ins.argval})"
        elif ins.arg is not None and ins.argval is not None:
            valpart = f" ({ins.argval})"
        lines.append(f"{mark} {ins.op_offset:>5} {ins.opname}{argpart}{valpart}")
    return "\n".join(lines) + "\n"


def to_dot_many(codes, device=None):
    """to_dot(analyze(code)[2]) for every code object of `codes`, on the device:
    list of dot texts or exception instances."""
    from .api import run_arena
    from .arena import pack

    codes = list(codes)
    if not codes:
        return []
    res = run_arena(pack(codes), None, device, output=1)
    out = res.values()
    for v in out:
        if isinstance(v, errors.DeviceCapacityError):
            raise v
    return out


def to_dot(code, device=None) -> str:
    """cfg.to_dot(analyze(code)[2]) for one code object."""
    v = to_dot_many([code], device)[0]
    if isinstance(v, BaseException):
        raise v
    return v
