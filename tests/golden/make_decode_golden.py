"""Golden vectors for the decoder stage, made by running the REAL reference's
`unpyre.disasm.decode_instructions` (disasm.py:71-172, incl. resolve_jump_targets
and its is_jump_target marking) on every object (roots and nested codes) of the
golden sets.  Run in the build container:

    python tests/golden/make_decode_golden.py

Each line of decode.jsonl: {"set", "obj", "minor", "status", ...} for object
index `obj` of `arena.pack(inputs)` where the inputs are the set's records
without a style (the same list tests/test_decode.py packs).  status "ok" adds
n (instructions), jt (number of jump targets) and sha: SHA-256 of the records
encoded exactly like the C ABI's upy_ins (include/upy.h:103-110):
<u32 offset, u32 arg (None -> 0; >= 2**32 -> 0xFFFFFFFF), u8 opcode,
u8 n_prefixes (<= 255), u8 cache_units, u8 flags = has_arg | saturated << 1 |
is_jump_target << 2>.  Errors carry the class name and str(exception).
"""
import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

import unpyre  # noqa: E402
from unpyre import disasm  # noqa: E402

from paper_2403_13839_b200 import arena  # noqa: E402
from paper_2403_13839_b200.synth import cases  # noqa: E402

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "c4big")


def records_bytes(instrs):
    out = bytearray()
    for ins in instrs:
        has = ins.arg is not None
        arg = ins.arg if has else 0
        sat = has and arg >= (1 << 32)
        flags = (1 if has else 0) | (2 if sat else 0) | (4 if ins.is_jump_target else 0)
        out += struct.pack("<IIBBBB", ins.offset, 0xFFFFFFFF if sat else arg, ins.opcode,
                           min(ins.n_prefixes, 255), ins.cache_units, flags)
    return bytes(out)


def set_records(name):
    if name == "c4big":
        return cases.C4BIG
    with open(os.path.join(HERE, f"{name}.jsonl")) as f:
        recs = [json.loads(line) for line in f]
    return [r for r in recs if not r.get("style")]


def main():
    path = os.path.join(HERE, "decode.jsonl")
    with open(path, "w") as f:
        for name in SETS:
            if name != "c4big" and not os.path.exists(os.path.join(HERE, f"{name}.jsonl")):
                continue
            recs = set_records(name)
            ar = arena.pack([cases.build(r) for r in recs])
            objs = arena.unpack(ar, unpyre.CodeObject, unpyre.Const, unpyre.VersionTag,
                                objects=range(ar.n_objs))
            n_ok = n_jt = 0
            for i, co in enumerate(objs):
                row = {"set": name, "obj": i, "minor": co.version.minor}
                try:
                    ins = disasm.decode_instructions(co)
                except Exception as e:  # noqa: BLE001
                    row.update(status=type(e).__name__, msg=str(e))
                else:
                    jt = sum(1 for x in ins if x.is_jump_target)
                    n_ok += 1
                    n_jt += jt > 0
                    row.update(status="ok", n=len(ins), jt=jt,
                               sha=hashlib.sha256(records_bytes(ins)).hexdigest()[:32])
                f.write(json.dumps(row) + "\n")
            print(f"{name}: {ar.n_objs} objects, {n_ok} decoded, {n_jt} with jump targets")
    print("->", path)


if __name__ == "__main__":
    main()
