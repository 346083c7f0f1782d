""".pyc loader corpus: valid .pyc images of the synthetic golden objects in
several marshal encodings, plus seeded mutants that exercise every failure
branch of the reference reader (pyc.py:36-352): truncation, damaged headers,
unknown/unsupported type bytes, negative and huge lengths, bad back-references,
undecodable text, text floats, out-of-range long digits, deep nesting and
3.11 localsplus kinds that do not round-trip.

A case is a small JSON-able record {"spec", "enc", "mut"}; `blob(rec)`
rebuilds its bytes deterministically.
"""
from __future__ import annotations

import random
import struct

from . import cases, marshal

ENCODINGS = ({}, {"refs": False}, {"long_tuples": True, "unicode_all": True},
             # equal bytes objects shared by back-reference (co_code, line tables and
             # bytes constants of different code objects alias one marshal object)
             {"share_bytes": True})

JUNK = (b"f\x031.5", b"f\x02xx", b"f\x041_00", b"f\x03inf", b"f\x05 -2e3", b"f\x04+nan", b"f\x021_",
        b"l\x02\x00\x00\x00\xff\xff\x00\x00", b"l\xfe\xff\xff\xff\x01\x00\x02\x00", b"l\x00\x00\x00\x00",
        b"u\x02\x00\x00\x00\xc3\x28", b"u\x03\x00\x00\x00\xed\xa0\x80", b"u\x04\x00\x00\x00\xf0\x9f\x98\x80",
        b"u\x02\x00\x00\x00\xc0\x80", b"r\x00\x00\x00\x00", b"r\xff\x00\x00\x00", b"r\xff\xff\xff\xff",
        b"\xa9\x00", b"(\x01\x00\x00\x00", b"a\x02\x00\x00\x00\xe9\xff", b"<\x00\x00\x00\x00", b"[", b"S",
        b"y" + struct.pack("<dd", 1.5, -0.0), b"g" + struct.pack("<d", float("nan")))


def blob(rec) -> bytes:
    co = cases.build(rec["spec"])
    b = bytearray(marshal.dump_pyc(co, **ENCODINGS[rec["enc"]]))
    mut = rec.get("mut")
    if mut is None:
        return bytes(b)
    kind, seed = mut
    rng = random.Random(seed)
    if kind == "truncate":
        b = b[:rng.randrange(len(b))]
    elif kind == "flip":
        i = rng.randrange(len(b))
        b[i] = rng.randrange(256)
    elif kind == "type":
        i = rng.randrange(16, len(b))
        b[i] = rng.choice(b"ilgfysutaAzZ()>cr[{<S0?NTF.\x00\x7f") | rng.choice([0, 0x80])
    elif kind == "int32":
        i = rng.randrange(16, max(17, len(b) - 4))
        b[i:i + 4] = struct.pack("<i", rng.choice([-1, -5, 2 ** 31 - 1, 300, 70000]))
    elif kind == "header":
        k = rng.randrange(4)
        if k == 0:
            b = b[:rng.randrange(16)]
        elif k == 1:
            b[2] = 0
        elif k == 2:
            b[0:2] = struct.pack("<H", rng.choice([3400, 3430, 3500, 0xFFFF, 0]))
        else:
            b[3] = ord("x")
    elif kind == "junk":
        i = rng.randrange(16, len(b))
        b[i:i] = rng.choice(JUNK)
    elif kind == "nest":
        # depth limit 256 (pyc.py:75,107); the reference itself hits Python's
        # recursion limit from ~245 levels, so only 256+ stays in the parity domain
        depth = rng.choice([256, 257, 300, 1000])
        b = b[:16] + b")\x01" * depth + b"N"
    elif kind == "dup":
        i = rng.randrange(16, len(b))
        j = min(len(b), i + rng.randrange(1, 12))
        b[i:i] = b[i:j]
    elif kind == "delete":
        i = rng.randrange(16, len(b))
        del b[i:min(len(b), i + rng.randrange(1, 8))]
    elif kind == "kinds":  # 3.11 localsplus kinds bits
        idx = [k for k in range(16, len(b) - 5) if b[k] == ord("s")]
        if idx:
            k = rng.choice(idx)
            ln = struct.unpack("<i", b[k + 1:k + 5])[0]
            if 0 < ln < 64 and k + 5 + ln <= len(b):
                p = k + 5 + rng.randrange(ln)
                b[p] ^= rng.choice([0x20, 0x40, 0x80, 0x60])
    else:
        raise KeyError(kind)
    return bytes(b)


MUTATIONS = ("truncate", "flip", "type", "int32", "header", "junk", "nest", "dup", "delete", "kinds")


def corpus(n_valid_per_set=24, n_mutants=600, seed=0x9C):
    """Case records: every encoding of a sample of each golden set, then mutants."""
    rng = random.Random(seed)
    specs = []
    for name in ("c1", "snippets", "fuzz", "c3"):
        specs += cases.GOLDEN_SETS[name][:n_valid_per_set]
    specs += [{"case": f"shared-bytes-3.{m}", "gen": "shared_bytes", "minor": m} for m in (8, 9, 10, 11)]
    out = []
    for i, spec in enumerate(specs):
        for e in range(len(ENCODINGS)):
            out.append({"case": f"pyc-valid-{i}-{e}", "spec": spec, "enc": e, "mut": None})
    for i in range(n_mutants):
        spec = rng.choice(specs)
        kind = MUTATIONS[i % len(MUTATIONS)]
        out.append({"case": f"pyc-mut-{i}", "spec": spec, "enc": rng.randrange(len(ENCODINGS)),
                    "mut": [kind, rng.randrange(1 << 30)]})
    return out
