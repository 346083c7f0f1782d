"""Decoder stage (decode_instructions, disasm.py:71-172) against the REAL
reference: tests/golden/decode.jsonl holds, for every object (roots and nested
codes) of the golden sets, the reference's records -- offset, arg, opcode,
n_prefixes, cache_units, has_arg / saturated / is_jump_target flags -- as a
digest of their upy_ins encoding, or the exception class and message
(tests/golden/make_decode_golden.py).

CPU tier: the scalar reference-order decoder (decode_scalar, built for the
host, the same source the device's lane-0 fallback runs).  GPU tier:
upy_decode_batch through the C ABI -- the TMA-pipelined warp path (3.8-3.10),
the warp 3.11 path and the scalar fallback -- record for record.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from helpers import inputs

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "c4big")


def _golden():
    out = {}
    with open(os.path.join(GOLDEN, "decode.jsonl")) as f:
        for line in f:
            r = json.loads(line)
            out.setdefault(r["set"], []).append(r)
    return out


GOLD = _golden()


def _arena(gset):
    from paper_2403_13839_b200 import arena

    from paper_2403_13839_b200.synth import cases

    recs = cases.C4BIG if gset == "c4big" else [r for r in load_golden(gset) if not r.get("style")]
    return arena.pack(inputs(recs))


def decode_error(ar, o, status, a0, a1):
    """(class, message) of a device decode status (aux conventions: csrc/decode.h)."""
    from paper_2403_13839_b200._optables import TABLES

    if status == 2:
        return "UnknownOpcode", f"unknown opcode {a0} at offset {a1}"
    if status == 4:
        return "BadJumpTarget", f"jump at offset {a0} targets {a1}, not an instruction boundary"
    if status == 3:
        if a0 == 1:
            return "TruncatedCode", "empty code object"
        if a0 == 2:
            return "TruncatedCode", "odd code length"
        if a0 == 3:
            return "TruncatedCode", f"code ends inside EXTENDED_ARG run at {a1}"
        if a0 == 4:
            ob = ar.section("objs")[o]
            op = int(ar.section("bytes")[int(ob["code_off"]) + a1 - 2])
            return "TruncatedCode", f"code ends inside inline cache of {TABLES[int(ob['minor'])][op][0]} at {a1}"
        return "TruncatedCode", "code holds no instruction"
    return f"status{status}", ""


def compare(gset, ar, ins, dec):
    objs = ar.section("objs")
    gold = GOLD[gset]
    assert len(gold) == ar.n_objs
    bad = []
    for g in gold:
        o = g["obj"]
        st = int(dec[o]["status"])
        if g["status"] != "ok":
            got = decode_error(ar, o, st, int(dec[o]["aux0"]), int(dec[o]["aux1"])) if st else ("ok", "")
            if got != (g["status"], g["msg"]):
                bad.append((gset, o, g["status"], g["msg"], got))
            continue
        if st != 0 or int(dec[o]["n_instrs"]) != g["n"]:
            bad.append((gset, o, "ok", g["n"], st, int(dec[o]["n_instrs"])))
            continue
        base = int(objs[o]["code_off"]) >> 1
        rec = ins[base:base + g["n"]]
        if hashlib.sha256(rec.tobytes()).hexdigest()[:32] != g["sha"]:
            jt = int(np.count_nonzero(rec["flags"] & 4))
            bad.append((gset, o, "records differ", f"jump targets {jt} vs {g['jt']}"))
    return bad


@pytest.mark.parametrize("gset", SETS)
def test_decode_scalar_matches_reference(gset):
    from paper_2403_13839_b200 import hostcheck

    ar = _arena(gset)
    ins, dec = hostcheck.decode(ar)
    bad = compare(gset, ar, ins, dec)
    assert not bad, bad[:5]


def test_decode_golden_covers_jump_targets():
    n = sum(1 for rs in GOLD.values() for r in rs if r.get("jt"))
    assert n > 10000  # the flag the round-1 kernel never wrote is exercised


def device_decode(ar):
    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.arena import DECODED_DTYPE, INS_DTYPE
    import torch

    da = DeviceArena(ar)
    da.upload()
    da.run(mode="decode")
    torch.cuda.synchronize()
    units = ar.total_code_units + 1
    dec_off = (units * 12 + 255) & ~255
    ws = da.ws.cpu().numpy()
    ins = ws[:units * 12].view(INS_DTYPE)
    dec = ws[dec_off:dec_off + 24 * ar.n_objs].view(DECODED_DTYPE)
    return ins, dec


@pytest.mark.gpu
@pytest.mark.parametrize("gset", SETS)
def test_decode_kernel_matches_reference(gset):
    ar = _arena(gset)
    ins, dec = device_decode(ar)
    bad = compare(gset, ar, ins, dec)
    assert not bad, bad[:5]


@pytest.mark.gpu
@pytest.mark.parametrize("gset", ["c2", "c4", "fuzz", "mutant2"])
def test_decode_kernel_tiled_matches_reference(gset):
    """The same objects tiled x8: more groups per warp, so the TMA ring runs
    across object and group boundaries with other objects' chunks in flight."""
    from paper_2403_13839_b200 import arena

    ar = _arena(gset)
    reps = 8
    big = arena.tile(ar, reps)
    ins, dec = device_decode(big)
    n = ar.n_objs
    for r in (0, reps // 2, reps - 1):
        sub_dec = dec[r * n:(r + 1) * n]
        shift = int(big.section("objs")["code_off"][r * n] - ar.section("objs")["code_off"][0]) >> 1
        sub_ins = ins[shift:shift + ar.total_code_units + 1]
        bad = compare(gset, ar, sub_ins, sub_dec)
        assert not bad, (r, bad[:5])
