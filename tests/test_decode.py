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


def _lane_edge_codes():
    """3.11 objects around the lane kernel's limits (decode_kernel.cu: <= 4096 code
    bytes, no EXTENDED_ARG, no jump) plus ones it must hand back, interleaved with
    3.10 objects: straight-line code of random known opcodes with their cache units,
    at lengths 2046-2050 units; variants with an EXTENDED_ARG, a forward jump, an
    unknown opcode and a cache run past the end."""
    import random

    from paper_2403_13839_b200._optables import TABLES
    from paper_2403_13839_b200.model import CodeObject, VersionTag

    rng = random.Random(0x311)
    t11 = TABLES[11]
    plain = [op for op, v in t11.items() if v and v[2] == "none" and op not in (0, 144)]
    jumps = [op for op, v in t11.items() if v and v[2] == "jump_rel"]

    def body(units, variant):
        out = bytearray()
        while len(out) < 2 * units:
            op = rng.choice(plain)
            out += bytes([op, rng.randrange(256) if t11[op][1] else 0])
            out += bytes(2 * t11[op][3])
        out = out[:2 * units]
        if variant == "cut" and len(out) >= 2:
            out[-2:] = bytes([next(op for op in plain if t11[op][3] > 0), 1])  # caches past the end
        k = 2 * rng.randrange(1, max(2, units // 2))
        # re-align k to an instruction start by walking the instruction chain
        i = 0
        while i + 2 <= len(out) and i < k:
            i += 2 * (1 + t11.get(out[i], ("", False, "", 0))[3]) if out[i] in t11 and t11[out[i]] else 2
        k = min(i, len(out) - 4)
        if variant == "ext" and k >= 0:
            out[k:k + 4] = bytes([144, 0, rng.choice([op for op in plain if t11[op][1] and t11[op][3] == 0]), 1])
        elif variant == "jump" and k >= 0:
            out[k:k + 2] = bytes([jumps[0], 0])
        elif variant == "unknown" and k >= 0:
            out[k] = next(op for op in range(256) if op not in t11 or not t11[op])
        return bytes(out)

    def obj(minor, code):
        return CodeObject(VersionTag(3, minor), 0, 0, 0, 0, 0, 0, code, (), (), (), (), (), "f", "f.py", 1)

    codes = []
    for units in (1, 7, 8, 200, 2046, 2047, 2048, 2049, 2050):
        for variant in ("plain", "plain", "ext", "jump", "unknown", "cut"):
            codes.append(obj(11, body(units, variant)))
            codes.append(obj(10, bytes([100, 0, 83, 0])))  # LOAD_CONST 0; RETURN_VALUE
    return codes


@pytest.mark.gpu
def test_decode_lane_kernel_edges_match_scalar():
    """The 3.11 lane kernel and its hand-back path against the reference-order
    scalar decoder (decode_scalar on the host, pinned to the reference above) on
    objects at and past the lane kernel's size limit, with EXTENDED_ARG, jumps,
    unknown opcodes and truncated caches, tiled so every warp mixes them."""
    from paper_2403_13839_b200 import arena, hostcheck

    ar = arena.tile(arena.pack(_lane_edge_codes()), 5)
    want_ins, want_dec = hostcheck.decode(ar)
    ins, dec = device_decode(ar)
    objs = ar.section("objs")
    bad = []
    for o in range(ar.n_objs):
        if tuple(dec[o]) != tuple(want_dec[o]):
            bad.append((o, tuple(dec[o]), tuple(want_dec[o])))
            continue
        if int(dec[o]["status"]) == 0:
            base, n = int(objs[o]["code_off"]) >> 1, int(dec[o]["n_instrs"])
            if ins[base:base + n].tobytes() != want_ins[base:base + n].tobytes():
                bad.append((o, "records differ"))
    assert not bad, bad[:5]
    assert int(np.count_nonzero(dec["status"] == 0)) > ar.n_objs // 2
