"""instruction listings and the CFG dot export -- against the REAL
reference: tests/golden/disasm.jsonl holds, for every object (roots and nested
codes) of the golden sets, the reference's `format_listing(decode_instructions(co))`
and `to_dot(analyze(co)[2])` (digest + length, or exception class and message;
tests/golden/make_disasm_golden.py).

CPU tier: records from the host build of the decoder + host argval resolution /
formatting (`disasm.instructions`, `format_listing`); the dot text from the host
build of csrc/dot.h.  GPU tier: the decode kernel's records and the device dot
kernel (upy_options.output = 1) through the C ABI.
"""
import hashlib
import json
import os

import pytest

from conftest import GOLDEN, load_golden
from helpers import PY_INTERNAL, inputs

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "c4big")


def _golden():
    out = {}
    with open(os.path.join(GOLDEN, "disasm.jsonl")) as f:
        for line in f:
            r = json.loads(line)
            out.setdefault(r["set"], []).append(r)
    return out


GOLD = _golden()


def _objects(gset):
    """(arena with every object as a root, the objects as model CodeObjects)."""
    from paper_2403_13839_b200 import arena
    from paper_2403_13839_b200.synth import cases

    recs = cases.C4BIG if gset == "c4big" else [r for r in load_golden(gset) if not r.get("style")]
    ar = arena.pack(inputs(recs))
    objs = arena.unpack(ar, objects=range(ar.n_objs))
    return arena.with_roots(ar, range(ar.n_objs)), objs


def _check(want, got, what):
    """got: text or exception instance."""
    if isinstance(got, BaseException):
        cls, msg = type(got).__name__, str(got)
        if want["status"] == cls and (want["msg"] == msg or cls in PY_INTERNAL):
            return None
        return (what, want["status"], want.get("msg"), cls, msg)
    if want["status"] != "ok":
        return (what, want["status"], want.get("msg"), "ok", got[:200])
    b = got.encode("utf-8", "surrogatepass")
    if hashlib.sha256(b).hexdigest()[:32] == want["sha"] and len(b) == want["n"]:
        return None
    return (what, "text differs", want.get("text", "")[:300], got[:300])


def _listings_from(ar, objs, ins, dec):
    from paper_2403_13839_b200 import disasm

    o_rows = ar.section("objs")
    out = []
    for i, co in enumerate(objs):
        d = dec[i]
        st = int(d["status"])
        if st:
            out.append(disasm.decode_exception(co, st, int(d["aux0"]), int(d["aux1"])))
            continue
        base = int(o_rows[i]["code_off"]) >> 1
        out.append(disasm.format_listing(disasm.instructions(co, ins[base:base + int(d["n_instrs"])])))
    return out


@pytest.mark.parametrize("gset", SETS)
def test_listing_host_matches_reference(gset):
    from paper_2403_13839_b200 import hostcheck

    ar, objs = _objects(gset)
    ins, dec = hostcheck.decode(ar)
    got = _listings_from(ar, objs, ins, dec)
    bad = [b for g, x in zip(GOLD[gset], got) if (b := _check(g["listing"], x, g["obj"]))]
    assert not bad, bad[:3]


def _dot_outcomes(res):
    from paper_2403_13839_b200.errors import make_exception

    return [s if st == 0 else make_exception(st, s, aux) for st, s, aux in res]


@pytest.mark.parametrize("gset", SETS)
def test_dot_host_matches_reference(gset):
    from paper_2403_13839_b200 import hostcheck

    ar, objs = _objects(gset)
    got = _dot_outcomes(hostcheck.run(ar, output=1, text_cap=64 * ar.code_bytes + (1 << 20)))
    bad = [b for g, x in zip(GOLD[gset], got) if (b := _check(g["dot"], x, g["obj"]))]
    assert not bad, bad[:3]


def test_dot_covers_loop_back_and_exception_edges():
    """The digest-pinned C4 graphs carry both re-tagged back edges and dashed
    exception edges (so both branches of dot.h are under parity)."""
    from paper_2403_13839_b200 import hostcheck

    ar, _objs = _objects("c4")
    texts = [s for st, s, _ in hostcheck.run(ar, output=1, text_cap=64 * ar.code_bytes + (1 << 20)) if st == 0]
    assert sum("loop_back" in t for t in texts) > 10 and sum("style=dashed" in t for t in texts) > 10


@pytest.mark.gpu
@pytest.mark.parametrize("gset", SETS)
def test_listing_device_matches_reference(gset):
    from paper_2403_13839_b200 import disasm

    _ar, objs = _objects(gset)
    got = [v if isinstance(v, BaseException) else disasm.format_listing(v) for v in disasm.decode_many(objs)]
    bad = [b for g, x in zip(GOLD[gset], got) if (b := _check(g["listing"], x, g["obj"]))]
    assert not bad, bad[:3]


@pytest.mark.gpu
@pytest.mark.parametrize("gset", SETS)
def test_dot_device_matches_reference(gset):
    from paper_2403_13839_b200.api import run_arena

    ar, _objs = _objects(gset)
    res = run_arena(ar, output=1)
    got = _dot_outcomes([(*res.item(i), res.aux[i]) for i in range(len(res.status))])
    bad = [b for g, x in zip(GOLD[gset], got) if (b := _check(g["dot"], x, g["obj"]))]
    assert not bad, bad[:3]
