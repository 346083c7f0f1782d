"""Stack-depth scan (north-star subsystem 3; csrc/stackscan.h, stackscan_kernel.cu)
against depths recorded from the REAL reference's symbolic simulation
(tests/golden/stack.jsonl, make_stack_golden.py: per simulated block its entry
depth E and, after each transfer function, the depth relative to E).

A block starting at instruction j lies inside one scan segment, so the scan
predicts depth(i) - E = S(i) - S(j-1) (S(j-1) = 0 when j starts a segment).
Positions whose segment holds a contents-dependent effect before them (flag
bit1), and blocks split by a leader the scan does not know (3.11 yield-from
rewriting), are skipped; the test asserts how much is covered.

CPU tier: the host build of the scalar scan.  GPU tier: the warp kernel, against
the golden and bit-for-bit against the host scan on large corpora."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from helpers import inputs

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz")


def _golden():
    out = {}
    with open(os.path.join(GOLDEN, "stack.jsonl")) as f:
        for line in f:
            r = json.loads(line)
            out.setdefault(r["set"], {})[r["obj"]] = r["blocks"]
    return out


GOLD = _golden()


def _arena(gset):
    from paper_2403_13839_b200 import arena

    return arena.pack(inputs([r for r in load_golden(gset) if not r.get("style")]))


def compare(gset, ar, offsets_of, scan_of):
    """offsets_of(o) -> instruction offsets; scan_of(o) -> upy_stackrec array."""
    checked = skipped = 0
    bad = []
    for o, blocks in GOLD[gset].items():
        offs = offsets_of(o)
        if offs is None:
            continue
        idx = {int(x): i for i, x in enumerate(offs)}
        rec = scan_of(o)
        for lo, _e, calls, _fall in blocks:
            j = idx.get(lo)
            for off, d in calls:
                i = idx.get(off)
                if j is None or i is None:
                    skipped += 1
                    continue
                seg_inside = i > j and (rec["flags"][j + 1:i + 1] & 1).any()
                base_unknown = j > 0 and not (rec["flags"][j] & 1) and (rec["flags"][j - 1] & 2)
                if seg_inside or base_unknown or (rec["flags"][i] & 2):
                    skipped += 1
                    continue
                base = 0 if (j == 0 or rec["flags"][j] & 1) else int(rec["depth"][j - 1])
                checked += 1
                if int(rec["depth"][i]) - base != d:
                    bad.append((o, lo, off, d, int(rec["depth"][i]) - base))
    return checked, skipped, bad


def _host(ar):
    from paper_2403_13839_b200 import hostcheck

    ins, dec = hostcheck.decode(ar)
    recs, info = hostcheck.stackscan(ar)
    objs = ar.section("objs")

    def offsets_of(o):
        if int(dec[o]["status"]):
            return None
        base = int(objs[o]["code_off"]) >> 1
        return ins["offset"][base:base + int(dec[o]["n_instrs"])]

    def scan_of(o):
        base = int(objs[o]["code_off"]) >> 1
        return recs[base:base + int(dec[o]["n_instrs"])]

    return offsets_of, scan_of, recs, info, ins, dec


MIN_COVERED = {"c1": 0.99, "c2": 0.97, "c3": 0.99, "c4": 0.97, "snippets": 0.95, "fuzz": 0.99}


@pytest.mark.parametrize("gset", SETS)
def test_stackscan_host_matches_reference_simulation(gset):
    ar = _arena(gset)
    offsets_of, scan_of, *_ = _host(ar)
    checked, skipped, bad = compare(gset, ar, offsets_of, scan_of)
    assert not bad, bad[:5]
    assert checked / max(1, checked + skipped) >= MIN_COVERED[gset], (checked, skipped)


def test_stackscan_summary_consistent():
    ar = _arena("c4")
    _o, _s, recs, info, ins, dec = _host(ar)
    objs = ar.section("objs")
    for o in range(ar.n_objs):
        if int(info[o]["status"]):
            continue
        base = int(objs[o]["code_off"]) >> 1
        r = recs[base:base + int(dec[o]["n_instrs"])]
        known = (r["flags"] & 2) == 0
        assert int(info[o]["n_segments"]) == int((r["flags"] & 1).sum())
        assert int(info[o]["max_depth"]) == max(0, int(r["depth"][known].max(initial=0)))
        assert int(info[o]["min_depth"]) == min(0, int(r["depth"][known].min(initial=0)))


@pytest.mark.gpu
@pytest.mark.parametrize("gset", SETS)
def test_stackscan_kernel_matches_reference_simulation(gset):
    import torch

    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.arena import STACKINFO_DTYPE, STACKREC_DTYPE

    ar = _arena(gset)
    offsets_of, _scan_host, host_recs, host_info, _ins, dec = _host(ar)
    da = DeviceArena(ar)
    da.upload()
    da.run(mode="decode")
    stack, info = da.stackscan()
    torch.cuda.synchronize()
    recs = stack.cpu().numpy().view(STACKREC_DTYPE)
    inf = info.cpu().numpy().view(STACKINFO_DTYPE)
    objs = ar.section("objs")

    def scan_of(o):
        base = int(objs[o]["code_off"]) >> 1
        return recs[base:base + int(dec[o]["n_instrs"])]

    checked, skipped, bad = compare(gset, ar, offsets_of, scan_of)
    assert not bad, bad[:5]
    assert checked / max(1, checked + skipped) >= MIN_COVERED[gset]
    # bit-for-bit against the host scan on every decoded object
    assert np.array_equal(inf, host_info)
    for o in range(ar.n_objs):
        if int(dec[o]["status"]) == 0:
            base = int(objs[o]["code_off"]) >> 1
            n = int(dec[o]["n_instrs"])
            assert np.array_equal(recs[base:base + n], host_recs[base:base + n]), o


@pytest.mark.gpu
@pytest.mark.parametrize("minor", [10, 11])
def test_stackscan_kernel_matches_host_on_c3_corpus(minor):
    """65,536 distinct C3 objects (native generator): kernel == host scan."""
    import torch

    from paper_2403_13839_b200 import hostcheck
    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.arena import STACKINFO_DTYPE, STACKREC_DTYPE
    from paper_2403_13839_b200.synth import c3fast

    ar = c3fast.c3_arena(65536, minor)
    da = DeviceArena(ar)
    da.upload()
    da.run(mode="decode")
    stack, info = da.stackscan()
    torch.cuda.synchronize()
    h_recs, h_info = hostcheck.stackscan(ar)
    assert np.array_equal(info.cpu().numpy().view(STACKINFO_DTYPE), h_info)
    d_recs = stack.cpu().numpy().view(STACKREC_DTYPE)
    dec = da.decoded()
    objs = ar.section("objs")
    mask = np.zeros(len(h_recs), dtype=bool)
    for o in range(ar.n_objs):  # only record slots of real instructions are defined
        base = int(objs[o]["code_off"]) >> 1
        mask[base:base + int(dec[o]["n_instrs"])] = True
    assert np.array_equal(d_recs[mask], h_recs[mask])


def test_stack_descriptor_table_equals_switch():
    """The kernel's per-(version, opcode) descriptors (stack_desc) give the same
    effect and unknown flag as the reference-order switch (stack_effect) for every
    table entry and every 16-bit arg (plus wide ones)."""
    import ctypes

    from paper_2403_13839_b200 import hostcheck

    lib = hostcheck.lib()
    lib.upyh_stack_desc_selfcheck.restype = ctypes.c_uint64
    assert lib.upyh_stack_desc_selfcheck(ctypes.c_uint32(1 << 16)) == 0
