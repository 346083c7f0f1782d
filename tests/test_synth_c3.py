"""The C3 bench corpus: the native generator (synth/c3fast.py +
c3gen.cpp) must lay out exactly the arena `arena.pack` builds from the Python
generator's objects, and the committed reference digest blocks
(tests/golden/c3_digests_3*.json, made by make_c3_digests.py with the real
reference) must match what the decompiler produces for the same seeds."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.mark.parametrize("minor", [10, 11])
@pytest.mark.parametrize("first,n", [(0, 600), (997, 40), (99_990, 25)])
def test_native_c3_generator_is_byte_identical_to_pack(minor, first, n):
    from paper_2403_13839_b200 import arena
    from paper_2403_13839_b200.synth import c3fast, corpus

    a = c3fast.c3_arena(n, minor, first)
    b = arena.pack([corpus.c3(i, minor) for i in range(first, first + n)])
    assert a.offsets == b.offsets and a.counts == b.counts
    assert (a.max_code_len, a.total_code_units) == (b.max_code_len, b.total_code_units)
    assert np.array_equal(a.blob, b.blob)


def _blocks(minor):
    path = os.path.join(GOLDEN, f"c3_digests_3{minor}.json")
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("minor", [10, 11])
def test_c3_digest_blocks_match_host_build(minor):
    """First two 1024-object blocks decompiled by the host build of the device
    sources, hashed the way bench.py hashes the device's outputs."""
    from paper_2403_13839_b200 import hostcheck
    from paper_2403_13839_b200.synth import c3fast

    d = _blocks(minor)
    assert d["spec"]["n"] >= 1 << 20 and d["spec"]["n_ok"] == d["spec"]["n"]
    block = d["spec"]["block"]
    res = hostcheck.run(c3fast.c3_arena(2 * block, minor))
    lines = [f"ok:{hashlib.sha256(s.encode('utf-8', 'surrogatepass')).hexdigest()[:24]}\n"
             for st, s, _ in res if st == 0]
    assert len(lines) == 2 * block
    for b in range(2):
        got = hashlib.sha256("".join(lines[b * block:(b + 1) * block]).encode()).hexdigest()[:32]
        assert got == d["blocks"][b], b
