"""CPU tier: the decompiler's C++ sources (host build, test-only) against the
reference's golden outputs.  Same code the sm_100a kernels compile."""
import pytest

from helpers import inputs, mismatches, style_of, ST_NAMES
from conftest import golden_cases
from paper_2403_13839_b200 import arena, hostcheck


@pytest.mark.parametrize("gset", ["c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "mutant3"])
def test_host_build_matches_reference(gset):
    recs = golden_cases([gset])
    assert recs
    by_style = {}
    for r in recs:
        by_style.setdefault(repr(r.get("style")), []).append(r)
    bad = []
    for _, group in by_style.items():
        res = hostcheck.run(arena.pack(inputs(group)), style_of(group[0]))
        got = [(ST_NAMES.get(st, str(st)), text) for st, text, _ in res]
        bad += mismatches(group, got)
    assert not bad, bad[:3]
