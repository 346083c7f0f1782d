"""CPU tier: pin the oracle (CPU restatement of the reference algorithm) to
vectors the REAL reference produced: every golden case and every pool digest."""
import hashlib
import json
import os

import pytest

from conftest import GOLDEN, golden_cases
from helpers import inputs, style_of
from oracle import port


@pytest.mark.parametrize("gset", ["c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant"])
def test_oracle_matches_reference_goldens(gset):
    recs = golden_cases([gset])
    bad = []
    for r, co in zip(recs, inputs(recs)):
        got = port.outcome(co, style_of(r))
        if got != (r["status"], r["text"]):
            bad.append((r["case"], r["status"], got[0], r["text"][:200], got[1][:200]))
    assert not bad, bad[:3]


@pytest.mark.parametrize("pool,limit", [("c3_310", 512), ("c3_311", 256), ("c4_310", 4)])
def test_oracle_matches_reference_pool_digests(pool, limit):
    from paper_2403_13839_b200.bench_pools import pool_objects

    with open(os.path.join(GOLDEN, "pools.json")) as f:
        ref = json.load(f)[pool]
    bad = 0
    for i, co in enumerate(pool_objects(pool, 0, limit)):
        st, text = port.outcome(co)
        h = hashlib.sha256(text.encode("utf-8", "surrogatepass")).hexdigest()[:24]
        bad += (st, h) != (ref["status"][i], ref["sha"][i])
    assert bad == 0
