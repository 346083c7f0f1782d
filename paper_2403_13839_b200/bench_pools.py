"""Benchmark pools: the distinct synthetic objects a benchmark corpus is tiled
from (BASELINE.json configs C3/C4/C5).  Pool digests of the reference's
output live in tests/golden/pools.json."""
from __future__ import annotations

from .synth import corpus

POOLS = {
    # C3 / C5: ~200-unit straight-line objects (3.10), seeds splitmix64(0xC3 ^ i)
    "c3_310": {"gen": "c3", "minor": 10, "size": 4096},
    "c3_311": {"gen": "c3", "minor": 11, "size": 1024},
    # C4: ~10K-unit nested control flow (3.10)
    "c4_310": {"gen": "c4", "minor": 10, "size": 64, "units": 10000},
    "c4_311": {"gen": "c4", "minor": 11, "size": 32, "units": 10000},
    # C2: the reference's 110-module syntax corpus compiled to 3.10 (fixture
    # tests/golden/c2.jsonl, made by make_c2_golden.py); roots are modules
    "c2_310": {"gen": "c2", "minor": 10, "size": 110},
    "c2_311": {"gen": "c2", "minor": 11, "size": 110},
    "c2_39": {"gen": "c2", "minor": 9, "size": 110},
    "c2_38": {"gen": "c2", "minor": 8, "size": 110},
}


def _c2_trees(minor):
    import json
    import os

    from .synth import codejson

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c2.jsonl")
    with open(path) as f:
        recs = [json.loads(line) for line in f]
    return [codejson.from_json(r["tree"]) for r in recs if not r.get("style") and r["minor"] == minor]


def pool_objects(name, lo=0, hi=None):
    spec = POOLS[name]
    hi = spec["size"] if hi is None else hi
    if spec["gen"] == "c2":
        return _c2_trees(spec["minor"])[lo:hi]
    if spec["gen"] == "c3":
        return [corpus.c3(i, spec["minor"]) for i in range(lo, hi)]
    return [corpus.c4(i, spec["minor"], spec["units"]) for i in range(lo, hi)]
