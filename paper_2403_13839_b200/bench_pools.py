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
}


def pool_objects(name, lo=0, hi=None):
    spec = POOLS[name]
    hi = spec["size"] if hi is None else hi
    if spec["gen"] == "c3":
        return [corpus.c3(i, spec["minor"]) for i in range(lo, hi)]
    return [corpus.c4(i, spec["minor"], spec["units"]) for i in range(lo, hi)]
