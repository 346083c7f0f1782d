"""Reference digests for the benchmark pools (run in the build container):

    python tests/golden/make_pools.py [pool ...]   # default: all pools

bench.py tiles a pool of distinct synthetic objects up to the configured
corpus size and checks EVERY device output against these SHA-256 digests of
the REAL reference's text (unpyre.decompile_source), so the full-size run is
verified byte-exact without the reference on the GPU box.
"""
import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_2403_13839_b200.bench_pools import POOLS, pool_objects  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest_range(args):
    import unpyre

    from paper_2403_13839_b200 import arena

    name, lo, hi = args
    objs = pool_objects(name, lo, hi)
    refs = arena.unpack(arena.pack(objs), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)
    out = []
    for co in refs:
        try:
            text = unpyre.decompile_source(co)
            st = "ok"
        except Exception as e:  # noqa: BLE001
            text, st = str(e), type(e).__name__
        out.append((st, hashlib.sha256(text.encode("utf-8", "surrogatepass")).hexdigest()[:24]))
    return out


def main():
    only = sys.argv[1:]
    res = {}
    if only:
        with open(os.path.join(HERE, "pools.json")) as f:
            res = json.load(f)
    with Pool(os.cpu_count()) as p:
        for name, spec in POOLS.items():
            if only and name not in only:
                continue
            t0 = time.time()
            n = spec["size"]
            step = max(1, n // (4 * os.cpu_count()))
            parts = p.map(_digest_range, [(name, lo, min(n, lo + step)) for lo in range(0, n, step)])
            flat = [x for part in parts for x in part]
            res[name] = {"spec": spec, "status": [s for s, _ in flat], "sha": [h for _, h in flat]}
            ok = sum(s == "ok" for s, _ in flat)
            print(f"{name}: {n} objects, {ok} ok, {time.time() - t0:.1f}s")
    with open(os.path.join(HERE, "pools.json"), "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    main()
