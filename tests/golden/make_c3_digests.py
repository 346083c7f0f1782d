"""Reference digests for the full C3 bench corpus (1M distinct
objects, seed_i = splitmix64(0xC3 ^ i), i < 1M), made by running the REAL
reference's `decompile_source` on every object in the build container:

    python tests/golden/make_c3_digests.py [--minor 10|11] [--n 1048576] [--procs 8]

Per object the digest is SHA-256(text)[:24] (status "ok") or of "Class: message";
per block of 1024 consecutive objects the committed value is
SHA-256 over the block's "<status>:<digest>\\n" lines.  bench.py recomputes the
block hashes from the device's outputs and compares all of them (a checksum of
checksums: 1M objects checked with a 25 KB fixture).  Inputs come from the
Python generator (synth/corpus.py c3), the same seeds the native generator
(synth/c3fast.py) lays out byte-identically.
"""
import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))

BLOCK = 1024


def _work(args):
    minor, lo, hi = args
    import unpyre

    from paper_2403_13839_b200 import arena
    from paper_2403_13839_b200.synth import corpus

    out = []
    for i in range(lo, hi):
        co = corpus.c3(i, minor)
        ref = arena.unpack(arena.pack([co]), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)[0]
        try:
            text, st = unpyre.decompile_source(ref), "ok"
        except Exception as e:  # noqa: BLE001
            text, st = f"{type(e).__name__}: {e}", type(e).__name__
        out.append(f"{st}:{hashlib.sha256(text.encode('utf-8', 'surrogatepass')).hexdigest()[:24]}\n")
    return lo, out


def block_hash(lines):
    return hashlib.sha256("".join(lines).encode()).hexdigest()[:32]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minor", type=int, default=10)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    assert a.n % BLOCK == 0
    t0 = time.time()
    chunks = [(a.minor, lo, lo + BLOCK) for lo in range(0, a.n, BLOCK)]
    lines = [None] * a.n
    n_ok = 0
    with mp.Pool(a.procs) as pool:
        for k, (lo, out) in enumerate(pool.imap_unordered(_work, chunks)):
            lines[lo:lo + BLOCK] = out
            if k % 64 == 0:
                print(f"{k}/{len(chunks)} blocks, {time.time() - t0:.0f}s", flush=True)
    n_ok = sum(1 for x in lines if x.startswith("ok:"))
    blocks = [block_hash(lines[lo:lo + BLOCK]) for lo in range(0, a.n, BLOCK)]
    path = os.path.join(HERE, f"c3_digests_3{a.minor}.json")
    with open(path, "w") as f:
        json.dump({"spec": {"gen": "c3", "minor": a.minor, "n": a.n, "block": BLOCK, "n_ok": n_ok,
                            "seconds": round(time.time() - t0, 1), "procs": a.procs},
                   "blocks": blocks}, f)
    print(f"-> {path}: {a.n} objects ({n_ok} ok) in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
