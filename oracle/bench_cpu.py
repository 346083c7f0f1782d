"""TEST INFRASTRUCTURE ONLY -- CPU baseline timing on every host core of the
reference itself (`unpyre.decompile_source` from the staged copy oracle/_ref,
kind "reference") or of the oracle (the reference algorithm restated in Python,
kind "port") when the reference is absent.

Each forked worker decompiles its share of a bounded sample of the benchmark
pool in a loop for `seconds`; the rate is total objects / wall time.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

_POOL = None


def _decompile_fn(kind):
    if kind == "reference":
        import unpyre

        def run(co):
            try:
                unpyre.decompile_source(co)
            except unpyre.UnpyreError:
                pass
        return run
    from oracle import port

    return port.outcome


def _worker(args):
    lo, hi, seconds, kind = args
    fn = _decompile_fn(kind)
    objs = _POOL[lo:hi]
    done = 0
    t0 = time.perf_counter()
    while True:
        for co in objs:
            fn(co)
            done += 1
        if time.perf_counter() - t0 >= seconds:
            break
    return done, time.perf_counter() - t0


def run(pool, seconds=10.0, cores=None, kind="port"):
    """(objects/s, cores used, sample description).  kind "reference": `pool`
    holds the reference's own CodeObjects and `unpyre` is importable."""
    global _POOL
    _POOL = list(pool)
    cores = cores or os.cpu_count() or 1
    n = len(_POOL)
    per = max(1, n // cores)
    jobs = [(i * per % n, min(n, i * per % n + per), seconds, kind) for i in range(cores)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as p:
        res = p.map(_worker, jobs)
    wall = time.perf_counter() - t0
    total = sum(d for d, _ in res)
    slowest = max(t for _, t in res)
    rate = total / max(slowest, 1e-9)
    what = "unpyre.decompile_source (the reference)" if kind == "reference" else "the oracle port"
    sample = (f"{what} on {n} distinct objects of the workload, {cores} forked workers x ~{seconds:.0f}s each, "
              f"{total} decompiles in {wall:.1f}s wall (rate uses the slowest worker's time)")
    return rate, cores, sample
