"""Per-stage thread-cycle split of the decompile kernel (profiling variant).

    tools/build_variant.sh prof -DUPY_PHASE_PROF
    UPY_LIB=paper_2403_13839_b200/_variants/prof.so python tools/stage_prof.py c3_310 c4_310 [--objects N]

Prints, per pool, the share of thread-cycles spent in validate / analyze (decode
check + CFG, dominators, loops) / structure (structurer + symbolic simulation +
canonicalize) / finish (def recovery incl. nested bodies, scope decls) / emit.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pools", nargs="+")
    ap.add_argument("--objects", type=int, default=0)
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--arena-bytes", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_2403_13839_b200 import _lib, arena as arena_mod
    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.bench_pools import pool_objects

    lib = _lib.load()
    lib.upy_prof_read.restype = C.c_int
    names = ["validate", "analyze", "structure", "finish", "emit"]
    for name in a.pools:
        pool = pool_objects(name)
        ar = arena_mod.pack(pool)
        if a.objects:
            ar = arena_mod.tile(ar, max(1, a.objects // len(pool)))
        da = DeviceArena(ar, slots=a.slots, arena_bytes=a.arena_bytes)
        da.upload()
        da.run(mode="decode")
        da.run(mode="structure")
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * 8)()
        lib.upy_prof_read(buf, 1)
        da.run(mode="structure")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        lib.upy_prof_read(buf, 1)
        ev[0].record()
        da.run(mode="structure")
        ev[1].record()
        torch.cuda.synchronize()
        n = lib.upy_prof_read(buf, 1)
        tot = sum(buf[i] for i in range(n))
        ms = ev[0].elapsed_time(ev[1])
        print(f"{name}: {ar.n_roots} roots, decompile {ms:.1f} ms, thread-cycles/root {tot / ar.n_roots:.3e}")
        for i in range(n):
            print(f"  {names[i]:<10} {100.0 * buf[i] / tot:6.2f}%  {buf[i] / ar.n_roots:.3e} cycles/root")


if __name__ == "__main__":
    main()
