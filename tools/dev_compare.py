"""Dev loop: diff the host build of the device sources against the live reference.

    python tools/dev_compare.py [corpus ...]

Only usable in the build container (imports /root/reference).
"""
import sys
import time
import traceback

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/repo")

import unpyre  # noqa: E402

from paper_2403_13839_b200 import arena, hostcheck  # noqa: E402
from paper_2403_13839_b200.synth import corpus  # noqa: E402


def ref_objs(objs):
    return arena.unpack(arena.pack(objs), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)


def ref_run(objs, style=None):
    out = []
    rs = None if style is None else unpyre.EmitStyle(style.indent, style.header, style.tool)
    for co in ref_objs(objs):
        try:
            out.append(("ok", unpyre.decompile_source(co, rs)))
        except Exception as e:  # noqa: BLE001
            out.append((type(e).__name__, str(e)))
    return out


ST_NAMES = {0: "ok", 1: "UnpyreError", 2: "UnknownOpcode", 3: "TruncatedCode", 4: "BadJumpTarget",
            5: "MalformedExceptionTable", 6: "StackUnderflow", 7: "UnsupportedOpcode",
            8: "StackDepthMismatch", 9: "StructuringFailed", 10: "InternalMarkerLeak", 20: "IndexError",
            21: "AttributeError", 22: "TypeError", 23: "KeyError", 24: "ValueError", 25: "RecursionError"}


def compare(objs, label, style=None, show=3):
    t0 = time.time()
    ref = ref_run(objs, style)
    t1 = time.time()
    got = hostcheck.run(arena.pack(objs), style)
    t2 = time.time()
    bad = 0
    for i, ((rk, rt), (st, gt, aux)) in enumerate(zip(ref, got)):
        gk = ST_NAMES.get(st, f"status{st}")
        if rk != gk or rt != gt:
            bad += 1
            if bad <= show:
                print(f"--- {label}[{i}] ref={rk} got={gk}")
                if rk == gk:
                    import difflib
                    for line in list(difflib.unified_diff(rt.splitlines(), gt.splitlines(), lineterm=""))[:40]:
                        print(line)
                else:
                    print("REF:", rt[:800])
                    print("GOT:", gt[:800])
    print(f"{label}: {len(objs) - bad}/{len(objs)} match  (ref {t1 - t0:.2f}s, host {t2 - t1:.3f}s)")
    return bad


def main():
    which = sys.argv[1:] or ["fig1", "c3", "c4"]
    for w in which:
        if w == "fig1":
            for m in (10, 11):
                compare(corpus.fig1(m), f"fig1/3.{m}")
        elif w == "c3":
            for m in (10, 11):
                compare([corpus.c3(s, m) for s in range(200)], f"c3/3.{m}")
        elif w == "c4":
            for m in (10, 11):
                compare([corpus.c4(s, m, 800) for s in range(60)], f"c4/3.{m}")


if __name__ == "__main__":
    main()
