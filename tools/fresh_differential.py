"""Fresh-seed differential: the real reference vs the host build of the device
sources on synthetic programs whose seeds no golden set uses (build container only:
imports /root/reference).

    python tools/fresh_differential.py valid 10000 500        # structured fuzz programs
    python tools/fresh_differential.py valid 20000 250 80     # larger ones (size=80)
    python tools/fresh_differential.py mutant 7000 250        # byte mutants

Prints the reference's outcome classes and every mismatch (Python-internal failures
compare by class only, the parity domain of DESIGN.md §4; a reference run longer than
20 s counts as TIMEOUT and is skipped).
"""
import sys, collections, multiprocessing as mp
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2403_13839_b200.synth import cases
from paper_2403_13839_b200 import arena, hostcheck
from paper_2403_13839_b200.errors import make_exception

def ref_outcome(rec):
    import unpyre, signal
    co = cases.build(rec)
    ref = arena.unpack(arena.pack([co]), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)[0]
    def h(s, f): raise TimeoutError()
    signal.signal(signal.SIGALRM, h); signal.alarm(20)
    try:
        return ("ok", unpyre.decompile_source(ref))
    except TimeoutError:
        return ("TIMEOUT", "")
    except RecursionError as e:
        return ("RecursionError", str(e))
    except Exception as e:
        return (type(e).__name__, str(e))
    finally:
        signal.alarm(0)

def main(mode, first, n, size):
    recs = []
    for m in (8, 9, 10, 11):
        for s in range(first, first + n):
            kw = {} if mode == "valid" else {"mode": mode}
            if size: kw["size"] = size
            recs.append({"case": f"{mode}-3.{m}-{s}", "gen": "fuzz", "minor": m, "seed": s, "kw": kw})
    with mp.Pool(8) as p:
        want = p.map(ref_outcome, recs, chunksize=8)
    got = hostcheck.run(arena.pack([cases.build(r) for r in recs]))
    PY = {"IndexError", "AttributeError", "TypeError", "KeyError", "ValueError", "RecursionError"}
    c = collections.Counter(); bad = []
    for r, w, (st, s, aux) in zip(recs, want, got):
        e = None if st == 0 else make_exception(st, s, aux)
        g = ("ok", s) if st == 0 else (type(e).__name__, str(e))
        c[w[0]] += 1
        if w[0] == "TIMEOUT": continue
        if g == w: continue
        if w[0] in PY and g[0] == w[0]: c["py_msg_differs"] += 1; continue
        bad.append((r["case"], w[0], g[0], w[1][:300], g[1][:300]))
    print(mode, first, n, size, dict(c), "mismatches:", len(bad))
    for b in bad[:10]: print("  ", b)

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 0)
