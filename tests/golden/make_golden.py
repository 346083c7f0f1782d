"""Generate golden vectors by running the REAL reference (unpyre, imported from
/root/reference/pkg/src) on the synthetic corpora.  Run in the build container:

    python tests/golden/make_golden.py

Each line of <name>.jsonl: {"case", "gen", "minor", "seed", "kw", "input_sha",
"status", "text"} where status is "ok" or the reference exception class and
text is the decompiled source or str(exception).  The inputs are regenerated
from (gen, minor, seed, kw) by paper_2403_13839_b200.synth; input_sha pins the
generator so drift is detected instead of silently re-baselined.
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import unpyre  # noqa: E402

from paper_2403_13839_b200 import arena  # noqa: E402
from paper_2403_13839_b200.synth import cases  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def input_sha(co):
    h = hashlib.sha256()
    stack = [co]
    while stack:
        c = stack.pop()
        h.update(bytes([c.version.minor]))
        h.update(c.code)
        h.update(repr([(k.kind, k.value if k.kind != "code" else None) for k in c.consts]).encode())
        h.update(repr((c.names, c.varnames, c.freevars, c.cellvars, c.name, c.argcount, c.flags)).encode())
        h.update(c.exceptiontable)
        stack.extend(k.value for k in c.consts if k.kind == "code")
    return h.hexdigest()[:16]


def run_ref(co, style=None):
    ref = arena.unpack(arena.pack([co]), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)[0]
    rs = None if style is None else unpyre.EmitStyle(**style)
    try:
        return "ok", unpyre.decompile_source(ref, rs)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e)


def main(only=None):
    for name, specs in cases.GOLDEN_SETS.items():
        if only and name not in only:
            continue
        path = os.path.join(HERE, f"{name}.jsonl")
        n_ok = 0
        with open(path, "w") as f:
            for spec in specs:
                co = cases.build(spec)
                status, text = run_ref(co, spec.get("style"))
                n_ok += status == "ok"
                rec = dict(spec)
                rec.update(input_sha=input_sha(co), status=status, text=text)
                f.write(json.dumps(rec, ensure_ascii=False) + "\n")
        print(f"{name}: {len(specs)} cases, {n_ok} ok -> {path}")


if __name__ == "__main__":
    main(sys.argv[1:])
