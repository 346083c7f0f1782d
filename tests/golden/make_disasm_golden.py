"""Golden vectors for the secondary outputs of SURVEY §8 f4, made by running the
REAL reference on every object (roots and nested codes) of the golden sets:

* listing: `format_listing(decode_instructions(code))` (disasm.py:224-236, 71-172)
* dot:     `to_dot(analyze(code)[2])` (cfg.py:331-344, pipeline.py:17-54) -- what
           `unpyre disasm --cfg --dot` prints per code object (cli.py:103-105)

Run in the build container:

    python tests/golden/make_disasm_golden.py

Each line of disasm.jsonl: {"set", "obj", "minor", "listing": OUT, "dot": OUT} for
object index `obj` of `arena.pack(inputs)` (the set's records without a style, as
tests/test_decode.py packs them); OUT is {"status": "ok", "sha": SHA-256[:32] of the
UTF-8 text, "n": its length} or {"status": class name, "msg": str(exception)}.  The
first few texts (<= 2 KB) of each set are kept verbatim under "text" for readable diffs.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

import unpyre  # noqa: E402
from unpyre import cfg as ref_cfg  # noqa: E402
from unpyre import disasm as ref_disasm  # noqa: E402
from unpyre import pipeline as ref_pipeline  # noqa: E402

from paper_2403_13839_b200 import arena  # noqa: E402
from paper_2403_13839_b200.synth import cases  # noqa: E402

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "c4big")
VERBATIM = 3


def set_records(name):
    if name == "c4big":
        return cases.C4BIG
    with open(os.path.join(HERE, f"{name}.jsonl")) as f:
        recs = [json.loads(line) for line in f]
    return [r for r in recs if not r.get("style")]


def outcome(fn, keep):
    try:
        text = fn()
    except RecursionError as e:  # noqa: BLE001
        return {"status": "RecursionError", "msg": str(e)}
    except Exception as e:  # noqa: BLE001
        return {"status": type(e).__name__, "msg": str(e)}
    b = text.encode("utf-8", "surrogatepass")
    out = {"status": "ok", "sha": hashlib.sha256(b).hexdigest()[:32], "n": len(b)}
    if keep and len(b) <= 2048:
        out["text"] = text
    return out


def main():
    path = os.path.join(HERE, "disasm.jsonl")
    with open(path, "w") as f:
        for name in SETS:
            if name != "c4big" and not os.path.exists(os.path.join(HERE, f"{name}.jsonl")):
                continue
            recs = set_records(name)
            ar = arena.pack([cases.build(r) for r in recs])
            objs = arena.unpack(ar, unpyre.CodeObject, unpyre.Const, unpyre.VersionTag,
                                objects=range(ar.n_objs))
            n_l = n_d = 0
            for i, co in enumerate(objs):
                keep = i < VERBATIM
                row = {"set": name, "obj": i, "minor": co.version.minor,
                       "listing": outcome(lambda: ref_disasm.format_listing(ref_disasm.decode_instructions(co)), keep),
                       "dot": outcome(lambda: ref_cfg.to_dot(ref_pipeline.analyze(co)[2]), keep)}
                n_l += row["listing"]["status"] == "ok"
                n_d += row["dot"]["status"] == "ok"
                f.write(json.dumps(row) + "\n")
            print(f"{name}: {ar.n_objs} objects, {n_l} listings, {n_d} dot graphs")
    print("->", path)


if __name__ == "__main__":
    main()
