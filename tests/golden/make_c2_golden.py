"""C2 golden vectors (BASELINE.json configs[1]): the
reference's syntax corpus `pkg/corpus/<category>/*.py` (110 modules) compiled
to CPython 3.8-3.11 code objects by the in-repo code generators
(paper_2403_13839_b200/synth/pycodegen38.py, pycodegen39.py, pycodegen.py, pycodegen311.py), then decompiled by the REAL
reference (unpyre.decompile_source, imported from /root/reference/pkg/src).
Run in the build container:

    python tests/golden/make_c2_golden.py

The corpus sources exist only here, so each line of c2.jsonl carries its
input as a lossless JSON code tree (synth/codejson.py) plus input_sha (the
same digest as make_golden.py) and the reference outcome (status/text).  The
reference's own .pyc reader (unpyre.pyc.load_pyc) is also run on the .pyc
image synth/marshal.py writes for each module and must give back the same
tree, so the fixture doubles as a loader corpus of realistic modules.
"""
import glob
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import unpyre  # noqa: E402
from unpyre.pyc import load_pyc  # noqa: E402

from helpers import code_key_sha  # noqa: E402
from make_golden import input_sha, run_ref  # noqa: E402
from paper_2403_13839_b200 import arena  # noqa: E402
from paper_2403_13839_b200.synth import (codejson, marshal, pycodegen, pycodegen38, pycodegen39,  # noqa: E402
                                         pycodegen311)

HERE = os.path.dirname(os.path.abspath(__file__))
CORPUS = "/root/reference/pkg/corpus"
STYLES = [None, {"indent": "    ", "header": True, "tool": "unpyre"}]


def _ref_tree_sha(ref_co):
    """code_key_sha of a reference CodeObject, via our model types."""
    from paper_2403_13839_b200 import model

    mine = arena.unpack(arena.pack([ref_co]), model.CodeObject, model.Const, model.VersionTag)[0]
    return code_key_sha(mine)


def main():
    files = sorted(glob.glob(os.path.join(CORPUS, "*", "*.py")))
    path = os.path.join(HERE, "c2.jsonl")
    n_ok = n = 0
    with open(path, "w") as f:
        for minor, compile_source in ((8, pycodegen38.compile_source), (9, pycodegen39.compile_source),
                                     (10, pycodegen.compile_source),
                                     (11, pycodegen311.compile_source)):
            for fn in files:
                rel = os.path.relpath(fn, CORPUS)
                with open(fn, encoding="utf-8") as src:
                    co = compile_source(src.read(), rel)
                _, ref_loaded = load_pyc(marshal.dump_pyc(co))
                assert _ref_tree_sha(ref_loaded) == code_key_sha(co), rel
                for style in STYLES:
                    status, text = run_ref(co, style)
                    rec = {"case": f"c2-3.{minor}-{rel[:-3]}" + ("-header" if style else ""), "gen": "c2", "minor": minor,
                           "tree": codejson.to_json(co), "input_sha": input_sha(co), "status": status, "text": text}
                    if style:
                        rec["style"] = style
                    f.write(json.dumps(rec) + "\n")
                    n += 1
                    n_ok += status == "ok"
    print(f"c2: {n} cases ({len(files)} modules x 4 versions x {len(STYLES)} styles), {n_ok} ok -> {path}")


if __name__ == "__main__":
    main()
