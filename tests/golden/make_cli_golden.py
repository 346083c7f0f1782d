"""Golden runs of the REAL reference CLI (unpyre.cli.main, imported from
/root/reference/pkg/src) for the batch CLI (paper_2403_13839_b200/cli.py,
SURVEY.md §8 f2).  Run in the build container:

    python tests/golden/make_cli_golden.py

Inputs are C2 modules (tests/golden/c2.jsonl) written as .pyc images
(synth/marshal.py) and JSON dumps (jsondump.dumps), plus broken files (a
truncated .pyc, an unknown magic, schema errors), a missing path, and a verify
corpus (py310/ with goldens that match, differ or are missing, and a failing
case).  Each line of cli.jsonl: {"case", "files": {relpath: base64}, "argv",
"rc", "stdout", "stderr", "out_files": {relpath: text}}; paths are relative to
a scratch directory that the test recreates.
"""
import base64
import contextlib
import io
import json
import os
import shutil
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import unpyre  # noqa: E402
from unpyre import cli as ref_cli  # noqa: E402

from paper_2403_13839_b200 import arena, jsondump  # noqa: E402
from paper_2403_13839_b200.synth import codejson, marshal  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MODS = ["classes/class_inherit_kw", "comprehensions/nested_listcomp", "control/for_break_continue",
        "exceptions/try_except_else_finally", "functions/nested_defs", "generators_ctx/with_two_items",
        "modules/module_level_code", "strings/fstring_format_spec", "bool_flow/and_or_values",
        "functions/lambda_uses"]


def _trees(minor=10):
    with open(os.path.join(HERE, "c2.jsonl")) as f:
        recs = [json.loads(line) for line in f]
    by = {r["case"][len(f"c2-3.{minor}-"):]: codejson.from_json(r["tree"]) for r in recs
          if not r.get("style") and r["minor"] == minor}
    return [(m.split("/")[1], by[m]) for m in MODS]


def _run(files, argv):
    d = tempfile.mkdtemp()
    try:
        for rel, data in files.items():
            p = os.path.join(d, rel)
            os.makedirs(os.path.dirname(p), exist_ok=True)
            with open(p, "wb") as f:
                f.write(data)
        out, err = io.StringIO(), io.StringIO()
        cwd = os.getcwd()
        os.chdir(d)
        os.environ["UNPYRE_COLOR"] = "never"
        try:
            with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                rc = ref_cli.main(argv)
        finally:
            os.chdir(cwd)
        produced = {}
        if os.path.isdir(os.path.join(d, "outdir")):
            for fn in sorted(os.listdir(os.path.join(d, "outdir"))):
                with open(os.path.join(d, "outdir", fn), encoding="utf-8") as f:
                    produced[f"outdir/{fn}"] = f.read()
        return rc, out.getvalue(), err.getvalue(), produced
    finally:
        shutil.rmtree(d)


def main():
    trees = _trees()
    pyc = {f"{n}.pyc": marshal.dump_pyc(co) for n, co in trees}
    js = {f"{n}.json": jsondump.dumps(co).encode() for n, co in trees}
    bad = {
        "trunc.pyc": marshal.dump_pyc(trees[0][1])[:40],
        "magic.pyc": b"\x00\x00\x0d\x0a" + bytes(12),
        "schema.json": json.dumps({"format_version": 1, "python_version": [3, 10], "root": {"argcount": 0}}).encode(),
        "notjson.json": b"{ nope",
        "badver.json": json.dumps({"format_version": 1, "python_version": [3, 12], "root": {}}).encode(),
    }
    names = [n for n, _ in trees]
    # a module whose nested `f` fails validation (stacksize < 0): plain decompile
    # reports it, --function decompiles f without validating (cli.py:75-78)
    import dataclasses

    from paper_2403_13839_b200.model import Const
    from paper_2403_13839_b200.synth import corpus as synth_corpus

    mod = synth_corpus.shared_bytes(10)
    f_code = dataclasses.replace(mod.consts[0].value, stacksize=-1)
    invalid = {"invalid.pyc": marshal.dump_pyc(dataclasses.replace(
        mod, consts=(Const("code", f_code),) + tuple(mod.consts[1:])))}
    cases = [
        ("pyc-all", pyc, ["decompile", *pyc]),
        ("json-all-noheader", js, ["decompile", "--no-header", *js]),
        ("mixed-with-errors", {**pyc, **js, **bad}, ["decompile", *list(pyc)[:3], *bad, *list(js)[3:6]]),
        ("missing-after-bad", {**pyc, **bad}, ["decompile", "trunc.pyc", list(pyc)[1], "nothere.pyc", list(pyc)[2]]),
        ("missing-first", pyc, ["decompile", "nothere.pyc", *list(pyc)[:2]]),
        ("out-dir", pyc, ["decompile", "--out", "outdir", *list(pyc)[:4]]),
        ("function", pyc, ["decompile", "--function", "<module>.outer.middle", f"{names[4]}.pyc"]),
        ("function-missing", pyc, ["decompile", "--function", "nope", f"{names[0]}.pyc", f"{names[1]}.pyc"]),
        ("function-module", pyc, ["decompile", "--function", "<module>", f"{names[6]}.pyc", f"{names[8]}.pyc"]),
        ("invalid-nested", invalid, ["decompile", "invalid.pyc"]),
        ("function-invalid-nested", invalid, ["decompile", "--function", "<module>.f", "invalid.pyc"]),
        ("version-override", js, ["decompile", "--version-override", "3.10", *list(js)[:2]]),
        ("version-override-bad", js, ["decompile", "--version-override", "3.x", *list(js)[:2]]),
        ("usage", {}, ["decompile"]),
    ]
    # disasm (cli.py:95-116): listings and the --cfg --dot export, incl. 3.11
    # (exception tables), a code error inside a nested code object, bad inputs
    by311 = _trees(11)
    pyc311 = {f"{n}_311.pyc": marshal.dump_pyc(co) for n, co in by311}
    broken = {"brokennested.pyc": marshal.dump_pyc(dataclasses.replace(
        mod, consts=(Const("code", dataclasses.replace(mod.consts[0].value, code=b"\x00\x00")),)
        + tuple(mod.consts[1:])))}
    cases += [
        ("disasm-pyc", pyc, ["disasm", f"{names[4]}.pyc"]),
        ("disasm-json", js, ["disasm", f"{names[0]}.json"]),
        ("disasm-cfg-dot", pyc, ["disasm", "--cfg", "--dot", f"{names[3]}.pyc"]),
        ("disasm-cfg-dot-loops", pyc, ["disasm", "--cfg", "--dot", f"{names[2]}.pyc"]),
        ("disasm-cfg-only", pyc, ["disasm", "--cfg", f"{names[1]}.pyc"]),
        ("disasm-dot-only", pyc, ["disasm", "--dot", f"{names[7]}.pyc"]),
        ("disasm-311", pyc311, ["disasm", f"{by311[3][0]}_311.pyc"]),
        ("disasm-311-dot", pyc311, ["disasm", "--cfg", "--dot", f"{by311[3][0]}_311.pyc"]),
        ("disasm-311-dot-gen", pyc311, ["disasm", "--cfg", "--dot", f"{by311[5][0]}_311.pyc"]),
        ("disasm-nested-error", broken, ["disasm", "brokennested.pyc"]),
        ("disasm-nested-error-dot", broken, ["disasm", "--cfg", "--dot", "brokennested.pyc"]),
        ("disasm-bad-pyc", bad, ["disasm", "trunc.pyc"]),
        ("disasm-schema", bad, ["disasm", "schema.json"]),
        ("disasm-missing", {}, ["disasm", "nothere.pyc"]),
        ("disasm-version-override", js, ["disasm", "--version-override", "3.10", f"{names[5]}.json"]),
        ("disasm-version-override-bad", js, ["disasm", "--version-override", "x", f"{names[5]}.json"]),
    ]
    # verify corpus: py310/<case>.json + <case>.expected.py
    corpus = {}
    for i, (n, co) in enumerate(trees):
        corpus[f"corp/py310/{n}.json"] = jsondump.dumps(co).encode()
        ref = arena.unpack(arena.pack([co]), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)[0]
        text = unpyre.decompile_source(ref, unpyre.EmitStyle(header=True))
        if i == 2:
            text += "# drift\n"
        if i != 5:
            corpus[f"corp/py310/{n}.expected.py"] = text.encode()
    corpus["corp/py310/zz_schema.json"] = bad["schema.json"]
    good = {k: v for k, v in corpus.items() if not k.startswith("corp/py310/zz") and "with_two" not in k
            and "for_break" not in k}
    cases += [
        ("verify", corpus, ["verify", "corp"]),
        ("verify-json", corpus, ["verify", "--json-report", "corp"]),
        ("verify-clean", good, ["verify", "corp"]),
        ("verify-notdir", {}, ["verify", "nodir"]),
    ]
    path = os.path.join(HERE, "cli.jsonl")
    with open(path, "w") as f:
        for name, files, argv in cases:
            rc, out, err, produced = _run(files, argv)
            f.write(json.dumps({"case": name, "files": {k: base64.b64encode(v).decode() for k, v in files.items()},
                                "argv": argv, "rc": rc, "stdout": out, "stderr": err, "out_files": produced}) + "\n")
            print(f"{name}: rc={rc} stdout={len(out)}B stderr={len(err)}B")
    print(f"-> {path}")


if __name__ == "__main__":
    main()
