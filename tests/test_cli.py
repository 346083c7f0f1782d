"""Batch CLI (paper_2403_13839_b200/cli.py) against runs of the
REAL reference CLI recorded in tests/golden/cli.jsonl (make_cli_golden.py):
same exit codes, stdout, stderr and written files.  verify's elapsed-time
line / field is masked.  GPU tier (the decompile batches run on the device);
the JSON-dump reader is checked on CPU."""
import base64
import contextlib
import io
import json
import os
import re

import pytest

from conftest import load_golden


def _mask(s):
    s = re.sub(r"total (\d+) cases in [0-9.]+s", r"total \1 cases in Xs", s)
    return re.sub(r'"elapsed_seconds": [0-9.]+', '"elapsed_seconds": X', s)


def _run(tmp_path, rec):
    from paper_2403_13839_b200 import cli

    for rel, b64 in rec["files"].items():
        p = tmp_path / rel
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_bytes(base64.b64decode(b64))
    out, err = io.StringIO(), io.StringIO()
    cwd = os.getcwd()
    os.chdir(tmp_path)
    os.environ["UNPYRE_COLOR"] = "never"
    try:
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            rc = cli.main(rec["argv"])
    finally:
        os.chdir(cwd)
    produced = {}
    if (tmp_path / "outdir").is_dir():
        for fn in sorted(os.listdir(tmp_path / "outdir")):
            produced[f"outdir/{fn}"] = (tmp_path / "outdir" / fn).read_text(encoding="utf-8")
    return rc, out.getvalue(), err.getvalue(), produced


@pytest.mark.gpu
@pytest.mark.parametrize("rec", load_golden("cli"), ids=lambda r: r["case"])
def test_cli_matches_reference_cli(tmp_path, rec):
    rc, out, err, produced = _run(tmp_path, rec)
    assert rc == rec["rc"]
    assert _mask(out) == _mask(rec["stdout"])
    assert _mask(err) == _mask(rec["stderr"])
    assert produced == rec["out_files"]


def test_json_dump_reader_roundtrip_and_schema_errors():
    from paper_2403_13839_b200 import errors, jsondump
    from paper_2403_13839_b200.synth import codejson

    from helpers import code_key

    recs = [r for r in load_golden("c2") if not r.get("style")][:20]
    for r in recs:
        co = codejson.from_json(r["tree"])
        (back,) = jsondump.load_json_dump(jsondump.dumps(co))
        assert code_key(back) == code_key(co)
    # the schema errors the reference's CLI reported for the broken dumps
    want = {}
    for rec in load_golden("cli"):
        for line in rec["stderr"].splitlines():
            m = re.match(r"(\w+\.json): SchemaError: (.*)$", line)
            if m:
                want[m.group(1)] = (m.group(2), base64.b64decode(rec["files"][m.group(1)]))
    assert len(want) >= 3
    for name, (msg, data) in want.items():
        with pytest.raises(errors.SchemaError) as ei:
            jsondump.load_json_dump(data.decode())
        assert str(ei.value) == msg, name


def test_json_dump_reader_matches_reference_on_schema_mutants():
    """tests/golden/json.jsonl: the reference reader's outcome (tree digest or
    SchemaError/UnsupportedVersion message) on 720 seeded schema mutants."""
    from conftest import GOLDEN
    from paper_2403_13839_b200 import jsondump
    from paper_2403_13839_b200.synth import jsonfuzz

    from helpers import code_key_sha

    docs = jsonfuzz.base_docs(GOLDEN)
    bad = []
    for rec in load_golden("json"):
        text = jsonfuzz.mutate(docs[rec["base"]], rec["seed"])
        try:
            (co,) = jsondump.load_json_dump(text)
            got = ("ok", code_key_sha(co))
        except Exception as e:  # noqa: BLE001
            got = (type(e).__name__, str(e))
        if got != (rec["status"], rec["text"]):
            bad.append((rec["base"], rec["seed"], rec["status"], rec["text"], got))
    assert not bad, bad[:3]


@pytest.mark.parametrize("case", ["function", "function-module", "invalid-nested", "function-invalid-nested"])
def test_cli_function_path_host_build(tmp_path, case, monkeypatch):
    """--function renders emit_module([function_tree(target)]) with no
    validation (cli.py:75-78), also for '<module>' and for nested code that fails
    validation: CPU tier with the host build of the device sources standing in
    for the device batch."""
    from paper_2403_13839_b200 import api, hostcheck

    rec = next(r for r in load_golden("cli") if r["case"] == case)
    if not any(a.endswith(".pyc") for a in rec["argv"]):
        pytest.skip("no inputs")
    monkeypatch.setattr(api, "decompile_many", lambda codes, style=None, function_tree=False, **kw:
                        hostcheck.decompile_many(codes, style, function_tree=function_tree))
    from paper_2403_13839_b200 import arena, loader

    def pyc_many(blobs, style=None, **kw):
        ar, per = loader.load_pyc_batch(blobs)
        objs = arena.unpack(ar)
        return [v if isinstance(v, BaseException) else hostcheck.decompile_many([objs[v]], style)[0] for v in per]

    monkeypatch.setattr(loader, "decompile_pyc_many", pyc_many)
    rc, out, err, produced = _run(tmp_path, rec)
    assert (rc, out, err) == (rec["rc"], rec["stdout"], rec["stderr"])


def _host_backends(monkeypatch):
    """disasm's two device calls served by the test-only host build of the same
    sources (so the CLI's host logic runs on CPU)."""
    from paper_2403_13839_b200 import arena, disasm, hostcheck
    from paper_2403_13839_b200.errors import make_exception

    def decode_many(codes, device=None):
        ar = arena.pack(codes)
        ins, dec = hostcheck.decode(ar)
        objs, roots = ar.section("objs"), ar.section("roots")
        out = []
        for co, o in zip(codes, roots):
            d = dec[int(o)]
            if int(d["status"]):
                out.append(disasm.decode_exception(co, int(d["status"]), int(d["aux0"]), int(d["aux1"])))
            else:
                base = int(objs[int(o)]["code_off"]) >> 1
                out.append(disasm.instructions(co, ins[base:base + int(d["n_instrs"])]))
        return out

    def to_dot_many(codes, device=None):
        ar = arena.pack(codes)
        res = hostcheck.run(ar, output=1, text_cap=64 * ar.code_bytes + (1 << 20))
        return [s if st == 0 else make_exception(st, s, aux) for st, s, aux in res]

    monkeypatch.setattr(disasm, "decode_many", decode_many)
    monkeypatch.setattr(disasm, "to_dot_many", to_dot_many)


@pytest.mark.parametrize("rec", [r for r in load_golden("cli") if r["argv"][0] == "disasm"], ids=lambda r: r["case"])
def test_disasm_cli_host_matches_reference_cli(tmp_path, monkeypatch, rec):
    _host_backends(monkeypatch)
    rc, out, err, produced = _run(tmp_path, rec)
    assert (rc, out, err) == (rec["rc"], rec["stdout"], rec["stderr"])
