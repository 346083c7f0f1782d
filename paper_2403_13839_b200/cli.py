"""Batch command line front end on the GPU path.

    python -m paper_2403_13839_b200 decompile FILE... [--out DIR] [--function QUALNAME]
                                              [--version-override 3.X] [--no-header]
    python -m paper_2403_13839_b200 verify CORPUS_DIR [--json-report]
    python -m paper_2403_13839_b200 disasm FILE [--cfg] [--dot] [--version-override 3.X]

Restates the reference CLI's `decompile` and `verify` commands
(/root/reference/pkg/src/unpyre/cli.py:54-174, parser :177-217) with the same
arguments, stdout/stderr text, `UNPYRE_COLOR` handling and exit codes
(0 all good, 1 any processing failure, 2 usage or I/O error) -- but where the
reference decompiles one file after another, every input is loaded first
(.pyc images by the native loader in one multi-threaded call, JSON dumps by
jsondump.py) and all roots go to the device in ONE decompile_many batch.
Diagnostics are then emitted in input order, so the output matches the
serial reference byte for byte (verify's elapsed-time line aside).

`disasm` (cli.py:95-116) prints the instruction listing of every
code object from the decode kernel's records, or with --cfg --dot the Graphviz
CFG written by the device (csrc/dot.h).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

from . import errors
from .model import EmitStyle, VersionTag, flatten_nested_codes


def _color_mode():
    return os.environ.get("UNPYRE_COLOR", "auto")


def _diag(msg):
    """cli.py:26-35."""
    mode = _color_mode()
    if mode == "always" or (mode == "auto" and sys.stderr.isatty()):
        msg = f"\x1b[31m{msg}\x1b[0m"
    print(msg, file=sys.stderr)


def _parse_version(text):
    try:
        major, minor = text.split(".")
        return VersionTag(int(major), int(minor))
    except (ValueError, errors.UnpyreError):
        raise SystemExit(2)


def _is_json(path: Path, data: bytes):
    return path.suffix == ".json" or data[:1] in (b"{", b" ")


class _Loaded:
    """One input after loading: the roots as CodeObjects, or (for .pyc files on
    the plain decompile path) the image, decompiled straight from bytes."""

    def __init__(self, name, path, roots=None, pyc=None, error=None):
        self.name, self.path, self.roots, self.pyc, self.error = name, path, roots, pyc, error


def _load_all(items, override, want_objects):
    """Load every (name, path, data) triple: JSON dumps on the host, .pyc images
    in one native loader call.  Errors are kept per input (cli.py:61-89)."""
    from . import loader
    from .jsondump import load_json_dump

    out = []
    pyc_idx = []
    for name, path, data in items:
        if _is_json(path, data):
            try:
                out.append(_Loaded(name, path, roots=load_json_dump(data.decode("utf-8"), override)))
            except errors.UnpyreError as exc:
                out.append(_Loaded(name, path, error=exc))
        else:
            out.append(_Loaded(name, path, pyc=data))
            pyc_idx.append(len(out) - 1)
    if pyc_idx:
        arena, per_file = loader.load_pyc_batch([out[i].pyc for i in pyc_idx])
        objs = None
        for i, v in zip(pyc_idx, per_file):
            if isinstance(v, BaseException):
                out[i].error, out[i].pyc = v, None
            elif want_objects:
                if objs is None:
                    from .arena import unpack

                    objs = unpack(arena)
                out[i].roots, out[i].pyc = [objs[v]], None
    return out


def _decompile_loaded(loaded, style, function=None):
    """One device batch for every root of every loaded input.  Returns per input
    either the joined text or the first exception (reference order)."""
    from . import api, loader

    jobs = []   # (input index, CodeObject) in reference order
    pre = {}    # input index -> exception raised before decompiling
    for k, ld in enumerate(loaded):
        if ld.error is not None or ld.pyc is not None:
            continue
        for root in ld.roots:
            if function:
                flat = dict(flatten_nested_codes(root))
                if function not in flat:
                    pre.setdefault(k, errors.UnpyreError(f"no code object named {function!r}; have: "
                                                  + ", ".join(sorted(flat))))
                    break
                jobs.append((k, flat[function]))
            else:
                jobs.append((k, root))
    vals = api.decompile_many([c for _, c in jobs], style, function_tree=bool(function)) if jobs else []
    pyc_k = [k for k, ld in enumerate(loaded) if ld.pyc is not None]
    pyc_vals = loader.decompile_pyc_many([loaded[k].pyc for k in pyc_k], style) if pyc_k else []
    texts = {k: [] for k in range(len(loaded))}
    errs = {}
    for (k, _), v in zip(jobs, vals):
        if k in errs or k in pre:
            continue
        if isinstance(v, BaseException):
            errs[k] = v
        else:
            texts[k].append(v)
    for k, v in zip(pyc_k, pyc_vals):
        if isinstance(v, BaseException):
            errs[k] = v
        else:
            texts[k].append(v)
    result = []
    for k, ld in enumerate(loaded):
        e = ld.error or pre.get(k) or errs.get(k)
        result.append(e if e is not None else "".join(texts[k]))
    return result


def cmd_decompile(args) -> int:
    """cli.py:54-92.  The reference stops at the first missing input after having
    processed (and reported the failures of) the inputs before it; the batch
    keeps that order: inputs up to the first missing one go to the device,
    their diagnostics are printed, then the missing-file error, exit 2."""
    style = EmitStyle(header=not args.no_header)
    items = []
    missing = None
    override = None
    for name in args.inputs:
        path = Path(name)
        if not path.exists():
            missing = name
            break
        override = _parse_version(args.version_override) if args.version_override else None
        items.append((name, path, path.read_bytes()))
    loaded = _load_all(items, override, want_objects=bool(args.function))
    results = _decompile_loaded(loaded, style, args.function) if items else []
    failures = 0
    outputs = []
    for (name, path, _), r in zip(items, results):
        if isinstance(r, errors.UnpyreError):
            _diag(f"{name}: {type(r).__name__}: {r}")
            failures += 1
        elif isinstance(r, BaseException):
            raise r
        else:
            outputs.append((path, r))
    if missing is not None:
        _diag(f"{missing}: no such file")
        return 2
    for path, text in outputs:
        if args.out:
            dest = Path(args.out) / (path.stem + ".py")
            dest.parent.mkdir(parents=True, exist_ok=True)
            dest.write_text(text, encoding="utf-8")
        else:
            sys.stdout.write(text)
    return 1 if failures else 0


def cmd_verify(args) -> int:
    """cli.py:119-174: per-version pass table (or JSON report) of a corpus of
    JSON dumps against their .expected.py goldens, all cases in one batch."""
    t0 = time.monotonic()
    base = Path(args.corpus_dir)
    if not base.is_dir():
        _diag(f"{args.corpus_dir}: not a directory")
        return 2
    style = EmitStyle(header=True)
    cases = []
    for vdir in sorted(base.glob("py3*")):
        for case in sorted(vdir.glob("*.json")):
            cases.append((vdir.name, case))
    loaded = _load_all([(str(c), c, c.read_bytes()) for _, c in cases], None, want_objects=False)
    results = _decompile_loaded(loaded, style)
    table = {}
    failures = []
    total = 0
    for vdir in sorted(base.glob("py3*")):
        table[vdir.name] = [0, 0]
    for (version, case), r in zip(cases, results):
        total += 1
        table[version][1] += 1
        name = f"{version}/{case.stem}"
        if isinstance(r, errors.UnpyreError):
            failures.append((name, f"{type(r).__name__}: {r}"))
            continue
        if isinstance(r, BaseException):
            raise r
        expected = case.with_suffix("").with_suffix(".expected.py")
        if not expected.exists():
            failures.append((name, "missing golden"))
            continue
        if r == expected.read_text(encoding="utf-8"):
            table[version][0] += 1
        else:
            failures.append((name, "output differs from golden"))
    elapsed = time.monotonic() - t0
    if args.json_report:
        report = {
            "versions": {v: {"passed": ok, "total": n} for v, (ok, n) in table.items()},
            "failures": [{"case": c, "reason": r} for c, r in failures],
            "elapsed_seconds": round(elapsed, 3),
        }
        json.dump(report, sys.stdout, indent=2)
        print()
    else:
        if not table:
            print("0 cases")
        width = max((len(v) for v in table), default=8)
        for version, (ok, n) in table.items():
            pct = 100.0 * ok / n if n else 100.0
            print(f"{version:<{width}}  {pct:6.1f}%  ({ok}/{n})")
        for case, reason in failures:
            _diag(f"FAIL {case}: {reason}")
        print(f"total {total} cases in {elapsed:.2f}s")
    return 1 if failures else 0


def cmd_disasm(args) -> int:
    """cli.py:95-116: an instruction listing per code object (flatten order), or
    with --cfg --dot the CFG export.  All code objects of the input go to the
    device in one batch (decode kernel for listings, the CFG kernel for dot);
    output and the first error are then reported in reference order."""
    from . import disasm

    path = Path(args.input)
    if not path.exists():
        _diag(f"{args.input}: no such file")
        return 2
    try:
        override = _parse_version(args.version_override) if args.version_override else None
        ld = _load_all([(args.input, path, path.read_bytes())], override, want_objects=True)[0]
        if ld.error is not None:
            raise ld.error
        flat = [qc for root in ld.roots for qc in flatten_nested_codes(root)]
        dot = args.cfg and args.dot
        codes = [c for _, c in flat]
        results = disasm.to_dot_many(codes) if dot else disasm.decode_many(codes)
        for (qualname, _code), v in zip(flat, results):
            if not dot:
                print(f"-- {qualname}")
            if isinstance(v, BaseException):
                raise v
            sys.stdout.write(v if dot else disasm.format_listing(v))
    except errors.UnpyreError as exc:
        _diag(f"{args.input}: {type(exc).__name__}: {exc}")
        return 1
    return 0


def build_parser():
    """cli.py:177-202."""
    parser = argparse.ArgumentParser(prog="unpyre", description="CPython bytecode decompiler")
    sub = parser.add_subparsers(dest="command", required=True)
    d = sub.add_parser("decompile", help="decompile .pyc files or JSON dumps")
    d.add_argument("inputs", nargs="+")
    d.add_argument("--out", help="write one .py per input into this directory")
    d.add_argument("--function", help="decompile only this qualified code object")
    d.add_argument("--version-override", help="force MAJ.MIN for JSON dumps")
    d.add_argument("--no-header", action="store_true", help="omit the provenance header comment")
    d.set_defaults(func=cmd_decompile)
    s = sub.add_parser("disasm", help="print an instruction listing")
    s.add_argument("input")
    s.add_argument("--cfg", action="store_true")
    s.add_argument("--dot", action="store_true")
    s.add_argument("--version-override")
    s.set_defaults(func=cmd_disasm)
    v = sub.add_parser("verify", help="check fixture corpus against goldens")
    v.add_argument("corpus_dir")
    v.add_argument("--json-report", action="store_true")
    v.set_defaults(func=cmd_verify)
    return parser


def main(argv=None) -> int:
    """cli.py:205-217."""
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 2 if exc.code not in (0, None) else 0
    try:
        return args.func(args)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 2
    except BrokenPipeError:
        return 1
