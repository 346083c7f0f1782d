"""Native .pyc loader (csrc/pyc_loader.cpp, `upy_pyc_load`) against the real
reference's `load_pyc` + `decompile_source` outcomes (tests/golden/pyc.jsonl,
made by tests/golden/make_pyc_golden.py): valid images in three marshal
encodings and ~600 seeded mutants covering every reader failure branch.

CPU tier: the loader is host code, so the loaded CodeObject trees (every field)
and the loader exceptions (class, message, offset / magic) are checked here.
GPU tier: the same images end to end through decompile_pyc_many.
"""
import hashlib
import os

import pytest

from conftest import ROOT, load_golden
from helpers import code_key_sha, outcome

LIB = os.path.join(ROOT, "paper_2403_13839_b200", "libupy_cuda.so")
needs_lib = pytest.mark.skipif(not os.path.exists(LIB), reason="CUDA library not built")


def _cases():
    # RecursionError: the reference hits Python's recursion limit (outside the parity domain)
    return [r for r in load_golden("pyc") if r["load_status"] != "RecursionError"]


def _blobs(recs):
    from paper_2403_13839_b200.synth import pycfuzz

    out = []
    for r in recs:
        b = pycfuzz.blob(r)
        assert hashlib.sha256(b).hexdigest()[:16] == r["blob_sha"], r["case"]
        out.append(b)
    return out


def _load_outcome(v):
    if isinstance(v, BaseException):
        return (type(v).__name__, str(v), getattr(v, "offset", None), getattr(v, "magic", None))
    return v


@needs_lib
def test_native_loader_matches_reference_load_pyc():
    from paper_2403_13839_b200 import arena, loader

    recs = _cases()
    ar, per_file = loader.load_pyc_batch(_blobs(recs))
    roots = arena.unpack(ar)
    bad = []
    n_ok = 0
    for r, v in zip(recs, per_file):
        if r["load_status"] == "ok":
            got = "ok" if isinstance(v, BaseException) else code_key_sha(roots[v])
            n_ok += 1
            if got != r["key_sha"]:
                bad.append((r["case"], "ok", _load_outcome(v)))
        else:
            want = (r["load_status"], r["load_text"], r["load_offset"], r["load_magic"])
            if _load_outcome(v) != want:
                bad.append((r["case"], want, _load_outcome(v)))
    assert n_ok > 300
    assert not bad, bad[:3]


@needs_lib
def test_native_loader_threads_agree():
    from paper_2403_13839_b200 import loader

    blobs = _blobs(_cases()[:200])
    a1, p1 = loader.load_pyc_batch(blobs, n_threads=1)
    a8, p8 = loader.load_pyc_batch(blobs, n_threads=8)
    assert (a1.blob == a8.blob).all()
    assert [_load_outcome(x) for x in p1] == [_load_outcome(x) for x in p8]


@needs_lib
def test_load_pyc_single_file_api():
    from paper_2403_13839_b200 import errors, loader

    r = next(x for x in _cases() if x["load_status"] == "ok")
    version, co = loader.load_pyc(_blobs([r])[0])
    assert code_key_sha(co) == r["key_sha"] and version.minor == co.version.minor
    with pytest.raises(errors.TruncatedHeader) as ei:
        loader.load_pyc(b"\x6f\x0d\x0d\x0a")
    assert str(ei.value) == "pyc header needs 16 bytes, got 4"
    with pytest.raises(errors.UnknownMagic) as ei:
        loader.load_pyc(b"\x00\x00\x0d\x0a" + bytes(12))
    assert ei.value.magic == 0 and str(ei.value) == "unknown pyc magic 0x0000 (unsupported interpreter version)"


@pytest.mark.gpu
def test_gpu_decompile_pyc_matches_reference():
    from paper_2403_13839_b200 import loader

    recs = _cases()
    got = loader.decompile_pyc_many(_blobs(recs))
    bad = []
    for r, v in zip(recs, got):
        if r["load_status"] != "ok":
            want = (r["load_status"], r["load_text"])
        else:
            want = (r["status"], r["text"])
        if outcome(v) != want:
            bad.append((r["case"], want[0], outcome(v)[0], want[1][:200], outcome(v)[1][:200]))
    assert not bad, bad[:3]
