"""Drop-in boundary: the reference's own CLI (`unpyre.cli.main`,
cli.py:54-92,205-216) with this package patched in as INTEGRATION.md §1 shows,
over a mixed batch of good and failing inputs, must behave exactly like the
plain reference: same exit code, same stdout, same stderr.  This holds only if
`decompile` raises the reference's exception classes (errors.bind), so
`except UnpyreError` in cmd_decompile catches them.

CPU tier: the patched-in backend is the host build of the device sources
(tests only); needs the reference tree, so it is skipped where that is absent
(the GPU box).  The GPU tier runs the same check through the CUDA path.
"""
import contextlib
import io
import os
import sys

import pytest

from conftest import golden_cases
from helpers import inputs

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.make_ref import ref_path  # noqa: E402

REF = ref_path()  # /root/reference/pkg/src here, the staged oracle/_ref copy on the GPU box
pytestmark = pytest.mark.skipif(REF is None, reason="reference not present")


def _files(tmp_path):
    from paper_2403_13839_b200 import jsondump

    recs = [r for r in golden_cases(["c1", "snippets", "mutant"]) if not r.get("style")]
    picks = [r for r in recs if r["status"] == "ok"][:6] + \
            [r for r in recs if r["status"] in ("StackUnderflow", "BadJumpTarget", "UnknownOpcode",
                                                "TruncatedCode", "StructuringFailed")][:6]
    paths = []
    for i, (r, co) in enumerate(zip(picks, inputs(picks))):
        p = tmp_path / f"in{i:02d}.json"
        p.write_text(jsondump.dumps(co))
        paths.append(str(p))
    return paths


def _run_cli(argv):
    import unpyre.cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = unpyre.cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def _check(tmp_path, backend):
    sys.path.insert(0, REF)
    import unpyre
    import unpyre.cli
    import unpyre.errors

    from paper_2403_13839_b200 import errors

    files = _files(tmp_path)
    want = _run_cli(["decompile", *files])
    assert want[0] == 1 and want[2].count("\n") >= 3 and want[1]  # a mixed batch: some inputs fail
    errors.bind(unpyre.errors)
    saved = unpyre.cli.decompile_source
    try:
        assert errors.bound() and errors.StackUnderflow is unpyre.errors.StackUnderflow
        unpyre.cli.decompile_source = backend
        got = _run_cli(["decompile", *files])
    finally:
        unpyre.cli.decompile_source = saved
        errors.bind(None)
    assert got == want


def test_reference_cli_with_host_build_patched_in(tmp_path):
    from paper_2403_13839_b200 import arena, hostcheck
    from paper_2403_13839_b200.errors import make_exception

    def host_decompile(code, style=None):
        ((st, text, aux),) = hostcheck.run(arena.pack([code]), style)
        if st:
            raise make_exception(st, text, aux)
        return text

    _check(tmp_path, host_decompile)


@pytest.mark.gpu
def test_reference_cli_with_cuda_path_patched_in(tmp_path):
    from paper_2403_13839_b200 import api

    _check(tmp_path, api.decompile)


def test_emitstyle_any_length_host():
    """EmitStyle.indent / tool longer than 64 bytes (accepted by the reference,
    emitter.py:46-50) go through the ABI by pointer."""
    from paper_2403_13839_b200 import _abi
    from paper_2403_13839_b200.model import EmitStyle

    st = EmitStyle(indent="\t" * 100, header=True, tool="t" * 300)
    o = _abi.options(st)
    assert o.indent_len == 100 and o.tool_len == 300 and o.indent == b"\t" * 100
