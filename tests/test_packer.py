"""The native arena packer (csrc/packer.cpp, `arena.pack`) against the Python
restatement of the same layout (`arena.pack_py`): byte-identical images on every
golden input set, on the reference's own CodeObject instances, and on the edge
cases of the int clamping and const kinds."""
import dataclasses

import numpy as np
import pytest

from conftest import golden_cases
from helpers import inputs


def _same(a, b):
    assert a.offsets == b.offsets and a.counts == b.counts
    assert (a.max_code_len, a.total_code_units) == (b.max_code_len, b.total_code_units)
    assert np.array_equal(a.blob, b.blob)


@pytest.mark.parametrize("gset", ["c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2"])
def test_native_pack_matches_python_pack(gset):
    from paper_2403_13839_b200 import arena

    codes = inputs([r for r in golden_cases([gset]) if not r.get("style")])
    _same(arena.pack(codes), arena.pack_py(codes))


def test_native_pack_edge_values():
    from paper_2403_13839_b200 import arena
    from paper_2403_13839_b200.model import Const
    from paper_2403_13839_b200.synth import corpus

    base = corpus.c3(5)
    inner = corpus.c3(6)
    consts = (Const("int", -(1 << 200) - 7), Const("int", 0), Const("bool", True), Const("float", -0.0),
              Const("complex", complex(1.5, -2.0)), Const("str", "a\udc80€"), Const("bytes", b"\x00\xff"),
              Const("tuple", (Const("int", 3), Const("tuple", ()), Const("code", inner))),
              Const("frozenset", (Const("str", "x"),)), Const("code", inner), Const("ellipsis"), Const("none"))
    odd = dataclasses.replace(base, consts=consts, flags=(1 << 63) | 0x43, argcount=1 << 70,
                              stacksize=-(1 << 65), firstlineno=True, linetable=b"\x01\x02",
                              exceptiontable=b"\x80\x01", names=("g", "h", "é"), qualname="")
    roots = [odd, base, odd, inner]  # shared objects are packed once
    _same(arena.pack(roots), arena.pack_py(roots))


def test_native_pack_reference_objects():
    import sys

    from oracle import make_ref

    path = make_ref.ref_path()
    if path is None:
        pytest.skip("reference not available")
    sys.path.insert(0, path)
    import unpyre

    from paper_2403_13839_b200 import arena

    codes = inputs([r for r in golden_cases(["c2"]) if not r.get("style")])[:60]
    ref = arena.unpack(arena.pack_py(codes), unpyre.CodeObject, unpyre.Const, unpyre.VersionTag)
    _same(arena.pack(ref), arena.pack_py(ref))


def test_native_pack_errors_are_python_exceptions():
    from paper_2403_13839_b200 import arena
    from paper_2403_13839_b200.model import Const
    from paper_2403_13839_b200.synth import corpus

    bad = dataclasses.replace(corpus.c3(1), consts=(Const("none"), object()))
    with pytest.raises(AttributeError):
        arena.pack([bad])
