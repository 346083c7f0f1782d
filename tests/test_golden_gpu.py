"""GPU tier: the CUDA path (C ABI -> decode + decompile kernels) against the
reference's golden outputs, byte for byte."""
import pytest

from conftest import golden_cases
from helpers import inputs, mismatches, outcome, style_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gset", ["c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2"])
def test_gpu_matches_reference(gset):
    from paper_2403_13839_b200 import api

    recs = golden_cases([gset])
    by_style = {}
    for r in recs:
        by_style.setdefault(repr(r.get("style")), []).append(r)
    bad = []
    for _, group in by_style.items():
        got = [outcome(v) for v in api.decompile_many(inputs(group), style_of(group[0]))]
        bad += mismatches(group, got)
    assert not bad, bad[:3]


def test_gpu_single_decompile_raises_reference_class():
    from paper_2403_13839_b200 import api, errors
    from paper_2403_13839_b200.synth import snippets

    with pytest.raises(errors.StackUnderflow) as ei:
        api.decompile(snippets.underflow(10))
    assert str(ei.value) == "evaluation stack underflow at offset 0 (RETURN_VALUE)"
    assert ei.value.offset == 0


def test_gpu_c2_from_pyc_images_matches_reference():
    """C2 modules as .pyc images (synth/marshal.py) through the native loader and
    the kernels: same text as the reference decompiling the compiled tree."""
    from paper_2403_13839_b200 import loader
    from paper_2403_13839_b200.synth import marshal

    recs = [r for r in golden_cases(["c2"]) if not r.get("style")]
    got = [outcome(v) for v in loader.decompile_pyc_many([marshal.dump_pyc(co) for co in inputs(recs)])]
    assert not mismatches(recs, got)
