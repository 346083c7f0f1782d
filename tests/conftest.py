import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}.jsonl")) as f:
        return [json.loads(line) for line in f]


GOLDEN_SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz", "mutant", "mutant2", "mutant3")


def golden_cases(sets=GOLDEN_SETS):
    out = []
    for s in sets:
        if os.path.exists(os.path.join(GOLDEN, f"{s}.jsonl")):
            out.extend(load_golden(s))
    return out


@pytest.fixture(scope="session")
def all_golden():
    return golden_cases()
