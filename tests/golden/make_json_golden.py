"""Golden outcomes of the REAL reference's JSON dump reader
(`unpyre.pyc.load_json_dump`, pyc.py:378-508) on seeded schema mutants
(paper_2403_13839_b200/synth/jsonfuzz.py) of dumps of a few golden objects.

    python tests/golden/make_json_golden.py

json.jsonl: {"base", "seed", "status", "text"}: status "ok" with text = the
structural digest of the loaded tree (tests/helpers.code_key_sha), or the
exception class and message.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

from unpyre import pyc  # noqa: E402

from helpers import code_key_sha  # noqa: E402
from paper_2403_13839_b200.synth import jsonfuzz  # noqa: E402

N_SEEDS = 120


def main():
    docs = jsonfuzz.base_docs(HERE)
    n = 0
    with open(os.path.join(HERE, "json.jsonl"), "w") as f:
        for b, doc in enumerate(docs):
            for seed in range(N_SEEDS):
                text = jsonfuzz.mutate(doc, seed)
                try:
                    (co,) = pyc.load_json_dump(text)
                    status, out = "ok", code_key_sha(co)
                except Exception as e:  # noqa: BLE001
                    status, out = type(e).__name__, str(e)
                n += status != "ok"
                f.write(json.dumps({"base": b, "seed": seed, "status": status, "text": out}) + "\n")
    print(f"{len(docs)} bases x {N_SEEDS} seeds, {n} errors")


if __name__ == "__main__":
    main()
