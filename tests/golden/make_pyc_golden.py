"""Golden vectors for the native .pyc loader, produced by the REAL reference
(unpyre.pyc.load_pyc + unpyre.decompile_source, imported from
/root/reference/pkg/src) on the corpus of paper_2403_13839_b200.synth.pycfuzz:

    python tests/golden/make_pyc_golden.py

Each line of pyc.jsonl: the case record (rebuilt into bytes by pycfuzz.blob),
blob_sha (pins the generator), the loader outcome (load_status = "ok" or the
exception class, load_text = str(exception), load_offset / load_magic
attributes, key_sha = digest of the loaded CodeObject tree, see
tests/helpers.code_key) and, for loadable files, the decompile outcome
(status/text as in the other golden sets).  Files on which the reference dies
with RecursionError (marshal nesting beyond ~245 levels hits Python's
recursion limit before the reader's own 256 limit) are recorded as such and
excluded from parity (loader).
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import unpyre  # noqa: E402
from unpyre.pyc import load_pyc  # noqa: E402

from helpers import code_key_sha  # noqa: E402
from paper_2403_13839_b200.synth import pycfuzz  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    recs = pycfuzz.corpus()
    path = os.path.join(HERE, "pyc.jsonl")
    stats = {}
    with open(path, "w") as f:
        for rec in recs:
            b = pycfuzz.blob(rec)
            out = dict(rec)
            out["blob_sha"] = hashlib.sha256(b).hexdigest()[:16]
            try:
                _, co = load_pyc(b)
            except RecursionError:
                out.update(load_status="RecursionError", load_text="", load_offset=None, load_magic=None)
            except Exception as e:  # noqa: BLE001
                out.update(load_status=type(e).__name__, load_text=str(e),
                           load_offset=getattr(e, "offset", None), load_magic=getattr(e, "magic", None))
            else:
                out.update(load_status="ok", load_text="", load_offset=None, load_magic=None,
                           key_sha=code_key_sha(co))
                try:
                    out.update(status="ok", text=unpyre.decompile_source(co))
                except Exception as e:  # noqa: BLE001
                    out.update(status=type(e).__name__, text=str(e))
            stats[out["load_status"]] = stats.get(out["load_status"], 0) + 1
            f.write(json.dumps(out, ensure_ascii=False) + "\n")
    print(f"pyc: {len(recs)} cases {stats} -> {path}")


if __name__ == "__main__":
    main()
