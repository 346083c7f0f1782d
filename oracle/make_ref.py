"""TEST INFRASTRUCTURE ONLY -- stage the real reference for the GPU box.

The reference (`unpyre`, /root/reference/pkg/src/unpyre) is pure Python, so
"building" it is a copy: into oracle/_ref/unpyre, which is git-ignored (never
committed) but travels with the gpurun snapshot like the built .so files.
There it is (a) the `bench.py --impl reference` arm and the cpu_baseline
(kind "reference"), and (b) the reference CLI the drop-in test patches.  Run by
`__graft_entry__.build()` / `python -m paper_2403_13839_b200.build` whenever
/root/reference exists; a no-op elsewhere (the box uses the staged copy).
"""
import os
import shutil

SRC = "/root/reference/pkg/src/unpyre"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_ref", "unpyre")


def ref_path():
    """Directory to put on sys.path to import the real `unpyre`, or None."""
    if os.path.isdir(os.path.dirname(SRC)):
        return os.path.dirname(SRC)
    if os.path.isdir(DST):
        return os.path.dirname(DST)
    return None


def stage():
    if not os.path.isdir(SRC):
        return None
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return DST


if __name__ == "__main__":
    print(stage())
