"""In-tree build of the sm_100a library (and the test-only host harness).

    python -m paper_2403_13839_b200.build [--force]

libupy_cuda.so is compiled with nvcc for sm_100a only.  The decompile kernel
is one large, recursive, divergent function: full ptxas -O3 on it takes >10
minutes for little gain on pointer-chasing code, so ptxas runs at -O2 (cicc
stays at -O3).  See DESIGN.md "Build".
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libupy_cuda.so")
# Measured on B200 (C3, 1M objects): cicc -O3 / ptxas -O1  2.75M obj/s (build ~5 min)
#                                    cicc -O3 / ptxas -O3  2.55M obj/s (build ~6 min)
#                                    cicc -O1 / ptxas -O1  1.67M obj/s (build ~30 s)
# UPY_FAST_BUILD=1 selects the last one for edit-compile-test loops.
CICC_OPT = "-O1" if os.environ.get("UPY_FAST_BUILD") else "-O3"
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xcicc", CICC_OPT, "-Xptxas", "-O1",
              "-diag-suppress", "550"]


def _deps():
    out = [os.path.join(ROOT, "include", "upy.h")]
    out += [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]
    return out


def _digest(deps, flags):
    import hashlib

    h = hashlib.sha256(" ".join(flags).encode())
    for d in deps:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def up_to_date(target, deps, flags=()):
    """Content-addressed: a stamp next to the library records the digest of
    the sources and flags it was built from (mtimes do not survive copies)."""
    stamp = target + ".stamp"
    if not os.path.exists(target) or not os.path.exists(stamp):
        return False
    with open(stamp) as f:
        return f.read().strip() == _digest(deps, flags)


def build_cuda(force=False, verbose=True):
    deps = _deps()
    if not force and up_to_date(LIB, deps, NVCC_FLAGS):
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp", os.path.join(CSRC, "upy.cu")]
    if verbose:
        print("[build]", " ".join(cmd), flush=True)
    digest = _digest(deps, NVCC_FLAGS)  # of the sources as they were when compilation started
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    with open(LIB + ".stamp", "w") as f:
        f.write(digest)
    return LIB


def build_host(force=False):
    from . import hostcheck

    return hostcheck.build(force=force)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    build_cuda(force)
    build_host(force)


if __name__ == "__main__":
    main()
