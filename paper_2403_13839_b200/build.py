"""In-tree build of the sm_100a library (and the test-only host harness).

    python -m paper_2403_13839_b200.build [--force]

libupy_cuda.so is linked from two nvcc objects compiled for sm_100a only:

* ``decode_kernel.o`` -- the HBM-bound decode kernel, full -O3;
* ``upy.o`` -- the decompile kernel and the C ABI.  The decompile kernel is one
  large, recursive, divergent function: ptxas -O3 on it takes >10 minutes for
  less speed than -O1 (measured below), so ptxas runs at -O1 there.

Each object is content-addressed (a stamp holds the digest of its sources and
flags), so tuning the decode kernel does not rebuild the decompile kernel.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJDIR = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libupy_cuda.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Measured on B200 (C3, 1M objects): cicc -O3 / ptxas -O1  2.75M obj/s (build ~5 min)
#                                    cicc -O3 / ptxas -O3  2.55M obj/s (build ~6 min)
#                                    cicc -O1 / ptxas -O1  1.67M obj/s (build ~30 s)
# UPY_FAST_BUILD=1 selects the last one for edit-compile-test loops.
CICC_OPT = "-O1" if os.environ.get("UPY_FAST_BUILD") else "-O3"
COMMON = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "550"]
BASE_DEPS = ["../../include/upy.h", "common.h", "optables.h", "unicode_tables.h"]
OBJECTS = {
    "decode_kernel": {"src": "decode_kernel.cu", "deps": BASE_DEPS + ["decode.h", "tma.h"],
                      "flags": COMMON + ["-Xptxas", "-O3"]},
    "stackscan_kernel": {"src": "stackscan_kernel.cu", "deps": BASE_DEPS + ["stackscan.h", "tma.h"],
                         "flags": COMMON + ["-Xptxas", "-O3"]},
    "pyc_loader": {"src": "pyc_loader.cpp", "deps": None, "flags": COMMON},
    "upy": {"src": "upy.cu", "deps": None,  # every header but decode.h / stackscan.h (their own kernels)
            "flags": COMMON + ["-Xcicc", CICC_OPT, "-Xptxas", "-O1"]},
}
LINK_FLAGS = [*ARCH, "-shared", "-Xcompiler", "-fPIC"]
NVCC_FLAGS = OBJECTS["upy"]["flags"]  # kept for tools that print the main flags


def _obj_deps(spec):
    if spec["deps"] is None:
        deps = [os.path.join(ROOT, "include", "upy.h")]
        deps += [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".h") and f not in ("decode.h", "stackscan.h", "tma.h")]
    else:
        deps = [os.path.normpath(os.path.join(CSRC, d)) for d in spec["deps"]]
    return deps + [os.path.join(CSRC, spec["src"])]


def _deps():
    out = [os.path.join(ROOT, "include", "upy.h")]
    out += [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]
    return out


def _digest(deps, flags):
    h = hashlib.sha256(" ".join(flags).encode())
    for d in deps:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def up_to_date(target, deps, flags=()):
    """Content-addressed: a stamp next to the target records the digest of the
    sources and flags it was built from (mtimes do not survive copies)."""
    stamp = target + ".stamp"
    if not os.path.exists(target) or not os.path.exists(stamp):
        return False
    with open(stamp) as f:
        return f.read().strip() == _digest(deps, flags)


def _run(cmd, verbose):
    if verbose:
        print("[build]", " ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def _stamp(target, digest):
    with open(target + ".stamp", "w") as f:
        f.write(digest)


def build_cuda(force=False, verbose=True):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJDIR, exist_ok=True)
    objs, link_digest = [], hashlib.sha256(" ".join(LINK_FLAGS).encode())
    for name, spec in OBJECTS.items():
        obj = os.path.join(OBJDIR, name + ".o")
        deps, flags = _obj_deps(spec), spec["flags"]
        digest = _digest(deps, flags)  # of the sources as they were when compilation started
        if force or not up_to_date(obj, deps, flags):
            _run([nvcc, *flags, "-c", "-o", obj + ".tmp", os.path.join(CSRC, spec["src"])], verbose)
            os.replace(obj + ".tmp", obj)
            _stamp(obj, digest)
        objs.append(obj)
        link_digest.update(digest.encode())
    link_digest = link_digest.hexdigest()
    if not force and os.path.exists(LIB) and os.path.exists(LIB + ".stamp"):
        with open(LIB + ".stamp") as f:
            if f.read().strip() == link_digest:
                return LIB
    _run([nvcc, *LINK_FLAGS, "-o", LIB + ".tmp", *objs], verbose)
    os.replace(LIB + ".tmp", LIB)
    _stamp(LIB, link_digest)
    return LIB


def build_packer(force=False, verbose=True):
    """The native arena packer (csrc/packer.cpp), a CPython extension built in-tree
    next to the package (g++ against this interpreter's Python.h)."""
    import sysconfig

    src = os.path.join(CSRC, "packer.cpp")
    target = os.path.join(HERE, "_packer" + sysconfig.get_config_var("EXT_SUFFIX"))
    flags = ["-O2", "-std=c++17", "-shared", "-fPIC", "-I" + sysconfig.get_paths()["include"]]
    if force or not up_to_date(target, [src], flags):
        digest = _digest([src], flags)
        _run([os.environ.get("CXX", "g++"), *flags, "-o", target + ".tmp", src], verbose)
        os.replace(target + ".tmp", target)
        _stamp(target, digest)
    return target


def build_host(force=False):
    from . import hostcheck

    return hostcheck.build(force=force)


def stage_reference():
    """Test infrastructure: copy the pure-Python reference into the git-ignored
    oracle/_ref (oracle/make_ref.py) when /root/reference exists."""
    sys.path.insert(0, ROOT)
    from oracle import make_ref

    return make_ref.stage()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    build_cuda(force)
    build_packer(force)
    build_host(force)
    stage_reference()


if __name__ == "__main__":
    main()
