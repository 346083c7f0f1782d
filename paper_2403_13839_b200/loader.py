"""Native .pyc loading: the reference's `load_pyc(data) -> (VersionTag,
CodeObject)` (pyc.py:50-52) and a batched path that parses many .pyc images
in C++ (csrc/pyc_loader.cpp, `upy_pyc_load`) straight into the arena the
decompile kernel reads, skipping Python object construction entirely.

    arena, errors = load_pyc_batch(blobs)        # host, multi-threaded C++
    texts = decompile_pyc_many(blobs, style)     # + one H2D copy + the GPU path

Loader failures are the reference's exception classes (UnknownMagic,
TruncatedHeader, MalformedMarshal) with identical messages and attributes.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _abi, _lib
from .arena import SECTIONS, Arena, unpack
from .errors import ST_OK, make_exception


def load_pyc_batch(blobs, n_threads=0, pinned=False):
    """Parse .pyc images into one Arena.  Returns (arena, per_file) where
    per_file[i] is the root position of file i in the arena or the exception
    instance the reference's load_pyc raises for it.  pinned=True writes the
    image into page-locked memory (torch's caching host allocator, reused across
    calls) so the H2D copy is a direct DMA."""
    lib = _lib.load()
    blobs = [bytes(b) for b in blobs]
    n = len(blobs)
    bufs = [C.create_string_buffer(b, len(b)) if b else C.create_string_buffer(1) for b in blobs]
    ptrs = (C.c_void_p * max(n, 1))(*[C.addressof(x) for x in bufs])
    sizes = (C.c_uint64 * max(n, 1))(*[len(b) for b in blobs])
    return _load(lib, ptrs, sizes, n, n_threads, pinned)


def load_pyc_buffer(buf, offsets, sizes, n_threads=0, pinned=False):
    """load_pyc_batch over files stored back to back in one buffer (numpy uint8 /
    bytes) at `offsets` with `sizes`: no per-file Python objects at all."""
    lib = _lib.load()
    base = np.frombuffer(buf, dtype=np.uint8)
    offsets = np.asarray(offsets, dtype=np.uint64)
    sizes = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
    ptrs = np.ascontiguousarray(offsets + np.uint64(base.ctypes.data))
    return _load(lib, ptrs.ctypes.data_as(C.POINTER(C.c_void_p)), sizes.ctypes.data_as(C.POINTER(C.c_uint64)),
                 len(sizes), n_threads, pinned)


def _load(lib, ptrs, sizes, n, n_threads, pinned):
    out = C.POINTER(_abi.UpyPycBatch)()
    rc = lib.upy_pyc_load(ptrs, sizes, n, int(n_threads), _abi.PYC_DEFER_IMAGE if pinned else 0, C.byref(out))
    _lib.check(rc, "upy_pyc_load")
    b = out.contents
    host = None
    if pinned:
        import torch

        host = torch.empty(int(b.image_bytes), dtype=torch.uint8, pin_memory=True)
        _lib.check(lib.upy_pyc_write_image(out, C.c_void_p(host.data_ptr()), C.c_uint64(host.numel())),
                   "upy_pyc_write_image")
        image = host.numpy()
    else:
        # the arena views the library's image (no copy); freed with the arena
        image = np.ctypeslib.as_array(C.cast(b.image, C.POINTER(C.c_uint8)), shape=(int(b.image_bytes),))
    offsets = {s: int(b.section_off[i]) for i, s in enumerate(SECTIONS)}
    counts = {s: int(b.section_count[i]) for i, s in enumerate(SECTIONS)}
    arena = Arena(image, offsets, counts, int(b.max_code_len), int(b.total_code_units))
    arena.pinned = host  # torch pinned tensor (DeviceArena uploads from it directly) or None
    status = np.ctypeslib.as_array(b.file_status, shape=(n,)).copy() if n else np.zeros(0, np.int32)
    per_file = []
    if n and (status == ST_OK).all():
        per_file = np.ctypeslib.as_array(b.file_root, shape=(n,)).tolist()
    else:
        msgs = C.string_at(b.messages, int(sum(b.msg_len[i] for i in range(n)))) if n else b""
        for i in range(n):
            if status[i] == ST_OK:
                per_file.append(int(b.file_root[i]))
            else:
                o, ln = int(b.msg_off[i]), int(b.msg_len[i])
                per_file.append(make_exception(int(status[i]), msgs[o:o + ln].decode("utf-8", "replace"),
                                               (int(b.file_aux[i]), 0)))
    if pinned:
        lib.upy_pyc_free(out)
    else:
        weakref.finalize(arena, lib.upy_pyc_free, out)
    return arena, per_file


def load_pyc(data: bytes):
    """Drop-in for unpyre.pyc.load_pyc (pyc.py:50-52): (VersionTag, CodeObject)."""
    arena, per_file = load_pyc_batch([data], n_threads=1)
    v = per_file[0]
    if isinstance(v, BaseException):
        raise v
    code = unpack(arena)[v]
    return code.version, code


def decompile_pyc_many(blobs, style=None, device=None, n_threads=0, chunk_files=1 << 18):
    """Decompile a batch of .pyc images on the GPU: one entry per file, the text
    or the exception the reference's `load_pyc` + `decompile_source` raise.

    Large batches run as a pipeline of sub-batches of `chunk_files` files: the
    native loader (all host threads) parses sub-batch i+1 while the device
    decompiles sub-batch i."""
    blobs = [bytes(b) for b in blobs]
    out = []
    for lo, per_file, res in decompile_pyc_chunks(
            lambda a, b: load_pyc_batch(blobs[a:b], n_threads, pinned=True), len(blobs), style, device,
            chunk_files):
        vals = res.values() if res is not None else []
        for v in per_file:
            out.append(v if isinstance(v, BaseException) else vals[v])
    return out


def decompile_pyc_chunks(load, n_files, style=None, device=None, chunk_files=1 << 18):
    """Pipelined driver: `load(lo, hi)` -> (arena, per_file) for files [lo, hi) runs
    on a worker thread (the native loader releases the GIL and uses every host
    core) one sub-batch ahead of the device.  Yields (lo, per_file, BatchResult or
    None) in order."""
    from concurrent.futures import ThreadPoolExecutor

    from .api import run_arena

    chunk_files = max(1, int(chunk_files))
    bounds = [(lo, min(n_files, lo + chunk_files)) for lo in range(0, n_files, chunk_files)]
    if not bounds:
        return
    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(load, *bounds[0])
        for i, (lo, _hi) in enumerate(bounds):
            arena, per_file = fut.result()
            if i + 1 < len(bounds):
                fut = ex.submit(load, *bounds[i + 1])
            res = run_arena(arena, style, device) if arena.n_roots else None
            del arena
            yield lo, per_file, res
