"""B200-native batched decompiler for CPython 3.8-3.11 code objects.

Drop-in for the reference's hot path `unpyre.decompile_source(code, style)`
(/root/reference/pkg/src/unpyre/pipeline.py:143-160): `decompile` has the same
signature, text and exception classes; `decompile_many` batches any number of
code objects into one device arena.  `load_pyc` / `decompile_pyc_many` read
.pyc images natively (pyc.py:36-352) straight into that arena.
"""
from .errors import (BadJumpTarget, InternalMarkerLeak, MalformedExceptionTable, MalformedMarshal,
                     StackDepthMismatch, StackUnderflow, StructuringFailed, TruncatedCode, TruncatedHeader,
                     UnknownMagic, UnknownOpcode, UnpyreError, UnsupportedOpcode, UnsupportedVersion)
from .model import CodeObject, Const, EmitStyle, VersionTag, flatten_nested_codes

__all__ = [
    "BadJumpTarget", "CodeObject", "Const", "EmitStyle", "InternalMarkerLeak", "MalformedExceptionTable",
    "MalformedMarshal", "StackDepthMismatch", "StackUnderflow", "StructuringFailed", "TruncatedCode",
    "TruncatedHeader", "UnknownMagic", "UnknownOpcode", "UnpyreError", "UnsupportedOpcode",
    "UnsupportedVersion", "VersionTag", "decompile", "decompile_many", "decompile_source",
    "decompile_pyc_many", "flatten_nested_codes", "load_pyc", "load_pyc_batch",
]
__version__ = "0.1.0"


def __getattr__(name):
    # the API module needs torch + the CUDA library; import it lazily so the
    # model / packer can be used (and tested) without a GPU
    if name in ("decompile", "decompile_many", "decompile_source", "run_arena", "DeviceArena"):
        from . import api

        return getattr(api, name)
    if name in ("load_pyc", "load_pyc_batch", "decompile_pyc_many"):
        from . import loader

        return getattr(loader, name)
    raise AttributeError(name)
