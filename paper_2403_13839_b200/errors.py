"""Error hierarchy of the decompile path, mirroring the reference's class names
one to one so callers can `except` the same types.

Reference: /root/reference/pkg/src/unpyre/errors.py:8-102.  The device reports a
status code per object plus a message it formatted itself; `make_exception`
turns that into the matching exception instance (attributes from the aux
words the kernel wrote).

Drop-in interop: when the reference package (`unpyre`) is importable, the
classes below are REPLACED by the reference's own class objects (`bind`), so
`except unpyre.UnpyreError` around `decompile(...)` -- e.g. the reference CLI's
`cmd_decompile` (cli.py:82) with this package patched in -- catches exactly
what it catches around `unpyre.decompile_source`.  Without the reference the
package's own mirror hierarchy is used.
"""


class UnpyreError(Exception):
    """Base class for all decompiler errors (errors.py:8)."""


class UnsupportedVersion(UnpyreError):
    def __init__(self, major, minor):
        super().__init__(f"unsupported Python version {major}.{minor} (supported: 3.8-3.11)")
        self.major = major
        self.minor = minor


# ---------------------------------------------------------------- loaders (errors.py:19-34)

class UnknownMagic(UnpyreError):
    def __init__(self, magic):
        super().__init__(f"unknown pyc magic {magic:#06x} (unsupported interpreter version)")
        self.magic = magic


class TruncatedHeader(UnpyreError):
    pass


class MalformedMarshal(UnpyreError):
    def __init__(self, message, offset):
        super().__init__(f"{message} (at byte offset {offset})")
        self.offset = offset


class SchemaError(UnpyreError):
    """JSON code-object dump does not match the schema (errors.py:37-40)."""

    def __init__(self, message, path):
        super().__init__(f"{message} (at {path})")
        self.path = path


class UnknownOpcode(UnpyreError):
    def __init__(self, opcode, offset):
        super().__init__(f"unknown opcode {opcode} at offset {offset}")
        self.opcode = opcode
        self.offset = offset


class TruncatedCode(UnpyreError):
    pass


class BadJumpTarget(UnpyreError):
    def __init__(self, offset, target):
        super().__init__(f"jump at offset {offset} targets {target}, not an instruction boundary")
        self.offset = offset
        self.target = target


class MalformedExceptionTable(UnpyreError):
    pass


class StackUnderflow(UnpyreError):
    def __init__(self, offset, opname=""):
        super().__init__(f"evaluation stack underflow at offset {offset}" + (f" ({opname})" if opname else ""))
        self.offset = offset


class UnsupportedOpcode(UnpyreError):
    def __init__(self, opname, offset):
        super().__init__(f"no lifting rule for {opname} at offset {offset}")
        self.opname = opname
        self.offset = offset


class StackDepthMismatch(UnpyreError):
    def __init__(self, block_id, depths):
        super().__init__(f"predecessors of block {block_id} disagree on stack depth: {depths}")
        self.block_id = block_id


class StructuringFailed(UnpyreError):
    def __init__(self, block_id, reason):
        super().__init__(f"cannot structure region at block {block_id}: {reason}")
        self.block_id = block_id
        self.reason = reason


class InternalMarkerLeak(UnpyreError):
    """A control-flow marker survived structuring."""


class DeviceCapacityError(RuntimeError):
    """A device-side capacity limit (arena, recursion guard) was hit even after
    the host's retry with a larger arena.  Not a reference error class."""


# status codes written by the device (keep in sync with include/upy.h)
ST_OK = 0
ST_UNPYRE = 1
ST_UNKNOWN_OPCODE = 2
ST_TRUNCATED_CODE = 3
ST_BAD_JUMP_TARGET = 4
ST_MALFORMED_EXCTABLE = 5
ST_STACK_UNDERFLOW = 6
ST_UNSUPPORTED_OPCODE = 7
ST_STACK_DEPTH_MISMATCH = 8
ST_STRUCTURING_FAILED = 9
ST_MARKER_LEAK = 10
ST_UNKNOWN_MAGIC = 11
ST_TRUNCATED_HEADER = 12
ST_MALFORMED_MARSHAL = 13
ST_PY_INDEX_ERROR = 20
ST_PY_ATTRIBUTE_ERROR = 21
ST_PY_TYPE_ERROR = 22
ST_PY_KEY_ERROR = 23
ST_PY_VALUE_ERROR = 24
ST_PY_RECURSION_ERROR = 25
ST_ARENA_OVERFLOW = 30
ST_OUTPUT_OVERFLOW = 31
ST_DEPTH_LIMIT = 32
ST_INTERNAL = 33
ST_NOT_RUN = 34

# capacity statuses the host re-runs with larger limits (ST_DEPTH_LIMIT is the
# device's recursion guard, sized to the kernel stack: a retry cannot pass it)
RETRYABLE = (ST_ARENA_OVERFLOW, ST_OUTPUT_OVERFLOW)


def _bare(cls, message):
    e = cls.__new__(cls)
    Exception.__init__(e, message)
    return e


def make_exception(status, message, aux):
    """Exception instance for a device status (message formatted on device)."""
    a0, a1 = int(aux[0]), int(aux[1])
    if status == ST_UNPYRE:
        return UnpyreError(message)
    if status == ST_UNKNOWN_OPCODE:
        e = _bare(UnknownOpcode, message)
        e.opcode, e.offset = a0, a1
        return e
    if status == ST_TRUNCATED_CODE:
        return TruncatedCode(message)
    if status == ST_BAD_JUMP_TARGET:
        e = _bare(BadJumpTarget, message)
        e.offset, e.target = a0, a1
        return e
    if status == ST_MALFORMED_EXCTABLE:
        return MalformedExceptionTable(message)
    if status == ST_STACK_UNDERFLOW:
        e = _bare(StackUnderflow, message)
        e.offset = a0
        return e
    if status == ST_UNSUPPORTED_OPCODE:
        e = _bare(UnsupportedOpcode, message)
        e.offset = a0
        e.opname = message[len("no lifting rule for "):message.rfind(" at offset ")]
        return e
    if status == ST_STACK_DEPTH_MISMATCH:
        e = _bare(StackDepthMismatch, message)
        e.block_id = a0
        return e
    if status == ST_STRUCTURING_FAILED:
        e = _bare(StructuringFailed, message)
        e.block_id = a0
        e.reason = message.split(": ", 1)[1] if ": " in message else ""
        return e
    if status == ST_MARKER_LEAK:
        return InternalMarkerLeak(message)
    if status == ST_UNKNOWN_MAGIC:
        e = _bare(UnknownMagic, message)
        e.magic = a0
        return e
    if status == ST_TRUNCATED_HEADER:
        return TruncatedHeader(message)
    if status == ST_MALFORMED_MARSHAL:
        e = _bare(MalformedMarshal, message)
        e.offset = a0
        return e
    py = {
        ST_PY_INDEX_ERROR: IndexError,
        ST_PY_ATTRIBUTE_ERROR: AttributeError,
        ST_PY_TYPE_ERROR: TypeError,
        ST_PY_KEY_ERROR: KeyError,
        ST_PY_VALUE_ERROR: ValueError,
        ST_PY_RECURSION_ERROR: RecursionError,
    }.get(status)
    if py is KeyError:
        # the device formats the missing key as repr(key); KeyError(key) has str == repr(key)
        try:
            return KeyError(int(message))
        except ValueError:
            return KeyError(message)
    if py is not None:
        return py(message)
    return DeviceCapacityError(f"device status {status}: {message}")


# ---------------------------------------------------------------- interop
CLASS_NAMES = ("UnpyreError", "UnsupportedVersion", "UnknownMagic", "TruncatedHeader", "MalformedMarshal",
               "SchemaError", "UnknownOpcode", "TruncatedCode", "BadJumpTarget", "MalformedExceptionTable",
               "StackUnderflow", "UnsupportedOpcode", "StackDepthMismatch", "StructuringFailed",
               "InternalMarkerLeak")
_OWN = {n: globals()[n] for n in CLASS_NAMES}


def bind(module=None):
    """Use `module`'s exception classes (the reference's `unpyre.errors`, or any
    module defining the same names) for every exception this package raises;
    `bind(None)` restores the package's own hierarchy.  Returns the module bound."""
    import sys

    g = globals()
    for n in CLASS_NAMES:
        cls = getattr(module, n, None) if module is not None else None
        g[n] = cls if cls is not None else _OWN[n]
    pkg = sys.modules.get(__package__)
    if pkg is not None:  # the package re-exports the classes
        for n in CLASS_NAMES:
            if hasattr(pkg, n):
                setattr(pkg, n, g[n])
    return module


def bound():
    """True when the reference's classes are in use."""
    return UnpyreError is not _OWN["UnpyreError"]


def _auto_bind():
    import importlib
    import os

    if os.environ.get("UPY_BIND_REFERENCE_ERRORS", "1") == "0":
        return
    try:
        ref = importlib.import_module("unpyre.errors")
    except ImportError:
        return
    bind(ref)


_auto_bind()
