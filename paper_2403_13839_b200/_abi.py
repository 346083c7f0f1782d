"""ctypes mirror of include/upy.h (the C ABI).  Layouts are checked against
upy_abi_sizeof() when a library is loaded."""
from __future__ import annotations

import ctypes as C

c_u8p = C.POINTER(C.c_uint8)


class UpyArena(C.Structure):
    _fields_ = [
        ("objs", C.c_void_p), ("n_objs", C.c_int64),
        ("consts", C.c_void_p), ("n_consts", C.c_int64),
        ("strs", C.c_void_p), ("n_strs", C.c_int64),
        ("refs", C.c_void_p), ("n_refs", C.c_int64),
        ("limbs", C.c_void_p), ("n_limbs", C.c_int64),
        ("bytes", C.c_void_p), ("n_bytes", C.c_int64),
        ("roots", C.c_void_p), ("n_roots", C.c_int64),
        ("max_code_len", C.c_uint64),
        ("total_code_units", C.c_uint64),
    ]


class UpyOptions(C.Structure):
    _fields_ = [
        ("indent", C.c_char_p), ("indent_len", C.c_uint64),
        ("tool", C.c_char_p), ("tool_len", C.c_uint64),
        ("header", C.c_int32),
        ("threads_per_block", C.c_int32),
        ("slots", C.c_int32),
        ("decode_only", C.c_int32),
        ("arena_bytes", C.c_uint64),
        ("skip_decode", C.c_int32),
        ("schedule", C.c_int32),
        ("max_depth", C.c_int32),
        ("function_tree", C.c_int32),
        ("output", C.c_int32),
        ("pad0", C.c_int32),
        ("order", C.c_void_p),
    ]


class UpyOut(C.Structure):
    _fields_ = [
        ("text", C.c_void_p), ("text_cap", C.c_uint64),
        ("text_used", C.c_void_p),
        ("text_off", C.c_void_p),
        ("text_len", C.c_void_p),
        ("status", C.c_void_p),
        ("aux", C.c_void_p),
    ]


class UpyPycBatch(C.Structure):
    _fields_ = [
        ("image", C.c_void_p), ("image_bytes", C.c_uint64),
        ("section_off", C.c_uint64 * 7), ("section_count", C.c_int64 * 7),
        ("max_code_len", C.c_uint64), ("total_code_units", C.c_uint64),
        ("n_files", C.c_int64),
        ("file_status", C.POINTER(C.c_int32)),
        ("file_root", C.POINTER(C.c_int32)),
        ("file_aux", C.POINTER(C.c_int64)),
        ("messages", C.c_void_p),
        ("msg_off", C.POINTER(C.c_uint64)),
        ("msg_len", C.POINTER(C.c_uint32)),
    ]


SIZES = {0: 152, 1: 40, 2: 16, 3: C.sizeof(UpyArena), 4: C.sizeof(UpyOptions), 5: C.sizeof(UpyOut),
         6: 12, 7: 24, 8: 4, 9: 24}

# symbols declared by include/upy.h
EXPORTS = ("upy_abi_sizeof", "upy_abi_version", "upy_query_workspace", "upy_decompile_batch",
           "upy_decode_batch", "upy_stackscan_batch", "upy_last_error", "upy_launch_count", "upy_pyc_load", "upy_pyc_write_image", "upy_pyc_free")
PYC_DEFER_IMAGE = 1


def arena_struct(arena, base_ptr: int) -> UpyArena:
    """UpyArena whose pointers address `arena`'s sections at base_ptr (host or device)."""
    a = UpyArena()
    for name, cnt in (("objs", "objs"), ("consts", "consts"), ("strs", "strs"), ("refs", "refs"),
                      ("limbs", "limbs"), ("bytes", "bytes"), ("roots", "roots")):
        setattr(a, name, base_ptr + arena.offsets[name])
        setattr(a, "n_" + name, arena.counts[cnt])
    a.max_code_len = arena.max_code_len
    a.total_code_units = arena.total_code_units
    return a


def options(style=None, **kw) -> UpyOptions:
    """upy_options for an EmitStyle (any indent / tool length; the encoded
    strings are kept alive on the returned struct)."""
    o = UpyOptions()
    indent = "    " if style is None else style.indent
    tool = "unpyre" if style is None else style.tool
    o._keep = (indent.encode("utf-8", "surrogatepass"), tool.encode("utf-8", "surrogatepass"))
    o.indent, o.indent_len = o._keep[0], len(o._keep[0])
    o.tool, o.tool_len = o._keep[1], len(o._keep[1])
    o.header = 1 if (style is not None and style.header) else 0
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def check_layout(lib):
    lib.upy_abi_sizeof.restype = C.c_size_t
    lib.upy_abi_sizeof.argtypes = [C.c_int]
    for k, v in SIZES.items():
        got = lib.upy_abi_sizeof(k)
        if got != v:
            raise RuntimeError(f"ABI layout mismatch for struct #{k}: library {got}, binding {v}")
