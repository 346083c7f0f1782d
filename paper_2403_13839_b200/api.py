"""Public host API: the reference's `decompile_source(code, style=None) -> str`
surface (pipeline.py:143-160) as `decompile`, plus the batched
`decompile_many(codes, style=None) -> list[str | UnpyreError]`.

Host work is limited to packing CodeObjects into the arena image, one H2D copy,
the C-ABI call (decode kernel + decompile kernel on the current CUDA stream),
and reading back the flat text buffer.  Objects that hit a device capacity
limit (per-thread arena, output buffer) are re-run on device with larger
limits; nothing is ever computed on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _abi, _lib
from .arena import Arena, pack
from .errors import RETRYABLE, ST_OK, DeviceCapacityError, make_exception




def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_13839_b200 requires a CUDA device (sm_100a); none is visible")
    return torch


@dataclass
class BatchResult:
    status: np.ndarray      # int32 [n_roots]
    text_off: np.ndarray    # uint64
    text_len: np.ndarray    # uint32
    aux: np.ndarray         # int64 [n_roots, 2]
    text: np.ndarray        # flat UTF-8 buffer (uint8; a view of page-locked host memory)

    def item(self, i):
        s = self.text[int(self.text_off[i]):int(self.text_off[i]) + int(self.text_len[i])]
        return int(self.status[i]), bytes(s).decode("utf-8", "surrogatepass")

    def values(self):
        """One str (or exception instance) per root.  When the whole text buffer is
        ASCII (the usual case) it is decoded once and sliced by the byte offsets,
        instead of one decode per root."""
        tb = self.text.tobytes() if len(self.text) else b""
        if tb.isascii():
            whole = tb.decode("ascii")
            offs = self.text_off.tolist()
            lens = self.text_len.tolist()
            sts = self.status.tolist()
            out = [whole[o:o + n] for o, n in zip(offs, lens)]
            for i, st in enumerate(sts):
                if st != ST_OK:
                    out[i] = make_exception(st, out[i], self.aux[i])
            return out
        out = []
        for i in range(len(self.status)):
            st, s = self.item(i)
            out.append(s if st == ST_OK else make_exception(st, s, self.aux[i]))
        return out


class DeviceArena:
    """An arena resident in HBM plus the workspace/output buffers to decompile it.

    `run()` is stream-ordered and leaves every result on the device;
    `fetch()` copies them back.  Used by the API and by bench.py (which times
    `run()` on HBM-resident inputs and `upload()+run()+fetch()` end to end)."""

    def __init__(self, arena: Arena, style=None, device=None, text_cap=None, arena_bytes=0, slots=0,
                 threads_per_block=0, pinned=None, function_tree=False, output=0, schedule="input"):
        torch = _torch()
        self.torch = torch
        self.lib = _lib.load()
        self.arena = arena
        self.device = torch.device(device or "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        if pinned is None:
            pinned = getattr(arena, "pinned", None)  # image already page-locked (loader.load_pyc_batch)
        self.host = pinned if pinned is not None else torch.from_numpy(arena.blob).pin_memory()
        self.dev = torch.empty(self.host.numel(), dtype=torch.uint8, device=self.device)
        self.A = _abi.arena_struct(arena, self.dev.data_ptr())
        # schedule="cost": roots are taken largest code-object tree first (longest-
        # processing-time order: big objects do not start last and form the batch's
        # tail, and lanes of a warp get objects of similar size).  The order is
        # computed on the device from the uploaded arena at every run (cost_order)
        # and handed to the kernel as upy_options.order; results stay in input order.
        base_sched, _, mode = schedule.partition("+")
        if base_sched not in ("input", "cost", "similar", "shape", "dshape1", "dshape2", "dshape4") or \
                mode not in ("", "thread", "sync", "coemit", "split", "split3"):
            raise ValueError(f"schedule must be input|cost|similar|shape[+thread|+sync|+coemit|+split|+split3], "
                             f"not {schedule!r}")
        self.schedule = base_sched if arena.n_roots > 1 else "input"
        # kernel schedule (upy_options.schedule): 0 each thread takes the next root,
        # 1 warp-synchronous, 2 warp-synchronous with statement-parallel emission,
        # 3 split (a tree kernel, then an emit kernel, per chunk of positions).
        # Unspecified: statement-parallel emission for long objects (mean root tree of
        # COEMIT_MIN_BYTES of code or more: C4 +26%); for short ones the split
        # schedule (C3 +11%, C3-3.11 +10%: each kernel's code is one part of the
        # pipeline) when the batch is past the latency-mode size and free memory holds
        # arena slots for chunks of SPLIT_MIN_WAVES objects per resident thread (or all
        # roots), three kernels (split3) when the roots carry nested code, else per-thread.
        self.output = output
        if not mode:
            if mean_tree_code_bytes(arena) >= COEMIT_MIN_BYTES:
                mode = "coemit"
            elif output == 0 and not slots and not arena_bytes and self._split_fits(arena):
                # roots with nested code (modules, classes): validate + analyze in a
                # kernel of their own as well (C2x +10%; flat C3 objects: +0.3 / -0.8%)
                mode = "split3" if arena.n_objs > SPLIT3_MIN_OBJS_PER_ROOT * arena.n_roots else "split"
            else:
                mode = "thread"
        self.warp_sync = {"thread": 0, "sync": 1, "coemit": 2, "split": 3, "split3": 4}[mode]
        self.mode = mode
        if self.schedule in ("similar", "shape"):  # experiments: host-computed orders
            fn = root_similarity_order if self.schedule == "similar" else root_shape_order
            self._order = torch.from_numpy(fn(arena).astype(np.int32)).to(self.device)
        roots = arena.section("roots")
        self._trees_contiguous = bool(len(roots) < 2 or np.all(np.diff(roots.astype(np.int64)) > 0))
        if self.schedule not in ("similar", "shape"):
            self._order = None
        if not slots and not arena_bytes:
            slots = self._memory_slots(arena, split=self.warp_sync in (3, 4))
        self.opts = _abi.options(style, arena_bytes=arena_bytes, slots=slots,
                                 threads_per_block=threads_per_block, function_tree=1 if function_tree else 0,
                                 output=output, schedule=self.warp_sync)
        ws = C.c_size_t(0)
        with torch.cuda.device(self.device):  # sizing reads the device's SM count
            _lib.check(self.lib.upy_query_workspace(C.byref(self.A), C.byref(self.opts), C.byref(ws)),
                       "upy_query_workspace")
        self.ws_bytes = ws.value
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=self.device)
        n = max(arena.n_roots, 1)
        # source text is ~1.5-4.5x co_code; the CFG export lists every instruction (~12x)
        per_byte, per_root = (8, 512) if output == 0 else (32, 1024)
        cap = text_cap or max(1 << 16, per_byte * arena.code_bytes + per_root * arena.n_roots)
        self.text = torch.empty(cap, dtype=torch.uint8, device=self.device)
        # meta layout: [used u64 | pad][off u64 n][aux i64 2n][len u32 n][status i32 n]
        self.out = _abi.UpyOut()
        self.out.text = self.text.data_ptr()
        self.out.text_cap = cap
        self.meta = torch.zeros(64 + 32 * n, dtype=torch.uint8, device=self.device)
        m = self.meta.data_ptr()
        self.out.text_used = m
        self.out.text_off = m + 64
        self.out.aux = m + 64 + 8 * n
        self.out.text_len = m + 64 + 24 * n
        self.out.status = m + 64 + 28 * n
        self.n = arena.n_roots

    @property
    def schedule_spec(self):
        """The resolved schedule as a `schedule=` argument ("order+mode")."""
        return f"{self.schedule}+{self.mode}"

    def _split_fits(self, arena):
        sms = self.torch.cuda.get_device_properties(self.device).multi_processor_count
        if arena.n_roots <= sms * 32:  # the library's latency mode (upy.cu layout)
            return False
        slots = self._memory_slots(arena, split=True)
        # chunks of at least SPLIT_MIN_WAVES objects per resident thread (C5, 16M roots in
        # 26 chunks of 669K: +24% over per-thread), or all roots in one
        return slots == 0 or slots >= min(arena.n_roots, SPLIT_MIN_WAVES * sms * 1024)

    DECODE_KERNELS = ("upy_decode311_lane_kernel", "upy_decode_kernel")  # upy_decode_batch's two launches

    def kernel_names(self):
        """The kernels one run() launches (per chunk for the split schedule): the
        decode kernels, then the decompile kernels."""
        dec = list(self.DECODE_KERNELS)
        if self.output == 1:
            return dec + ["upy_cfgdot_kernel"]
        if self.warp_sync == 3:
            return dec + ["upy_tree_kernel", "upy_emit_kernel"]
        if self.warp_sync == 4:
            return dec + ["upy_analyze_kernel", "upy_structure_kernel", "upy_emit_kernel"]
        return dec + ["upy_decompile_kernel"]

    def _memory_slots(self, arena, split=False):
        """Concurrent per-thread arenas when the library's default 40 GB budget
        would bind (long objects: C4's ~3 MB slots allow only ~13K threads):
        size the slot count from the device's free memory instead (70% of it;
        the text buffer needs the rest).  0 = library
        default.  Measured on C4 (profiles/r02/bench_c4_slots_*.json): 12,288
        slots 2,726 objects/s, 24,576 2,965, 49,152 3,542."""
        full = self.torch.cuda.get_device_properties(self.device).multi_processor_count * 1024
        if split:
            # schedule 3: one arena slot per position of a chunk (upy.cu layout_split):
            # as many positions as 80% of free memory holds after the other buffers
            # (records, per-object decode results, per-thread scratch, text, meta)
            sb = split_slot_bytes(arena) + 256  # + its SplitState
            if (40 << 30) // sb >= arena.n_roots:
                # the library's default 40 GB budget holds every root: no device query
                # (cudaMemGetInfo waits behind other host threads' pinned allocations,
                # e.g. the .pyc loader's next sub-batch)
                return 0
            others = (12 * (arena.total_code_units + 1) + 24 * arena.n_objs + full * (68 << 10)
                      + 8 * arena.code_bytes + 544 * arena.n_roots + (64 << 20))
            free, _ = self.torch.cuda.mem_get_info(self.device)
            free += self.torch.cuda.memory_reserved(self.device) - self.torch.cuda.memory_allocated(self.device)
            return int(max(1, min(arena.n_roots, (int(free * 0.8) - others) // sb)))
        else:
            sb = default_slot_bytes(arena) + (68 << 10) + 256  # + the slot header (upy.cu SLOT_HEADER)
            want = min(arena.n_roots, full)
        if (40 << 30) // sb >= want:
            return 0
        free, _ = self.torch.cuda.mem_get_info(self.device)
        # blocks torch's caching allocator holds but no tensor uses are free to us too
        free += self.torch.cuda.memory_reserved(self.device) - self.torch.cuda.memory_allocated(self.device)
        return int(max(1, min(want, int(free * 0.7) // sb)))

    def upload(self, stream=None):
        with self.torch.cuda.device(self.device):
            self.dev.copy_(self.host, non_blocking=True)

    def run(self, stream=None, mode="full"):
        """mode: "full" (decode + decompile), "decode" (decode kernel only) or
        "structure" (decompile kernel on the records of a previous "decode")."""
        torch = self.torch
        s = stream or torch.cuda.current_stream(self.device)
        self.opts.decode_only = 1 if mode == "decode" else 0
        self.opts.skip_decode = 1 if mode == "structure" else 0
        with torch.cuda.device(self.device):  # the C ABI launches on the current device
            if mode != "decode":
                self.meta[:8].zero_()
                if self.schedule == "cost":
                    with torch.cuda.stream(s):
                        self._order = cost_order(self.dev, self.arena.offsets, self.arena.counts,
                                                 self._trees_contiguous)
                elif self.schedule.startswith("dshape"):  # experiment: device opcode-shape order
                    with torch.cuda.stream(s):
                        self._order = shape_order(self.dev, self.arena.offsets, self.arena.counts,
                                                  int(self.schedule[6:]))
                self.opts.order = self._order.data_ptr() if self._order is not None else None
                self.opts.schedule = self.warp_sync
            rc = self.lib.upy_decompile_batch(C.byref(self.A), C.byref(self.opts), C.byref(self.out),
                                              C.c_void_p(self.ws.data_ptr()), C.c_size_t(self.ws_bytes),
                                              C.c_void_p(s.cuda_stream))
        _lib.check(rc, "upy_decompile_batch")

    def stackscan(self, stream=None):
        """Stack-depth scan (csrc/stackscan_kernel.cu) over the
        records of the last decode on this workspace.  Returns device tensors
        (records: int32 view of upy_stackrec per code unit slot, info: upy_stackinfo
        bytes per object); stream-ordered."""
        from .arena import DECODED_DTYPE, INS_DTYPE

        torch = self.torch
        s = stream or torch.cuda.current_stream(self.device)
        units = self.arena.total_code_units + 1
        if getattr(self, "_stack", None) is None:
            self._stack = torch.empty(4 * units, dtype=torch.uint8, device=self.device)
            self._stack_info = torch.empty(24 * max(self.arena.n_objs, 1), dtype=torch.uint8, device=self.device)
        ws = self.ws.data_ptr()
        dec_off = (units * INS_DTYPE.itemsize + 255) & ~255
        assert DECODED_DTYPE.itemsize == 24
        with torch.cuda.device(self.device):
            rc = self.lib.upy_stackscan_batch(C.byref(self.A), C.c_void_p(ws), C.c_void_p(ws + dec_off),
                                              C.c_void_p(self._stack.data_ptr()),
                                              C.c_void_p(self._stack_info.data_ptr()), C.c_void_p(s.cuda_stream))
        _lib.check(rc, "upy_stackscan_batch")
        return self._stack, self._stack_info

    def decoded(self):
        """Per-object decode results (upy_decoded: status, n_instrs, aux) of the
        last decode on this workspace (layout: upy.cu WsLayout)."""
        from .arena import DECODED_DTYPE, INS_DTYPE

        units = self.arena.total_code_units + 1
        off = (units * INS_DTYPE.itemsize + 255) & ~255
        n = DECODED_DTYPE.itemsize * self.arena.n_objs
        return self.ws[off:off + n].cpu().numpy().view(DECODED_DTYPE)

    def fetch(self) -> BatchResult:
        n = self.n
        meta = self.meta.cpu().numpy()
        used = int(meta[:8].view(np.uint64)[0])
        used = min(used, self.out.text_cap)
        off = meta[64:64 + 8 * n].view(np.uint64).copy()
        aux = meta[64 + 8 * n:64 + 24 * n].view(np.int64).reshape(n, 2).copy()
        ln = meta[64 + 24 * n:64 + 28 * n].view(np.uint32).copy()
        st = meta[64 + 28 * n:64 + 32 * n].view(np.int32).copy()
        if used:
            # page-locked destination (torch's caching host allocator reuses it across
            # calls): a direct DMA instead of a pageable copy plus a bytes() copy
            host = self.torch.empty(used, dtype=self.torch.uint8, pin_memory=True)
            host.copy_(self.text[:used])
            text = host.numpy()
        else:
            text = np.zeros(0, dtype=np.uint8)
        return BatchResult(st, off, ln, aux, text)


COEMIT_MIN_BYTES = 4096
SPLIT_MIN_WAVES = 4
SPLIT3_MIN_OBJS_PER_ROOT = 1.25


def mean_tree_code_bytes(arena: Arena) -> float:
    """Mean code bytes per root tree (all objects over the roots)."""
    return float(arena.code_bytes) / max(1, arena.n_roots)


def cost_order(blob, offsets, counts, trees_contiguous):
    """Largest-tree-first order of the root positions (int32 tensor on blob's
    device), from the arena image itself: a root's cost is the code bytes of its
    tree -- the run of objects from the root to the next root when the roots are
    in packing order (pack / tile lay each tree out contiguously), else the root's
    own code length.  Stable, so equal costs keep input order."""
    import torch

    from .arena import OBJ_DTYPE

    n_objs, n_roots = int(counts["objs"]), int(counts["roots"])
    o0, r0 = int(offsets["objs"]), int(offsets["roots"])
    rec = OBJ_DTYPE.itemsize
    cl_at = OBJ_DTYPE.fields["code_len"][1]
    objs = blob[o0:o0 + n_objs * rec].view(n_objs, rec)
    lens = objs[:, cl_at:cl_at + 4].contiguous().view(torch.int32).view(-1).to(torch.int64)
    roots = blob[r0:r0 + 4 * n_roots].view(torch.int32).to(torch.int64)
    if trees_contiguous:
        csum = torch.zeros(n_objs + 1, dtype=torch.int64, device=blob.device)
        csum[1:] = torch.cumsum(lens, 0)
        ends = torch.cat([roots[1:], torch.full((1,), n_objs, dtype=torch.int64, device=blob.device)])
        cost = csum[ends] - csum[roots]
    else:
        cost = lens[roots]
    return torch.sort(cost, descending=True, stable=True).indices.to(torch.int32)


def root_shape_order(arena: Arena, prefix=64):
    """Experiment: root positions sorted by their first `prefix` OPCODES (args
    ignored), so neighbouring roots share the longest possible run of identical
    control flow through the transfer functions (profiles/r02/schedule/)."""
    objs = arena.section("objs")
    roots = arena.section("roots").astype(np.int64)
    offs = objs["code_off"].astype(np.int64)[roots]
    lens = objs["code_len"].astype(np.int64)[roots]
    by = arena.section("bytes")
    j = np.arange(prefix, dtype=np.int64)
    idx = np.minimum(offs[:, None] + 2 * j[None, :], len(by) - 1)
    pre = np.where(2 * j[None, :] < lens[:, None], by[idx], 0).astype(np.uint8)
    words = pre.reshape(len(roots), prefix // 8, 8)
    keys = [lens]
    for w in range(prefix // 8 - 1, -1, -1):
        keys.append(words[:, w, :].copy().view(">u8").ravel())
    return np.lexsort(keys)


def root_similarity_order(arena: Arena, prefix=32):
    """Experiment: root positions sorted by the first `prefix` bytes of their
    co_code (then by length), so neighbouring roots start with the same
    instructions (profiles/r02/schedule/)."""
    objs = arena.section("objs")
    roots = arena.section("roots").astype(np.int64)
    offs = objs["code_off"].astype(np.int64)[roots]
    lens = objs["code_len"].astype(np.int64)[roots]
    by = arena.section("bytes")
    j = np.arange(prefix, dtype=np.int64)
    idx = np.minimum(offs[:, None] + j[None, :], len(by) - 1)
    pre = np.where(j[None, :] < lens[:, None], by[idx], 0).astype(np.uint8)
    words = pre.reshape(len(roots), prefix // 8, 8)
    keys = [lens]
    for w in range(prefix // 8 - 1, -1, -1):  # lexsort: last key is primary
        keys.append(words[:, w, :].copy().view(">u8").ravel())
    return np.lexsort(keys)


def shape_order(blob, offsets, counts, n_words):
    """Device form of the opcode-shape order: roots sorted by their first
    8 * n_words opcodes (args ignored), most significant first, via n_words chained
    stable sorts of 64-bit keys (int32 tensor on blob's device)."""
    import torch

    from .arena import OBJ_DTYPE

    n_objs, n_roots = int(counts["objs"]), int(counts["roots"])
    o0, r0, b0 = int(offsets["objs"]), int(offsets["roots"]), int(offsets["bytes"])
    n_bytes = int(counts["bytes"])
    rec = OBJ_DTYPE.itemsize
    co_at = OBJ_DTYPE.fields["code_off"][1]
    cl_at = OBJ_DTYPE.fields["code_len"][1]
    objs = blob[o0:o0 + n_objs * rec].view(n_objs, rec)
    roots = blob[r0:r0 + 4 * n_roots].view(torch.int32).to(torch.int64)
    code_off = objs[:, co_at:co_at + 8].contiguous().view(torch.int64).view(-1)[roots]
    code_len = objs[:, cl_at:cl_at + 4].contiguous().view(torch.int32).view(-1).to(torch.int64)[roots]
    by = blob[b0:b0 + n_bytes]
    j = torch.arange(8 * n_words, device=blob.device, dtype=torch.int64)
    idx = (code_off[:, None] + 2 * j[None, :]).clamp_(max=max(n_bytes - 1, 0))
    ops = torch.where(2 * j[None, :] < code_len[:, None], by[idx], torch.zeros((), dtype=torch.uint8,
                                                                                     device=blob.device))
    perm = torch.arange(n_roots, device=blob.device)
    weights = (256 ** torch.arange(7, -1, -1, device=blob.device, dtype=torch.int64))
    for w in range(n_words - 1, -1, -1):  # least significant word first (stable)
        word = ops[:, 8 * w:8 * w + 8].to(torch.int64)
        # big-endian 8 bytes as a signed 64-bit key, top byte offset by -128 so the
        # signed order is the unsigned (lexicographic) one
        key = (word[:, 0] - 128) * weights[0] + (word[:, 1:] * weights[1:]).sum(1)
        k = key[perm]
        perm = perm[torch.sort(k, stable=True).indices]
    return perm.to(torch.int32)


def root_cost_order(arena: Arena):
    """Host (numpy) restatement of cost_order, for tests."""
    objs = arena.section("objs")
    roots = arena.section("roots").astype(np.int64)
    lens = objs["code_len"].astype(np.int64)
    if len(roots) < 2 or np.all(np.diff(roots) > 0):
        csum = np.concatenate([[0], np.cumsum(lens)])
        ends = np.concatenate([roots[1:], [len(lens)]])
        cost = csum[ends] - csum[roots]
    else:
        cost = lens[roots]
    return np.argsort(-cost, kind="stable")


def default_slot_bytes(arena: Arena) -> int:
    """The per-thread arena size upy_query_workspace picks (upy.cu layout())."""
    return (64 << 10) + 160 * arena.max_code_len


def split_slot_bytes(arena: Arena) -> int:
    """The per-position arena size of the split schedule (upy.cu layout_split())."""
    return ((32 << 10) + 16 * arena.max_code_len + 255) & ~255


def tree_sizes(arena: Arena, roots) -> tuple:
    """(code bytes, str/bytes constant payload bytes) of the code-object trees
    under the given root positions (roots and every nested code constant)."""
    from .arena import KIND_ID

    objs = arena.section("objs")
    consts = arena.section("consts")
    refs = arena.section("refs")
    root_obj = arena.section("roots")
    seen = set()
    stack = [int(root_obj[i]) for i in roots]
    code = payload = 0
    while stack:
        o = stack.pop()
        if o in seen:
            continue
        seen.add(o)
        r = objs[o]
        code += int(r["code_len"])
        todo = [int(c) for c in refs[int(r["consts_off"]):int(r["consts_off"]) + int(r["n_consts"])]]
        while todo:
            c = consts[todo.pop()]
            k = int(c["kind"])
            if k == KIND_ID["code"]:
                stack.append(int(c["off"]))
            elif k in (KIND_ID["str"], KIND_ID["bytes"]):
                payload += int(c["n"])
            elif k in (KIND_ID["tuple"], KIND_ID["frozenset"]):
                todo.extend(int(x) for x in refs[int(c["off"]):int(c["off"]) + int(c["n"])])
    return code, payload


DEFAULT_SCHEDULE = os.environ.get("UPY_SCHEDULE", "cost")


def run_arena(arena: Arena, style=None, device=None, retries=3, function_tree=False, output=0,
              schedule=None, first_arena_bytes=0, first_text_cap=None) -> BatchResult:
    """Decompile every root of a packed arena on the GPU.

    Roots that hit a device capacity limit (per-thread arena, output buffer) are
    re-run on the device with 4x larger limits per attempt, sized from the
    retried roots' own trees and capped by the device's free memory.  output=1
    writes each root's CFG export (to_dot, csrc/dot.h) instead of its source.
    first_arena_bytes / first_text_cap override the first attempt's capacities
    (tests use them to drive the retry path)."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    with torch.cuda.device(dev):
        da = DeviceArena(arena, style, dev, function_tree=function_tree, output=output,
                         schedule=schedule or DEFAULT_SCHEDULE, arena_bytes=first_arena_bytes,
                         text_cap=first_text_cap)
        da.upload()
        da.run()
        res = da.fetch()
        del da
        slot = default_slot_bytes(arena)
        for attempt in range(1, retries + 1):
            redo = np.nonzero(np.isin(res.status, RETRYABLE))[0]
            if not len(redo):
                break
            scale = 4 ** attempt
            slot_bytes = slot * scale
            code, payload = tree_sizes(arena, redo)
            text_cap = scale * (8 * code + 2 * payload + 512 * len(redo)) + (1 << 16)
            free, _ = torch.cuda.mem_get_info(dev)
            budget = max(0, int(free * 0.6) - text_cap - 2 * len(arena.blob))
            slots = int(min(len(redo), 4096, budget // slot_bytes))
            if slots < 1:
                break  # not even one slot fits: the statuses stay (DeviceCapacityError)
            sub = _subset(arena, redo)
            db = DeviceArena(sub, style, dev, text_cap=text_cap, arena_bytes=slot_bytes, slots=slots,
                             function_tree=function_tree, output=output)
            db.upload()
            db.run()
            r2 = db.fetch()
            del db
            # splice retried results back
            base = len(res.text)
            res.text = np.concatenate([res.text, r2.text])
            for j, i in enumerate(redo):
                res.status[i] = r2.status[j]
                res.text_off[i] = base + int(r2.text_off[j])
                res.text_len[i] = r2.text_len[j]
                res.aux[i] = r2.aux[j]
    return res


def _subset(arena: Arena, idx) -> Arena:
    """Same objects, roots restricted to positions `idx` (a new roots section)."""
    from .arena import with_roots

    return with_roots(arena, arena.section("roots")[idx])


def decompile_many(codes, style=None, device=None, devices=None, function_tree=False):
    """Batched decompile_source: one entry per input, text or the exception
    instance the reference would raise (the batch keeps going, like the CLI).

    `devices` (e.g. ["cuda:0", "cuda:1"]) shards the batch: contiguous root
    ranges balanced by code bytes (shard.shard_bounds), one packed arena and
    one host thread per device, results gathered back in input order.  There
    is no cross-device traffic: every root (with its nested codes) is
    decompiled on one device.  function_tree=True renders each input as
    emit_module([function_tree(code)]) without validation (the reference CLI's
    --function path, cli.py:75-78) instead of decompile_source."""
    codes = list(codes)
    if not codes:
        return []
    if devices is not None and len(devices) > 1:
        return _decompile_sharded(codes, style, list(devices), function_tree)
    if devices:
        device = devices[0]
    res = run_arena(pack(codes), style, device, function_tree=function_tree)
    return _values(res)


def _values(res):
    out = res.values()
    for v in out:
        if isinstance(v, DeviceCapacityError):
            raise v
    return out


def shard_plan(codes, n_devices):
    """Contiguous [lo, hi) ranges of `codes` per device, balanced by the code
    bytes of each root's tree (the decompile cost grows with it)."""
    from .shard import shard_bounds

    def tree_code(co, seen):
        if id(co) in seen:
            return 0
        seen.add(id(co))
        n = len(co.code)
        todo = list(co.consts)
        while todo:
            c = todo.pop()
            if c.kind == "code":
                n += tree_code(c.value, seen)
            elif c.kind in ("tuple", "frozenset"):
                todo.extend(c.value)
        return n

    return shard_bounds([tree_code(co, set()) for co in codes], n_devices)


def _decompile_sharded(codes, style, devices, function_tree=False):
    from concurrent.futures import ThreadPoolExecutor

    plan = shard_plan(codes, len(devices))

    def work(k):
        lo, hi = plan[k]
        if lo == hi:
            return []
        return _values(run_arena(pack(codes[lo:hi]), style, devices[k], function_tree=function_tree))

    with ThreadPoolExecutor(len(devices)) as ex:
        parts = list(ex.map(work, range(len(devices))))
    return [v for part in parts for v in part]


def _value(triple):
    st, text, aux = triple
    if st == ST_OK:
        return text
    v = make_exception(st, text, aux)
    if isinstance(v, DeviceCapacityError):
        raise v
    return v


def decompile_many_distributed(codes, style=None, gather=True, device=None, backend=None):
    """Multi-process form of decompile_many (one process per GPU, under
    torch.distributed): every rank passes the same `codes`; rank r decompiles
    the contiguous shard shard_plan(codes, world)[r] on its own device, with no
    communication.  gather=True then all-gathers the per-root (status, text,
    aux) triples so every rank returns the full list in input order (the
    optional final gather of SURVEY §8e); gather=False returns (lo, hi,
    values of the rank's own shard).  `backend(codes, style) -> [(status,
    text, aux)]` replaces the device run (tests use the host build)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = shard_plan(codes, world)[rank]
    if hi == lo:
        triples = []
    elif backend is not None:
        triples = backend(codes[lo:hi], style)
    else:
        res = run_arena(pack(codes[lo:hi]), style, device)
        triples = [(*res.item(i), (int(res.aux[i][0]), int(res.aux[i][1]))) for i in range(len(res.status))]
    if not gather:
        return lo, hi, [_value(t) for t in triples]
    parts = [None] * world
    dist.all_gather_object(parts, triples)
    return [_value(t) for part in parts for t in part]


def decompile(code, style=None, device=None) -> str:
    """Drop-in for unpyre.decompile_source(code, style) (pipeline.py:143)."""
    v = decompile_many([code], style, device)[0]
    if isinstance(v, BaseException):
        raise v
    return v


decompile_source = decompile
