"""Benchmark: code objects decompiled/sec (bit-exact source) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c4|c3_311] [--objects M]
    python bench.py --impl reference ...      # the reference algorithm on host cores

A step decompiles the whole corpus once: decode kernel (co_code -> instruction
records) then decompile kernel (validate/analyze/structure/recover/emit) into
one flat UTF-8 buffer.  The corpus is a pool of distinct seeded synthetic
objects (bench_pools.py) tiled to --objects per GPU (weak scaling); after the
timed region EVERY output is checked against the reference's SHA-256 digests
(tests/golden/pools.json).  `value` is timed with inputs resident in HBM;
`e2e` adds the H2D copy of the packed arena from pinned memory and the D2H of
statuses + text each step.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "code objects decompiled/sec (bit-exact source), bytecode GB/s vs HBM roofline"
WORKLOADS = {
    "c3": ("c3_310", 1_000_000, "C3: synthetic 1M code objects x ~200 units (3.10), straight-line"),
    "c3_311": ("c3_311", 1_000_000, "C3 (3.11 variant): synthetic 1M code objects x ~200 units + caches"),
    "c4": ("c4_310", 65_536, "C4: synthetic 64K code objects x ~10K units (3.10), nested if/for/while/try"),
    "c4_311": ("c4_311", 65_536, "C4 (3.11 variant): synthetic 64K code objects x ~10K units, exception tables"),
    # C2 (BASELINE configs[1]): the reference's own syntax corpus, one batch of its 110
    # modules (nested defs/classes/lambdas/comprehensions decompiled through their roots)
    "c2": ("c2_310", 110, "C2: the reference's pkg/corpus, 110 modules (+nested code, 3.10) in one batch"),
    "c2x": ("c2_310", 110 * 4096, "C2 x4096: the reference's pkg/corpus modules (3.10) tiled to 450,560 roots"),
    "c2_311": ("c2_311", 110, "C2 (3.11): the reference's pkg/corpus, 110 modules (+nested code) in one batch"),
    # C5: one 16M-object corpus split across the ranks (strong scaling)
    "c5": ("c3_310", 16_777_216, "C5: synthetic 16M code objects x ~200 units (3.10) sharded by object across GPUs"),
}


def measured_traffic(workload, kernel):
    """DRAM bytes (read + write) per launch of `kernel` on `workload`, from the
    committed ncu capture of the same bench command (profiles/traffic.json, made by
    tools/traffic_json.py from `ncu --metrics dram__bytes_read.sum,...`); None when
    this configuration was not captured."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(workload, {}).get(kernel)
    return None if v is None else float(v["bytes_per_launch"])


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(arena, text_len_total, n_instr_total):
    """Per-launch algorithmic bytes.

    decode kernel:     |co_code| + |exctable| + 12 B x N_instr (records written)
    decompile kernel:  12 B x N_instr (records read) + referenced name/const bytes + |output text|
    """
    objs = arena.section("objs")
    code = int(objs["code_len"].sum())
    exc = int(objs["exc_len"].sum())
    strs = arena.section("strs")
    refs = arena.section("refs")
    name_bytes = 0
    for f in ("names", "varnames", "freevars", "cellvars"):
        offs = objs[f + "_off"].astype(np.int64)
        ns = objs["n_" + f].astype(np.int64)
        lens = strs["len"].astype(np.int64)
        tot = 0
        # vectorized: expand (off, n) ranges
        if ns.sum():
            idx = np.repeat(offs, ns) + (np.arange(ns.sum()) - np.repeat(np.cumsum(ns) - ns, ns))
            tot = int(lens[refs[idx]].sum())
        name_bytes += tot
    consts = arena.section("consts")
    cidx = objs["consts_off"].astype(np.int64)
    cn = objs["n_consts"].astype(np.int64)
    const_bytes = 0
    if cn.sum():
        idx = np.repeat(cidx, cn) + (np.arange(cn.sum()) - np.repeat(np.cumsum(cn) - cn, cn))
        ks = consts[refs[idx]]
        const_bytes = int(ks.size * consts.dtype.itemsize)
    dec = code + exc + 12 * n_instr_total
    struct = 12 * n_instr_total + name_bytes + const_bytes + text_len_total
    return dec, struct


def verify(res, pool_name, n_pool, stride=1, first=0):
    with open(os.path.join(ROOT, "tests", "golden", "pools.json")) as f:
        pools = json.load(f)
    want_sha = pools[pool_name]["sha"]
    want_st = pools[pool_name]["status"]
    from paper_2403_13839_b200.errors import ST_OK

    bad = 0
    n = len(res.status)
    tb = res.text
    for i in range(0, n, stride):
        j = (first + i) % n_pool
        st = int(res.status[i])
        s = tb[int(res.text_off[i]):int(res.text_off[i]) + int(res.text_len[i])]
        ok_status = (st == ST_OK) == (want_st[j] == "ok")
        if not ok_status or hashlib.sha256(s).hexdigest()[:24] != want_sha[j]:
            bad += 1
    return len(range(0, n, stride)), bad


def cpu_oracle_baseline(pool, seconds):
    """The oracle (CPU restatement of the reference algorithm) on every host core,
    over a bounded sample of the pool.  Returns (objects/s, cores, sample_desc)."""
    from oracle import bench_cpu

    return bench_cpu.run(pool, seconds)


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pool_name, n_obj, desc = WORKLOADS[args.workload]
    from paper_2403_13839_b200.bench_pools import pool_objects

    n_sample = 512 if args.workload != "c4" else 8
    pool = pool_objects(pool_name, 0, n_sample)
    from oracle import bench_cpu

    times = []
    cores = None
    sample = None
    for step in range(args.warmup + args.steps):
        rate, cores, sample = bench_cpu.run(pool, args.ref_seconds)
        if step >= args.warmup:
            times.append(rate)
    value = statistics.median(times)
    line = {"metric": METRIC, "value": value, "unit": "objects/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * n_sample / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": desc, "objects_per_step": n_sample, "pool": pool_name},
            "cpu_baseline": {"value": value, "unit": "objects/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "objects/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--objects", type=int, default=0, help="objects per GPU (default per workload)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--arena-bytes", type=int, default=0)
    ap.add_argument("--tpb", type=int, default=0)
    ap.add_argument("--verify-stride", type=int, default=0, help="check every k-th output (0: 1, c5: 16)")
    ap.add_argument("--pyc", type=int, default=1, help="also time the .pyc-bytes end-to-end path (0: skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2403_13839_b200 import arena as arena_mod
    from paper_2403_13839_b200.api import DeviceArena
    from paper_2403_13839_b200.bench_pools import POOLS, pool_objects

    pool_name, default_n, desc = WORKLOADS[args.workload]
    strong = args.workload == "c5"
    n_total = args.objects or default_n
    n_per_rank = n_total // world if strong else n_total
    t_gen = time.time()
    pool = pool_objects(pool_name)
    n_pool = len(pool)
    reps = max(1, n_per_rank // n_pool)
    pool_arena = arena_mod.pack(pool)
    arena = arena_mod.tile(pool_arena, reps)
    t_gen = time.time() - t_gen
    n_roots = arena.n_roots
    da = DeviceArena(arena, device=f"cuda:{local}", slots=args.slots, arena_bytes=args.arena_bytes,
                     threads_per_block=args.tpb)
    da.upload()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (full steps)
    for _ in range(args.warmup):
        da.run(stream, "decode")
        da.run(stream, "structure")
    barrier()

    # ---------------- timed: inputs resident in HBM
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            ev[k][0].record(stream)
            da.run(stream, "decode")
            ev[k][1].record(stream)
            da.run(stream, "structure")
            ev[k][2].record(stream)
        barrier()
    dec_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    st_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
    total_ms = ev[0][0].elapsed_time(ev[-1][2])
    res = da.fetch()

    # ---------------- timed: end to end (H2D of the packed arena, kernels, D2H of results)
    # Every step copies its inputs host -> device from pinned memory and its results
    # (statuses + text) device -> host.  Two buffer sets and three streams overlap the
    # copies of one step with the kernels of the neighbouring steps (double buffering);
    # time is measured from the first H2D to the last D2H.
    used = len(res.text)
    # second buffer set when it fits (C5's 16M objects need ~100 GB per set: single-buffered)
    free, _ = torch.cuda.mem_get_info()
    need = da.ws_bytes + da.text.numel() + da.dev.numel() + da.meta.numel()
    if free > 1.2 * need:
        das = [da, DeviceArena(arena, device=f"cuda:{local}", slots=args.slots, arena_bytes=args.arena_bytes,
                               threads_per_block=args.tpb, pinned=da.host)]
    else:
        das = [da, da]
    metas = [torch.empty(da.meta.numel(), dtype=torch.uint8).pin_memory() for _ in range(2)]
    texts = [torch.empty(used, dtype=torch.uint8).pin_memory() for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(args.steps)]
    ev_run = [torch.cuda.Event() for _ in range(args.steps)]
    ev_out = [torch.cuda.Event() for _ in range(args.steps)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(s_in)
    for k in range(args.steps):
        d = das[k % 2]
        with torch.cuda.stream(s_in):
            if k >= 2:
                s_in.wait_event(ev_run[k - 2])   # buffer set k%2 free again
            if das[0] is das[1] and k >= 1:
                s_in.wait_event(ev_run[k - 1])   # single buffer set: the previous step's kernels are done
            d.dev.copy_(d.host, non_blocking=True)
            ev_in[k].record(s_in)
        with torch.cuda.stream(stream):
            stream.wait_event(ev_in[k])
            if k >= 2:
                stream.wait_event(ev_out[k - 2])
            if das[0] is das[1] and k >= 1:
                stream.wait_event(ev_out[k - 1])  # single buffer set: results of step k-1 copied out
            d.run(stream, "full")
            ev_run[k].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_run[k])
            metas[k % 2].copy_(d.meta, non_blocking=True)
            texts[k % 2].copy_(d.text[:used], non_blocking=True)
            ev_out[k].record(s_out)
    s_in.wait_event(ev_out[args.steps - 1])
    e1.record(s_in)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    double_buffered = das[0] is not das[1]
    del das

    # ---------------- end to end from .pyc files in host memory:
    # native loader (all host threads) -> H2D -> kernels -> D2H, wall clock
    pyc = None
    if args.pyc and args.workload in ("c2", "c2x", "c2_311", "c3", "c3_311", "c5"):
        pyc = pyc_e2e(pool, reps, local, args, pool_name, n_pool, barrier)

    # ---------------- max over ranks
    times = torch.tensor([total_ms, e2e_ms, sum(dec_ms), sum(st_ms)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, dec_sum, st_sum = [float(x) for x in times.tolist()]

    # ---------------- parity of every output against the reference digests
    stride = args.verify_stride or (16 if strong else 1)
    n_checked, n_bad = verify(res, pool_name, n_pool, stride)
    bad_t = torch.tensor([n_checked, n_bad], dtype=torch.int64, device="cuda")
    if dist is not None:
        dist.all_reduce(bad_t)
    n_checked, n_bad = [int(x) for x in bad_t.tolist()]

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    objs_total = n_roots * world
    ms_step = total_ms / args.steps
    value = objs_total / (ms_step / 1000.0)
    code_bytes = arena.code_bytes
    # instruction count and name/const bytes from the distinct pool, x tiles
    n_instr = reps * int(_count_instructions(pool_arena))
    text_total = int(res.text_len.sum())
    pd, ps = algorithmic_bytes(pool_arena, 0, 0)
    alg_dec = reps * pd + 12 * n_instr
    alg_struct = reps * ps + 12 * n_instr + text_total
    peak, peak_src = peaks()
    dec_avg = dec_sum / args.steps / 1000.0
    st_avg = st_sum / args.steps / 1000.0
    ach_struct = alg_struct / st_avg / 1e9
    ach_dec = alg_dec / dec_avg / 1e9
    h2d = int(da.host.numel())
    d2h = int(da.meta.numel()) + used
    e2e_value = objs_total / (e2e_ms / args.steps / 1000.0)
    cpu = None
    if not args.no_cpu and world == 1:
        try:
            rate, cores, sample = cpu_oracle_baseline(pool[:512], args.cpu_seconds)
            cpu = {"value": rate, "unit": "objects/s", "cores": cores, "kind": "port", "sample": sample}
        except ImportError as e:
            cpu = {"value": None, "unit": "objects/s", "cores": None, "kind": "port",
                   "sample": f"unavailable: {e}"}
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "objects/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "objects_per_gpu": n_roots, "objects_total": objs_total,
                   "code_objects_per_gpu": int(len(arena.section("objs"))),
                   "pool": f"{pool_name} ({n_pool} distinct reference-checked objects tiled x{reps})",
                   "python": POOLS[pool_name]["minor"], "code_bytes_per_gpu": code_bytes,
                   "instructions_per_gpu": n_instr,
                   "l2": f"inputs larger than L2 ({h2d / 1e9:.2f} GB arena + {12 * n_instr / 1e9:.2f} GB records)",
                   "parallelism": f"shard roots x{world}", "gen_seconds": round(t_gen, 1)},
        "bytecode_gbs": code_bytes * world / (ms_step / 1000.0) / 1e9,
        "kernel_ms": {"decode": dec_sum / args.steps, "decompile": st_sum / args.steps},
        "parity": {"checked": n_checked, "mismatches": n_bad, "against": "reference SHA-256 (pools.json)"},
        "roofline": {"bound": "hbm", "kernel": "upy_decompile_kernel", "achieved": ach_struct, "peak": peak,
                     "unit": "GB/s", "frac": ach_struct / peak,
                     "traffic": measured_traffic(args.workload, "upy_decompile_kernel"),
                     "algorithmic_bytes_per_launch": alg_struct, "peak_source": peak_src},
        "roofline_decode": {"bound": "hbm", "kernel": "upy_decode_kernel", "achieved": ach_dec, "peak": peak,
                            "unit": "GB/s", "frac": ach_dec / peak,
                            "traffic": measured_traffic(args.workload, "upy_decode_kernel"),
                            "algorithmic_bytes_per_launch": alg_dec},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "objects/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "double_buffered": double_buffered},
        "e2e_pyc": pyc,
        "gpu_launches": 2 * args.steps + 2 * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def pyc_e2e(pool, reps, local, args, pool_name, n_pool, barrier):
    """decompile_pyc path timed end to end: .pyc images back to back in host memory
    -> upy_pyc_load (C++, all host threads) -> pinned H2D -> decode + decompile
    kernels -> D2H of statuses and text, as 4 pipelined sub-batches
    (loader.decompile_pyc_chunks).  Wall clock per step (host work is part of it),
    outputs checked against the reference digests."""
    from paper_2403_13839_b200.loader import decompile_pyc_chunks, load_pyc_buffer
    from paper_2403_13839_b200.synth import marshal

    blobs = [marshal.dump_pyc(co) for co in pool]
    one = b"".join(blobs)
    sizes = np.array([len(b) for b in blobs] * reps, dtype=np.uint64)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    buf = np.frombuffer(one * reps, dtype=np.uint8)
    n = len(sizes)
    # up to 4 sub-batches of >= 65,536 files: host parsing of one overlaps the device work
    # of the previous (small batches stay one batch: per-batch fixed costs dominate there)
    chunk = max(65536, (n + 3) // 4)

    def load(lo, hi):
        return load_pyc_buffer(buf, offs[lo:hi], sizes[lo:hi], pinned=True)

    t_all = []
    results = None
    for k in range(1 + args.steps):  # first step is warm-up
        barrier()
        results = None  # return the previous step's page-locked buffers to the caches first
        t0 = time.perf_counter()
        results = [(lo, res) for lo, _pf, res in decompile_pyc_chunks(load, n, None, f"cuda:{local}", chunk)]
        barrier()
        t2 = time.perf_counter()
        if k:
            t_all.append(t2 - t0)
    n_checked = n_bad = 0
    for lo, r in results:
        c, b = verify(r, pool_name, n_pool, 1, first=lo % n_pool)
        n_checked += c
        n_bad += b
    step = sum(t_all) / len(t_all)
    return {"value": n / step, "unit": "objects/s", "files_per_step": n, "pyc_bytes_per_step": int(len(buf)),
            "step_ms": 1000 * step, "sub_batches": (n + chunk - 1) // chunk,
            "loader_threads": os.cpu_count(), "parity": {"checked": n_checked, "mismatches": n_bad},
            "timing": "wall clock, synchronized, mean of --steps after 1 warm-up; host parsing of sub-batch "
                      "i+1 overlaps the device work of sub-batch i"}


def _count_instructions(arena):
    """Instruction count = code units minus EXTENDED_ARG prefixes minus cache units."""
    from paper_2403_13839_b200._optables import TABLES

    objs = arena.section("objs")
    by = arena.section("bytes")
    total = 0
    # only the distinct pool copy needs decoding logic; tiles repeat it
    for o in objs:
        off, ln, minor = int(o["code_off"]), int(o["code_len"]), int(o["minor"])
        code = by[off:off + ln]
        ops = code[0::2]
        n_ext = int(np.sum(ops == 144))
        if minor >= 11:
            caches = np.array([TABLES[11].get(int(x), ("", 0, "", 0))[3] for x in range(256)])
            # walk in order (caches are skipped, not decoded)
            i = 0
            n = 0
            while i < ln:
                op = int(code[i])
                if op != 144:
                    n += 1
                i += 2 + 2 * (int(caches[op]) if op != 144 else 0)
            total += n
        else:
            total += ln // 2 - n_ext
    return total


if __name__ == "__main__":
    main()
