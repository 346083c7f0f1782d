"""CPU tier: packer round trips, ABI surface of the built libraries, sharding
logic under a 2-process gloo group."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_13839_b200 import _abi, arena, shard
from paper_2403_13839_b200.model import CodeObject, Const, VersionTag
from paper_2403_13839_b200.synth import corpus, snippets

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _all_objects():
    objs = corpus.fig1(10) + corpus.fig1(11) + [corpus.c3(3), corpus.c4(1, 10, 600)]
    objs += [fn(m) for fn in snippets.SNIPPETS.values() for m in fn.minors]
    return objs


def test_pack_unpack_roundtrip():
    objs = _all_objects()
    back = arena.unpack(arena.pack(objs))
    assert len(back) == len(objs)
    for a, b in zip(objs, back):
        assert a._key() == b._key()
        assert a.filename == b.filename and a.qualname == b.qualname and a.exceptiontable == b.exceptiontable


def test_pack_layout_alignment():
    a = arena.pack(_all_objects())
    objs = a.section("objs")
    assert all(int(o) % 16 == 0 for o in objs["code_off"])
    for s in arena.SECTIONS:
        assert a.offsets[s] % 256 == 0


def test_tile_shares_pools_and_copies_code():
    a = arena.pack([corpus.c3(i) for i in range(5)])
    t = arena.tile(a, 3)
    assert t.n_roots == 15 and t.code_bytes == 3 * a.code_bytes
    back = arena.unpack(t)
    for k in range(3):
        for i in range(5):
            assert back[5 * k + i]._key() == back[i]._key()


def test_bigint_and_float_consts_roundtrip():
    c = Const("tuple", (Const("int", -(2 ** 200) + 7), Const("float", -0.0), Const("complex", complex(1, -2)),
                        Const("str", "\udc80x"), Const("bytes", b"\x00\xff"), Const("frozenset", (Const("int", 0),))))
    co = CodeObject(VersionTag(3, 10), 0, 0, 0, 0, 1, 0, b"d\x00S\x00", (c,), (), (), (), (), "f", "<s>", 1)
    back = arena.unpack(arena.pack([co]))[0]
    assert back.consts[0] == c


def _lib_path(name):
    return os.path.join(ROOT, "paper_2403_13839_b200", name)


@pytest.mark.skipif(not os.path.exists(_lib_path("libupy_cuda.so")), reason="CUDA library not built")
def test_cuda_library_exports_every_declared_symbol():
    import re

    lib = ctypes.CDLL(_lib_path("libupy_cuda.so"))
    declared = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        with open(os.path.join(ROOT, "include", h)) as f:
            declared |= set(re.findall(r"\b(upy_[a-z_]+)\s*\(", f.read()))
    assert declared == set(_abi.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym
    _abi.check_layout(lib)
    lib.upy_abi_version.restype = ctypes.c_int
    assert lib.upy_abi_version() == 4


def test_shard_bounds_partition_and_balance():
    w = np.random.default_rng(0).integers(1, 1000, size=1001)
    for world in (1, 2, 3, 8):
        b = shard.shard_bounds(w, world)
        assert b[0][0] == 0 and b[-1][1] == len(w)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        loads = [w[lo:hi].sum() for lo, hi in b]
        assert max(loads) - min(loads) <= 2 * w.max()


GLOO_WORKER = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
from paper_2403_13839_b200 import shard
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
weights = np.arange(1, 101)
lo, hi = shard.shard_bounds(weights, w)[r]
mx = shard.max_over_ranks([float(r + 1), float(hi - lo)])
tot = shard.sum_over_ranks([hi - lo])
assert mx[0] == w, mx
assert tot[0] == 100, tot
with open(os.path.join(sys.argv[2], f"ok_{r}"), "w") as f:  # files, not interleaved stdout
    f.write(f"{lo} {hi} {mx} {tot}")
dist.destroy_process_group()
"""


def test_gloo_world_size_2(tmp_path):
    import socket

    script = tmp_path / "w.py"
    script.write_text(GLOO_WORKER)
    with socket.socket() as sk:  # a free port (a fixed one can still be in TIME_WAIT from a previous run)
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script), ROOT, str(tmp_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert sorted(p.name for p in tmp_path.glob("ok_*")) == ["ok_0", "ok_1"]


SHARD_WORKER = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
import torch.distributed as dist
from paper_2403_13839_b200 import api, arena, hostcheck
from conftest import golden_cases
from helpers import inputs, mismatches, outcome
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
recs = [x for x in golden_cases(["c2", "c3", "c4", "mutant"]) if not x.get("style")]
codes = inputs(recs)
backend = lambda cs, style: hostcheck.run(arena.pack(cs), style)
lo, hi, mine = api.decompile_many_distributed(codes, gather=False, backend=backend)
full = api.decompile_many_distributed(codes, backend=backend)
bad = mismatches(recs, [outcome(v) for v in full])
own = mismatches(recs[lo:hi], [outcome(v) for v in mine])
with open(os.path.join(sys.argv[2], f"ok_{r}"), "w") as f:
    json.dump({"lo": lo, "hi": hi, "n": len(full), "bad": len(bad), "own_bad": len(own)}, f)
dist.destroy_process_group()
"""


def test_gloo_sharded_decompile_and_gather(tmp_path):
    """The multi-process path over gloo, world size 2: roots partitioned by tree
    code bytes (shard_plan), each rank decompiles only its shard (host build as
    the per-rank worker), the all-gather returns every result in input order,
    byte-identical to the reference's goldens."""
    import json
    import socket

    script = tmp_path / "w.py"
    script.write_text(SHARD_WORKER)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script), ROOT, str(tmp_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = [json.loads((tmp_path / f"ok_{r}").read_text()) for r in range(2)]
    assert res[0]["lo"] == 0 and res[0]["hi"] == res[1]["lo"] and res[1]["hi"] == res[0]["n"]
    assert 0 < res[0]["hi"] < res[0]["n"]  # both ranks got work
    assert all(x["bad"] == 0 and x["own_bad"] == 0 for x in res), res


def test_cost_order_matches_host_restatement():
    """The device-side largest-tree-first order (api.cost_order, torch ops, run here
    on a CPU tensor) equals its numpy restatement, for contiguous trees (pack /
    tile layout) and for a roots array in arbitrary order."""
    import numpy as np
    import torch

    from conftest import golden_cases
    from helpers import inputs
    from paper_2403_13839_b200 import api, arena

    ar = arena.tile(arena.pack(inputs([r for r in golden_cases(["c2"]) if not r.get("style")])), 3)
    for a in (ar, arena.with_roots(ar, ar.section("roots")[::-1].copy())):
        roots = a.section("roots").astype(np.int64)
        contiguous = bool(np.all(np.diff(roots) > 0))
        got = api.cost_order(torch.from_numpy(a.blob), a.offsets, a.counts, contiguous).numpy()
        assert np.array_equal(got, api.root_cost_order(a))
        assert sorted(got.tolist()) == list(range(a.n_roots))


def test_shape_order_is_lexicographic_on_opcodes():
    """api.shape_order (torch, chained stable sorts of 64-bit keys; run here on a
    CPU tensor) equals a numpy lexsort of the roots' first 8*n opcodes, input
    order breaking ties."""
    import numpy as np
    import torch

    from paper_2403_13839_b200 import api
    from paper_2403_13839_b200.synth import c3fast

    a = c3fast.c3_arena(3000, 11)
    objs, roots = a.section("objs"), a.section("roots").astype(np.int64)
    offs = objs["code_off"].astype(np.int64)[roots]
    lens = objs["code_len"].astype(np.int64)[roots]
    by = a.section("bytes")
    for nw in (1, 2, 4):
        j = np.arange(8 * nw)
        ops = np.where(2 * j[None, :] < lens[:, None], by[np.minimum(offs[:, None] + 2 * j[None, :], len(by) - 1)], 0)
        want = np.lexsort([np.arange(len(roots))] + [ops[:, c] for c in range(8 * nw - 1, -1, -1)])
        got = api.shape_order(torch.from_numpy(a.blob), a.offsets, a.counts, nw).numpy()
        assert np.array_equal(got, want), nw


TENSOR_GATHER_WORKER = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
import numpy as np, torch
import torch.distributed as dist
from paper_2403_13839_b200 import api, arena, hostcheck
from paper_2403_13839_b200.errors import make_exception
from paper_2403_13839_b200.gather import gather_results
from conftest import golden_cases
from helpers import inputs, mismatches, outcome
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
recs = [x for x in golden_cases(["c2", "c4", "mutant"]) if not x.get("style")]
codes = inputs(recs)
lo, hi = api.shard_plan(codes, w)[r]
res = hostcheck.run(arena.pack(codes[lo:hi]))
# this rank's results as the tensors the device path gathers (text at rank-local offsets)
texts = [s.encode("utf-8", "surrogatepass") for _, s, _ in res]
offs = np.cumsum([0] + [len(t) + 16 for t in texts])[:-1]  # gaps, like the 16-B reservations
text = torch.zeros(int(offs[-1] + len(texts[-1])) if texts else 0, dtype=torch.uint8)
for o, t in zip(offs, texts):
    text[int(o):int(o) + len(t)] = torch.tensor(list(t), dtype=torch.uint8)
g = gather_results(torch.tensor(offs, dtype=torch.int64),
                   torch.tensor([list(a) for _, _, a in res], dtype=torch.int64).reshape(-1, 2),
                   torch.tensor([len(t) for t in texts], dtype=torch.int32),
                   torch.tensor([st for st, _, _ in res], dtype=torch.int32), text)
vals = []
for i in range(len(g.status)):
    st, s = g.item(i)
    vals.append(s if st == 0 else make_exception(st, s, g.aux[i]))
bad = mismatches(recs, [outcome(v) for v in vals])
# bench.time_gather on the same results laid out as a DeviceArena meta buffer
import types
import bench
n = len(res)
meta = torch.zeros(64 + 32 * n, dtype=torch.uint8)
meta[:8] = torch.tensor([text.numel()], dtype=torch.int64).view(torch.uint8)
meta[64:64 + 8 * n] = torch.tensor(offs, dtype=torch.int64).view(torch.uint8)
meta[64 + 8 * n:64 + 24 * n] = torch.tensor([list(a) for _, _, a in res], dtype=torch.int64).view(-1).view(torch.uint8)
meta[64 + 24 * n:64 + 28 * n] = torch.tensor([len(t) for t in texts], dtype=torch.int32).view(torch.uint8)
meta[64 + 28 * n:64 + 32 * n] = torch.tensor([st for st, _, _ in res], dtype=torch.int32).view(torch.uint8)
br = api.BatchResult(np.array([st for st, _, _ in res], np.int32), np.array(offs, np.uint64),
                     np.array([len(t) for t in texts], np.uint32),
                     np.array([list(a) for _, _, a in res], np.int64).reshape(-1, 2), text.numpy())
tg = bench.time_gather(types.SimpleNamespace(n=n, meta=meta, text=text), br, dist.barrier)
with open(os.path.join(sys.argv[2], f"ok_{r}"), "w") as f:
    json.dump({"n": len(vals), "want": len(recs), "bad": len(bad), "ranks": g.ranks,
               "bench_own": tg["own_slice_identical"], "bench_roots": tg["roots_gathered"]}, f)
dist.destroy_process_group()
"""


def test_gloo_tensor_gather(tmp_path):
    """gather.gather_results (the final all-gather of the sharded path, on the
    device tensors in production) over gloo with CPU tensors, world size 2:
    every rank ends up with all results in input order, equal to the goldens."""
    import json
    import socket

    script = tmp_path / "g.py"
    script.write_text(TENSOR_GATHER_WORKER)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script), ROOT, str(tmp_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = [json.loads((tmp_path / f"ok_{r}").read_text()) for r in range(2)]
    assert all(x["n"] == x["want"] and x["bad"] == 0 for x in res), res
    assert res[0]["ranks"][1][1] > 0  # rank 1 contributed
    assert all(x["bench_own"] and x["bench_roots"] == x["want"] for x in res), res
