"""Golden stack depths for the stack-depth scan (north star (3)),
recorded from the REAL reference's symbolic simulation.  Run in the build
container:

    python tests/golden/make_stack_golden.py

The reference has no stand-alone depth pass: depth is `len(st)` inside
`Simulator.simulate_block` (symexec.py:138-210).  This script instruments it
without copying it: it wraps `simulate_block` (entry depth, exit states) and every
`_op_*` transfer function (depth after the call and how many following
instructions it consumed, symexec.py:203-209), then runs `decompile_source` on
every root of the golden sets.  Each line of stack.jsonl:

    {"set", "obj", "blocks": [[lo, E, [[off, d], ...], fall], ...]}

for object `obj` of `arena.pack(inputs)` (the set's records without a style): per
simulated block (first instruction offset lo, entry depth E), the offset of the
LAST instruction each transfer function consumed with the depth after it
(relative: d = len(st) - E), and the fall-through exit depth (relative, or None).
Only objects whose decompile reached simulation are listed; a block simulated
several times (different entry stacks) appears once per distinct (lo, E).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

import unpyre  # noqa: E402
from unpyre import symexec  # noqa: E402

from paper_2403_13839_b200 import arena  # noqa: E402
from paper_2403_13839_b200.synth import cases  # noqa: E402

SETS = ("c1", "c2", "c3", "c4", "snippets", "fuzz")
TRACE = None   # list of blocks of the object being decompiled
TRACE_CODE = None  # ... and that object (nested bodies decompiled on the way are not traced)
_active = [0]  # nesting of transfer-function calls (only the outermost is recorded)


def _wrap_block(orig):
    def simulate_block(self, block, entry_state):
        st0 = entry_state.entries if isinstance(entry_state, symexec.StackState) else entry_state
        rec = None
        if TRACE is not None and self.code is TRACE_CODE and getattr(block, "instrs", None):
            rec = [block.instrs[0].offset, len(st0), [], None]
            TRACE.append(rec)
        res = orig(self, block, entry_state)
        if rec is not None and res.exit_fall is not None:
            rec[3] = len(res.exit_fall.entries) - rec[1]
        return res
    return simulate_block


def _wrap_op(orig):
    def op(self, ins, st, out, rest):
        _active[0] += 1
        try:
            consumed = orig(self, ins, st, out, rest)
        finally:
            _active[0] -= 1
        if TRACE is not None and self.code is TRACE_CODE and _active[0] == 0 and TRACE:
            last = rest[consumed - 1] if consumed else ins
            TRACE[-1][2].append([last.offset, len(st) - TRACE[-1][1]])
        return consumed
    return op


def instrument():
    sim = symexec.Simulator
    sim.simulate_block = _wrap_block(sim.simulate_block)
    for name in list(vars(sim)):
        if name.startswith("_op_") and callable(getattr(sim, name)):
            setattr(sim, name, _wrap_op(getattr(sim, name)))


def set_records(name):
    with open(os.path.join(HERE, f"{name}.jsonl")) as f:
        recs = [json.loads(line) for line in f]
    return [r for r in recs if not r.get("style")]


def main():
    global TRACE, TRACE_CODE
    instrument()
    path = os.path.join(HERE, "stack.jsonl")
    with open(path, "w") as f:
        for name in SETS:
            recs = set_records(name)
            ar = arena.pack([cases.build(r) for r in recs])
            objs = arena.unpack(ar, unpyre.CodeObject, unpyre.Const, unpyre.VersionTag, objects=range(ar.n_objs))
            n_calls = 0
            for i, co in enumerate(objs):
                TRACE, TRACE_CODE = [], co
                try:
                    unpyre.decompile_source(co)
                except Exception:  # noqa: BLE001 -- errors end the trace; what ran is still valid
                    pass
                blocks, seen = [], set()
                for lo, e, calls, fall in TRACE:
                    key = (lo, e, json.dumps(calls))
                    if key in seen:
                        continue
                    seen.add(key)
                    blocks.append([lo, e, calls, fall])
                    n_calls += len(calls)
                TRACE = None
                if blocks:
                    f.write(json.dumps({"set": name, "obj": i, "blocks": blocks}) + "\n")
            print(f"{name}: {ar.n_objs} objects, {n_calls} transfer-function depths")
    print("->", path)


if __name__ == "__main__":
    main()
