"""Seeded schema mutants of JSON code-object dumps (test inputs for the JSON
loader): a valid dump of a small code-object tree with one
structural edit -- a key removed, a value retyped, a base64 field corrupted,
a constant re-tagged, the envelope broken -- so every SchemaError branch of
the reference's reader (pyc.py:378-508) is reached.  Test infrastructure."""
from __future__ import annotations

import json
import random

_JUNK = [None, True, False, 0, -3, 7.5, "", "x", "!!not-b64!!", "QUJD", [], [1], {}, {"t": "none"},
         {"t": "bogus"}, {"t": "int", "v": "12"}, {"t": "float", "v": "0x1.8p1"}, {"t": "bytes", "v": 5}]


def _paths(node, prefix=()):
    yield prefix, node
    if isinstance(node, dict):
        for k, v in node.items():
            yield from _paths(v, prefix + (k,))
    elif isinstance(node, list):
        for i, v in enumerate(node):
            yield from _paths(v, prefix + (i,))


def _get(node, path):
    for p in path:
        node = node[p]
    return node


def mutate(doc: dict, seed: int) -> str:
    """One mutant (JSON text) of the parsed dump `doc` (not modified)."""
    rng = random.Random(seed)
    d = json.loads(json.dumps(doc))
    kind = rng.randrange(10)
    if kind == 0:  # envelope
        choice = rng.randrange(6)
        if choice == 0:
            return json.dumps(d)[:-rng.randrange(1, 20)]
        if choice == 1:
            return json.dumps([d])
        if choice == 2:
            d["format_version"] = rng.choice([2, "1", None, True])
        elif choice == 3:
            d["python_version"] = rng.choice([[3], [3, 12], [2, 7], "3.10", [3, "10"], [3, 10, 0], [3, True]])
        elif choice == 4:
            del d["root"]
        else:
            del d["python_version"]
        return json.dumps(d)
    paths = [p for p, _ in _paths(d["root"]) if p]
    path = rng.choice(paths)
    parent = _get(d["root"], path[:-1])
    key = path[-1]
    if kind in (1, 2):  # remove a key / element
        if isinstance(parent, dict):
            del parent[key]
        else:
            parent.pop(key)
    elif kind in (3, 4, 5):  # retype a value
        parent[key] = rng.choice(_JUNK)
    elif kind == 6:  # corrupt a base64 string
        v = parent[key]
        if isinstance(v, str) and v:
            i = rng.randrange(len(v))
            parent[key] = v[:i] + rng.choice("!*= \n") + v[i + 1:]
        else:
            parent[key] = "A"
    elif kind == 7:  # re-tag a constant
        consts = [p for p, v in _paths(d["root"]) if isinstance(v, dict) and "t" in v]
        if consts:
            c = _get(d["root"], rng.choice(consts))
            c["t"] = rng.choice(["none", "bool", "int", "float", "complex", "str", "bytes", "tuple",
                                 "frozenset", "code", "ellipsis", "set", 3, None])
    elif kind == 8:  # add junk keys / elements (usually harmless)
        if isinstance(parent, dict):
            parent["zz"] = rng.choice(_JUNK)
        else:
            parent.append(rng.choice(_JUNK))
    else:  # swap a string list for a non-string element
        for k in ("names", "varnames", "freevars", "cellvars"):
            if rng.random() < 0.3:
                d["root"][k] = list(d["root"][k]) + [rng.choice([1, None, ["a"], "ok"])]
    return json.dumps(d)


def base_docs(golden_dir):
    """Parsed dumps of the mutation bases: C2 modules with nested code and
    constant tuples, and snippets covering float/complex/bytes/bool consts."""
    import os

    from .. import jsondump
    from . import cases

    with open(os.path.join(golden_dir, "c2.jsonl")) as f:
        c2 = [json.loads(line) for line in f]
    c2 = [r for r in c2 if not r.get("style")]
    picks = [c2[i] for i in (0, 17, 45)]
    snips = {r["name"]: r for r in cases.GOLDEN_SETS["snippets"]}
    picks += [snips[n] for n in ("constants", "fstring", "nested_defs")]
    return [json.loads(jsondump.dumps(cases.build(r))) for r in picks]
