"""Oracle node model: the expression/statement vocabulary of ir.py:16-472 plus
the simulator/structurer-private kinds (symexec.py:93-101,947-959,
structurer.py:974-981), generated from one field table.  Equality is the
dataclass rule (same class, every field equal in declaration order); side
attributes (_pending_targets, _loop_iter, _source) live outside the fields.
"""
from __future__ import annotations


class Node:
    kind_fields = ()
    is_expr = False
    is_stmt = False

    def __init__(self, *args):
        fs = self.kind_fields
        for i, (name, default) in enumerate(fs):
            if i < len(args):
                v = args[i]
            else:
                v = default() if callable(default) else default
            object.__setattr__(self, name, v)

    def __eq__(self, other):
        if other.__class__ is not self.__class__:
            return NotImplemented
        for name, _ in self.kind_fields:
            a = getattr(self, name)
            b = getattr(other, name)
            if a is b:
                continue
            if not (a == b):
                return False
        return True

    __hash__ = None

    def __repr__(self):
        inner = ", ".join(f"{n}={getattr(self, n)!r}" for n, _ in self.kind_fields)
        return f"{type(self).__name__}({inner})"


_LIST = list
TABLE = {
    # expressions (ir.py)
    "ConstE": ("E", [("const", None)]),
    "Name": ("E", [("id", None), ("scope", "fast")]),
    "BinOp": ("E", [("op", None), ("left", None), ("right", None), ("inplace", False)]),
    "UnaryOp": ("E", [("op", None), ("operand", None)]),
    "Compare": ("E", [("left", None), ("ops", None), ("comparators", None)]),
    "BoolOp": ("E", [("op", None), ("values", None)]),
    "Call": ("E", [("func", None), ("args", _LIST), ("keywords", _LIST)]),
    "Attr": ("E", [("value", None), ("name", None)]),
    "Subscript": ("E", [("value", None), ("index", None)]),
    "SliceE": ("E", [("lower", None), ("upper", None), ("step", None)]),
    "TupleE": ("E", [("elts", None)]),
    "ListE": ("E", [("elts", None)]),
    "SetE": ("E", [("elts", None)]),
    "DictE": ("E", [("keys", None), ("values", None)]),
    "Starred": ("E", [("value", None)]),
    "FormattedValue": ("E", [("value", None), ("conversion", ""), ("format_spec", None)]),
    "FString": ("E", [("parts", None)]),
    "Ternary": ("E", [("cond", None), ("then", None), ("orelse", None)]),
    "Yield": ("E", [("value", None)]),
    "YieldFrom": ("E", [("value", None)]),
    "NamedExpr": ("E", [("target", None), ("value", None)]),
    "Lambda": ("E", [("params", None), ("body", None)]),
    "CompExpr": ("E", [("kind", None), ("elt", None), ("key", None), ("value", None), ("generators", None)]),
    "FuncExpr": ("E", [("code", None), ("defaults", _LIST), ("kwdefaults", _LIST), ("annotations", _LIST),
                       ("closure", ())]),
    "StackTemp": ("E", [("index", None)]),
    "NullSlot": ("E", []),
    "MethodSelf": ("E", []),
    "ExcValue": ("E", [("slot", 0)]),
    "FinallySentinel": ("E", []),
    "UnpackSlot": ("E", [("source", None), ("count", None), ("index", None), ("star_index", -1),
                         ("after_count", 0), ("group", None)]),
    "ImportExpr": ("E", [("module", None), ("fromlist", None), ("level", None)]),
    "ImportFromExpr": ("E", [("source", None), ("name", None)]),
    "BuildClass": ("E", []),
    "ForItem": ("E", [("iter", None)]),
    "WithExit": ("E", [("context", None)]),
    "WithEnter": ("E", [("context", None)]),
    # helper records
    "CompFor": ("X", [("target", None), ("iter", None), ("ifs", None)]),
    "ExceptHandler": ("X", [("type", None), ("name", None), ("body", _LIST)]),
    "WithItem": ("X", [("context", None), ("target", None)]),
    "Params": ("X", [("args", _LIST), ("posonly", 0), ("vararg", None), ("kwonly", _LIST), ("kwarg", None),
                     ("defaults", _LIST), ("kwdefaults", dict)]),
    "UnpackGroup": ("X", [("source", None), ("total", None), ("star_index", -1), ("targets", None),
                          ("parent", None)]),
    # statements
    "Assign": ("S", [("targets", None), ("value", None)]),
    "AugAssign": ("S", [("target", None), ("op", None), ("value", None)]),
    "ExprStmt": ("S", [("value", None)]),
    "Return": ("S", [("value", None)]),
    "Raise": ("S", [("exc", None), ("cause", None)]),
    "Delete": ("S", [("targets", None)]),
    "Import": ("S", [("module", None), ("asname", None)]),
    "ImportFrom": ("S", [("module", None), ("names", _LIST), ("level", 0)]),
    "ImportStar": ("S", [("module", None), ("level", 0)]),
    "Pass": ("S", []),
    "Global": ("S", [("names", None)]),
    "Nonlocal": ("S", [("names", None)]),
    "Assert": ("S", [("test", None), ("msg", None)]),
    "If": ("S", [("cond", None), ("then", None), ("orelse", _LIST)]),
    "While": ("S", [("cond", None), ("body", None), ("orelse", _LIST)]),
    "For": ("S", [("target", None), ("iter", None), ("body", None), ("orelse", _LIST)]),
    "Try": ("S", [("body", None), ("handlers", _LIST), ("orelse", _LIST), ("final", _LIST)]),
    "With": ("S", [("items", None), ("body", None)]),
    "FuncDef": ("S", [("name", None), ("params", None), ("body", None), ("decorators", _LIST),
                      ("is_async", False)]),
    "ClassDef": ("S", [("name", None), ("bases", None), ("keywords", None), ("body", None),
                       ("decorators", _LIST)]),
    "Break": ("S", []),
    "Continue": ("S", []),
    "JumpMarker": ("S", [("target", None)]),
    "CondJumpMarker": ("S", [("cond", None), ("jump_when", None), ("target", None), ("pops_on_jump", True)]),
    "CompAccum": ("S", [("kind", None), ("value", None), ("key", None), ("depth", 0)]),
    "_WhileShape": ("S", [("cond", None), ("body", None), ("orelse", None), ("tail_cond", None)]),
}

K = {}
for _name, (_cat, _fields) in TABLE.items():
    K[_name] = type(_name, (Node,), {"kind_fields": tuple(_fields), "is_expr": _cat == "E",
                                     "is_stmt": _cat == "S"})
globals().update(K)

MARKERS = (K["JumpMarker"], K["CondJumpMarker"])


def is_expr(x):
    return isinstance(x, Node) and x.is_expr


def is_stmt(x):
    return isinstance(x, Node) and x.is_stmt
