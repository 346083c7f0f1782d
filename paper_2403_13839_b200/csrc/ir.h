// ir.h -- expression / statement nodes (ir.py:16-472, symexec.py:93-101,947-959,
// structurer.py:974-981) with Python object semantics: nodes are mutable
// arena objects with identity, list fields are separately allocated mutable
// vectors (so aliasing such as TupleE(v.elts) behaves as in the reference),
// and node_eq() reproduces dataclass __eq__ (same class, all fields in order).
#pragma once
#include "model.h"

enum NodeKind : u8 {
  N_INVALID = 0,
  // ---- expressions (ir.Expr subclasses)
  E_CONST, E_NAME, E_BINOP, E_UNARY, E_COMPARE, E_BOOLOP, E_CALL, E_ATTR, E_SUBSCR, E_SLICE,
  E_TUPLE, E_LIST, E_SET, E_DICT, E_STARRED, E_FMTVAL, E_FSTRING, E_TERNARY, E_YIELD,
  E_YIELDFROM, E_NAMED, E_LAMBDA, E_COMP, E_FUNC, E_STACKTEMP, E_NULL, E_METHSELF, E_EXCVALUE,
  E_FINSENT, E_UNPACKSLOT, E_IMPORT, E_IMPORTFROM, E_BUILDCLASS, E_FORITEM, E_WITHEXIT,
  E_WITHENTER,
  E__END,
  // ---- helper records (not Expr, not Stmt)
  X_STRPART,   // str element of FString.parts
  X_KWPAIR,    // (name | None, Expr) tuple: Call.keywords, FuncExpr.kwdefaults/annotations
  X_NAMEPAIR,  // (name, asname | None) tuple: ImportFrom.names
  X_COMPFOR, X_HANDLER, X_WITHITEM, X_PARAMS, X_GROUP,
  X__END,
  // ---- statements (ir.Stmt subclasses)
  S_ASSIGN, S_AUGASSIGN, S_EXPR, S_RETURN, S_RAISE, S_DELETE, S_IMPORT, S_IMPORTFROM,
  S_IMPORTSTAR, S_PASS, S_GLOBAL, S_NONLOCAL, S_ASSERT, S_IF, S_WHILE, S_FOR, S_TRY, S_WITH,
  S_FUNCDEF, S_CLASSDEF, S_BREAK, S_CONTINUE, S_JUMP, S_CONDJUMP, S_COMPACCUM, S_WHILESHAPE,
  S__END
};

// binary / unary / bool / compare operator ids
enum BinOpId : u8 { BO_ADD, BO_AND, BO_FLOORDIV, BO_LSHIFT, BO_MATMUL, BO_MUL, BO_MOD, BO_OR,
                    BO_POW, BO_RSHIFT, BO_SUB, BO_TRUEDIV, BO_XOR, BO__N };
enum UnOpId : u8 { UO_NOT, UO_NEG, UO_POS, UO_INV };
enum CmpId : u8 { CO_LT, CO_LE, CO_EQ, CO_NE, CO_GT, CO_GE, CO_IN, CO_NOTIN, CO_IS, CO_ISNOT,
                  CO_EXCMATCH, CO_BAD, CO_NONE /* cmp_op out of range -> None */ };
enum ScopeId : u8 { SC_FAST, SC_GLOBAL, SC_DEREF, SC_NAME, SC_CELL };

struct Node;
typedef Vec<Node*> NV;

// Field usage per kind (reference field order in comments):
//  E_CONST     cid
//  E_NAME      s=id, op=scope
//  E_BINOP     op, a=left, b=right, f&1=inplace
//  E_UNARY     op, a=operand
//  E_COMPARE   a=left, l1=ops (X-less: Node* encodes CmpId via i), l2=comparators
//  E_BOOLOP    op (0 and, 1 or), l1=values
//  E_CALL      a=func, l1=args, l2=keywords(X_KWPAIR)
//  E_ATTR      a=value, s=name
//  E_SUBSCR    a=value, b=index
//  E_SLICE     a=lower?, b=upper?, c=step?
//  E_TUPLE/LIST/SET  l1=elts;  E_DICT l1=keys (nullptr = **), l2=values
//  E_STARRED   a=value
//  E_FMTVAL    a=value, op=conversion (0 '',1 s,2 r,3 a), b=format_spec?
//  E_FSTRING   l1=parts (X_STRPART | E_FMTVAL)
//  E_TERNARY   a=cond, b=then, c=orelse
//  E_YIELD     a=value?   E_YIELDFROM a=value
//  E_NAMED     a=target(Name), b=value
//  E_LAMBDA    p=params(X_PARAMS), a=body
//  E_COMP      op=kind(0 list,1 set,2 dict,3 gen), a=elt, b=key, c=value, l1=generators(X_COMPFOR)
//  E_FUNC      cid=code object index, l1=defaults, l2=kwdefaults(X_KWPAIR), l3=annotations(X_KWPAIR),
//              sl=closure (Vec<Str>)
//  E_STACKTEMP i=index
//  E_EXCVALUE  i=slot
//  E_UNPACKSLOT a=source, i=count, j=index, k=star_index, m=after_count, p=group(X_GROUP)
//  E_IMPORT    s=module, sl=fromlist (nullptr = None), i=level const id (const), f&2 = fromlist present
//  E_IMPORTFROM a=source, s=name
//  E_FORITEM   a=iter?    E_WITHEXIT/E_WITHENTER a=context
//  X_STRPART   s
//  X_KWPAIR    s=name (p==nullptr -> None), a=value?
//  X_NAMEPAIR  s=name, s2=asname?
//  X_COMPFOR   a=target, b=iter, l1=ifs
//  X_HANDLER   a=type?, s=name?, l1=body
//  X_WITHITEM  a=context, b=target?
//  X_PARAMS    sl=args, i=posonly, s=vararg?, sl2=kwonly, s2=kwarg?, l1=defaults, l2=kwdefaults(X_KWPAIR)
//  X_GROUP     a=source, i=total, k=star_index, l1=targets (nullptr = None), p=parent group?, j=parent index
//  S_ASSIGN    l1=targets, a=value
//  S_AUGASSIGN a=target, op, b=value
//  S_EXPR/S_RETURN a=value;  S_RAISE a=exc?, b=cause?;  S_DELETE l1=targets
//  S_IMPORT    s=module, s2=asname?;  S_IMPORTFROM s=module, l1=names(X_NAMEPAIR), i=level, src=_source
//  S_IMPORTSTAR s=module, i=level;  S_GLOBAL/S_NONLOCAL sl=names;  S_ASSERT a=test, b=msg?
//  S_IF        a=cond, l1=then, l2=orelse
//  S_WHILE     a=cond, l1=body, l2=orelse
//  S_FOR       a=target, b=iter, l1=body, l2=orelse
//  S_TRY       l1=body, l2=handlers(X_HANDLER), l3=orelse, l4=final
//  S_WITH      l1=items(X_WITHITEM), l2=body
//  S_FUNCDEF   s=name, p=params, l1=body, l2=decorators, f&4 is_async
//  S_CLASSDEF  s=name, l1=bases, l2=keywords(X_KWPAIR), l3=body, l4=decorators
//  S_JUMP      i=target;  S_CONDJUMP a=cond, f&1 jump_when, i=target, f&2 pops_on_jump
//  S_COMPACCUM op=kind(0 list,1 set,2 map), a=value, b=key?, i=depth
//  S_WHILESHAPE a=cond, l1=body, l2=orelse, b=tail_cond?
// Fields are ordered by how many kinds use them and a node is allocated with
// only the prefix its kind touches (node_bytes), so the common expression
// nodes take 24-72 bytes instead of the full record.  Code may only read a
// field that its node's kind uses (the per-kind table above).
struct Node {
  u8 k;
  u8 op;
  u8 f;       // flag bits (see above); bit7 = _loop_iter side attribute
  u8 pad;
  i32 i;
  u32 cid;
  i32 j;
  NV* pend;   // _pending_targets side attribute (nullptr = absent)   [all expressions]
  Str s;
  Node* a;
  Node* b;
  NV* l1;
  NV* l2;
  Node* c;
  Node* p;
  NV* l3;
  NV* l4;
  Vec<Str>* sl;
  Vec<Str>* sl2;
  Str s2;
  i32 kk, m;
  Node* src;  // ImportFrom._source side attribute
};

#define F_LOOP_ITER 0x80

HD inline bool is_expr(const Node* n) { return n && n->k > N_INVALID && n->k < E__END; }
HD inline bool is_stmt(const Node* n) { return n && n->k > X__END && n->k < S__END; }
HD inline bool is_k(const Node* n, u8 k) { return n && n->k == k; }

#define NODE_END(f) (offsetof(Node, f) + sizeof(((Node*)0)->f))
// bytes of the Node prefix a kind uses (see the field table above)
HD constexpr u32 node_bytes_sw(u8 k) {
  switch (k) {
    case E_CONST: case E_STACKTEMP: case E_NULL: case E_METHSELF: case E_EXCVALUE: case E_FINSENT:
    case E_BUILDCLASS:
      return NODE_END(pend);
    case E_NAME: return NODE_END(s);
    case E_UNARY: case E_STARRED: case E_YIELD: case E_YIELDFROM: case E_FORITEM: case E_WITHEXIT:
    case E_WITHENTER: case E_ATTR: case E_IMPORTFROM: case X_STRPART: case X_KWPAIR: case S_EXPR:
    case S_RETURN: case S_CONDJUMP:
      return NODE_END(a);
    case E_BINOP: case E_SUBSCR: case E_FMTVAL: case E_NAMED: case X_WITHITEM: case S_AUGASSIGN: case S_RAISE:
    case S_ASSERT: case S_COMPACCUM:
      return NODE_END(b);
    case E_BOOLOP: case E_TUPLE: case E_LIST: case E_SET: case E_FSTRING: case X_COMPFOR: case X_HANDLER:
    case S_ASSIGN: case S_DELETE:
      return NODE_END(l1);
    case E_COMPARE: case E_CALL: case E_DICT: case S_IF: case S_WHILE: case S_FOR: case S_WITH:
    case S_WHILESHAPE:
      return NODE_END(l2);
    case E_SLICE: case E_TERNARY: case E_COMP: return NODE_END(c);
    case E_LAMBDA: case S_FUNCDEF: return NODE_END(p);
    case S_TRY: case S_CLASSDEF: return NODE_END(l4);
    case E_FUNC: case E_IMPORT: case S_GLOBAL: case S_NONLOCAL: return NODE_END(sl);
    case X_NAMEPAIR: case S_IMPORT: return NODE_END(s2);
    case E_UNPACKSLOT: case X_GROUP: case X_PARAMS: return NODE_END(m);
    case S_JUMP: case S_PASS: case S_BREAK: case S_CONTINUE: return NODE_END(j);
  }
  return sizeof(Node);  // S_IMPORTSTAR (cid), S_IMPORTFROM (src), anything else: full record
}
// ... as a 256-entry table (mk() is inlined at hundreds of sites; a switch there
// was an out-of-line call per node)
struct NodeSizeTable {
  u8 v[256];
  HD constexpr NodeSizeTable() : v() {
    for (int k = 0; k < 256; k++) v[k] = (u8)node_bytes_sw((u8)k);
  }
};
static_assert(sizeof(Node) <= 255, "node sizes are stored as u8");
#ifdef __CUDA_ARCH__
__constant__ NodeSizeTable NODE_SIZES;
#else
static constexpr NodeSizeTable NODE_SIZES;
#endif
HD inline u32 node_bytes(u8 k) { return NODE_SIZES.v[k]; }

#ifndef UPY_MK_TABLE
// The size comes from the constexpr switch, so at the (inlined) call sites with a
// literal kind it folds to a constant, and the node is cleared with straight-line
// 16-B stores (predicated when the kind is only known at run time) instead of a
// __constant__ table read followed by a loop.
HD FORCEINL Node* mk(Dc* C, u8 k) {
  const u32 r = (node_bytes_sw(k) + 15) & ~15u;
  Node* n = (Node*)alloc_raw(C, r, false);
#ifdef __CUDA_ARCH__
  uint4* q = (uint4*)n;
  const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (u32 i = 0; i < (sizeof(Node) + 15) / 16; i++)
    if (i * 16 < r) q[i] = z;
#else
  memset(n, 0, r);
#endif
  n->k = k;
  if (k == E_FUNC || k == E_BUILDCLASS) C->n_defs++;
  return n;
}
#else
HD ALLOCFN Node* mk(Dc* C, u8 k) {
  Node* n = (Node*)zalloc(C, node_bytes(k));
  n->k = k;
  if (k == E_FUNC || k == E_BUILDCLASS) C->n_defs++;
  return n;
}
#endif
HD inline Node* mk_const(Dc* C, u32 cid) {
  Node* n = mk(C, E_CONST);
  n->cid = cid;
  return n;
}
HD inline Node* mk_name(Dc* C, Str id, u8 scope) {
  Node* n = mk(C, E_NAME);
  n->s = id;
  n->op = scope;
  return n;
}
HD inline Node* mk1(Dc* C, u8 k, Node* a) {
  Node* n = mk(C, k);
  n->a = a;
  return n;
}
HD inline Node* mk2(Dc* C, u8 k, Node* a, Node* b) {
  Node* n = mk(C, k);
  n->a = a;
  n->b = b;
  return n;
}
HD inline NV* nv1(Dc* C, Node* x) {
  NV* v = vnew<Node*>(C, 1);
  vpush(C, v, x);
  return v;
}
HD inline NV* nv2(Dc* C, Node* x, Node* y) {
  NV* v = vnew<Node*>(C, 2);
  vpush(C, v, x);
  vpush(C, v, y);
  return v;
}
HD inline Node* mk_cmpop(Dc* C, u8 cmp) {  // element of Compare.ops
  Node* n = mk(C, X_STRPART);
  n->op = cmp;
  n->i = 1;  // marks "compare op" flavour
  return n;
}
HD inline Node* mk_compare(Dc* C, Node* left, u8 cmp, Node* right) {
  Node* n = mk(C, E_COMPARE);
  n->a = left;
  n->l1 = nv1(C, mk_cmpop(C, cmp));
  n->l2 = nv1(C, right);
  return n;
}
HD inline Node* mk_unary(Dc* C, u8 op, Node* a) {
  Node* n = mk1(C, E_UNARY, a);
  n->op = op;
  return n;
}
HD inline Node* mk_binop(Dc* C, u8 op, Node* l, Node* r, bool inplace) {
  Node* n = mk2(C, E_BINOP, l, r);
  n->op = op;
  n->f = inplace ? 1 : 0;
  return n;
}
HD inline Node* mk_assign(Dc* C, NV* targets, Node* value) {
  Node* n = mk(C, S_ASSIGN);
  n->l1 = targets;
  n->a = value;
  return n;
}
HD inline Node* mk_if(Dc* C, Node* cond, NV* then, NV* orelse) {
  Node* n = mk(C, S_IF);
  n->a = cond;
  n->l1 = then;
  n->l2 = orelse ? orelse : vnew<Node*>(C);
  return n;
}
HD inline Node* mk_kwpair(Dc* C, Str name, Node* v) {
  Node* n = mk(C, X_KWPAIR);
  n->s = name;
  n->a = v;
  return n;
}

// Python class name of the reference object a node stands for (for the
// reference's AttributeError messages, "'X' object has no attribute 'y'").
HD inline const char* py_type_name(const Node* n) {
  if (!n) return "NoneType";
  switch (n->k) {
    case E_CONST: return "ConstE"; case E_NAME: return "Name"; case E_BINOP: return "BinOp";
    case E_UNARY: return "UnaryOp"; case E_COMPARE: return "Compare"; case E_BOOLOP: return "BoolOp";
    case E_CALL: return "Call"; case E_ATTR: return "Attr"; case E_SUBSCR: return "Subscript";
    case E_SLICE: return "SliceE"; case E_TUPLE: return "TupleE"; case E_LIST: return "ListE";
    case E_SET: return "SetE"; case E_DICT: return "DictE"; case E_STARRED: return "Starred";
    case E_FMTVAL: return "FormattedValue"; case E_FSTRING: return "FString"; case E_TERNARY: return "Ternary";
    case E_YIELD: return "Yield"; case E_YIELDFROM: return "YieldFrom"; case E_NAMED: return "NamedExpr";
    case E_LAMBDA: return "Lambda"; case E_COMP: return "CompExpr"; case E_FUNC: return "FuncExpr";
    case E_STACKTEMP: return "StackTemp"; case E_NULL: return "NullSlot"; case E_METHSELF: return "MethodSelf";
    case E_EXCVALUE: return "ExcValue"; case E_FINSENT: return "FinallySentinel";
    case E_UNPACKSLOT: return "UnpackSlot"; case E_IMPORT: return "ImportExpr";
    case E_IMPORTFROM: return "ImportFromExpr"; case E_BUILDCLASS: return "BuildClass";
    case E_FORITEM: return "ForItem"; case E_WITHEXIT: return "WithExit"; case E_WITHENTER: return "WithEnter";
    case X_STRPART: return "str"; case X_KWPAIR: case X_NAMEPAIR: return "tuple";
    case X_COMPFOR: return "CompFor"; case X_HANDLER: return "ExceptHandler"; case X_WITHITEM: return "WithItem";
    case X_PARAMS: return "Params"; case X_GROUP: return "UnpackGroup";
  }
  return "Stmt";
}
HD inline void py_attr_error(Dc* C, const Node* n, const char* attr) {
  Text t;
  if (!fail_begin(C, UPY_ST_PY_ATTRIBUTE_ERROR, 0, 0, &t)) return;
  m_puts(C, &t, "'");
  m_puts(C, &t, py_type_name(n));
  m_puts(C, &t, "' object has no attribute '");
  m_puts(C, &t, attr);
  m_puts(C, &t, "'");
  fail_end(C, &t);
}

// ------------------------------------------------------------ equality
HD bool node_eq(Dc* C, const Node* a, const Node* b);

HD inline bool nv_eq(Dc* C, const NV* a, const NV* b) {
  u32 na = a ? a->n : 0, nb = b ? b->n : 0;
  if (na != nb) return false;
  for (u32 i = 0; i < na; i++) {
    if (a->d[i] == b->d[i]) continue;  // list equality tries identity first
    if (!node_eq(C, a->d[i], b->d[i])) return false;
    if (C->err) return false;
  }
  return true;
}
HD inline bool sv_eq(const Vec<Str>* a, const Vec<Str>* b) {
  if (!a || !b) return a == b;
  if (a->n != b->n) return false;
  for (u32 i = 0; i < a->n; i++)
    if (!s_eq(a->d[i], b->d[i])) return false;
  return true;
}
// Python `x == y` on Const fields: Const.__eq__ (or None == None)
HD inline bool cid_eq(Dc* C, u32 a, u32 b) {
  if (a == CID_INVALID || b == CID_INVALID) return a == b;
  return const_key_eq(C, a, b);
}
// dict equality for Params.kwdefaults (order-insensitive, last duplicate wins)
HD inline const Node* kw_lookup(const NV* kws, Str name) {
  const Node* hit = nullptr;
  for (u32 i = 0; kws && i < kws->n; i++)
    if (s_eq(kws->d[i]->s, name)) hit = kws->d[i];
  return hit;
}
HD inline bool kwdict_eq(Dc* C, const NV* a, const NV* b) {
  u32 ua = 0, ub = 0;  // count distinct keys
  for (u32 i = 0; a && i < a->n; i++) {
    if (kw_lookup(a, a->d[i]->s) != a->d[i]) continue;
    ua++;
    const Node* o = kw_lookup(b, a->d[i]->s);
    if (!o) return false;
    if (o->a != a->d[i]->a && !node_eq(C, a->d[i]->a, o->a)) return false;
  }
  for (u32 i = 0; b && i < b->n; i++)
    if (kw_lookup(b, b->d[i]->s) == b->d[i]) ub++;
  return ua == ub;
}

HD NOINL bool node_eq(Dc* C, const Node* x, const Node* y) {
  if (x == y) return true;
  if (!x || !y) return false;
  if (x->k != y->k) return false;
  GUARD(C);
  CKR(C, false);
#define EQN(f) (x->f == y->f || node_eq(C, x->f, y->f))
#define EQL(f) nv_eq(C, x->f, y->f)
  switch (x->k) {
    case E_CONST: return cid_eq(C, x->cid, y->cid);
    case E_NAME: return s_eq(x->s, y->s) && x->op == y->op;
    case E_BINOP: return x->op == y->op && EQN(a) && EQN(b) && (x->f & 1) == (y->f & 1);
    case E_UNARY: return x->op == y->op && EQN(a);
    case E_COMPARE: return EQN(a) && EQL(l1) && EQL(l2);
    case E_BOOLOP: return x->op == y->op && EQL(l1);
    case E_CALL: return EQN(a) && EQL(l1) && EQL(l2);
    case E_ATTR: return EQN(a) && s_eq(x->s, y->s);
    case E_SUBSCR: return EQN(a) && EQN(b);
    case E_SLICE: return EQN(a) && EQN(b) && EQN(c);
    case E_TUPLE: case E_LIST: case E_SET: return EQL(l1);
    case E_DICT: return EQL(l1) && EQL(l2);
    case E_STARRED: return EQN(a);
    case E_FMTVAL: return EQN(a) && x->op == y->op && EQN(b);
    case E_FSTRING: return EQL(l1);
    case E_TERNARY: return EQN(a) && EQN(b) && EQN(c);
    case E_YIELD: case E_YIELDFROM: return EQN(a);
    case E_NAMED: return EQN(a) && EQN(b);
    case E_LAMBDA: return EQN(p) && EQN(a);
    case E_COMP: return x->op == y->op && EQN(a) && EQN(b) && EQN(c) && EQL(l1);
    case E_FUNC:
      return code_full_eq(C, x->cid, y->cid) && EQL(l1) && EQL(l2) && EQL(l3) && sv_eq(x->sl, y->sl);
    case E_STACKTEMP: return x->i == y->i;
    case E_NULL: case E_METHSELF: case E_FINSENT: case E_BUILDCLASS: return true;
    case E_EXCVALUE: return x->i == y->i;
    case E_UNPACKSLOT:
      return EQN(a) && x->i == y->i && x->j == y->j && x->kk == y->kk && x->m == y->m && EQN(p);
    case E_IMPORT:
      return s_eq(x->s, y->s) && (x->f & 2) == (y->f & 2) && ((x->f & 2) == 0 || sv_eq(x->sl, y->sl)) &&
             cid_eq(C, x->cid, y->cid);
    case E_IMPORTFROM: return EQN(a) && s_eq(x->s, y->s);
    case E_FORITEM: case E_WITHEXIT: case E_WITHENTER: return EQN(a);
    case X_STRPART: return x->i == y->i && (x->i ? x->op == y->op : s_eq(x->s, y->s));
    case X_KWPAIR: return s_eq(x->s, y->s) && EQN(a);
    case X_NAMEPAIR: return s_eq(x->s, y->s) && s_eq(x->s2, y->s2);
    case X_COMPFOR: return EQN(a) && EQN(b) && EQL(l1);
    case X_HANDLER: return EQN(a) && s_eq(x->s, y->s) && EQL(l1);
    case X_WITHITEM: return EQN(a) && EQN(b);
    case X_PARAMS:
      return sv_eq(x->sl, y->sl) && x->i == y->i && s_eq(x->s, y->s) && sv_eq(x->sl2, y->sl2) &&
             s_eq(x->s2, y->s2) && EQL(l1) && kwdict_eq(C, x->l2, y->l2);
    case X_GROUP:
      return EQN(a) && x->i == y->i && x->kk == y->kk && EQL(l1) && EQN(p) && x->j == y->j;
    case S_ASSIGN: return EQL(l1) && EQN(a);
    case S_AUGASSIGN: return EQN(a) && x->op == y->op && EQN(b);
    case S_EXPR: case S_RETURN: return EQN(a);
    case S_RAISE: return EQN(a) && EQN(b);
    case S_DELETE: return EQL(l1);
    case S_IMPORT: return s_eq(x->s, y->s) && s_eq(x->s2, y->s2);
    case S_IMPORTFROM: return s_eq(x->s, y->s) && EQL(l1) && x->i == y->i;
    case S_IMPORTSTAR: return s_eq(x->s, y->s) && x->i == y->i;
    case S_PASS: case S_BREAK: case S_CONTINUE: return true;
    case S_GLOBAL: case S_NONLOCAL: return sv_eq(x->sl, y->sl);
    case S_ASSERT: return EQN(a) && EQN(b);
    case S_IF: case S_WHILE: return EQN(a) && EQL(l1) && EQL(l2);
    case S_FOR: return EQN(a) && EQN(b) && EQL(l1) && EQL(l2);
    case S_TRY: return EQL(l1) && EQL(l2) && EQL(l3) && EQL(l4);
    case S_WITH: return EQL(l1) && EQL(l2);
    case S_FUNCDEF: return s_eq(x->s, y->s) && EQN(p) && EQL(l1) && EQL(l2) && (x->f & 4) == (y->f & 4);
    case S_CLASSDEF: return s_eq(x->s, y->s) && EQL(l1) && EQL(l2) && EQL(l3) && EQL(l4);
    case S_JUMP: return x->i == y->i;
    case S_CONDJUMP: return EQN(a) && (x->f & 3) == (y->f & 3) && x->i == y->i;
    case S_COMPACCUM: return x->op == y->op && EQN(a) && EQN(b) && x->i == y->i;
    case S_WHILESHAPE: return EQN(a) && EQL(l1) && EQL(l2) && EQN(b);
  }
#undef EQN
#undef EQL
  return false;
}
