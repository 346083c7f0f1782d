// recover.h -- nested-code recovery and the per-object body pipeline
// (recover.py:25-357, pipeline.py:90-140).  Nested code constants are
// decompiled recursively on the same thread, at the same points and in the
// same order as the reference, so hoist order and __lambda_<k> numbering match.
#pragma once
#include "structurer.h"

HD NV* decompile_body(Dc* C, u32 oi);

// params_from_code (ir.py:432-450)
HD inline Node* params_from_code(Dc* C, u32 oi, NV* defaults, NV* kwdefaults) {
  const upy_obj* o = obj_at(C, oi);
  Node* p = mk(C, X_PARAMS);
  i64 nv = o->n_varnames;
  auto slice = [&](i64 a, i64 b) {  // names[a:b] with Python clamping
    if (a < 0) { a += nv; if (a < 0) a = 0; }
    if (b < 0) { b += nv; if (b < 0) b = 0; }
    if (a > nv) a = nv;
    if (b > nv) b = nv;
    Vec<Str>* v = vnew<Str>(C, b > a ? (u32)(b - a) : 0);
    for (i64 q = a; q < b; q++) vpush(C, v, obj_tab(C, o->varnames_off, (u32)q));
    return v;
  };
  i64 n = o->argcount;
  p->sl = slice(0, n);
  p->i = (i32)o->posonlyargcount;
  p->sl2 = slice(n, n + o->kwonlyargcount);
  p->l1 = defaults ? defaults : vnew<Node*>(C);
  p->l2 = kwdefaults ? kwdefaults : vnew<Node*>(C);
  p->s = Snone();
  p->s2 = Snone();
  i64 i = n + o->kwonlyargcount;
  auto at = [&](i64 k, Str* out) {
    if (k < 0) k += nv;
    if (k < 0 || k >= nv) {
      py_error(C, UPY_ST_PY_INDEX_ERROR, "tuple index out of range");
      return;
    }
    *out = obj_tab(C, o->varnames_off, (u32)k);
  };
  if (o->flags & 0x4) {
    at(i, &p->s);
    i++;
  }
  if (o->flags & 0x8) at(i, &p->s2);
  return p;
}

HD inline bool code_is_str_doc(Dc* C, u32 oi) {
  const upy_obj* o = obj_at(C, oi);
  return o->n_consts && ckind(C, obj_const_id(C, oi, 0)) == UPY_C_STR;
}
// Python type of a FuncExpr's `code` when MAKE_FUNCTION popped a non-code
// constant (FuncExpr.code = code_const.const.value, symexec.py:820-821): the
// node keeps that constant's kind in `j`.
HD inline const char* py_value_type(i32 kind) {
  switch (kind) {
    case UPY_C_BOOL: return "bool"; case UPY_C_INT: return "int"; case UPY_C_FLOAT: return "float";
    case UPY_C_COMPLEX: return "complex"; case UPY_C_STR: return "str"; case UPY_C_BYTES: return "bytes";
    case UPY_C_TUPLE: case UPY_C_FROZENSET: return "tuple";
  }
  return "NoneType";
}
HD inline void py_value_attr_error(Dc* C, i32 kind, const char* attr) {
  Text t;
  if (!fail_begin(C, UPY_ST_PY_ATTRIBUTE_ERROR, 0, 0, &t)) return;
  m_puts(C, &t, "'");
  m_puts(C, &t, py_value_type(kind));
  m_puts(C, &t, "' object has no attribute '");
  m_puts(C, &t, attr);
  m_puts(C, &t, "'");
  fail_end(C, &t);
}
// `fe.code.name` of a FuncExpr node
HD inline Str code_name_checked(Dc* C, const Node* fe) {
  if (fe->cid == CID_INVALID) {
    py_value_attr_error(C, fe->j, "name");
    return Snone();
  }
  return obj_name(C, fe->cid);
}

struct Recovery {
  Dc* C;
  u32 oi;
  NV* hoisted;
  i64 lambda_counter;

  HD Node* map_expr(Node* e);
  HD Node* map_pair(Node* x);
  HD NV* map_list(NV* v);
  HD Node* pre_expr(Node* e);
  HD Node* post_expr(Node* e);
  HD Node* hoist(Node* fe);
  HD Node* make_funcdef(Str name, Node* fe);
  HD Node* make_classdef(Str name, Node* call);
  HD Node* make_lambda(Node* fe);
  HD Node* make_comp(int kind, u32 code, Node* iter_arg);
  HD Node* match_def(Node* target, Node* value);
  HD NV* rewrite_stmt(Node* s);
  HD NV* rewrite_block(NV* stmts);
  HD void stmt_exprs(Node* s);
};

// _map_pair (recover.py:53-60)
HD inline Node* Recovery::map_pair(Node* x) {
  if (is_k(x, X_KWPAIR) && is_expr(x->a)) return mk_kwpair(C, x->s, map_expr(x->a));
  if (is_k(x, X_COMPFOR)) {
    x->a = map_expr(x->a);
    x->b = map_expr(x->b);
    NV* ifs = vnew<Node*>(C, x->l1->n);
    for (u32 q = 0; q < x->l1->n; q++) vpush(C, ifs, map_expr(x->l1->d[q]));
    x->l1 = ifs;
  }
  return x;
}
HD inline NV* Recovery::map_list(NV* v) {
  NV* out = vnew<Node*>(C, v ? v->n : 0);
  for (u32 q = 0; v && q < v->n && !C->err; q++) {
    Node* x = v->d[q];
    vpush(C, out, is_expr(x) ? map_expr(x) : map_pair(x));
  }
  return out;
}

// map_expr (recover.py:25-50): pre may replace a subtree, fields in dataclass order, post last
HD NOINL Node* Recovery::map_expr(Node* e) {
  if (!is_expr(e)) return e;
  GUARD(C);
  CKR(C, e);
  Node* r = pre_expr(e);
  CKR(C, e);
  if (r) return r;
#define MX(f) \
  if (is_expr(e->f)) e->f = map_expr(e->f)
#define ML(f) e->f = map_list(e->f)
  switch (e->k) {
    case E_BINOP: MX(a); MX(b); break;
    case E_UNARY: MX(a); break;
    case E_COMPARE: MX(a); ML(l1); ML(l2); break;
    case E_BOOLOP: ML(l1); break;
    case E_CALL: MX(a); ML(l1); ML(l2); break;
    case E_ATTR: MX(a); break;
    case E_SUBSCR: MX(a); MX(b); break;
    case E_SLICE: MX(a); MX(b); MX(c); break;
    case E_TUPLE: case E_LIST: case E_SET: ML(l1); break;
    case E_DICT: ML(l1); ML(l2); break;
    case E_STARRED: MX(a); break;
    case E_FMTVAL: MX(a); MX(b); break;
    case E_FSTRING: ML(l1); break;
    case E_TERNARY: MX(a); MX(b); MX(c); break;
    case E_YIELD: case E_YIELDFROM: MX(a); break;
    case E_NAMED: MX(a); MX(b); break;
    case E_LAMBDA: MX(a); break;
    case E_COMP: MX(a); MX(b); MX(c); ML(l1); break;
    case E_FUNC: ML(l1); ML(l2); ML(l3); break;
    case E_UNPACKSLOT: MX(a); break;
    case E_IMPORTFROM: MX(a); break;
    case E_FORITEM: case E_WITHEXIT: case E_WITHENTER: MX(a); break;
    default: break;
  }
#undef MX
#undef ML
  CKR(C, e);
  return post_expr(e);
}

HD inline int comp_kind_of(Str name) {  // COMP_NAMES (recover.py:17-22)
  if (s_eqc(name, "<listcomp>")) return 0;
  if (s_eqc(name, "<setcomp>")) return 1;
  if (s_eqc(name, "<dictcomp>")) return 2;
  if (s_eqc(name, "<genexpr>")) return 3;
  return -1;
}

HD inline Node* Recovery::pre_expr(Node* e) {  // recover.py:176-189
  if (is_k(e, E_CALL) && is_k(e->a, E_FUNC)) {
    Str nm = code_name_checked(C, e->a);
    CKR(C, nullptr);
    int kind = comp_kind_of(nm);
    if (kind >= 0 && e->l1->n == 1 && e->l2->n == 0) {
      Node* arg = map_expr(e->l1->d[0]);
      CKR(C, nullptr);
      Node* comp = make_comp(kind, e->a->cid, arg);
      CKR(C, nullptr);
      if (comp) return comp;
    }
  }
  if (is_k(e, E_FUNC)) {
    Str nm = code_name_checked(C, e);
    CKR(C, nullptr);
    if (s_eqc(nm, "<lambda>")) {
      Node* lam = make_lambda(e);
      CKR(C, nullptr);
      if (lam) return lam;
    }
  }
  return nullptr;
}
HD inline Node* Recovery::post_expr(Node* e) {
  if (is_k(e, E_FUNC)) return hoist(e);
  return e;
}
HD inline Node* Recovery::hoist(Node* fe) {  // recover.py:221-227
  Str name = code_name_checked(C, fe);
  CKR(C, fe);
  if (s_eqc(name, "<lambda>")) {
    Node* nm = mk_name_syn(C, "__lambda_", lambda_counter, SC_FAST);
    lambda_counter++;
    name = nm->s;
  }
  Node* d = make_funcdef(name, fe);
  CKR(C, fe);
  vpush(C, hoisted, d);
  return mk_name(C, name, SC_FAST);
}
HD NOINL Node* Recovery::make_funcdef(Str name, Node* fe) {  // recover.py:150-159
  GUARD(C);
  CKR(C, nullptr);
  if (fe->cid == CID_INVALID) {
    py_value_attr_error(C, fe->j, "varnames");
    return nullptr;
  }
  NV* defs = vnew<Node*>(C, fe->l1->n);
  for (u32 q = 0; q < fe->l1->n; q++) vpush(C, defs, map_expr(fe->l1->d[q]));
  NV* kwd = vnew<Node*>(C, fe->l2->n);
  for (u32 q = 0; q < fe->l2->n; q++) vpush(C, kwd, mk_kwpair(C, fe->l2->d[q]->s, map_expr(fe->l2->d[q]->a)));
  CKR(C, nullptr);
  Node* params = params_from_code(C, fe->cid, defs, kwd);
  CKR(C, nullptr);
  NV* body = decompile_body(C, fe->cid);
  CKR(C, nullptr);
  if (code_is_str_doc(C, fe->cid)) {
    NV* b2 = nv1(C, mk1(C, S_EXPR, mk_const(C, obj_const_id(C, fe->cid, 0))));
    vextend(C, b2, body);
    body = b2;
  }
  Node* d = mk(C, S_FUNCDEF);
  d->s = name;
  d->p = params;
  d->l1 = or_pass(C, body);
  d->l2 = vnew<Node*>(C);
  return d;
}

// _clean_class_body (recover.py:282-301)
HD inline NV* clean_class_body(Dc* C, NV* body) {
  NV* out = vnew<Node*>(C, body->n);
  for (u32 q = 0; q < body->n; q++) {
    Node* s = body->d[q];
    if (is_k(s, S_ASSIGN) && s->l1->n == 1 && is_k(s->l1->d[0], E_NAME)) {
      Str tid = s->l1->d[0]->s;
      if (s_eqc(tid, "__module__") && is_k(s->a, E_NAME)) continue;
      if (s_eqc(tid, "__qualname__") && is_k(s->a, E_CONST)) continue;
      if (s_eqc(tid, "__classcell__")) continue;
      if (s_eqc(tid, "__doc__") && is_k(s->a, E_CONST)) {
        vpush(C, out, mk1(C, S_EXPR, s->a));
        continue;
      }
    }
    if (is_k(s, S_RETURN)) continue;
    vpush(C, out, s);
  }
  return out;
}

HD NOINL Node* Recovery::make_classdef(Str name, Node* call) {  // recover.py:161-172
  NV* args = call->l1;
  if (args->n < 2 || !is_k(args->d[0], E_FUNC)) return nullptr;
  u32 cls_code = args->d[0]->cid;
  if (cls_code == CID_INVALID) {
    py_value_attr_error(C, args->d[0]->j, "code");
    return nullptr;
  }
  NV* bases = vnew<Node*>(C, args->n - 2);
  for (u32 q = 2; q < args->n; q++) vpush(C, bases, map_expr(args->d[q]));
  NV* kws = vnew<Node*>(C, call->l2->n);
  for (u32 q = 0; q < call->l2->n; q++) vpush(C, kws, mk_kwpair(C, call->l2->d[q]->s, map_expr(call->l2->d[q]->a)));
  CKR(C, nullptr);
  NV* body = decompile_body(C, cls_code);
  CKR(C, nullptr);
  body = clean_class_body(C, body);
  Node* d = mk(C, S_CLASSDEF);
  d->s = name;
  d->l1 = bases;
  d->l2 = kws;
  d->l3 = or_pass(C, body);
  d->l4 = vnew<Node*>(C);
  return d;
}

HD inline Node* Recovery::make_lambda(Node* fe) {  // recover.py:199-204
  NV* body = decompile_body(C, fe->cid);
  CKR(C, nullptr);
  if (body->n == 1 && is_k(body->d[0], S_RETURN)) {
    Node* params = params_from_code(C, fe->cid, fe->l1, fe->l2);
    CKR(C, nullptr);
    Node* lam = mk(C, E_LAMBDA);
    lam->p = params;
    lam->a = body->d[0]->a;
    return lam;
  }
  return nullptr;
}

// _match_comp_body (recover.py:230-279); returns accum (CompAccum or yield value)
HD inline bool match_comp_body(Dc* C, NV* body, Node** accum, NV** gens_out) {
  u32 n = body->n;
  if (n && is_k(body->d[n - 1], S_RETURN)) n--;
  if (n != 1 || !is_k(body->d[0], S_FOR)) return false;
  Node* node = body->d[0];
  NV* gens = vnew<Node*>(C, 2);
  while (!C->err) {
    if (node->l2->n) return false;
    Node* gen = mk(C, X_COMPFOR);
    gen->a = node->a;
    gen->b = node->b;
    gen->l1 = vnew<Node*>(C);
    vpush(C, gens, gen);
    NV* inner = node->l1;
    while (!C->err) {
      if (inner->n >= 2 && is_k(inner->d[0], S_IF) && inner->d[0]->l1->n == 1 &&
          is_k(inner->d[0]->l1->d[0], S_CONTINUE) && !inner->d[0]->l2->n) {
        vpush(C, gen->l1, negate(C, inner->d[0]->a));
        inner = vcopy<Node*>(C, inner, 1);
        continue;
      }
      if (inner->n == 1 && is_k(inner->d[0], S_IF) && !inner->d[0]->l2->n &&
          !(inner->d[0]->l1->n == 1 && is_k(inner->d[0]->l1->d[0], S_CONTINUE))) {
        vpush(C, gen->l1, inner->d[0]->a);
        inner = inner->d[0]->l1;
        continue;
      }
      break;
    }
    if (inner->n == 1 && is_k(inner->d[0], S_FOR)) {
      node = inner->d[0];
      continue;
    }
    if (inner->n == 1 && is_k(inner->d[0], S_COMPACCUM)) {
      *accum = inner->d[0];
      *gens_out = gens;
      return true;
    }
    if (inner->n == 1 && is_k(inner->d[0], S_EXPR) && is_k(inner->d[0]->a, E_YIELD)) {
      *accum = inner->d[0]->a->a;
      *gens_out = gens;
      return true;
    }
    return false;
  }
  return false;
}

HD NOINL Node* Recovery::make_comp(int kind, u32 code, Node* iter_arg) {  // recover.py:206-219
  NV* body = decompile_body(C, code);
  CKR(C, nullptr);
  Node* accum = nullptr;
  NV* gens = nullptr;
  if (!match_comp_body(C, body, &accum, &gens)) return nullptr;
  gens->d[0]->b = iter_arg;
  Node* c = mk(C, E_COMP);
  c->op = (u8)kind;
  c->l1 = gens;
  if (kind == 2) {
    if (!is_k(accum, S_COMPACCUM) || accum->op != 2) return nullptr;
    c->b = accum->b;
    c->c = accum->a;
    return c;
  }
  c->a = is_k(accum, S_COMPACCUM) ? accum->a : accum;
  return c;
}

HD NOINL Node* Recovery::match_def(Node* target, Node* value) {  // recover.py:123-148
  NV* decorators = vnew<Node*>(C);
  Node* inner = value;
  while (is_k(inner, E_CALL) && inner->l1->n == 1 && inner->l2->n == 0 && !is_k(inner->a, E_BUILDCLASS)) {
    vpush(C, decorators, inner->a);
    inner = inner->l1->d[0];
  }
  if (is_k(inner, E_CALL) && is_k(inner->a, E_BUILDCLASS)) {
    Node* made = make_classdef(target->s, inner);
    CKR(C, nullptr);
    if (made) {
      NV* ds = vnew<Node*>(C, decorators->n);
      for (u32 q = 0; q < decorators->n; q++) vpush(C, ds, map_expr(decorators->d[q]));
      made->l4 = ds;
      return made;
    }
    return nullptr;
  }
  if (is_k(inner, E_FUNC)) {
    Str nm = code_name_checked(C, inner);
    CKR(C, nullptr);
    if (s_eq(nm, target->s)) {
      Node* made = make_funcdef(target->s, inner);
      CKR(C, nullptr);
      NV* ds = vnew<Node*>(C, decorators->n);
      for (u32 q = 0; q < decorators->n; q++) vpush(C, ds, map_expr(decorators->d[q]));
      made->l2 = ds;
      return made;
    }
  }
  return nullptr;
}

// _stmt_exprs (recover.py:63-78), dataclass field order per statement kind
HD NOINL void Recovery::stmt_exprs(Node* s) {
  auto mx = [&](Node** f) {
    if (is_expr(*f)) *f = map_expr(*f);
  };
  auto ml = [&](NV** f) {  // list of Expr (non-empty, all Expr) -> new mapped list
    NV* v = *f;
    if (!v || !v->n) return;
    for (u32 q = 0; q < v->n; q++)
      if (!is_expr(v->d[q])) return;
    NV* out = vnew<Node*>(C, v->n);
    for (u32 q = 0; q < v->n; q++) vpush(C, out, map_expr(v->d[q]));
    *f = out;
  };
  switch (s->k) {
    case S_ASSIGN: ml(&s->l1); mx(&s->a); break;
    case S_AUGASSIGN: mx(&s->a); mx(&s->b); break;
    case S_EXPR: case S_RETURN: mx(&s->a); break;
    case S_RAISE: mx(&s->a); mx(&s->b); break;
    case S_DELETE: ml(&s->l1); break;
    case S_ASSERT: mx(&s->a); mx(&s->b); break;
    case S_IF: case S_WHILE: mx(&s->a); break;
    case S_FOR: mx(&s->a); mx(&s->b); break;
    case S_WITH:
      for (u32 q = 0; q < s->l1->n; q++) {
        Node* it = s->l1->d[q];
        it->a = map_expr(it->a);
        if (it->b) it->b = map_expr(it->b);
      }
      break;
    case S_FUNCDEF: ml(&s->l2); break;
    case S_CLASSDEF: {
      ml(&s->l1);
      NV* v = s->l2;
      for (u32 q = 0; v && q < v->n; q++) {
        Node* x = v->d[q];
        if (!is_k(x, X_KWPAIR) || !is_expr(x->a)) continue;
        u32 idx = q;  // v.index(x): first equal element
        for (u32 w = 0; w < v->n; w++)
          if (v->d[w] == x || node_eq(C, v->d[w], x)) {
            idx = w;
            break;
          }
        v->d[idx] = mk_kwpair(C, x->s, map_expr(x->a));
      }
      ml(&s->l4);
      break;
    }
    case S_CONDJUMP: mx(&s->a); break;
    case S_COMPACCUM: mx(&s->a); mx(&s->b); break;
    case S_WHILESHAPE: mx(&s->a); mx(&s->b); break;
    default: break;
  }
}

HD NOINL NV* Recovery::rewrite_stmt(Node* s) {  // recover.py:99-121
  GUARD(C);
  CKR(C, nullptr);
  if (is_k(s, S_ASSIGN) && s->l1->n == 1 && is_k(s->l1->d[0], E_NAME)) {
    Node* made = match_def(s->l1->d[0], s->a);
    CKR(C, nullptr);
    if (made) return nv1(C, made);
  }
  for (int f = 0; f < 4; f++) {
    NV** sub = stmt_field(s, f);
    if (sub && *sub && (*sub)->n && is_stmt((*sub)->d[0])) *sub = rewrite_block(*sub);
    CKR(C, nullptr);
  }
  if (is_k(s, S_TRY))
    for (u32 h = 0; h < s->l2->n; h++) s->l2->d[h]->l1 = rewrite_block(s->l2->d[h]->l1);
  if (is_k(s, S_WITH)) s->l2 = rewrite_block(s->l2);
  CKR(C, nullptr);
  stmt_exprs(s);
  CKR(C, nullptr);
  return nv1(C, s);
}
HD inline NV* Recovery::rewrite_block(NV* stmts) {
  NV* out = vnew<Node*>(C, stmts->n);
  for (u32 q = 0; q < stmts->n && !C->err; q++) {
    NV* rep = rewrite_stmt(stmts->d[q]);
    CKR(C, out);
    vextend(C, out, hoisted);
    hoisted = vnew<Node*>(C);
    vextend(C, out, rep);
  }
  return out;
}

// add_scope_decls (recover.py:304-357)
struct ScopeScan {
  Dc* C;
  const upy_obj* o;
  Vec<Str>* globals_seen;
  Vec<Str>* nonlocals_seen;
  HD bool in_free(Str id) {
    for (u32 q = 0; q < o->n_freevars; q++)
      if (s_eq(obj_tab(C, o->freevars_off, q), id)) return true;
    return false;
  }
  HD static bool has(Vec<Str>* v, Str s) {
    for (u32 q = 0; q < v->n; q++)
      if (s_eq(v->d[q], s)) return true;
    return false;
  }
  HD void note(Node* e) {
    if (!is_k(e, E_NAME)) return;
    if (e->op == SC_GLOBAL && !has(globals_seen, e->s)) vpush(C, globals_seen, e->s);
    if (e->op == SC_DEREF && in_free(e->s) && !has(nonlocals_seen, e->s)) vpush(C, nonlocals_seen, e->s);
  }
  HD void target(Node* t) {
    GUARD(C);
    CK(C);
    if (is_k(t, E_NAME)) note(t);
    else if (is_k(t, E_TUPLE) || is_k(t, E_LIST))
      for (u32 q = 0; q < t->l1->n; q++) target(t->l1->d[q]);
    else if (is_k(t, E_STARRED)) target(t->a);
  }
  HD void scan(NV* stmts) {
    GUARD(C);
    CK(C);
    for (u32 q = 0; stmts && q < stmts->n; q++) {
      Node* s = stmts->d[q];
      if (is_k(s, S_FUNCDEF) || is_k(s, S_CLASSDEF)) continue;
      if (is_k(s, S_ASSIGN) || is_k(s, S_DELETE)) {
        for (u32 t = 0; t < s->l1->n; t++) target(s->l1->d[t]);
      } else if (is_k(s, S_AUGASSIGN) || is_k(s, S_FOR)) {
        target(s->a);
      }
      // _child_blocks (ir.py:461-472)
      switch (s->k) {
        case S_IF: scan(s->l1); scan(s->l2); break;
        case S_WHILE: case S_FOR: scan(s->l1); scan(s->l2); break;
        case S_TRY:
          scan(s->l1);
          for (u32 h = 0; h < s->l2->n; h++) scan(s->l2->d[h]->l1);
          scan(s->l3);
          scan(s->l4);
          break;
        case S_WITH: scan(s->l2); break;
      }
    }
  }
};
HD NOINL NV* add_scope_decls(Dc* C, NV* body, u32 oi) {
  ScopeScan sc;
  sc.C = C;
  sc.o = obj_at(C, oi);
  sc.globals_seen = vnew<Str>(C);
  sc.nonlocals_seen = vnew<Str>(C);
  sc.scan(body);
  CKR(C, body);
  if (!sc.globals_seen->n && !sc.nonlocals_seen->n) return body;
  u32 insert = (body->n && is_k(body->d[0], S_EXPR) && is_k(body->d[0]->a, E_CONST)) ? 1 : 0;
  NV* out = vnew<Node*>(C, body->n + 2);
  vextend(C, out, body, 0, insert);
  if (sc.globals_seen->n) {
    Node* g = mk(C, S_GLOBAL);
    g->sl = sc.globals_seen;
    vpush(C, out, g);
  }
  if (sc.nonlocals_seen->n) {
    Node* g = mk(C, S_NONLOCAL);
    g->sl = sc.nonlocals_seen;
    vpush(C, out, g);
  }
  vextend(C, out, body, insert);
  return out;
}

HD inline bool is_return_none(Dc* C, Node* s) {  // pipeline.py:113-118
  if (!is_k(s, S_RETURN) || !is_k(s->a, E_CONST)) return false;
  return node_ckind(C, s->a) == UPY_C_NONE;
}

// decompile_body (pipeline.py:90-110), as stages so the kernel can run a root
// object's stages in warp lockstep (upy.cu); nested bodies run them back to back.
struct BodyJob {
  u32 oi;
  u32 defs_before;
  Code* K;
  Cfg* G;
  NV* stmts;
};
HD NOINL bool body_analyze(Dc* C, BodyJob* J) {  // decode check + CFG (pipeline.py:92, 17-54)
  J->K = anew<Code>(C);
  CKR(C, false);
  J->defs_before = C->n_defs;
  if (!load_instructions(C, J->K, J->oi)) return false;
  J->G = analyze(C, J->K);
  return !C->err;
}
HD NOINL bool body_structure(Dc* C, BodyJob* J) {  // Structurer + canonicalize (pipeline.py:93-95)
  Structurer* S_ = make_structurer(C, J->K, J->G);
  CKR(C, false);
  NV* stmts = S_->structure();
  CKR(C, false);
  J->stmts = canonicalize_tree(C, stmts);
  return !C->err;
}
HD NOINL bool body_finish(Dc* C, BodyJob* J) {  // DefRecovery, scope decls, implicit return (:96-110)
  NV* stmts = J->stmts;
  // DefRecovery (recover.py:81-227) only ever changes a tree through FuncExpr
  // and BuildClass nodes (pre/post hooks, _match_def); everything else it does
  // is rebuilding lists with identical contents.  When the simulation of this
  // object created neither, the pass is skipped: the output is identical.
  if (C->n_defs != J->defs_before) {
    Recovery R;
    R.C = C;
    R.oi = J->oi;
    R.hoisted = vnew<Node*>(C);
    R.lambda_counter = 0;
    stmts = R.rewrite_block(stmts);
    CKR(C, false);
  }
  stmts = add_scope_decls(C, stmts, J->oi);
  CKR(C, false);
  const upy_obj* o = obj_at(C, J->oi);
  if (o->flags & (0x20 | 0x200)) {
    while (stmts->n && is_return_none(C, vlast(stmts))) stmts->n--;
  } else if (stmts->n && is_return_none(C, vlast(stmts))) {
    stmts->n--;
  }
  J->stmts = stmts;
  return !C->err;
}
HD NOINL NV* decompile_body(Dc* C, u32 oi) {
  GUARD(C);
  CKR(C, nullptr);
  BodyJob J;
  J.oi = oi;
  if (!body_analyze(C, &J) || !body_structure(C, &J) || !body_finish(C, &J)) return nullptr;
  return J.stmts;
}
