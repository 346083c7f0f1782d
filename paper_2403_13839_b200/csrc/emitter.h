// emitter.h -- source text rendering (emitter.py:19-551): 16-level precedence,
// statements streamed straight into the object's text buffer, constants via
// numfmt.h, plus the dataclass repr the reference puts in InternalMarkerLeak.
#pragma once
#include "recover.h"
#include "numfmt.h"

enum {
  P_LAMBDA = 1, P_TERNARY, P_OR, P_AND, P_NOT, P_COMPARE, P_BITOR, P_BITXOR, P_BITAND, P_SHIFT,
  P_ARITH, P_TERM, P_UNARY, P_POWER, P_AWAIT, P_ATOM
};
HD inline int binop_prec(u8 op) {
  switch (op) {
    case BO_OR: return P_BITOR;
    case BO_XOR: return P_BITXOR;
    case BO_AND: return P_BITAND;
    case BO_LSHIFT: case BO_RSHIFT: return P_SHIFT;
    case BO_ADD: case BO_SUB: return P_ARITH;
    case BO_POW: return P_POWER;
  }
  return P_TERM;
}
HD inline const char* binop_str(u8 op) {
  switch (op) {
    case BO_ADD: return "+"; case BO_AND: return "&"; case BO_FLOORDIV: return "//";
    case BO_LSHIFT: return "<<"; case BO_MATMUL: return "@"; case BO_MUL: return "*";
    case BO_MOD: return "%"; case BO_OR: return "|"; case BO_POW: return "**";
    case BO_RSHIFT: return ">>"; case BO_SUB: return "-"; case BO_TRUEDIV: return "/";
  }
  return "^";
}
HD inline const char* cmp_str(u8 c) {
  if (c < UPY_NCMP_ALL) return T_CMPOP[c];
  return "None";
}
HD inline const char* unary_str(u8 op) {
  switch (op) {
    case UO_NOT: return "not"; case UO_NEG: return "-"; case UO_POS: return "+";
  }
  return "~";
}

struct Emitter {
  Dc* C;
  Text* out;
  int depth;
  Str indent;

  // ---------------------------------------------------------- dataclass repr
  HD void r_str(Text* t, Str s) {
    if (s_is_none(s)) t_puts(C, t, "None");
    else t_str_repr(C, t, s);
  }
  HD void r_const_value(Text* t, u32 cid);
  HD void r_const(Text* t, u32 cid) {  // Const.__repr__ (code_model.py:94-97)
    if (cid == CID_INVALID) {
      t_puts(C, t, "None");
      return;
    }
    u32 k = ckind(C, cid);
    const char* kn = k == UPY_C_NONE ? "none" : k == UPY_C_BOOL ? "bool" : k == UPY_C_INT ? "int"
                     : k == UPY_C_FLOAT ? "float" : k == UPY_C_COMPLEX ? "complex" : k == UPY_C_STR ? "str"
                     : k == UPY_C_BYTES ? "bytes" : k == UPY_C_TUPLE ? "tuple" : k == UPY_C_FROZENSET ? "frozenset"
                     : k == UPY_C_CODE ? "code" : "ellipsis";
    t_puts(C, t, "Const(");
    t_puts(C, t, kn);
    if (k != UPY_C_NONE && k != UPY_C_ELLIPSIS) {
      t_puts(C, t, ", ");
      r_const_value(t, cid);
    }
    t_put(C, t, ')');
  }
  HD void r_list(Text* t, NV* v, bool tuple = false) {
    t_put(C, t, tuple ? '(' : '[');
    for (u32 q = 0; v && q < v->n; q++) {
      if (q) t_puts(C, t, ", ");
      r_node(t, v->d[q]);
    }
    if (tuple && v && v->n == 1) t_put(C, t, ',');
    t_put(C, t, tuple ? ')' : ']');
  }
  HD void r_strlist(Text* t, Vec<Str>* v, bool tuple) {
    t_put(C, t, tuple ? '(' : '[');
    for (u32 q = 0; v && q < v->n; q++) {
      if (q) t_puts(C, t, ", ");
      r_str(t, v->d[q]);
    }
    if (tuple && v && v->n == 1) t_put(C, t, ',');
    t_put(C, t, tuple ? ')' : ']');
  }
  HD void r_field(Text* t, const char* name, bool first) {
    if (!first) t_puts(C, t, ", ");
    t_puts(C, t, name);
    t_put(C, t, '=');
  }
  HD void r_node(Text* t, const Node* n);

  // ---------------------------------------------------------- constants
  HD void render_float(Text* t, double v) {  // _render_float (emitter.py:83-90)
    if (d_isnan(v)) { t_puts(C, t, "float('nan')"); return; }
    if (d_isinf(v)) { t_puts(C, t, v > 0 ? "float('inf')" : "float('-inf')"); return; }
    t_float_repr(C, t, v);
  }
  HD void imag_literal(Text* t, double im) {  // _imag_literal (emitter.py:105-109)
    if (d_isinf(im)) {
      t_puts(C, t, "complex(0.0, ");
      render_float(t, im);
      t_put(C, t, ')');
      return;
    }
    t_float_repr(C, t, im);
    t_put(C, t, 'j');
  }
  HD NOINL void render_constant(Text* t, u32 cid) {  // emitter.py:53-80
    GUARD(C);
    CK(C);
    if (cid == CID_INVALID) {
      py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'kind'");
      return;
    }
    u32 k = ckind(C, cid);
    switch (k) {
      case UPY_C_NONE: t_puts(C, t, "None"); return;
      case UPY_C_BOOL: t_puts(C, t, cbool(C, cid) ? "True" : "False"); return;
      case UPY_C_ELLIPSIS: t_puts(C, t, "..."); return;
      case UPY_C_INT: {
        const upy_const* c = cget(C, cid);
        t_int_repr(C, t, c->ival, C->limbs + c->off, c->n);
        return;
      }
      case UPY_C_FLOAT: render_float(t, cget(C, cid)->re); return;
      case UPY_C_COMPLEX: {  // _render_complex (emitter.py:93-102)
        double re = cget(C, cid)->re, im = cget(C, cid)->im;
        if (re == 0.0 && !d_signbit(re) && !d_isnan(im)) {
          imag_literal(t, im);
          return;
        }
        if (d_isnan(re) || d_isinf(re) || d_isnan(im) || d_isinf(im)) {
          t_puts(C, t, "complex(");
          render_float(t, re);
          t_puts(C, t, ", ");
          render_float(t, im);
          t_put(C, t, ')');
          return;
        }
        t_put(C, t, '(');
        render_float(t, re);
        if (!d_signbit(im)) {
          t_puts(C, t, " + ");
          imag_literal(t, im);
        } else {
          t_puts(C, t, " - ");
          imag_literal(t, -im);
        }
        t_put(C, t, ')');
        return;
      }
      case UPY_C_STR: t_str_repr(C, t, cstr(C, cid)); return;
      case UPY_C_BYTES: {
        const upy_const* c = cget(C, cid);
        t_bytes_repr(C, t, C->bytes + c->off, c->n);
        return;
      }
      case UPY_C_TUPLE: {
        u32 n = cnelem(C, cid);
        if (!n) { t_puts(C, t, "()"); return; }
        t_put(C, t, '(');
        for (u32 q = 0; q < n && !C->err; q++) {
          if (q) t_puts(C, t, ", ");
          render_constant(t, celem(C, cid, q));
        }
        t_puts(C, t, n == 1 ? ",)" : ")");
        return;
      }
      case UPY_C_FROZENSET: {
        u32 n = cnelem(C, cid);
        if (!n) { t_puts(C, t, "frozenset()"); return; }
        t_puts(C, t, "frozenset({");
        for (u32 q = 0; q < n && !C->err; q++) {
          if (q) t_puts(C, t, ", ");
          render_constant(t, celem(C, cid, q));
        }
        t_puts(C, t, "})");
        return;
      }
    }
    // code constants cannot be rendered inline (emitter.py:80)
    Text m;
    if (fail_begin(C, UPY_ST_MARKER_LEAK, 0, 0, &m)) {
      m_puts(C, &m, "constant kind code cannot be rendered inline");
      fail_end(C, &m);
    }
  }
  HD bool const_text_negative(u32 cid) {  // text.startswith("-")
    u32 k = ckind(C, cid);
    if (k == UPY_C_INT) return cget(C, cid)->ival < 0 && cget(C, cid)->n > 0;
    if (k == UPY_C_FLOAT) {
      double v = cget(C, cid)->re;
      return d_signbit(v) && !d_isnan(v) && !d_isinf(v);
    }
    return false;
  }

  // ---------------------------------------------------------- lines
  HD void line_start() {
    for (int q = 0; q < depth; q++) t_str(C, out, indent);
  }
  HD void line_end() { t_put(C, out, '\n'); }
  HD void simple_line(const char* s) {
    line_start();
    t_puts(C, out, s);
    line_end();
  }
  HD void block(NV* stmts) {
    depth++;
    if (!stmts || !stmts->n) simple_line("pass");
    for (u32 q = 0; stmts && q < stmts->n && !C->err; q++) stmt(stmts->d[q]);
    depth--;
  }
  HD void stmt(Node* s);
  HD NOINL void funcdef_head(Node* s) {  // decorators and the def line (emitter.py:285-295)
    for (u32 q = 0; q < s->l2->n && !C->err; q++) {
      line_start();
      t_put(C, out, '@');
      concat_none(sub(out, s->l2->d[q]));
      line_end();
    }
    line_start();
    t_puts(C, out, "def ");
    t_str(C, out, s->s);
    t_put(C, out, '(');
    params(out, s->p);
    t_puts(C, out, "):");
    line_end();
  }
  HD void emit_if(Node* s, const char* kw);
  HD void params(Text* t, Node* p);
  // Python-None text.  In the reference a Name whose id is None (an
  // out-of-range name index) renders as the None object: f-strings print
  // "None", but str.join / "+" / .startswith on it raise.  expr(), target()
  // and callarg() return true when their result is that None object.
  struct Join {
    i64 bad;
    u32 i;
  };
  HD static Join join0() { return Join{-1, 0}; }
  HD static void join_item(Join& j, bool none) {
    if (none && j.bad < 0) j.bad = j.i;
    j.i++;
  }
  HD FORCEINL void join_end(const Join& j) {  // str.join: items are all evaluated first
    if (j.bad >= 0) join_fail(j);
  }
  HD NOINL void join_fail(const Join& j) {
    Text m;
    if (fail_begin(C, UPY_ST_PY_TYPE_ERROR, 0, 0, &m)) {
      m_puts(C, &m, "sequence item ");
      m_i64(C, &m, j.bad);
      m_puts(C, &m, ": expected str instance, NoneType found");
      fail_end(C, &m);
    }
  }
  HD void concat_none(bool none) {  // "..." + None
    if (none) py_error(C, UPY_ST_PY_TYPE_ERROR, "can only concatenate str (not \"NoneType\") to str");
  }
  HD bool target(Text* t, Node* e, bool nested);
  HD int prec_of(const Node* e, bool* ok);
  HD bool expr(Text* t, Node* e, int parent = 0, bool right_side = false);
  // sub() with the leaf cases inline: names and None / small non-negative int
  // constants are atoms (never parenthesised, never None-text), so they skip the
  // recursive call (its register save/restore was the emitter's main cost).
  HD FORCEINL bool sub(Text* t, Node* e, int parent = 0, bool right_side = false) {
    if (e && !C->err) {
      if (e->k == E_NAME && !s_is_none(e->s)) {
        t_str(C, t, e->s);
        return false;
      }
      if (e->k == E_CONST && e->cid < CID_NONE_SYN) {
        const upy_const* c = cget(C, e->cid);
        if (c->kind == UPY_C_INT && c->n == 1 && c->ival >= 0) {
          t_u32(C, t, C->limbs[c->off]);
          return false;
        }
        if (c->kind == UPY_C_NONE) {
          t_puts(C, t, "None");
          return false;
        }
      }
    }
    return expr(t, e, parent, right_side);
  }
  HD void expr_body(Text* t, Node* e);
  HD bool callarg(Text* t, Node* a) {
    if (is_k(a, E_STARRED)) {
      t_put(C, t, '*');
      concat_none(sub(t, a->a, P_LAMBDA));
      return false;
    }
    return sub(t, a, P_LAMBDA);
  }
  HD void index(Text* t, Node* idx);
  HD void slice(Text* t, Node* s);
  HD void format_part(Text* t, Node* fv);
  HD void format_spec(Text* t, Node* spec);
  HD void name_text(Text* t, Str s) {
    if (s_is_none(s)) t_puts(C, t, "None");
    else t_str(C, t, s);
  }
};

// ------------------------------------------------------------ repr
HD inline void Emitter::r_const_value(Text* t, u32 cid) {
  u32 k = ckind(C, cid);
  switch (k) {
    case UPY_C_BOOL: t_puts(C, t, cbool(C, cid) ? "True" : "False"); return;
    case UPY_C_INT: {
      const upy_const* c = cget(C, cid);
      t_int_repr(C, t, c->ival, C->limbs + c->off, c->n);
      return;
    }
    case UPY_C_FLOAT: t_float_repr(C, t, cget(C, cid)->re); return;
    case UPY_C_COMPLEX: t_complex_repr(C, t, cget(C, cid)->re, cget(C, cid)->im); return;
    case UPY_C_STR: t_str_repr(C, t, cstr(C, cid)); return;
    case UPY_C_BYTES: t_bytes_repr(C, t, C->bytes + cget(C, cid)->off, cget(C, cid)->n); return;
    case UPY_C_TUPLE:
    case UPY_C_FROZENSET: {
      u32 n = cnelem(C, cid);
      t_put(C, t, '(');
      for (u32 q = 0; q < n; q++) {
        if (q) t_puts(C, t, ", ");
        r_const(t, celem(C, cid, q));
      }
      if (n == 1) t_put(C, t, ',');
      t_put(C, t, ')');
      return;
    }
    case UPY_C_CODE: t_puts(C, t, "CodeObject(...)"); return;
  }
  t_puts(C, t, "None");
}

HD NOINL void Emitter::r_node(Text* t, const Node* n) {
  GUARD(C);
  CK(C);
  if (!n) {
    t_puts(C, t, "None");
    return;
  }
#define RN(name, f, first) r_field(t, name, first); r_node(t, n->f)
#define RL(name, f, first) r_field(t, name, first); r_list(t, n->f)
#define RS(name, f, first) r_field(t, name, first); r_str(t, n->f)
#define RI(name, f, first) r_field(t, name, first); t_i64(C, t, n->f)
  switch (n->k) {
    case E_CONST: t_puts(C, t, "ConstE("); r_field(t, "const", true); r_const(t, n->cid); break;
    case E_NAME: {
      t_puts(C, t, "Name("); RS("id", s, true);
      const char* sc = n->op == SC_FAST ? "fast" : n->op == SC_GLOBAL ? "global" : n->op == SC_DEREF ? "deref"
                       : n->op == SC_NAME ? "name" : "cell";
      r_field(t, "scope", false); t_str_repr(C, t, S(sc));
      break;
    }
    case E_BINOP:
      t_puts(C, t, "BinOp("); r_field(t, "op", true); t_str_repr(C, t, S(binop_str(n->op)));
      RN("left", a, false); RN("right", b, false);
      r_field(t, "inplace", false); t_puts(C, t, (n->f & 1) ? "True" : "False");
      break;
    case E_UNARY:
      t_puts(C, t, "UnaryOp("); r_field(t, "op", true); t_str_repr(C, t, S(unary_str(n->op))); RN("operand", a, false);
      break;
    case E_COMPARE: t_puts(C, t, "Compare("); RN("left", a, true); RL("ops", l1, false); RL("comparators", l2, false); break;
    case E_BOOLOP:
      t_puts(C, t, "BoolOp("); r_field(t, "op", true); t_str_repr(C, t, S(n->op ? "or" : "and")); RL("values", l1, false);
      break;
    case E_CALL: t_puts(C, t, "Call("); RN("func", a, true); RL("args", l1, false); RL("keywords", l2, false); break;
    case E_ATTR: t_puts(C, t, "Attr("); RN("value", a, true); RS("name", s, false); break;
    case E_SUBSCR: t_puts(C, t, "Subscript("); RN("value", a, true); RN("index", b, false); break;
    case E_SLICE: t_puts(C, t, "SliceE("); RN("lower", a, true); RN("upper", b, false); RN("step", c, false); break;
    case E_TUPLE: t_puts(C, t, "TupleE("); RL("elts", l1, true); break;
    case E_LIST: t_puts(C, t, "ListE("); RL("elts", l1, true); break;
    case E_SET: t_puts(C, t, "SetE("); RL("elts", l1, true); break;
    case E_DICT: t_puts(C, t, "DictE("); RL("keys", l1, true); RL("values", l2, false); break;
    case E_STARRED: t_puts(C, t, "Starred("); RN("value", a, true); break;
    case E_FMTVAL: {
      t_puts(C, t, "FormattedValue("); RN("value", a, true);
      const char* cv = n->op == 1 ? "s" : n->op == 2 ? "r" : n->op == 3 ? "a" : "";
      r_field(t, "conversion", false); t_str_repr(C, t, S(cv)); RN("format_spec", b, false);
      break;
    }
    case E_FSTRING: t_puts(C, t, "FString("); RL("parts", l1, true); break;
    case E_TERNARY: t_puts(C, t, "Ternary("); RN("cond", a, true); RN("then", b, false); RN("orelse", c, false); break;
    case E_YIELD: t_puts(C, t, "Yield("); RN("value", a, true); break;
    case E_YIELDFROM: t_puts(C, t, "YieldFrom("); RN("value", a, true); break;
    case E_NAMED: t_puts(C, t, "NamedExpr("); RN("target", a, true); RN("value", b, false); break;
    case E_LAMBDA: t_puts(C, t, "Lambda("); RN("params", p, true); RN("body", a, false); break;
    case E_COMP: {
      t_puts(C, t, "CompExpr(");
      const char* kd = n->op == 0 ? "list" : n->op == 1 ? "set" : n->op == 2 ? "dict" : "gen";
      r_field(t, "kind", true); t_str_repr(C, t, S(kd));
      RN("elt", a, false); RN("key", b, false); RN("value", c, false); RL("generators", l1, false);
      break;
    }
    case E_FUNC:
      t_puts(C, t, "FuncExpr("); r_field(t, "code", true); t_puts(C, t, "CodeObject(...)");
      RL("defaults", l1, false); RL("kwdefaults", l2, false); RL("annotations", l3, false);
      r_field(t, "closure", false); r_strlist(t, n->sl, true);
      break;
    case E_STACKTEMP: t_puts(C, t, "StackTemp("); RI("index", i, true); break;
    case E_NULL: t_puts(C, t, "NullSlot("); break;
    case E_METHSELF: t_puts(C, t, "MethodSelf("); break;
    case E_EXCVALUE: t_puts(C, t, "ExcValue("); RI("slot", i, true); break;
    case E_FINSENT: t_puts(C, t, "FinallySentinel("); break;
    case E_UNPACKSLOT:
      t_puts(C, t, "UnpackSlot("); RN("source", a, true); RI("count", i, false); RI("index", j, false);
      RI("star_index", kk, false); RI("after_count", m, false); RN("group", p, false);
      break;
    case E_IMPORT:
      t_puts(C, t, "ImportExpr("); RS("module", s, true); r_field(t, "fromlist", false);
      if (n->f & 2) r_strlist(t, n->sl, true); else t_puts(C, t, "None");
      r_field(t, "level", false);
      if (n->cid != CID_INVALID && ckind(C, n->cid) != UPY_C_NONE) r_const_value(t, n->cid); else t_puts(C, t, "None");
      break;
    case E_IMPORTFROM: t_puts(C, t, "ImportFromExpr("); RN("source", a, true); RS("name", s, false); break;
    case E_BUILDCLASS: t_puts(C, t, "BuildClass("); break;
    case E_FORITEM: t_puts(C, t, "ForItem("); RN("iter", a, true); break;
    case E_WITHEXIT: t_puts(C, t, "WithExit("); RN("context", a, true); break;
    case E_WITHENTER: t_puts(C, t, "WithEnter("); RN("context", a, true); break;
    case X_STRPART:
      if (n->i) t_str_repr(C, t, S(cmp_str(n->op))); else t_str_repr(C, t, n->s);
      return;
    case X_KWPAIR:
      t_put(C, t, '('); r_str(t, n->s); t_puts(C, t, ", "); r_node(t, n->a); t_put(C, t, ')');
      return;
    case X_NAMEPAIR:
      t_put(C, t, '('); r_str(t, n->s); t_puts(C, t, ", "); r_str(t, n->s2); t_put(C, t, ')');
      return;
    case X_COMPFOR: t_puts(C, t, "CompFor("); RN("target", a, true); RN("iter", b, false); RL("ifs", l1, false); break;
    case X_HANDLER: t_puts(C, t, "ExceptHandler("); RN("type", a, true); RS("name", s, false); RL("body", l1, false); break;
    case X_WITHITEM: t_puts(C, t, "WithItem("); RN("context", a, true); RN("target", b, false); break;
    case X_PARAMS: {
      t_puts(C, t, "Params("); r_field(t, "args", true); r_strlist(t, n->sl, false);
      RI("posonly", i, false); RS("vararg", s, false); r_field(t, "kwonly", false); r_strlist(t, n->sl2, false);
      RS("kwarg", s2, false); RL("defaults", l1, false); r_field(t, "kwdefaults", false);
      t_put(C, t, '{');
      bool first = true;
      for (u32 q = 0; n->l2 && q < n->l2->n; q++) {
        if (kw_lookup(n->l2, n->l2->d[q]->s) != n->l2->d[q]) continue;
        if (!first) t_puts(C, t, ", ");
        first = false;
        r_str(t, n->l2->d[q]->s); t_puts(C, t, ": "); r_node(t, n->l2->d[q]->a);
      }
      t_put(C, t, '}');
      break;
    }
    case X_GROUP: {
      t_puts(C, t, "UnpackGroup("); RN("source", a, true); RI("total", i, false); RI("star_index", kk, false);
      RL("targets", l1, false); r_field(t, "parent", false);
      if (n->p) { t_put(C, t, '('); r_node(t, n->p); t_puts(C, t, ", "); t_i64(C, t, n->j); t_put(C, t, ')'); }
      else t_puts(C, t, "None");
      break;
    }
    case S_ASSIGN: t_puts(C, t, "Assign("); RL("targets", l1, true); RN("value", a, false); break;
    case S_AUGASSIGN:
      t_puts(C, t, "AugAssign("); RN("target", a, true); r_field(t, "op", false); t_str_repr(C, t, S(binop_str(n->op)));
      RN("value", b, false);
      break;
    case S_EXPR: t_puts(C, t, "ExprStmt("); RN("value", a, true); break;
    case S_RETURN: t_puts(C, t, "Return("); RN("value", a, true); break;
    case S_RAISE: t_puts(C, t, "Raise("); RN("exc", a, true); RN("cause", b, false); break;
    case S_DELETE: t_puts(C, t, "Delete("); RL("targets", l1, true); break;
    case S_IMPORT: t_puts(C, t, "Import("); RS("module", s, true); RS("asname", s2, false); break;
    case S_IMPORTFROM:
      t_puts(C, t, "ImportFrom("); RS("module", s, true); RL("names", l1, false); r_field(t, "level", false);
      r_const_value(t, n->cid);
      break;
    case S_IMPORTSTAR:
      t_puts(C, t, "ImportStar("); RS("module", s, true); r_field(t, "level", false); r_const_value(t, n->cid);
      break;
    case S_PASS: t_puts(C, t, "Pass("); break;
    case S_GLOBAL: t_puts(C, t, "Global("); r_field(t, "names", true); r_strlist(t, n->sl, false); break;
    case S_NONLOCAL: t_puts(C, t, "Nonlocal("); r_field(t, "names", true); r_strlist(t, n->sl, false); break;
    case S_ASSERT: t_puts(C, t, "Assert("); RN("test", a, true); RN("msg", b, false); break;
    case S_IF: t_puts(C, t, "If("); RN("cond", a, true); RL("then", l1, false); RL("orelse", l2, false); break;
    case S_WHILE: t_puts(C, t, "While("); RN("cond", a, true); RL("body", l1, false); RL("orelse", l2, false); break;
    case S_FOR:
      t_puts(C, t, "For("); RN("target", a, true); RN("iter", b, false); RL("body", l1, false); RL("orelse", l2, false);
      break;
    case S_TRY:
      t_puts(C, t, "Try("); RL("body", l1, true); RL("handlers", l2, false); RL("orelse", l3, false);
      RL("final", l4, false);
      break;
    case S_WITH: t_puts(C, t, "With("); RL("items", l1, true); RL("body", l2, false); break;
    case S_FUNCDEF:
      t_puts(C, t, "FuncDef("); RS("name", s, true); RN("params", p, false); RL("body", l1, false);
      RL("decorators", l2, false); r_field(t, "is_async", false); t_puts(C, t, (n->f & 4) ? "True" : "False");
      break;
    case S_CLASSDEF:
      t_puts(C, t, "ClassDef("); RS("name", s, true); RL("bases", l1, false); RL("keywords", l2, false);
      RL("body", l3, false); RL("decorators", l4, false);
      break;
    case S_BREAK: t_puts(C, t, "Break("); break;
    case S_CONTINUE: t_puts(C, t, "Continue("); break;
    case S_JUMP: t_puts(C, t, "JumpMarker("); RI("target", i, true); break;
    case S_CONDJUMP:
      t_puts(C, t, "CondJumpMarker("); RN("cond", a, true); r_field(t, "jump_when", false);
      t_puts(C, t, (n->f & 1) ? "True" : "False"); RI("target", i, false);
      r_field(t, "pops_on_jump", false); t_puts(C, t, (n->f & 2) ? "True" : "False");
      break;
    case S_COMPACCUM: {
      t_puts(C, t, "CompAccum(");
      const char* kd = n->op == 0 ? "list" : n->op == 1 ? "set" : "map";
      r_field(t, "kind", true); t_str_repr(C, t, S(kd));
      RN("value", a, false); RN("key", b, false); RI("depth", i, false);
      break;
    }
    case S_WHILESHAPE:
      t_puts(C, t, "_WhileShape("); RN("cond", a, true); RL("body", l1, false); RL("orelse", l2, false);
      RN("tail_cond", b, false);
      break;
    default: t_puts(C, t, "<node"); break;
  }
  t_put(C, t, ')');
#undef RN
#undef RL
#undef RS
#undef RI
}

HD inline const char* class_name_of(const Node* n) {
  if (!n) return "NoneType";
  switch (n->k) {
    case E_SLICE: return "SliceE";
    case E_FMTVAL: return "FormattedValue";
    case E_FUNC: return "FuncExpr";
    case E_STACKTEMP: return "StackTemp";
    case E_NULL: return "NullSlot";
    case E_METHSELF: return "MethodSelf";
    case E_EXCVALUE: return "ExcValue";
    case E_FINSENT: return "FinallySentinel";
    case E_UNPACKSLOT: return "UnpackSlot";
    case E_IMPORT: return "ImportExpr";
    case E_IMPORTFROM: return "ImportFromExpr";
    case E_BUILDCLASS: return "BuildClass";
    case E_FORITEM: return "ForItem";
    case E_WITHEXIT: return "WithExit";
    case E_WITHENTER: return "WithEnter";
    case X_STRPART: return "str";
    case X_KWPAIR: case X_NAMEPAIR: return "tuple";
    case X_COMPFOR: return "CompFor";
    case X_HANDLER: return "ExceptHandler";
    case X_WITHITEM: return "WithItem";
    case X_PARAMS: return "Params";
    case X_GROUP: return "UnpackGroup";
  }
  return "Node";
}

// ------------------------------------------------------------ expressions
HD inline int Emitter::prec_of(const Node* e, bool* ok) {
  *ok = true;
  if (!e) { *ok = false; return 0; }
  switch (e->k) {
    case E_CONST: {
      if (e->cid == CID_INVALID) return P_ATOM;
      u32 k = ckind(C, e->cid);
      if (k == UPY_C_COMPLEX || const_text_negative(e->cid)) return P_UNARY;
      return P_ATOM;
    }
    case E_NAME: case E_STACKTEMP: return P_ATOM;
    case E_BINOP: return binop_prec(e->op);
    case E_UNARY: return e->op == UO_NOT ? P_NOT : P_UNARY;
    case E_COMPARE: return P_COMPARE;
    case E_BOOLOP: return e->op ? P_OR : P_AND;
    case E_TERNARY: return P_TERNARY;
    case E_LAMBDA: case E_NAMED: case E_STARRED: return P_LAMBDA;
    case E_CALL: case E_ATTR: case E_SUBSCR: case E_TUPLE: case E_LIST: case E_SET: case E_DICT:
    case E_YIELD: case E_YIELDFROM: case E_COMP: case E_FSTRING:
      return P_ATOM;
  }
  *ok = false;
  return 0;
}

HD NOINL bool Emitter::expr(Text* t, Node* e, int parent, bool right_side) {
  GUARD(C);
  CKR(C, false);
  bool ok;
  int prec = prec_of(e, &ok);
  if (!ok) {  // no emitter for this expression type (emitter.py:324-328)
    Text m;
    if (fail_begin(C, UPY_ST_MARKER_LEAK, 0, 0, &m)) {
      // the repr is rendered into a scratch text first, then copied
      m_puts(C, &m, "no emitter for expression ");
      m_puts(C, &m, class_name_of(e));
      m_puts(C, &m, ": ");
      u32 keep = m.n;
      C->err = 0;  // allow the repr scratch to allocate
      Text r = {nullptr, 0, 0};
      r_node(&r, e);
      int st2 = C->err;
      C->err = UPY_ST_MARKER_LEAK;
      if (!st2) m_putn(C, &m, r.d, r.n);
      (void)keep;
      fail_end(C, &m);
    }
    return false;
  }
  bool paren = prec < parent || (prec == parent && right_side && prec != P_ATOM);
  if (paren) t_put(C, t, '(');
  expr_body(t, e);
  if (paren) t_put(C, t, ')');
  return !paren && e->k == E_NAME && s_is_none(e->s);
}

HD FORCEINL void Emitter::expr_body(Text* t, Node* e) {  // only caller: sub()
  switch (e->k) {
    case E_CONST: render_constant(t, e->cid); return;
    case E_NAME: name_text(t, e->s); return;
    case E_STACKTEMP: t_puts(C, t, "__stack_"); t_i64(C, t, e->i); return;
    case E_BINOP: {
      int p = binop_prec(e->op);
      if (e->op == BO_POW) {
        sub(t, e->a, p, true);
        t_puts(C, t, " ** ");
        sub(t, e->b, p);
      } else {
        sub(t, e->a, p);
        t_put(C, t, ' ');
        t_puts(C, t, binop_str(e->op));
        t_put(C, t, ' ');
        sub(t, e->b, p, true);
      }
      return;
    }
    case E_UNARY:
      if (e->op == UO_NOT) {
        t_puts(C, t, "not ");
        sub(t, e->a, P_NOT);
      } else {
        t_puts(C, t, unary_str(e->op));
        sub(t, e->a, P_UNARY);
      }
      return;
    case E_COMPARE: {  // " ".join([left, op, operand, ...])
      Join j = join0();
      join_item(j, sub(t, e->a, P_COMPARE, true));
      u32 n = e->l1->n < e->l2->n ? e->l1->n : e->l2->n;
      for (u32 q = 0; q < n && !C->err; q++) {
        u8 c = e->l1->d[q]->op;
        join_item(j, c == CO_NONE);
        t_put(C, t, ' ');
        t_puts(C, t, cmp_str(c));
        t_put(C, t, ' ');
        join_item(j, sub(t, e->l2->d[q], P_COMPARE, true));
      }
      join_end(j);
      return;
    }
    case E_BOOLOP: {
      int p = e->op ? P_OR : P_AND;
      Join j = join0();
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        if (q) t_puts(C, t, e->op ? " or " : " and ");
        join_item(j, sub(t, e->l1->d[q], p, q > 0));
      }
      join_end(j);
      return;
    }
    case E_TERNARY:
      sub(t, e->b, P_TERNARY, true);
      t_puts(C, t, " if ");
      sub(t, e->a, P_TERNARY, true);
      t_puts(C, t, " else ");
      sub(t, e->c, P_TERNARY);
      return;
    case E_LAMBDA: {
      Text pt = {nullptr, 0, 0};
      params(&pt, e->p);
      CK(C);
      if (pt.n) {
        t_puts(C, t, "lambda ");
        t_putn(C, t, pt.d, pt.n);
        t_puts(C, t, ": ");
      } else {
        t_puts(C, t, "lambda: ");
      }
      concat_none(sub(t, e->a, P_LAMBDA));
      return;
    }
    case E_NAMED:
      if (!is_k(e->a, E_NAME)) {  // f"{e.target.id} := ..."
        py_attr_error(C, e->a, "id");
        return;
      }
      name_text(t, e->a->s);
      t_puts(C, t, " := ");
      sub(t, e->b, P_LAMBDA);
      return;
    case E_CALL: {
      sub(t, e->a, P_ATOM);
      t_put(C, t, '(');
      bool first = true;
      Join j = join0();
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        if (!first) t_puts(C, t, ", ");
        first = false;
        join_item(j, callarg(t, e->l1->d[q]));
      }
      for (u32 q = 0; q < e->l2->n && !C->err; q++) {
        if (!first) t_puts(C, t, ", ");
        first = false;
        Node* kw = e->l2->d[q];
        if (s_is_none(kw->s)) {
          t_puts(C, t, "**");
          concat_none(sub(t, kw->a, P_LAMBDA));
        } else {
          t_str(C, t, kw->s);
          t_put(C, t, '=');
          sub(t, kw->a, P_LAMBDA);
        }
        join_item(j, false);
      }
      join_end(j);
      t_put(C, t, ')');
      return;
    }
    case E_ATTR: {
      bool wrap = is_k(e->a, E_CONST) && e->a->cid != CID_INVALID && ckind(C, e->a->cid) == UPY_C_INT;
      if (is_k(e->a, E_CONST) && e->a->cid == CID_INVALID) {
        sub(t, e->a, P_ATOM);
        return;
      }
      if (wrap) t_put(C, t, '(');
      sub(t, e->a, P_ATOM);
      if (wrap) t_put(C, t, ')');
      t_put(C, t, '.');
      name_text(t, e->s);
      return;
    }
    case E_SUBSCR:
      sub(t, e->a, P_ATOM);
      t_put(C, t, '[');
      index(t, e->b);
      t_put(C, t, ']');
      return;
    case E_TUPLE: {
      u32 n = e->l1->n;
      if (!n) { t_puts(C, t, "()"); return; }
      t_put(C, t, '(');
      Join j = join0();
      for (u32 q = 0; q < n && !C->err; q++) {
        if (q) t_puts(C, t, ", ");
        join_item(j, callarg(t, e->l1->d[q]));
      }
      join_end(j);
      t_puts(C, t, n == 1 ? ",)" : ")");
      return;
    }
    case E_LIST: {
      t_put(C, t, '[');
      Join j = join0();
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        if (q) t_puts(C, t, ", ");
        join_item(j, callarg(t, e->l1->d[q]));
      }
      join_end(j);
      t_put(C, t, ']');
      return;
    }
    case E_SET: {
      if (!e->l1->n) { t_puts(C, t, "set()"); return; }
      t_put(C, t, '{');
      Join j = join0();
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        if (q) t_puts(C, t, ", ");
        join_item(j, callarg(t, e->l1->d[q]));
      }
      join_end(j);
      t_put(C, t, '}');
      return;
    }
    case E_DICT: {
      t_put(C, t, '{');
      u32 n = e->l1->n < e->l2->n ? e->l1->n : e->l2->n;
      for (u32 q = 0; q < n && !C->err; q++) {
        if (q) t_puts(C, t, ", ");
        Node* k = e->l1->d[q];
        if (!k) {
          t_puts(C, t, "**");
          concat_none(sub(t, e->l2->d[q], P_LAMBDA));
        } else {
          sub(t, k, P_LAMBDA);
          t_puts(C, t, ": ");
          sub(t, e->l2->d[q], P_LAMBDA);
        }
      }
      t_put(C, t, '}');
      return;
    }
    case E_STARRED:
      t_put(C, t, '*');
      concat_none(sub(t, e->a, P_LAMBDA));
      return;
    case E_YIELD: {
      bool bare = !e->a;
      if (!bare && is_k(e->a, E_CONST)) {
        u32 k = node_ckind(C, e->a);
        CK(C);
        bare = k == UPY_C_NONE;
      }
      if (bare) {
        t_puts(C, t, "(yield)");
        return;
      }
      t_puts(C, t, "(yield ");
      sub(t, e->a, P_LAMBDA);
      t_put(C, t, ')');
      return;
    }
    case E_YIELDFROM:
      t_puts(C, t, "(yield from ");
      sub(t, e->a, P_LAMBDA);
      t_put(C, t, ')');
      return;
    case E_COMP: {
      // generators are rendered first (emitter.py:479-485), then the element
      Text sp = {nullptr, 0, 0};
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        Node* g = e->l1->d[q];
        if (q) t_put(C, &sp, ' ');
        t_puts(C, &sp, "for ");
        target(&sp, g->a, false);
        t_puts(C, &sp, " in ");
        sub(&sp, g->b, P_TERNARY);
        for (u32 w = 0; w < g->l1->n && !C->err; w++) {
          t_puts(C, &sp, " if ");
          sub(&sp, g->l1->d[w], P_TERNARY);
        }
      }
      CK(C);
      if (e->op == 2) {
        t_put(C, t, '{');
        sub(t, e->b, P_TERNARY);
        t_puts(C, t, ": ");
        sub(t, e->c, P_TERNARY);
        t_put(C, t, ' ');
        t_putn(C, t, sp.d, sp.n);
        t_put(C, t, '}');
        return;
      }
      char open = e->op == 0 ? '[' : e->op == 1 ? '{' : '(';
      char close = e->op == 0 ? ']' : e->op == 1 ? '}' : ')';
      Text el = {nullptr, 0, 0};
      sub(&el, e->a, P_TERNARY);
      t_put(C, t, open);
      t_putn(C, t, el.d, el.n);
      t_put(C, t, ' ');
      t_putn(C, t, sp.d, sp.n);
      t_put(C, t, close);
      return;
    }
    case E_FSTRING: {
      Text body = {nullptr, 0, 0};
      for (u32 q = 0; q < e->l1->n && !C->err; q++) {
        Node* part = e->l1->d[q];
        if (is_k(part, X_STRPART)) {
          for (u32 w = 0; w < part->s.n; w++) {
            char ch = part->s.p[w];
            t_put(C, &body, ch);
            if (ch == '{' || ch == '}') t_put(C, &body, ch);
          }
        } else {
          format_part(&body, part);
        }
      }
      CK(C);
      bool sq = s_has(t_as_str(&body), '\''), dq = s_has(t_as_str(&body), '"');
      char quote = !sq ? '\'' : '"';
      t_put(C, t, 'f');
      if (sq && dq) {
        t_put(C, t, '\'');
        for (u32 w = 0; w < body.n; w++) {
          if (body.d[w] == '\'') t_put(C, t, '\\');
          t_put(C, t, body.d[w]);
        }
        t_put(C, t, '\'');
      } else {
        t_put(C, t, quote);
        t_putn(C, t, body.d, body.n);
        t_put(C, t, quote);
      }
      return;
    }
  }
}

HD NOINL void Emitter::format_part(Text* t, Node* fv) {  // emitter.py:510-519
  // Not a FormattedValue: the reference calls _format_part on it anyway, which
  // renders `fv.value` when the node has such a field and then fails on
  // `fv.conversion` (or on `.value` itself).
  Node* value = nullptr;
  bool fmt = is_k(fv, E_FMTVAL);
  if (fmt) value = fv->a;
  else if (is_k(fv, E_ATTR) || is_k(fv, E_SUBSCR) || is_k(fv, E_STARRED) || is_k(fv, E_YIELD) ||
           is_k(fv, E_YIELDFROM)) value = fv->a;
  else if (is_k(fv, E_NAMED)) value = fv->b;
  else if (is_k(fv, E_COMP)) value = fv->c;
  else {
    py_attr_error(C, fv, "value");
    return;
  }
  Text inner = {nullptr, 0, 0};
  bool none = sub(&inner, value, P_TERNARY);
  CK(C);
  if (none) {  // inner.startswith("{") on the None object
    py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'startswith'");
    return;
  }
  if (!fmt) {
    py_attr_error(C, fv, "conversion");
    return;
  }
  t_put(C, t, '{');
  if (inner.n && inner.d[0] == '{') t_put(C, t, ' ');
  t_putn(C, t, inner.d, inner.n);
  if (fv->op) {
    t_put(C, t, '!');
    t_put(C, t, fv->op == 1 ? 's' : fv->op == 2 ? 'r' : 'a');
  }
  if (fv->b) {
    t_put(C, t, ':');
    format_spec(t, fv->b);
  }
  t_put(C, t, '}');
}

HD inline void Emitter::format_spec(Text* t, Node* spec) {  // emitter.py:521-532
  if (is_k(spec, E_CONST)) {  // str(spec.const.value)
    u32 cid = spec->cid;
    if (cid == CID_INVALID) {
      py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'");
      return;
    }
    u32 k = ckind(C, cid);
    if (k == UPY_C_STR) t_str(C, t, cstr(C, cid));
    else if (k == UPY_C_NONE) t_puts(C, t, "None");
    else if (k == UPY_C_ELLIPSIS) t_puts(C, t, "Ellipsis");
    else r_const_value(t, cid);
    return;
  }
  if (is_k(spec, E_FSTRING)) {
    for (u32 q = 0; q < spec->l1->n && !C->err; q++) {
      Node* part = spec->l1->d[q];
      if (is_k(part, X_STRPART)) t_str(C, t, part->s);
      else format_part(t, part);
    }
    return;
  }
  t_put(C, t, '{');
  concat_none(sub(t, spec, P_TERNARY));
  t_put(C, t, '}');
}

HD inline void Emitter::index(Text* t, Node* idx) {  // emitter.py:420-430
  if (is_k(idx, E_SLICE)) {
    slice(t, idx);
    return;
  }
  if (is_k(idx, E_TUPLE) && idx->l1->n) {
    bool any = false;
    for (u32 q = 0; q < idx->l1->n; q++) any |= is_k(idx->l1->d[q], E_SLICE);
    if (any) {
      Join j = join0();
      for (u32 q = 0; q < idx->l1->n && !C->err; q++) {
        if (q) t_puts(C, t, ", ");
        Node* el = idx->l1->d[q];
        if (is_k(el, E_SLICE)) {
          slice(t, el);
          join_item(j, false);
        } else {
          join_item(j, sub(t, el));
        }
      }
      join_end(j);
      return;
    }
  }
  sub(t, idx);
}
HD inline void Emitter::slice(Text* t, Node* s) {
  if (s->a) sub(t, s->a, P_TERNARY);
  t_put(C, t, ':');
  if (s->b) sub(t, s->b, P_TERNARY);
  if (s->c) {
    t_put(C, t, ':');
    sub(t, s->c, P_TERNARY);
  }
}

HD inline bool Emitter::target(Text* t, Node* e, bool nested) {  // emitter.py:312-322
  GUARD(C);
  CKR(C, false);
  if ((is_k(e, E_TUPLE) || is_k(e, E_LIST)) && e->l1->n) {
    bool lst = is_k(e, E_LIST);
    if (lst) t_put(C, t, '[');
    else if (nested) t_put(C, t, '(');
    Join j = join0();
    for (u32 q = 0; q < e->l1->n && !C->err; q++) {
      if (q) t_puts(C, t, ", ");
      join_item(j, target(t, e->l1->d[q], true));
    }
    join_end(j);
    if (!lst && e->l1->n == 1) t_put(C, t, ',');
    if (lst) t_put(C, t, ']');
    else if (nested) t_put(C, t, ')');
    return false;
  }
  if (is_k(e, E_STARRED)) {
    t_put(C, t, '*');
    concat_none(target(t, e->a, nested));
    return false;
  }
  return sub(t, e);
}

HD NOINL void Emitter::params(Text* t, Node* p) {  // emitter.py:285-308
  bool first = true;
  auto sep = [&]() {
    if (!first) t_puts(C, t, ", ");
    first = false;
  };
  u32 nargs = p->sl->n;
  u32 nd = p->l1->n;
  for (u32 i = 0; i < nargs && !C->err; i++) {
    sep();
    t_str(C, t, p->sl->d[i]);
    i64 di = (i64)i - ((i64)nargs - (i64)nd);
    if (di >= 0) {
      t_put(C, t, '=');
      sub(t, p->l1->d[di]);
    }
    if (p->i && (i64)i + 1 == (i64)p->i) {
      sep();
      t_put(C, t, '/');
    }
  }
  if (!s_is_none(p->s) && p->s.n) {
    sep();
    t_put(C, t, '*');
    t_str(C, t, p->s);
  } else if (p->sl2->n) {
    sep();
    t_put(C, t, '*');
  }
  for (u32 q = 0; q < p->sl2->n && !C->err; q++) {
    sep();
    Str k = p->sl2->d[q];
    t_str(C, t, k);
    const Node* kd = kw_lookup(p->l2, k);
    if (kd) {
      t_put(C, t, '=');
      sub(t, kd->a);
    }
  }
  if (!s_is_none(p->s2) && p->s2.n) {
    sep();
    t_puts(C, t, "**");
    t_str(C, t, p->s2);
  }
}

// ------------------------------------------------------------ statements
HD NOINL void Emitter::emit_if(Node* s, const char* kw) {
  line_start();
  t_puts(C, out, kw);
  t_put(C, out, ' ');
  sub(out, s->a);
  t_put(C, out, ':');
  line_end();
  block(s->l1);
  if (!s->l2->n) return;
  if (s->l2->n == 1 && is_k(s->l2->d[0], S_IF)) {
    emit_if(s->l2->d[0], "elif");
    return;
  }
  simple_line("else:");
  block(s->l2);
}

HD NOINL void Emitter::stmt(Node* s) {  // emitter.py:136-283
  GUARD(C);
  CK(C);
  switch (s ? s->k : 0) {
    case S_JUMP: case S_CONDJUMP: case S_COMPACCUM: case S_WHILESHAPE: {
      Text m;
      if (fail_begin(C, UPY_ST_MARKER_LEAK, 0, 0, &m)) {
        m_puts(C, &m, "marker survived structuring: ");
        C->err = 0;
        Text r = {nullptr, 0, 0};
        r_node(&r, s);
        int st2 = C->err;
        C->err = UPY_ST_MARKER_LEAK;
        if (!st2) m_putn(C, &m, r.d, r.n);
        fail_end(C, &m);
      }
      return;
    }
    case S_ASSIGN: {
      line_start();
      Join j = join0();
      for (u32 q = 0; q < s->l1->n && !C->err; q++) {
        if (q) t_puts(C, out, " = ");
        join_item(j, target(out, s->l1->d[q], false));
      }
      join_end(j);
      t_puts(C, out, " = ");
      sub(out, s->a);
      line_end();
      return;
    }
    case S_AUGASSIGN:
      line_start();
      target(out, s->a, false);
      t_put(C, out, ' ');
      t_puts(C, out, binop_str(s->op));
      t_puts(C, out, "= ");
      sub(out, s->b);
      line_end();
      return;
    case S_EXPR:
      line_start();
      sub(out, s->a);
      line_end();
      return;
    case S_RETURN: {
      bool none_ = false;
      if (is_k(s->a, E_CONST)) {
        u32 k = node_ckind(C, s->a);
        CK(C);
        none_ = k == UPY_C_NONE;
      }
      line_start();
      if (none_) {
        t_puts(C, out, "return None");
      } else {
        t_puts(C, out, "return ");
        sub(out, s->a);
      }
      line_end();
      return;
    }
    case S_RAISE:
      line_start();
      if (!s->a) {
        t_puts(C, out, "raise");
      } else {
        t_puts(C, out, "raise ");
        sub(out, s->a);
        if (s->b) {
          t_puts(C, out, " from ");
          sub(out, s->b);
        }
      }
      line_end();
      return;
    case S_DELETE: {
      line_start();
      t_puts(C, out, "del ");
      Join j = join0();
      for (u32 q = 0; q < s->l1->n && !C->err; q++) {
        if (q) t_puts(C, out, ", ");
        join_item(j, target(out, s->l1->d[q], false));
      }
      join_end(j);
      line_end();
      return;
    }
    case S_PASS: simple_line("pass"); return;
    case S_BREAK: simple_line("break"); return;
    case S_CONTINUE: simple_line("continue"); return;
    case S_GLOBAL:
    case S_NONLOCAL:
      line_start();
      t_puts(C, out, s->k == S_GLOBAL ? "global " : "nonlocal ");
      {
        Join j = join0();
        for (u32 q = 0; q < s->sl->n; q++) {
          if (q) t_puts(C, out, ", ");
          name_text(out, s->sl->d[q]);
          join_item(j, s_is_none(s->sl->d[q]));
        }
        join_end(j);
      }
      line_end();
      return;
    case S_ASSERT:
      line_start();
      t_puts(C, out, "assert ");
      sub(out, s->a);
      if (s->b) {
        t_puts(C, out, ", ");
        sub(out, s->b);
      }
      line_end();
      return;
    case S_IMPORT:
      line_start();
      t_puts(C, out, "import ");
      name_text(out, s->s);
      if (!s_is_none(s->s2) && s->s2.n) {
        t_puts(C, out, " as ");
        t_str(C, out, s->s2);
      }
      line_end();
      return;
    case S_IMPORTFROM:
    case S_IMPORTSTAR: {
      // "." * level (level is the const's value)
      i64 level = 0;
      u32 lk = s->cid == CID_INVALID ? UPY_C_NONE : ckind(C, s->cid);
      if (lk == UPY_C_INT) {
        const upy_const* c = cget(C, s->cid);
        level = c->n ? (i64)C->limbs[c->off] * c->ival : 0;
      } else if (lk == UPY_C_BOOL) {
        level = cbool(C, s->cid);
      } else {
        Text m;
        if (fail_begin(C, UPY_ST_PY_TYPE_ERROR, 0, 0, &m)) {
          m_puts(C, &m, "can't multiply sequence by non-int of type '");
          m_puts(C, &m, lk == UPY_C_NONE ? "NoneType" : lk == UPY_C_FLOAT ? "float" : lk == UPY_C_STR ? "str"
                        : lk == UPY_C_BYTES ? "bytes" : lk == UPY_C_TUPLE || lk == UPY_C_FROZENSET ? "tuple"
                        : lk == UPY_C_COMPLEX ? "complex" : lk == UPY_C_ELLIPSIS ? "NoneType" : "CodeObject");
          m_puts(C, &m, "'");
          fail_end(C, &m);
        }
        return;
      }
      concat_none(s_is_none(s->s));  // "." * level + module
      CK(C);
      line_start();
      t_puts(C, out, "from ");
      for (i64 q = 0; q < level; q++) t_put(C, out, '.');
      name_text(out, s->s);
      if (s->k == S_IMPORTSTAR) {
        t_puts(C, out, " import *");
      } else {
        t_puts(C, out, " import ");
        Join j = join0();
        for (u32 q = 0; q < s->l1->n; q++) {
          if (q) t_puts(C, out, ", ");
          Node* pr = s->l1->d[q];
          name_text(out, pr->s);
          bool alias = !s_is_none(pr->s2) && pr->s2.n;
          if (alias) {
            t_puts(C, out, " as ");
            t_str(C, out, pr->s2);
          }
          join_item(j, !alias && s_is_none(pr->s));
        }
        join_end(j);
      }
      line_end();
      return;
    }
    case S_IF: emit_if(s, "if"); return;
    case S_WHILE:
      line_start();
      t_puts(C, out, "while ");
      sub(out, s->a);
      t_put(C, out, ':');
      line_end();
      block(s->l1);
      if (s->l2->n) {
        simple_line("else:");
        block(s->l2);
      }
      return;
    case S_FOR:
      line_start();
      t_puts(C, out, "for ");
      target(out, s->a, false);
      t_puts(C, out, " in ");
      sub(out, s->b);
      t_put(C, out, ':');
      line_end();
      block(s->l1);
      if (s->l2->n) {
        simple_line("else:");
        block(s->l2);
      }
      return;
    case S_TRY:
      simple_line("try:");
      block(s->l1);
      for (u32 h = 0; h < s->l2->n && !C->err; h++) {
        Node* hd = s->l2->d[h];
        line_start();
        if (!hd->a) {
          t_puts(C, out, "except:");
        } else {
          t_puts(C, out, "except ");
          sub(out, hd->a);
          if (!s_is_none(hd->s) && hd->s.n) {
            t_puts(C, out, " as ");
            t_str(C, out, hd->s);
          }
          t_put(C, out, ':');
        }
        line_end();
        block(hd->l1);
      }
      if (s->l3->n) {
        simple_line("else:");
        block(s->l3);
      }
      if (s->l4->n) {
        simple_line("finally:");
        block(s->l4);
      }
      return;
    case S_WITH: {
      line_start();
      t_puts(C, out, "with ");
      Join j = join0();
      for (u32 q = 0; q < s->l1->n && !C->err; q++) {
        if (q) t_puts(C, out, ", ");
        Node* it = s->l1->d[q];
        bool none = sub(out, it->a);
        if (it->b) {
          t_puts(C, out, " as ");
          target(out, it->b, true);
          if (none && !C->err)  // part += f" as ..." on the None object
            py_error(C, UPY_ST_PY_TYPE_ERROR, "unsupported operand type(s) for +=: 'NoneType' and 'str'");
          none = false;
        }
        join_item(j, none);
      }
      join_end(j);
      t_put(C, out, ':');
      line_end();
      block(s->l2);
      return;
    }
    case S_FUNCDEF:
      funcdef_head(s);
      block(s->l1);
      return;
    case S_CLASSDEF: {
      for (u32 q = 0; q < s->l4->n && !C->err; q++) {
        line_start();
        t_put(C, out, '@');
        concat_none(sub(out, s->l4->d[q]));
        line_end();
      }
      line_start();
      t_puts(C, out, "class ");
      t_str(C, out, s->s);
      u32 na = s->l1->n + s->l2->n;
      if (na) t_put(C, out, '(');
      bool first = true;
      Join j = join0();
      for (u32 q = 0; q < s->l1->n && !C->err; q++) {
        if (!first) t_puts(C, out, ", ");
        first = false;
        join_item(j, sub(out, s->l1->d[q]));
      }
      for (u32 q = 0; q < s->l2->n && !C->err; q++) {
        if (!first) t_puts(C, out, ", ");
        first = false;
        name_text(out, s->l2->d[q]->s);
        t_put(C, out, '=');
        sub(out, s->l2->d[q]->a);
      }
      join_end(j);
      if (na) t_put(C, out, ')');
      t_put(C, out, ':');
      line_end();
      block(s->l3);
      return;
    }
  }
  Text m;
  if (fail_begin(C, UPY_ST_MARKER_LEAK, 0, 0, &m)) {
    m_puts(C, &m, "no emitter for ");
    m_puts(C, &m, class_name_of(s));
    fail_end(C, &m);
  }
}
