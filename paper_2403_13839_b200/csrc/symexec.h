// symexec.h -- symbolic stack simulation of one basic block (symexec.py:128-1051).
// Stack states are NV* vectors treated as immutable once published (the
// reference copies on every StackState construction); the working stack of a
// block simulation is a private copy.
#pragma once
#include "ir.h"

struct Block {
  i32 id;
  u32 start, end;
  i32 lo, hi;              // instruction index range [lo, hi)
  Vec<i32>* succ;          // successor block ids (parallel with succ_kind)
  Vec<u8>* succ_kind;      // 0 jump_taken, 1 jump_not_taken, 2 fallthrough, 3 exception
  Vec<i32>* pred;
  bool alive;
};
enum { EK_TAKEN = 0, EK_NOT_TAKEN = 1, EK_FALL = 2, EK_EXC = 3 };

struct BlockResult {
  NV* stmts;
  NV* exit_fall;   // nullptr = None
  NV* exit_jump;
  i32 term;        // instruction index of the terminator, -1 = None
};

// One code object being decompiled: instructions + per-object simulator state.
struct Code {
  u32 oi;                  // object index
  int minor;
  const upy_obj* o;
  Ins* ins;
  i32 n_ins;
  bool has_kwnames;        // Simulator.kwnames (3.11 KW_NAMES pending)
  Vec<Str>* kwnames;
};

// The per-instruction helpers (pops, use_all, store, finish_call) are force-inlined
// into step: out of line, their prologue/epilogue register saves were the largest
// source of local-memory traffic (same-session A/B: C3 237.8 -> 223.1 ms).
#ifdef UPY_SYM_OUTLINE
#define SYMFN
#define SYMFN_NOINL NOINL
#else
#define SYMFN FORCEINL
#define SYMFN_NOINL FORCEINL
#endif

// The read-only part of Code the per-instruction transfer functions use, passed by
// value into the force-inlined step: the fields live in registers for the whole
// block instead of being reloaded through K after every arena store (which the
// compiler must assume may alias *K).
struct StepCtx {
  u32 oi;
  int minor;
  const upy_obj* o;
};

template <class KK>
HD FORCEINL Str argval_name(Dc* C, const KK* K, const Ins& in) {
  // kind == name (disasm.py:134-138)
  u64 idx = in.arg;
  if (K->minor >= 11 && in.op == OP_LOAD_GLOBAL) idx = in.arg >> 1;
  if ((in.flags & 2) || idx >= K->o->n_names) return Snone();
  return obj_tab(C, K->o->names_off, (u32)idx);
}
template <class KK>
HD FORCEINL Str argval_local(Dc* C, const KK* K, const Ins& in) {
  if (in.flags & 2) return Snone();
  if (K->minor <= 10) {
    if (in.arg >= K->o->n_varnames) return Snone();
    return obj_tab(C, K->o->varnames_off, in.arg);
  }
  bool ok;
  Str s = obj_localsplus(C, K->oi, in.arg, &ok);
  return ok ? s : Snone();
}
template <class KK>
HD FORCEINL Str argval_free(Dc* C, const KK* K, const Ins& in) {
  if (in.flags & 2) return Snone();
  bool ok;
  Str s = obj_deref_name(C, K->oi, in.arg, &ok);
  return ok ? s : Snone();
}
template <class KK>
HD FORCEINL u32 argval_const(Dc* C, const KK* K, const Ins& in) {
  if ((in.flags & 2) || in.arg >= K->o->n_consts) return CID_INVALID;
  return obj_const_id(C, K->oi, in.arg);
}
template <class KK>
HD inline u8 argval_cmp(Dc* C, const KK* K, const Ins& in) {
  if ((in.flags & 2) || (int)in.arg >= T_NCMP[K->minor - 8]) return CO_NONE;
  return (u8)in.arg;
}
// resolved jump target (disasm.py:157-164); decode validated it
HD inline u32 jump_target(const Code* K, const Ins& in) {
  u64 a = in.arg;
  if (in.kind == K_JUMP_ABS) return (u32)(K->minor == 10 ? a * 2 : a);
  if (in.kind == K_JUMP_BACK) return (u32)(ins_op_offset(in) + 2 - 2 * a);
  u64 delta = K->minor >= 10 ? a * 2 : a;
  return (u32)(ins_op_offset(in) + 2 + delta);
}

// ------------------------------------------------------------ helpers
HD inline NV* nv_copy(Dc* C, const NV* v) { return vcopy<Node*>(C, v); }
HD inline bool nv_contains_id(const NV* v, const Node* x, u32 hi) {
  for (u32 i = 0; i < hi && i < v->n; i++)
    if (v->d[i] == x) return true;
  return false;
}
// Python st[k] with negative/zero index semantics; nullptr + IndexError on failure
HD inline Node* py_index(Dc* C, NV* st, i64 k) {
  i64 n = st->n;
  if (k < 0) k += n;
  if (k < 0 || k >= n) {
    py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range");
    return nullptr;
  }
  return st->d[k];
}
HD inline i64 py_norm(i64 n, i64 k, bool* ok) {
  if (k < 0) k += n;
  *ok = k >= 0 && k < n;
  return k;
}
// ConstE.const.kind with the AttributeError of a None const
HD inline u32 node_ckind(Dc* C, const Node* e) {
  if (e->cid == CID_INVALID) {
    py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'kind'");
    return 0xFFFF;
  }
  return ckind(C, e->cid);
}
HD inline bool is_const_kind(Dc* C, const Node* e, u32 kind) {
  if (!is_k(e, E_CONST)) return false;
  return node_ckind(C, e) == kind;
}
HD inline Node* mk_name_syn(Dc* C, const char* stem, i64 k, u8 scope) {
  Text t = {nullptr, 0, 0};
  t_puts(C, &t, stem);
  t_i64(C, &t, k);
  return mk_name(C, t_as_str(&t), scope);
}

// is_effectful (symexec.py:120-125)
HD inline bool is_effectful(const Node* e) {
  if (!e) return true;
  switch (e->k) {
    case E_CONST: case E_FUNC: case E_LAMBDA: case E_NULL: case E_METHSELF: return false;
  }
  return true;
}

// negate (symexec.py:1002-1012)
HD inline u8 flip_cmp(u8 c, bool* ok) {
  *ok = true;
  switch (c) {
    case CO_EQ: return CO_NE;
    case CO_NE: return CO_EQ;
    case CO_LT: return CO_GE;
    case CO_GE: return CO_LT;
    case CO_GT: return CO_LE;
    case CO_LE: return CO_GT;
    case CO_IN: return CO_NOTIN;
    case CO_NOTIN: return CO_IN;
    case CO_IS: return CO_ISNOT;
    case CO_ISNOT: return CO_IS;
  }
  *ok = false;
  return c;
}
HD inline Node* negate(Dc* C, Node* e) {
  if (is_k(e, E_COMPARE) && e->l1->n == 1) {
    bool ok;
    u8 f = flip_cmp(e->l1->d[0]->op, &ok);
    if (ok) {
      Node* n = mk(C, E_COMPARE);
      n->a = e->a;
      n->l1 = nv1(C, mk_cmpop(C, f));
      n->l2 = e->l2;  // shares the comparators list object
      return n;
    }
  }
  if (is_k(e, E_UNARY) && e->op == UO_NOT) return e->a;
  return mk_unary(C, UO_NOT, e);
}

// _spread (symexec.py:991-999)
HD inline NV* spread(Dc* C, Node* v, bool as_set) {
  if (is_k(v, E_TUPLE) || is_k(v, E_LIST)) return nv_copy(C, v->l1);
  if (as_set && is_k(v, E_SET)) return nv_copy(C, v->l1);
  if (is_k(v, E_CONST)) {
    u32 k = node_ckind(C, v);
    CKR(C, nullptr);
    if (k == UPY_C_TUPLE || k == UPY_C_FROZENSET) {
      u32 n = cnelem(C, v->cid);
      NV* out = vnew<Node*>(C, n);
      for (u32 i = 0; i < n; i++) vpush(C, out, mk_const(C, celem(C, v->cid, i)));
      return out;
    }
  }
  return nv1(C, mk1(C, E_STARRED, v));
}

HD inline Node* attr_root(Node* e) {
  while (is_k(e, E_ATTR)) e = e->a;
  return e;
}
HD inline Node* none_to_null(Dc* C, Node* e) {
  if (is_k(e, E_CONST)) {
    u32 k = node_ckind(C, e);
    if (k == UPY_C_NONE) return nullptr;
  }
  return e;
}

// ------------------------------------------------------------ simulator
struct Sim {
  Dc* C;
  Code* K;

  HD FORCEINL Node* pop(NV* st, const Ins* ins) {
    if (st->n == 0) {
      fail_underflow(C, ins);
      return nullptr;
    }
    return st->d[--st->n];
  }
  // pop for expression use, folding pending walrus targets (symexec.py:217-228)
  HD FORCEINL Node* pop_value(NV* st, const Ins* ins) {
    Node* v = pop(st, ins);
    CKR(C, nullptr);
    NV* pend = v->pend;
    if (pend && pend->n) v = fold_pending(v);
    return v;
  }
  HD NOINL Node* fold_pending(Node* v) {  // walrus targets pending on a popped value
    NV* pend = v->pend;
    Node* target = pend->d[--pend->n];
    Node* inner = v;
    v->pend = nullptr;
    v = mk2(C, E_NAMED, target, inner);
    for (i32 i = (i32)pend->n - 1; i >= 0; i--) v = mk2(C, E_NAMED, pend->d[i], v);
    return v;
  }
  HD SYMFN NV* pops(NV* st, const Ins* ins, u64 n) {
    if (st->n < n) {
      fail_underflow(C, ins);
      return nullptr;
    }
    NV* vals = vcopy<Node*>(C, st, (u32)(st->n - n), st->n);
    st->n -= (u32)n;
    return vals;
  }
  HD Node* use(Node* v) {  // symexec.py:571-577
    NV* pend = v ? v->pend : nullptr;
    if (pend && pend->n) {
      v->pend = nullptr;
      for (i32 i = (i32)pend->n - 1; i >= 0; i--) v = mk2(C, E_NAMED, pend->d[i], v);
    }
    return v;
  }
  HD SYMFN NV* use_all(NV* vals) {
    NV* out = vnew<Node*>(C, vals ? vals->n : 0);
    for (u32 i = 0; vals && i < vals->n; i++) vpush(C, out, use(vals->d[i]));
    return out;
  }
  HD void push(NV* st, Node* x) { vpush(C, st, x); }

  HD bool in_comprehension() {
    Str n = obj_name(C, K->oi);
    return s_eqc(n, "<listcomp>") || s_eqc(n, "<setcomp>") || s_eqc(n, "<dictcomp>");
  }

  static HD bool is_scalar_store(u8 op) {
    return op == OP_STORE_FAST || op == OP_STORE_NAME || op == OP_STORE_GLOBAL || op == OP_STORE_DEREF;
  }
  static HD u8 store_scope(u8 op) {
    switch (op) {
      case OP_STORE_FAST: return SC_FAST;
      case OP_STORE_NAME: return SC_NAME;
      case OP_STORE_GLOBAL: return SC_GLOBAL;
      default: return SC_DEREF;
    }
  }
  template <class KK>
  HD FORCEINL Str store_name(const Ins& in, const KK* KX) {
    switch (in.op) {
      case OP_STORE_FAST: return argval_local(C, KX, in);
      case OP_STORE_DEREF: return argval_free(C, KX, in);
      default: return argval_name(C, KX, in);
    }
  }

  HD void complete_group(Node* group, NV* out) {  // symexec.py:401-410
    GUARD(C);
    CK(C);
    for (u32 i = 0; i < group->l1->n; i++)
      if (!group->l1->d[i]) return;
    NV* elts = nv_copy(C, group->l1);
    if (group->kk >= 0 && (u32)group->kk < elts->n) elts->d[group->kk] = mk1(C, E_STARRED, elts->d[group->kk]);
    Node* tup = mk(C, E_TUPLE);
    tup->l1 = elts;
    if (!group->p) {
      vpush(C, out, mk_assign(C, nv1(C, tup), group->a));
    } else {
      group->p->l1->d[group->j] = tup;
      complete_group(group->p, out);
    }
  }

  // _store (symexec.py:295-399); returns the number of following stores consumed
  HD SYMFN_NOINL int store(const Ins* ins, NV* st, NV* out, i32 idx, i32 hi, Node* target) {
    Node* v = pop(st, ins);
    CKR(C, 0);
    if (is_k(v, E_UNPACKSLOT)) {
      Node* group = v->p;
      group->l1->d[v->j] = target;
      complete_group(group, out);
      return 0;
    }
    // import statement recovery
    if (is_k(v, E_IMPORT) && !(v->f & 2)) {
      if (s_is_none(v->s)) {
        py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'split'");
        return 0;
      }
      Str root = v->s;
      u32 dot = 0;
      while (dot < root.n && root.p[dot] != '.') dot++;
      root.n = dot;
      Node* st_ = mk(C, S_IMPORT);
      st_->s = v->s;
      if (is_k(target, E_NAME) && s_eq(target->s, root)) {
        st_->s2 = Snone();
      } else {
        st_->s2 = is_k(target, E_NAME) ? target->s : Snone();
      }
      vpush(C, out, st_);
      return 0;
    }
    if (is_k(v, E_IMPORTFROM) && is_k(v->a, E_IMPORT)) {
      Node* imp = v->a;
      if (!(imp->f & 2)) {
        Node* s2 = mk(C, S_IMPORT);
        s2->s = imp->s;
        s2->s2 = is_k(target, E_NAME) ? target->s : Snone();
        vpush(C, out, s2);
        return 0;
      }
      Str asname = (is_k(target, E_NAME) && !s_eq(target->s, v->s)) ? target->s : Snone();
      Node* pair = mk(C, X_NAMEPAIR);
      pair->s = v->s;
      pair->s2 = asname;
      if (out->n && is_k(vlast(out), S_IMPORTFROM) && vlast(out)->src == imp) {
        vpush(C, vlast(out)->l1, pair);
      } else {
        Node* s3 = mk(C, S_IMPORTFROM);
        s3->s = imp->s;
        s3->l1 = nv1(C, pair);
        s3->cid = imp->cid;  // level
        s3->src = imp;
        vpush(C, out, s3);
      }
      return 0;
    }
    if (is_k(v, E_ATTR) && is_k(attr_root(v), E_IMPORT)) {
      Node* imp = attr_root(v);
      Node* s2 = mk(C, S_IMPORT);
      s2->s = imp->s;
      s2->s2 = is_k(target, E_NAME) ? target->s : Snone();
      vpush(C, out, s2);
      return 0;
    }
    // dup-twin still on the stack: walrus or chained assignment
    if (nv_contains_id(st, v, st->n)) {
      if (!v->pend) v->pend = vnew<Node*>(C);
      vpush(C, v->pend, target);
      return 0;
    }
    NV* targets = nv1(C, target);
    if (v->pend && v->pend->n) {
      targets = nv_copy(C, v->pend);
      vpush(C, targets, target);
      v->pend = nullptr;
    }
    // augmented assignment
    if (targets->n == 1 && is_k(v, E_BINOP) && (v->f & 1) && node_eq(C, v->a, target)) {
      CKR(C, 0);
      Node* s2 = mk(C, S_AUGASSIGN);
      s2->a = target;
      s2->op = v->op;
      s2->b = v->b;
      vpush(C, out, s2);
      return 0;
    }
    CKR(C, 0);
    // consecutive scalar stores = tuple swap assignment
    auto blocks_batch = [](const Node* t) {
      return is_k(t, E_UNPACKSLOT) || is_k(t, E_NULL) || is_k(t, E_METHSELF);
    };
    if (targets->n == 1 && is_scalar_store(ins->op) && idx + 1 < hi && is_scalar_store(K->ins[idx + 1].op) &&
        st->n && !blocks_batch(vlast(st)) && !vlast(st)->pend && !nv_contains_id(st, vlast(st), st->n - 1)) {
      NV* bt = nv1(C, target);
      NV* bv = nv1(C, v);
      int k = 0;
      while (idx + 1 + k < hi && is_scalar_store(K->ins[idx + 1 + k].op) && st->n && !blocks_batch(vlast(st))) {
        const Ins* nxt = &K->ins[idx + 1 + k];
        Node* t2 = mk_name(C, store_name(*nxt, K), store_scope(nxt->op));
        Node* u = pop(st, nxt);
        CKR(C, 0);
        vpush(C, bt, t2);
        vpush(C, bv, u);
        k++;
      }
      if (K->minor >= 11) {
        for (u32 a = 0, b = bt->n - 1; a < b; a++, b--) {
          Node* x = bt->d[a]; bt->d[a] = bt->d[b]; bt->d[b] = x;
          x = bv->d[a]; bv->d[a] = bv->d[b]; bv->d[b] = x;
        }
      }
      Node* tt = mk(C, E_TUPLE);
      tt->l1 = bt;
      Node* tv = mk(C, E_TUPLE);
      tv->l1 = bv;
      vpush(C, out, mk_assign(C, nv1(C, tt), tv));
      return k;
    }
    vpush(C, out, mk_assign(C, targets, v));
    return 0;
  }

  HD void push_unpack(NV* st, Node* src, u64 total, i32 star_index) {
    Node* group = mk(C, X_GROUP);
    group->a = src;
    group->i = (i32)total;
    group->kk = star_index;
    group->l1 = vnew<Node*>(C, (u32)(total < 0x100000 ? total : 0x100000));
    if (is_k(src, E_UNPACKSLOT)) {
      group->p = src->p;
      group->j = src->j;
    }
    for (u64 i = 0; i < total && !C->err; i++) vpush(C, group->l1, (Node*)nullptr);
    for (i64 index = (i64)total - 1; index >= 0 && !C->err; index--) {
      Node* slot = mk(C, E_UNPACKSLOT);
      slot->a = src;
      slot->i = (i32)total;
      slot->j = (i32)index;
      slot->kk = -1;
      slot->m = 0;
      slot->p = group;
      push(st, slot);
    }
  }

  HD FORCEINL void binop(NV* st, const Ins* ins, u8 op, bool inplace) {
    Node* r = pop_value(st, ins);
    CK(C);
    Node* l = pop_value(st, ins);
    CK(C);
    push(st, mk_binop(C, op, l, r, inplace));
  }

  HD Node* display_target(NV* st, const Ins* ins) {
    return py_index(C, st, -(i64)ins->arg);
  }

  HD SYMFN void finish_call(NV* st, const Ins* ins, NV* args, Vec<Str>* kwnames) {
    NV* kwargs = vnew<Node*>(C);
    if (kwnames && kwnames->n) {
      u32 n = kwnames->n;
      u32 na = args->n;
      u32 lo = n > na ? 0 : na - n;  // args[-n:]
      u32 cnt = na - lo;
      if (cnt > n) cnt = n;
      for (u32 i = 0; i < cnt; i++) vpush(C, kwargs, mk_kwpair(C, kwnames->d[i], args->d[lo + i]));
      args = vcopy<Node*>(C, args, 0, n >= na ? 0 : na - n);
    }
    Node* x = pop(st, ins);
    CK(C);
    Node* func;
    if (K->minor >= 11) {
      Node* y = pop(st, ins);
      CK(C);
      if (is_k(y, E_NULL)) {
        func = x;
      } else if (is_k(x, E_METHSELF)) {
        func = y;
      } else {
        func = y;
        NV* a2 = nv1(C, x);
        vextend(C, a2, args);
        args = a2;
      }
    } else {
      func = x;
    }
    Node* call = mk(C, E_CALL);
    call->a = func;
    call->l1 = args;
    call->l2 = kwargs;
    push(st, call);
  }

  // tuple of str values of a Const tuple (KW_NAMES, CALL_FUNCTION_KW)
  HD Vec<Str>* const_str_tuple(u32 cid) {
    if (cid == CID_INVALID) {
      py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'");
      return nullptr;
    }
    u32 k = ckind(C, cid);
    if (k != UPY_C_TUPLE && k != UPY_C_FROZENSET) {
      // `c.value for c in <const>.value` over a non-tuple value
      if ((k == UPY_C_STR || k == UPY_C_BYTES) && cget(C, cid)->n == 0) return vnew<Str>(C);
      if (k == UPY_C_STR) {
        py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'str' object has no attribute 'value'");
      } else if (k == UPY_C_BYTES) {
        py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'int' object has no attribute 'value'");
      } else {
        const char* tn = k == UPY_C_INT ? "'int'" : k == UPY_C_BOOL ? "'bool'" : k == UPY_C_FLOAT ? "'float'"
                         : k == UPY_C_COMPLEX ? "'complex'" : k == UPY_C_CODE ? "'CodeObject'" : "'NoneType'";
        Text m;
        if (fail_begin(C, UPY_ST_PY_TYPE_ERROR, 0, 0, &m)) {
          m_puts(C, &m, tn);
          m_puts(C, &m, " object is not iterable");
          fail_end(C, &m);
        }
      }
      return nullptr;
    }
    u32 n = cnelem(C, cid);
    Vec<Str>* v = vnew<Str>(C, n);
    for (u32 i = 0; i < n; i++) {
      u32 e = celem(C, cid, i);
      if (ckind(C, e) != UPY_C_STR) {
        py_error(C, UPY_ST_PY_TYPE_ERROR, "non-str name constant");
        return nullptr;
      }
      vpush(C, v, cstr(C, e));
    }
    return v;
  }
  HD u32 const_of(Node* e) {  // `e.const` of a ConstE, AttributeError otherwise
    if (!is_k(e, E_CONST)) {
      py_attr_error(C, e, "const");
      return CID_INVALID;
    }
    return e->cid;
  }

  // dispatch of one non-terminator instruction; returns consumed following instrs
  HD int step(const Ins* ins, i32 idx, i32 hi, NV* st, NV* out, const StepCtx& X);

  HD BlockResult simulate(const Block* b, const NV* entry);
};

#define BR_PUSH(x) push(st, (x))

// Inlined into simulate() (its only caller): as a call, its register save/restore
// was ~30% of the kernel's local-memory traffic (ncu source page, round 1).
HD FORCEINL int Sim::step(const Ins* ins, i32 idx, i32 hi, NV* st, NV* out, const StepCtx& X) {
  const Ins& in = *ins;
  switch (in.op) {
    // ------------------------------------------------ loads (symexec.py:239-268)
    case OP_LOAD_CONST: BR_PUSH(mk_const(C, argval_const(C, &X, in))); return 0;
    case OP_LOAD_FAST: BR_PUSH(mk_name(C, argval_local(C, &X, in), SC_FAST)); return 0;
    case OP_LOAD_GLOBAL:
      if (X.minor >= 11 && (in.arg & 1)) BR_PUSH(mk(C, E_NULL));
      BR_PUSH(mk_name(C, argval_name(C, &X, in), SC_GLOBAL));
      return 0;
    case OP_LOAD_NAME: BR_PUSH(mk_name(C, argval_name(C, &X, in), SC_NAME)); return 0;
    case OP_LOAD_DEREF:
    case OP_LOAD_CLASSDEREF: BR_PUSH(mk_name(C, argval_free(C, &X, in), SC_DEREF)); return 0;
    case OP_LOAD_CLOSURE: BR_PUSH(mk_name(C, argval_free(C, &X, in), SC_CELL)); return 0;
    case OP_LOAD_ASSERTION_ERROR: BR_PUSH(mk_name(C, S("AssertionError"), SC_GLOBAL)); return 0;
    case OP_LOAD_BUILD_CLASS: BR_PUSH(mk(C, E_BUILDCLASS)); return 0;
    case OP_PUSH_NULL: BR_PUSH(mk(C, E_NULL)); return 0;
    // ------------------------------------------------ stores (:272-291)
    case OP_STORE_FAST:
    case OP_STORE_NAME:
    case OP_STORE_GLOBAL:
    case OP_STORE_DEREF:
      return store(ins, st, out, idx, hi, mk_name(C, store_name(in, &X), store_scope(in.op)));
    case OP_STORE_ATTR: {
      Node* obj = pop(st, ins);
      CKR(C, 0);
      Node* t = mk1(C, E_ATTR, obj);
      t->s = argval_name(C, &X, in);
      return store(ins, st, out, idx, hi, t);
    }
    case OP_STORE_SUBSCR: {
      Node* i2 = pop(st, ins);
      CKR(C, 0);
      Node* obj = pop(st, ins);
      CKR(C, 0);
      return store(ins, st, out, idx, hi, mk2(C, E_SUBSCR, obj, i2));
    }
    case OP_UNPACK_SEQUENCE: {
      Node* src = pop(st, ins);
      CKR(C, 0);
      push_unpack(st, src, (in.flags & 2) ? 0xFFFFFFFFull : in.arg, -1);
      return 0;
    }
    case OP_UNPACK_EX: {
      Node* src = pop(st, ins);
      CKR(C, 0);
      u64 before = in.arg & 0xFF, after = in.arg >> 8;
      push_unpack(st, src, before + 1 + after, (i32)before);
      return 0;
    }
    // ------------------------------------------------ deletes (:433-451)
    case OP_DELETE_FAST:
    case OP_DELETE_NAME:
    case OP_DELETE_GLOBAL:
    case OP_DELETE_DEREF: {
      Str nm = in.op == OP_DELETE_FAST ? argval_local(C, &X, in)
               : in.op == OP_DELETE_DEREF ? argval_free(C, &X, in) : argval_name(C, &X, in);
      u8 sc = in.op == OP_DELETE_FAST ? SC_FAST : in.op == OP_DELETE_NAME ? SC_NAME
              : in.op == OP_DELETE_GLOBAL ? SC_GLOBAL : SC_DEREF;
      Node* d = mk(C, S_DELETE);
      d->l1 = nv1(C, mk_name(C, nm, sc));
      vpush(C, out, d);
      return 0;
    }
    case OP_DELETE_ATTR: {
      Node* o = pop(st, ins);
      CKR(C, 0);
      Node* t = mk1(C, E_ATTR, o);
      t->s = argval_name(C, &X, in);
      Node* d = mk(C, S_DELETE);
      d->l1 = nv1(C, t);
      vpush(C, out, d);
      return 0;
    }
    case OP_DELETE_SUBSCR: {
      Node* i2 = pop(st, ins);
      CKR(C, 0);
      Node* o = pop(st, ins);
      CKR(C, 0);
      Node* d = mk(C, S_DELETE);
      d->l1 = nv1(C, mk2(C, E_SUBSCR, o, i2));
      vpush(C, out, d);
      return 0;
    }
    // ------------------------------------------------ arithmetic (:455-484, 927-944)
    // the 26 binary / in-place operator cases share one inlined binop
    case OP_BINARY_ADD:
    case OP_BINARY_SUBTRACT:
    case OP_BINARY_MULTIPLY:
    case OP_BINARY_TRUE_DIVIDE:
    case OP_BINARY_FLOOR_DIVIDE:
    case OP_BINARY_MODULO:
    case OP_BINARY_POWER:
    case OP_BINARY_LSHIFT:
    case OP_BINARY_RSHIFT:
    case OP_BINARY_AND:
    case OP_BINARY_OR:
    case OP_BINARY_XOR:
    case OP_BINARY_MATRIX_MULTIPLY:
    case OP_INPLACE_ADD:
    case OP_INPLACE_SUBTRACT:
    case OP_INPLACE_MULTIPLY:
    case OP_INPLACE_TRUE_DIVIDE:
    case OP_INPLACE_FLOOR_DIVIDE:
    case OP_INPLACE_MODULO:
    case OP_INPLACE_POWER:
    case OP_INPLACE_LSHIFT:
    case OP_INPLACE_RSHIFT:
    case OP_INPLACE_AND:
    case OP_INPLACE_OR:
    case OP_INPLACE_XOR:
    case OP_INPLACE_MATRIX_MULTIPLY:
    {
      u8 bo = BO_ADD;
      switch (in.op) {
        case OP_BINARY_ADD: bo = BO_ADD; break;
        case OP_BINARY_SUBTRACT: bo = BO_SUB; break;
        case OP_BINARY_MULTIPLY: bo = BO_MUL; break;
        case OP_BINARY_TRUE_DIVIDE: bo = BO_TRUEDIV; break;
        case OP_BINARY_FLOOR_DIVIDE: bo = BO_FLOORDIV; break;
        case OP_BINARY_MODULO: bo = BO_MOD; break;
        case OP_BINARY_POWER: bo = BO_POW; break;
        case OP_BINARY_LSHIFT: bo = BO_LSHIFT; break;
        case OP_BINARY_RSHIFT: bo = BO_RSHIFT; break;
        case OP_BINARY_AND: bo = BO_AND; break;
        case OP_BINARY_OR: bo = BO_OR; break;
        case OP_BINARY_XOR: bo = BO_XOR; break;
        case OP_BINARY_MATRIX_MULTIPLY: bo = BO_MATMUL; break;
        case OP_INPLACE_ADD: bo = BO_ADD; break;
        case OP_INPLACE_SUBTRACT: bo = BO_SUB; break;
        case OP_INPLACE_MULTIPLY: bo = BO_MUL; break;
        case OP_INPLACE_TRUE_DIVIDE: bo = BO_TRUEDIV; break;
        case OP_INPLACE_FLOOR_DIVIDE: bo = BO_FLOORDIV; break;
        case OP_INPLACE_MODULO: bo = BO_MOD; break;
        case OP_INPLACE_POWER: bo = BO_POW; break;
        case OP_INPLACE_LSHIFT: bo = BO_LSHIFT; break;
        case OP_INPLACE_RSHIFT: bo = BO_RSHIFT; break;
        case OP_INPLACE_AND: bo = BO_AND; break;
        case OP_INPLACE_OR: bo = BO_OR; break;
        case OP_INPLACE_XOR: bo = BO_XOR; break;
        case OP_INPLACE_MATRIX_MULTIPLY: bo = BO_MATMUL; break;
        default: break;
      }
      const bool inplace = in.op == OP_INPLACE_ADD ||
                           in.op == OP_INPLACE_SUBTRACT ||
                           in.op == OP_INPLACE_MULTIPLY ||
                           in.op == OP_INPLACE_TRUE_DIVIDE ||
                           in.op == OP_INPLACE_FLOOR_DIVIDE ||
                           in.op == OP_INPLACE_MODULO ||
                           in.op == OP_INPLACE_POWER ||
                           in.op == OP_INPLACE_LSHIFT ||
                           in.op == OP_INPLACE_RSHIFT ||
                           in.op == OP_INPLACE_AND ||
                           in.op == OP_INPLACE_OR ||
                           in.op == OP_INPLACE_XOR ||
                           in.op == OP_INPLACE_MATRIX_MULTIPLY;
      binop(st, ins, bo, inplace);
      return 0;
    }
    case OP_BINARY_OP: {
      u64 arg = (in.flags & 2) ? 0xFFFFFFFFull : in.arg;
      bool inplace = arg >= 13;
      u64 k = inplace ? arg - 13 : arg;
      if (k >= 13) {
        py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range");
        return 0;
      }
      binop(st, ins, (u8)k, inplace);
      return 0;
    }
    case OP_BINARY_SUBSCR: {
      Node* i2 = pop_value(st, ins);
      CKR(C, 0);
      Node* o = pop_value(st, ins);
      CKR(C, 0);
      BR_PUSH(mk2(C, E_SUBSCR, o, i2));
      return 0;
    }
    case OP_COMPARE_OP:
    case OP_IS_OP:
    case OP_CONTAINS_OP: {
      Node* r = pop_value(st, ins);
      CKR(C, 0);
      Node* l = pop_value(st, ins);
      CKR(C, 0);
      u8 cmp = in.op == OP_COMPARE_OP ? argval_cmp(C, &X, in)
               : in.op == OP_IS_OP ? (in.arg ? CO_ISNOT : CO_IS) : (in.arg ? CO_NOTIN : CO_IN);
      BR_PUSH(mk_compare(C, l, cmp, r));
      return 0;
    }
    // ------------------------------------------------ shuffles (:488-546)
    case OP_POP_TOP: {
      Node* v = pop(st, ins);
      CKR(C, 0);
      switch (v->k) {
        case E_IMPORT: case E_NULL: case E_METHSELF: case E_EXCVALUE: case E_FINSENT: case E_WITHENTER:
          return 0;
      }
      if (v->f & F_LOOP_ITER) return 0;
      if (is_k(v, E_CALL) && is_k(v->a, E_WITHEXIT)) return 0;
      if (v->pend && v->pend->n) {
        NV* pend = v->pend;
        v->pend = nullptr;
        vpush(C, out, mk_assign(C, pend, v));
        return 0;
      }
      if (is_effectful(v)) vpush(C, out, mk1(C, S_EXPR, v));
      return 0;
    }
    case OP_ROT_TWO: {
      if (st->n < 2) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      Node** d = st->d + st->n;
      Node* t = d[-1]; d[-1] = d[-2]; d[-2] = t;
      return 0;
    }
    case OP_ROT_THREE: {
      if (st->n < 3) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      Node** d = st->d + st->n;
      Node *a1 = d[-1], *a2 = d[-2], *a3 = d[-3];
      d[-1] = a2; d[-2] = a3; d[-3] = a1;
      return 0;
    }
    case OP_ROT_FOUR: {
      if (st->n < 4) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      Node** d = st->d + st->n;
      Node *a1 = d[-1], *a2 = d[-2], *a3 = d[-3], *a4 = d[-4];
      d[-1] = a2; d[-2] = a3; d[-3] = a4; d[-4] = a1;
      return 0;
    }
    case OP_ROT_N: {
      if (st->n == 0) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      i64 n = (in.flags & 2) ? 0xFFFFFFFFll : (i64)in.arg;
      Node* top = st->d[--st->n];
      i64 len = st->n;
      i64 at = len - (n - 1);
      if (at < 0) { at += len; if (at < 0) at = 0; }
      if (at > len) at = len;
      vpush(C, st, (Node*)nullptr);
      CKR(C, 0);
      for (i64 q = len; q > at; q--) st->d[q] = st->d[q - 1];
      st->d[at] = top;
      return 0;
    }
    case OP_SWAP: {
      i64 i = (in.flags & 2) ? 0xFFFFFFFFll : (i64)in.arg;
      bool ok1, ok2;
      i64 n = st->n;
      i64 ki = py_norm(n, -i, &ok1);
      i64 k1 = py_norm(n, -1, &ok2);
      if (!ok1 || !ok2) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      Node* vi = st->d[ki];
      Node* v1 = st->d[k1];
      st->d[k1] = vi;
      st->d[ki] = v1;
      return 0;
    }
    case OP_COPY: {
      Node* v = py_index(C, st, -(i64)((in.flags & 2) ? 0xFFFFFFFFll : in.arg));
      CKR(C, 0);
      BR_PUSH(v);
      return 0;
    }
    case OP_DUP_TOP: {
      Node* v = py_index(C, st, -1);
      CKR(C, 0);
      BR_PUSH(v);
      return 0;
    }
    case OP_DUP_TOP_TWO: {
      u32 n = st->n;
      u32 lo = n >= 2 ? n - 2 : 0;
      for (u32 q = lo; q < n; q++) BR_PUSH(st->d[q]);
      return 0;
    }
    case OP_UNARY_NOT: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      BR_PUSH(negate(C, v));
      return 0;
    }
    case OP_UNARY_NEGATIVE:
    case OP_UNARY_POSITIVE:
    case OP_UNARY_INVERT: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      BR_PUSH(mk_unary(C, in.op == OP_UNARY_NEGATIVE ? UO_NEG : in.op == OP_UNARY_POSITIVE ? UO_POS : UO_INV, v));
      return 0;
    }
    // ------------------------------------------------ building (:550-708)
    case OP_BUILD_TUPLE:
    case OP_BUILD_LIST:
    case OP_BUILD_SET: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      Node* n = mk(C, in.op == OP_BUILD_TUPLE ? E_TUPLE : in.op == OP_BUILD_LIST ? E_LIST : E_SET);
      n->l1 = use_all(vals);
      BR_PUSH(n);
      return 0;
    }
    case OP_BUILD_MAP: {
      NV* kv = pops(st, ins, (in.flags & 2) ? 0x1FFFFFFFEull : 2ull * in.arg);
      CKR(C, 0);
      Node* n = mk(C, E_DICT);
      n->l1 = vnew<Node*>(C, kv->n / 2);
      n->l2 = vnew<Node*>(C, kv->n / 2);
      for (u32 q = 0; q < kv->n; q += 2) vpush(C, n->l1, use(kv->d[q]));
      for (u32 q = 1; q < kv->n; q += 2) vpush(C, n->l2, use(kv->d[q]));
      BR_PUSH(n);
      return 0;
    }
    case OP_BUILD_CONST_KEY_MAP: {
      Node* kc = pop(st, ins);
      CKR(C, 0);
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      NV* values = use_all(vals);
      u32 cid = const_of(kc);
      CKR(C, 0);
      if (cid == CID_INVALID) { py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'"); return 0; }
      u32 ck = ckind(C, cid);
      if (ck != UPY_C_TUPLE && ck != UPY_C_FROZENSET) { py_error(C, UPY_ST_PY_TYPE_ERROR, "const is not iterable"); return 0; }
      Node* n = mk(C, E_DICT);
      u32 ne = cnelem(C, cid);
      n->l1 = vnew<Node*>(C, ne);
      for (u32 q = 0; q < ne; q++) vpush(C, n->l1, mk_const(C, celem(C, cid, q)));
      n->l2 = values;
      BR_PUSH(n);
      return 0;
    }
    case OP_BUILD_SLICE: {
      NV* parts = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      if (parts->n < 2) { py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range"); return 0; }
      Node* n = mk(C, E_SLICE);
      n->a = none_to_null(C, parts->d[0]);
      n->b = none_to_null(C, parts->d[1]);
      if (in.arg == 3 && !(in.flags & 2)) n->c = none_to_null(C, parts->d[2]);
      BR_PUSH(n);
      return 0;
    }
    case OP_BUILD_STRING: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      NV* parts = vnew<Node*>(C, vals->n);
      for (u32 q = 0; q < vals->n; q++) {
        Node* v = vals->d[q];
        if (is_k(v, E_CONST) && v->cid != CID_INVALID && ckind(C, v->cid) == UPY_C_STR) {
          Node* sp = mk(C, X_STRPART);
          sp->s = cstr(C, v->cid);
          vpush(C, parts, sp);
        } else if (is_k(v, E_CONST) && v->cid == CID_INVALID) {
          py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'kind'");
          return 0;
        } else if (is_k(v, E_FSTRING)) {
          vextend(C, parts, v->l1);
        } else {
          vpush(C, parts, v);
        }
      }
      Node* n = mk(C, E_FSTRING);
      n->l1 = parts;
      BR_PUSH(n);
      return 0;
    }
    case OP_FORMAT_VALUE: {
      Node* spec = nullptr;
      if (in.arg & 4) {
        spec = pop(st, ins);
        CKR(C, 0);
      }
      Node* value = pop_value(st, ins);
      CKR(C, 0);
      Node* fv = mk2(C, E_FMTVAL, value, spec);
      fv->op = (u8)(in.arg & 3);
      Node* n = mk(C, E_FSTRING);
      n->l1 = nv1(C, fv);
      BR_PUSH(n);
      return 0;
    }
    case OP_LIST_APPEND:
    case OP_SET_ADD: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      if (in_comprehension()) {
        Node* a = mk(C, S_COMPACCUM);
        a->op = in.op == OP_LIST_APPEND ? 0 : 1;
        a->a = v;
        a->i = (i32)in.arg;
        vpush(C, out, a);
        return 0;
      }
      Node* target = display_target(st, ins);
      CKR(C, 0);
      u8 want = in.op == OP_LIST_APPEND ? E_LIST : E_SET;
      if (!is_k(target, want)) {
        fail_unsupported(C, in.op == OP_LIST_APPEND ? "LIST_APPEND outside display" : "SET_ADD outside display",
                         in.offset);
        return 0;
      }
      vpush(C, target->l1, v);
      return 0;
    }
    case OP_MAP_ADD: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      Node* k = pop_value(st, ins);
      CKR(C, 0);
      if (in_comprehension()) {
        Node* a = mk(C, S_COMPACCUM);
        a->op = 2;
        a->a = v;
        a->b = k;
        a->i = (i32)in.arg;
        vpush(C, out, a);
        return 0;
      }
      Node* target = display_target(st, ins);
      CKR(C, 0);
      if (!is_k(target, E_DICT)) {
        fail_unsupported(C, "MAP_ADD outside display", in.offset);
        return 0;
      }
      vpush(C, target->l1, k);
      vpush(C, target->l2, v);
      return 0;
    }
    case OP_LIST_EXTEND:
    case OP_SET_UPDATE: {
      Node* it = pop_value(st, ins);
      CKR(C, 0);
      Node* target = display_target(st, ins);
      CKR(C, 0);
      bool lst = in.op == OP_LIST_EXTEND;
      if (!is_k(target, lst ? E_LIST : E_SET)) {
        fail_unsupported(C, lst ? "LIST_EXTEND outside display" : "SET_UPDATE outside display", in.offset);
        return 0;
      }
      NV* sp = spread(C, it, !lst);
      CKR(C, 0);
      vextend(C, target->l1, sp);
      return 0;
    }
    case OP_DICT_UPDATE:
    case OP_DICT_MERGE: {
      Node* other = pop_value(st, ins);
      CKR(C, 0);
      Node* target = display_target(st, ins);
      CKR(C, 0);
      if (!is_k(target, E_DICT)) {
        fail_unsupported(C, "DICT_UPDATE outside display", in.offset);
        return 0;
      }
      bool all_keys = true;
      if (is_k(other, E_DICT))
        for (u32 q = 0; q < other->l1->n; q++)
          if (!other->l1->d[q]) all_keys = false;
      if (is_k(other, E_DICT) && other->l1->n <= 8 && all_keys) {
        vextend(C, target->l1, other->l1);
        vextend(C, target->l2, other->l2);
      } else {
        vpush(C, target->l1, (Node*)nullptr);
        vpush(C, target->l2, other);
      }
      return 0;
    }
    case OP_LIST_TO_TUPLE: {
      Node* v = pop(st, ins);
      CKR(C, 0);
      if (is_k(v, E_LIST)) {
        Node* t = mk(C, E_TUPLE);
        t->l1 = v->l1;  // shared list object
        BR_PUSH(t);
      } else {
        BR_PUSH(v);
      }
      return 0;
    }
    case OP_BUILD_TUPLE_UNPACK:
    case OP_BUILD_TUPLE_UNPACK_WITH_CALL:
    case OP_BUILD_LIST_UNPACK:
    case OP_BUILD_SET_UNPACK: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      bool as_set = in.op == OP_BUILD_SET_UNPACK;
      NV* parts = vnew<Node*>(C);
      for (u32 q = 0; q < vals->n; q++) {
        NV* sp = spread(C, vals->d[q], as_set);
        CKR(C, 0);
        vextend(C, parts, sp);
      }
      Node* n = mk(C, as_set ? E_SET : in.op == OP_BUILD_LIST_UNPACK ? E_LIST : E_TUPLE);
      n->l1 = parts;
      BR_PUSH(n);
      return 0;
    }
    case OP_BUILD_MAP_UNPACK:
    case OP_BUILD_MAP_UNPACK_WITH_CALL: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      Node* n = mk(C, E_DICT);
      n->l1 = vnew<Node*>(C);
      n->l2 = vnew<Node*>(C);
      for (u32 q = 0; q < vals->n; q++) {
        Node* v = vals->d[q];
        bool all_keys = is_k(v, E_DICT);
        if (all_keys)
          for (u32 r = 0; r < v->l1->n; r++)
            if (!v->l1->d[r]) all_keys = false;
        if (all_keys) {
          vextend(C, n->l1, v->l1);
          vextend(C, n->l2, v->l2);
        } else {
          vpush(C, n->l1, (Node*)nullptr);
          vpush(C, n->l2, v);
        }
      }
      BR_PUSH(n);
      return 0;
    }
    // ------------------------------------------------ access (:712-718)
    case OP_LOAD_ATTR: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      Node* t = mk1(C, E_ATTR, v);
      t->s = argval_name(C, &X, in);
      BR_PUSH(t);
      return 0;
    }
    case OP_LOAD_METHOD: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      Node* t = mk1(C, E_ATTR, v);
      t->s = argval_name(C, &X, in);
      BR_PUSH(t);
      BR_PUSH(mk(C, E_METHSELF));
      return 0;
    }
    // ------------------------------------------------ calls (:722-785)
    case OP_KW_NAMES: {
      Vec<Str>* kw = const_str_tuple(argval_const(C, &X, in));
      CKR(C, 0);
      K->kwnames = kw;
      K->has_kwnames = true;
      return 0;
    }
    case OP_CALL_FUNCTION: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      finish_call(st, ins, use_all(vals), nullptr);
      return 0;
    }
    case OP_CALL_FUNCTION_KW: {
      Node* kc = pop(st, ins);
      CKR(C, 0);
      u32 cid = const_of(kc);
      CKR(C, 0);
      Vec<Str>* kw = const_str_tuple(cid);
      CKR(C, 0);
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      finish_call(st, ins, use_all(vals), kw);
      return 0;
    }
    case OP_CALL_METHOD: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      NV* args = use_all(vals);
      pop(st, ins);
      CKR(C, 0);
      Node* meth = pop(st, ins);
      CKR(C, 0);
      Node* call = mk(C, E_CALL);
      call->a = meth;
      call->l1 = args;
      call->l2 = vnew<Node*>(C);
      BR_PUSH(call);
      return 0;
    }
    case OP_CALL: {
      NV* vals = pops(st, ins, (in.flags & 2) ? 0xFFFFFFFFull : in.arg);
      CKR(C, 0);
      NV* args = use_all(vals);
      Vec<Str>* kw = K->has_kwnames ? K->kwnames : nullptr;
      K->has_kwnames = false;
      K->kwnames = nullptr;
      finish_call(st, ins, args, kw);
      return 0;
    }
    case OP_CALL_FUNCTION_EX: {
      Node* kwargs = nullptr;
      if (in.arg & 1) {
        kwargs = pop_value(st, ins);
        CKR(C, 0);
      }
      Node* posargs = pop_value(st, ins);
      CKR(C, 0);
      Node* func = pop(st, ins);
      CKR(C, 0);
      if (X.minor >= 11 && st->n && is_k(vlast(st), E_NULL)) st->n--;
      NV* args = spread(C, posargs, false);
      CKR(C, 0);
      NV* kws = vnew<Node*>(C);
      if (kwargs) {
        if (is_k(kwargs, E_DICT)) {
          u32 n = kwargs->l1->n < kwargs->l2->n ? kwargs->l1->n : kwargs->l2->n;
          for (u32 q = 0; q < n; q++) {
            Node* k = kwargs->l1->d[q];
            Node* v = kwargs->l2->d[q];
            if (!k) {
              vpush(C, kws, mk_kwpair(C, Snone(), v));
            } else if (is_k(k, E_CONST) && is_const_kind(C, k, UPY_C_STR)) {
              vpush(C, kws, mk_kwpair(C, cstr(C, k->cid), v));
            } else {
              CKR(C, 0);
              Node* d = mk(C, E_DICT);
              d->l1 = nv1(C, k);
              d->l2 = nv1(C, v);
              vpush(C, kws, mk_kwpair(C, Snone(), d));
            }
          }
        } else {
          vpush(C, kws, mk_kwpair(C, Snone(), kwargs));
        }
      }
      Node* call = mk(C, E_CALL);
      call->a = func;
      call->l1 = args;
      call->l2 = kws;
      BR_PUSH(call);
      return 0;
    }
    // ------------------------------------------------ functions (:789-822)
    case OP_MAKE_FUNCTION: {
      u32 flags = in.arg;
      if (X.minor <= 10) {
        pop(st, ins);
        CKR(C, 0);
      }
      Node* code_const = pop(st, ins);
      CKR(C, 0);
      Node* fe = mk(C, E_FUNC);
      fe->l1 = vnew<Node*>(C);
      fe->l2 = vnew<Node*>(C);
      fe->l3 = vnew<Node*>(C);
      fe->sl = vnew<Str>(C);
      if (flags & 8) {
        Node* cells = pop(st, ins);
        CKR(C, 0);
        if (!(is_k(cells, E_TUPLE) || is_k(cells, E_LIST) || is_k(cells, E_SET))) {
          py_attr_error(C, cells, "elts");
          return 0;
        }
        for (u32 q = 0; q < cells->l1->n; q++) {
          Node* c = cells->l1->d[q];
          if (!is_k(c, E_NAME)) { py_attr_error(C, c, "id"); return 0; }
          vpush(C, fe->sl, c->s);
        }
      }
      if (flags & 4) {
        Node* ann = pop(st, ins);
        CKR(C, 0);
        if (is_k(ann, E_DICT)) {
          u32 n = ann->l1->n < ann->l2->n ? ann->l1->n : ann->l2->n;
          for (u32 q = 0; q < n; q++) {
            Node* k = ann->l1->d[q];
            if (!is_k(k, E_CONST) || k->cid == CID_INVALID || ckind(C, k->cid) != UPY_C_STR) {
              py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "annotation key is not a str constant");
              return 0;
            }
            vpush(C, fe->l3, mk_kwpair(C, cstr(C, k->cid), ann->l2->d[q]));
          }
        } else if (is_k(ann, E_CONST)) {
          Vec<Str>* names = const_str_tuple(ann->cid);
          CKR(C, 0);
          for (u32 q = 0; q < names->n; q++) vpush(C, fe->l3, mk_kwpair(C, names->d[q], nullptr));
        }
      }
      if (flags & 2) {
        Node* kwd = pop(st, ins);
        CKR(C, 0);
        if (!is_k(kwd, E_DICT)) { py_attr_error(C, kwd, "keys"); return 0; }
        u32 n = kwd->l1->n < kwd->l2->n ? kwd->l1->n : kwd->l2->n;
        for (u32 q = 0; q < n; q++) {
          Node* k = kwd->l1->d[q];
          if (!is_k(k, E_CONST) || k->cid == CID_INVALID || ckind(C, k->cid) != UPY_C_STR) {
            py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "kwdefault key is not a str constant");
            return 0;
          }
          vpush(C, fe->l2, mk_kwpair(C, cstr(C, k->cid), kwd->l2->d[q]));
        }
      }
      if (flags & 1) {
        Node* dflt = pop(st, ins);
        CKR(C, 0);
        if (is_k(dflt, E_TUPLE)) {
          fe->l1 = nv_copy(C, dflt->l1);
        } else {
          u32 cid = const_of(dflt);
          CKR(C, 0);
          if (cid == CID_INVALID) { py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'"); return 0; }
          u32 ck = ckind(C, cid);
          if (ck != UPY_C_TUPLE && ck != UPY_C_FROZENSET) { py_error(C, UPY_ST_PY_TYPE_ERROR, "const is not iterable"); return 0; }
          for (u32 q = 0; q < cnelem(C, cid); q++) vpush(C, fe->l1, mk_const(C, celem(C, cid, q)));
        }
      }
      u32 cc = const_of(code_const);
      CKR(C, 0);
      if (cc == CID_INVALID) { py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'"); return 0; }
      fe->cid = ckind(C, cc) == UPY_C_CODE ? (u32)cget(C, cc)->off : CID_INVALID;
      fe->j = (i32)ckind(C, cc);  // Python type of FuncExpr.code when it is not a code object
      BR_PUSH(fe);
      return 0;
    }
    // ------------------------------------------------ imports (:826-839)
    case OP_IMPORT_NAME: {
      Node* fromlist = pop(st, ins);
      CKR(C, 0);
      Node* level = pop(st, ins);
      CKR(C, 0);
      Node* n = mk(C, E_IMPORT);
      n->s = argval_name(C, &X, in);
      u32 fc = const_of(fromlist);
      CKR(C, 0);
      if (fc == CID_INVALID) { py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'kind'"); return 0; }
      if (ckind(C, fc) == UPY_C_TUPLE) {
        n->sl = const_str_tuple(fc);
        CKR(C, 0);
        n->f |= 2;
      }
      u32 lc = const_of(level);
      CKR(C, 0);
      if (lc == CID_INVALID) { py_error(C, UPY_ST_PY_ATTRIBUTE_ERROR, "'NoneType' object has no attribute 'value'"); return 0; }
      n->cid = lc;
      BR_PUSH(n);
      return 0;
    }
    case OP_IMPORT_FROM: {
      Node* top = py_index(C, st, -1);
      CKR(C, 0);
      Node* n = mk1(C, E_IMPORTFROM, top);
      n->s = argval_name(C, &X, in);
      BR_PUSH(n);
      return 0;
    }
    case OP_IMPORT_STAR: {
      Node* imp = pop(st, ins);
      CKR(C, 0);
      if (!is_k(imp, E_IMPORT)) { py_attr_error(C, imp, "module"); return 0; }
      Node* s2 = mk(C, S_IMPORTSTAR);
      s2->s = imp->s;
      s2->cid = imp->cid;
      vpush(C, out, s2);
      return 0;
    }
    // ------------------------------------------------ yields (:843-855)
    case OP_YIELD_VALUE: {
      Node* v = pop_value(st, ins);
      CKR(C, 0);
      BR_PUSH(mk1(C, E_YIELD, v));
      return 0;
    }
    case OP_YIELD_FROM:
    case OP_YIELD_FROM_311: {
      pop(st, ins);
      CKR(C, 0);
      Node* v = pop(st, ins);
      CKR(C, 0);
      BR_PUSH(mk1(C, E_YIELDFROM, v));
      return 0;
    }
    case OP_RETURN_GENERATOR: BR_PUSH(mk(C, E_NULL)); return 0;
    // ------------------------------------------------ exception plumbing (:859-917)
    case OP_SETUP_FINALLY: return 0;
    case OP_BEGIN_FINALLY: BR_PUSH(mk(C, E_FINSENT)); return 0;
    case OP_POP_FINALLY: {
      Node* preserve = nullptr;
      if (in.arg) {
        preserve = pop(st, ins);
        CKR(C, 0);
      }
      if (st->n && is_k(vlast(st), E_FINSENT)) st->n--;
      if (preserve) BR_PUSH(preserve);
      return 0;
    }
    case OP_POP_EXCEPT: {
      int n = X.minor >= 11 ? 1 : 3;
      for (int q = 0; q < n; q++)
        if (st->n) st->n--;
      return 0;
    }
    case OP_PUSH_EXC_INFO: {
      Node* exc = pop(st, ins);
      CKR(C, 0);
      Node* ev = mk(C, E_EXCVALUE);
      ev->i = 1;
      BR_PUSH(ev);
      BR_PUSH(exc);
      return 0;
    }
    case OP_CHECK_EXC_MATCH: {
      Node* ty = pop_value(st, ins);
      CKR(C, 0);
      Node* top = py_index(C, st, -1);
      CKR(C, 0);
      BR_PUSH(mk_compare(C, top, CO_EXCMATCH, ty));
      return 0;
    }
    case OP_SETUP_WITH:
    case OP_BEFORE_WITH: {
      Node* ctx = pop_value(st, ins);
      CKR(C, 0);
      BR_PUSH(mk1(C, E_WITHEXIT, ctx));
      BR_PUSH(mk1(C, E_WITHENTER, ctx));
      return 0;
    }
    case OP_WITH_CLEANUP_START: {
      if (st->n >= 2 && is_k(st->d[st->n - 1], E_FINSENT) && is_k(st->d[st->n - 2], E_WITHEXIT)) {
        Node* sent = st->d[st->n - 1];
        st->n -= 2;
        BR_PUSH(sent);
        BR_PUSH(mk(C, E_NULL));
        return 0;
      }
      fail_unsupported(C, opname_of(in.op), in.offset);
      return 0;
    }
    case OP_WITH_CLEANUP_FINISH: {
      if (st->n && is_k(vlast(st), E_NULL)) {
        st->n--;
        return 0;
      }
      fail_unsupported(C, opname_of(in.op), in.offset);
      return 0;
    }
    case OP_GET_LEN: {
      Node* top = py_index(C, st, -1);
      CKR(C, 0);
      Node* call = mk(C, E_CALL);
      call->a = mk_name(C, S("len"), SC_GLOBAL);
      call->l1 = nv1(C, top);
      call->l2 = vnew<Node*>(C);
      BR_PUSH(call);
      return 0;
    }
  }
  // no lifting rule (symexec.py:203-205), WITH_EXCEPT_START (:916-917)
  fail_unsupported(C, opname_of(in.op), in.offset);
  return 0;
}

HD inline bool is_async_op(u8 op) {  // symexec.py:35-38
  switch (op) {
    case OP_GET_AITER: case OP_GET_ANEXT: case OP_BEFORE_ASYNC_WITH: case OP_SETUP_ASYNC_WITH:
    case OP_END_ASYNC_FOR: case OP_GET_AWAITABLE: case OP_ASYNC_GEN_WRAP: case OP_SEND:
      return true;
  }
  return false;
}
HD inline bool is_nop_op(u8 op) {  // symexec.py:41-45
  switch (op) {
    case OP_NOP: case OP_RESUME: case OP_PRECALL: case OP_MAKE_CELL: case OP_COPY_FREE_VARS:
    case OP_GEN_START: case OP_SETUP_ANNOTATIONS: case OP_POP_BLOCK: case OP_GET_ITER:
    case OP_GET_YIELD_FROM_ITER: case OP_CALL_FINALLY:
      return true;
  }
  return false;
}
HD inline bool is_plain_jump(u8 op) {
  return op == OP_JUMP_FORWARD || op == OP_JUMP_ABSOLUTE || op == OP_JUMP_BACKWARD ||
         op == OP_JUMP_BACKWARD_NO_INTERRUPT;
}
// _COND_JUMPS (symexec.py:962-976): returns false when not a conditional jump
HD inline bool cond_jump_info(u8 op, bool* jump_when, int* none_test, bool* pops) {
  *none_test = -1;
  *pops = true;
  switch (op) {
    case OP_POP_JUMP_IF_FALSE: case OP_POP_JUMP_FORWARD_IF_FALSE: case OP_POP_JUMP_BACKWARD_IF_FALSE:
      *jump_when = false; return true;
    case OP_POP_JUMP_IF_TRUE: case OP_POP_JUMP_FORWARD_IF_TRUE: case OP_POP_JUMP_BACKWARD_IF_TRUE:
      *jump_when = true; return true;
    case OP_POP_JUMP_FORWARD_IF_NONE: case OP_POP_JUMP_BACKWARD_IF_NONE:
      *jump_when = true; *none_test = 1; return true;
    case OP_POP_JUMP_FORWARD_IF_NOT_NONE: case OP_POP_JUMP_BACKWARD_IF_NOT_NONE:
      *jump_when = true; *none_test = 0; return true;
    case OP_JUMP_IF_FALSE_OR_POP: *jump_when = false; *pops = false; return true;
    case OP_JUMP_IF_TRUE_OR_POP: *jump_when = true; *pops = false; return true;
  }
  return false;
}

HD inline Node* mk_condjump(Dc* C, Node* cond, bool jump_when, u32 target, bool pops) {
  Node* m = mk(C, S_CONDJUMP);
  m->a = cond;
  m->f = (jump_when ? 1 : 0) | (pops ? 2 : 0);
  m->i = (i32)target;
  return m;
}

// simulate_block (symexec.py:138-210)
HD NOINL BlockResult Sim::simulate(const Block* b, const NV* entry) {
  BlockResult R = {nullptr, nullptr, nullptr, -1};
  NV* st = nv_copy(C, entry);
  NV* out = vnew<Node*>(C);
  R.stmts = out;
  i32 i = b->lo;
  // loop invariants held in registers (the compiler must assume the arena stores of
  // every step may alias *K / *b and would reload them per instruction)
  const i32 hi_ = b->hi;
  const Ins* const ins_base = K->ins;
  const i64 depth_limit = K->o->stacksize + 6;
  const StepCtx X = {K->oi, K->minor, K->o};
  while (i < hi_) {
    CKR(C, R);
    const Ins* ins = &ins_base[i];
    u8 op = ins->op;
    if (is_async_op(op)) {
      fail_unsupported(C, opname_of(op), ins->offset);
      return R;
    }
    if (is_nop_op(op)) {
      i++;
      continue;
    }
    if (op == OP_RETURN_VALUE) {
      Node* v = pop(st, ins);
      CKR(C, R);
      vpush(C, out, mk1(C, S_RETURN, v));
      R.term = i;
      return R;
    }
    if (op == OP_RAISE_VARARGS) {
      Node *exc = nullptr, *cause = nullptr;
      u64 arg = (ins->flags & 2) ? 0xFFFFFFFFull : ins->arg;
      if (arg >= 2) {
        cause = pop(st, ins);
        CKR(C, R);
      }
      if (arg >= 1) {
        exc = pop(st, ins);
        CKR(C, R);
      }
      vpush(C, out, mk2(C, S_RAISE, exc, cause));
      R.term = i;
      return R;
    }
    if (op == OP_RERAISE) {
      R.term = i;
      return R;
    }
    if (is_plain_jump(op)) {
      Node* j = mk(C, S_JUMP);
      j->i = (i32)jump_target(K, *ins);
      vpush(C, out, j);
      R.exit_jump = st;
      R.term = i;
      return R;
    }
    bool jw, pops_;
    int nt;
    if (cond_jump_info(op, &jw, &nt, &pops_)) {
      u32 tgt = jump_target(K, *ins);
      if (pops_) {
        Node* cond = pop(st, ins);
        CKR(C, R);
        if (nt >= 0) cond = mk_compare(C, cond, nt ? CO_IS : CO_ISNOT, mk_const(C, CID_NONE_SYN));
        vpush(C, out, mk_condjump(C, cond, jw, tgt, true));
        R.exit_fall = st;
        R.exit_jump = st;
        R.term = i;
        return R;
      }
      Node* cond;
      if (st->n) {
        cond = vlast(st);
      } else {
        pop(st, ins);
        return R;
      }
      vpush(C, out, mk_condjump(C, cond, jw, tgt, false));
      NV* fall = nv_copy(C, st);
      fall->n--;
      R.exit_fall = fall;
      R.exit_jump = st;
      R.term = i;
      return R;
    }
    if (op == OP_JUMP_IF_NOT_EXC_MATCH) {
      Node* ty = pop(st, ins);
      CKR(C, R);
      Node* exc = pop(st, ins);
      CKR(C, R);
      vpush(C, out, mk_condjump(C, mk_compare(C, exc, CO_EXCMATCH, ty), false, jump_target(K, *ins), true));
      R.exit_fall = st;
      R.exit_jump = st;
      R.term = i;
      return R;
    }
    if (op == OP_FOR_ITER) {
      NV* fall = nv_copy(C, st);
      vpush(C, fall, mk1(C, E_FORITEM, st->n ? vlast(st) : nullptr));
      NV* jump = nv_copy(C, st);
      if (jump->n) jump->n--;
      R.exit_fall = fall;
      R.exit_jump = jump;
      R.term = i;
      return R;
    }
    if (op == OP_END_FINALLY) {
      if (st->n && is_k(vlast(st), E_FINSENT)) st->n--;
      R.exit_fall = st;
      R.term = i;
      return R;
    }
    int consumed = step(ins, i, hi_, st, out, X);
    CKR(C, R);
    i += 1 + consumed;
    if ((i64)st->n > depth_limit) {
      fail_depth(C, b->id, st->n, 0, false);
      return R;
    }
  }
  R.exit_fall = st;
  return R;
}
