// structurer.h -- region structuring (structurer.py:176-1197): the offset-segment
// walker that simulates blocks on demand and recovers if/elif/else, loops,
// try/except/finally, with, ternaries, and/or chains, chained compares, asserts,
// plus the tree passes (canonicalize_tree, strip_finally_copies).
#pragma once
#include "cfg.h"

enum { WX_FALL = 0, WX_JUMP = 1, WX_ENDED = 2, WX_NEXT = 3, WX_END_FINALLY = 4, WX_NONE = 5 };
struct WalkExit {
  u8 kind;
  i64 target;
  NV* stack;
};
HD inline WalkExit wx(u8 k, i64 t = -1, NV* s = nullptr) {
  WalkExit w;
  w.kind = k;
  w.target = t;
  w.stack = s;
  return w;
}

// Ctx (structurer.py:50-59); loop_exits is omitted: _resolve_jump treats a hit
// there exactly like the default case, so it never changes an outcome.
struct WCtx {
  i64 cont0, cont1;    // continue targets (-1 = absent)
  i64 brk;
  Vec<i64>* joins;
  i64 range_end;
};
HD inline bool ctx_is_cont(const WCtx* c, i64 t) { return t == c->cont0 || t == c->cont1; }
HD inline bool ctx_in_joins(const WCtx* c, i64 t) {
  for (u32 i = 0; c->joins && i < c->joins->n; i++)
    if (c->joins->d[i] == t) return true;
  return false;
}

struct Segs {
  int n;
  i64 s[2], e[2];
};
HD inline Segs seg1(i64 a, i64 b) {
  Segs s;
  s.n = 1;
  s.s[0] = a;
  s.e[0] = b;
  s.s[1] = s.e[1] = 0;
  return s;
}

HD inline NV* nv_pass(Dc* C) { return nv1(C, mk(C, S_PASS)); }
HD inline NV* or_pass(Dc* C, NV* v) { return (v && v->n) ? v : nv_pass(C); }

// _bool_join (structurer.py:1021-1028); BoolOp.op 0 = and, 1 = or
HD inline Node* bool_join(Dc* C, u8 op, Node* a, Node* b) {
  NV* parts = vnew<Node*>(C, 4);
  Node* ab[2] = {a, b};
  for (int q = 0; q < 2; q++) {
    Node* e = ab[q];
    if (is_k(e, E_BOOLOP) && e->op == op) vextend(C, parts, e->l1);
    else vpush(C, parts, e);
  }
  Node* n = mk(C, E_BOOLOP);
  n->op = op;
  n->l1 = parts;
  return n;
}

// block-list fields by attribute name (getattr(s, "then"/"orelse"/"body"/"final"))
enum { FLD_THEN = 0, FLD_ORELSE = 1, FLD_BODY = 2, FLD_FINAL = 3 };
HD inline NV** stmt_field(Node* s, int f) {
  switch (s->k) {
    case S_IF: return f == FLD_THEN ? &s->l1 : f == FLD_ORELSE ? &s->l2 : nullptr;
    case S_WHILE: case S_WHILESHAPE: return f == FLD_BODY ? &s->l1 : f == FLD_ORELSE ? &s->l2 : nullptr;
    case S_FOR: return f == FLD_BODY ? &s->l1 : f == FLD_ORELSE ? &s->l2 : nullptr;
    case S_TRY:
      return f == FLD_BODY ? &s->l1 : f == FLD_ORELSE ? &s->l3 : f == FLD_FINAL ? &s->l4 : nullptr;
    case S_WITH: return f == FLD_BODY ? &s->l2 : nullptr;
    case S_FUNCDEF: return f == FLD_BODY ? &s->l1 : nullptr;
    case S_CLASSDEF: return f == FLD_BODY ? &s->l3 : nullptr;
  }
  return nullptr;
}

// _strip_trailing_continue (structurer.py:992-1002), in place
HD inline NV* strip_trailing_continue(Dc* C, NV* body) {
  GUARD(C);
  CKR(C, body);
  while (body->n && is_k(vlast(body), S_CONTINUE)) body->n--;
  if (body->n && is_k(vlast(body), S_TRY)) {
    Node* t = vlast(body);
    strip_trailing_continue(C, t->l1);
    for (u32 h = 0; h < t->l2->n; h++) strip_trailing_continue(C, t->l2->d[h]->l1);
    if (t->l3->n) strip_trailing_continue(C, t->l3);
  }
  return body;
}

HD inline bool is_cleanup_pair(Dc* C, NV* st, u32 lo, Str name) {  // structurer.py:1058-1070
  Node* a = st->d[lo];
  Node* b = st->d[lo + 1];
  if (!is_k(a, S_ASSIGN) || a->l1->n != 1 || !is_k(a->l1->d[0], E_NAME) || !s_eq(a->l1->d[0]->s, name))
    return false;
  if (!is_k(a->a, E_CONST)) return false;
  if (node_ckind(C, a->a) != UPY_C_NONE) return false;
  if (!is_k(b, S_DELETE)) return false;
  if (b->l1->n == 0) {
    py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range");
    return false;
  }
  return is_k(b->l1->d[0], E_NAME) && s_eq(b->l1->d[0]->s, name);
}
HD inline NV* strip_as_cleanup(Dc* C, NV* body, Str name) {  // structurer.py:1073-1086
  if (s_is_none(name)) return body;
  if (body->n == 1 && is_k(body->d[0], S_TRY) && body->d[0]->l2->n == 0 && body->d[0]->l3->n == 0 &&
      body->d[0]->l4->n == 2 && is_cleanup_pair(C, body->d[0]->l4, 0, name))
    return body->d[0]->l1;
  CKR(C, body);
  if (body->n >= 2 && is_cleanup_pair(C, body, body->n - 2, name)) return vcopy<Node*>(C, body, 0, body->n - 2);
  return body;
}

// strip_finally_copies (structurer.py:1089-1112)
HD NOINL NV* strip_finally_copies(Dc* C, NV* stmts, NV* final) {
  GUARD(C);
  CKR(C, stmts);
  if (!final->n) return stmts;
  u32 n = final->n;
  NV* out = vnew<Node*>(C, stmts->n);
  u32 i = 0;
  while (i < stmts->n && !C->err) {
    bool eq = i + n <= stmts->n;
    for (u32 q = 0; eq && q < n; q++) eq = node_eq(C, stmts->d[i + q], final->d[q]);
    if (eq) {
      Node* nxt = i + n < stmts->n ? stmts->d[i + n] : nullptr;
      if (!nxt || is_k(nxt, S_RETURN) || is_k(nxt, S_BREAK) || is_k(nxt, S_CONTINUE)) {
        i += n;
        continue;
      }
    }
    Node* s = stmts->d[i];
    for (int f = 0; f < 4; f++) {
      NV** sub = stmt_field(s, f);
      if (sub && *sub) *sub = strip_finally_copies(C, *sub, final);
    }
    if (is_k(s, S_TRY))
      for (u32 h = 0; h < s->l2->n; h++) s->l2->d[h]->l1 = strip_finally_copies(C, s->l2->d[h]->l1, final);
    vpush(C, out, s);
    i++;
  }
  return out;
}

// ------------------------------------------------------------ canonicalize
HD NV* canonicalize_tree(Dc* C, NV* stmts);

HD inline Node* canon_children(Dc* C, Node* s) {
  for (int f = 0; f < 4; f++) {
    NV** sub = stmt_field(s, f);
    if (sub && *sub) *sub = canonicalize_tree(C, *sub);
  }
  if (is_k(s, S_TRY))
    for (u32 h = 0; h < s->l2->n; h++) s->l2->d[h]->l1 = canonicalize_tree(C, s->l2->d[h]->l1);
  return s;
}
HD inline Node* mk_while(Dc* C, Node* cond, NV* body, NV* orelse) {
  Node* w = mk(C, S_WHILE);
  w->a = cond;
  w->l1 = body;
  w->l2 = orelse;
  return w;
}
// _while_guard_merge (structurer.py:1138-1163)
HD inline Node* while_guard_merge(Dc* C, Node* cond, Node* shape) {
  NV* body = nv_copy(C, shape->l1);
  Node* tail = shape->b;
  while (!C->err) {
    if (tail && node_eq(C, tail, cond)) return mk_while(C, cond, or_pass(C, body), shape->l2);
    if (!body->n) return nullptr;
    Node* last = vlast(body);
    if (is_k(last, S_IF) && last->l2->n == 0 && last->l1->n == 1 && is_k(last->l1->d[0], S_BREAK)) {
      Node* piece = negate(C, last->a);
      tail = tail ? bool_join(C, 0, piece, tail) : piece;
      body->n--;
      continue;
    }
    return nullptr;
  }
  return nullptr;
}
HD NOINL Node* canon_one(Dc* C, Node* s) {  // structurer.py:1166-1197
  GUARD(C);
  CKR(C, s);
  if (is_k(s, S_IF) && s->l1->n == 1 && is_k(s->l1->d[0], S_WHILESHAPE) && s->l2->n == 0) {
    Node* merged = while_guard_merge(C, s->a, s->l1->d[0]);
    if (merged) return canon_children(C, merged);
  }
  if (is_k(s, S_WHILESHAPE)) {
    NV* body = s->l1;
    if (s->b) {
      body = nv_copy(C, s->l1);
      vpush(C, body, mk_if(C, negate(C, s->b), nv1(C, mk(C, S_BREAK)), nullptr));
    }
    return canon_children(C, mk_while(C, s->a, body, s->l2));
  }
  s = canon_children(C, s);
  if (is_k(s, S_IF)) {
    if (s->l1->n == 1 && is_k(s->l1->d[0], S_IF) && s->l2->n == 0 && s->l1->d[0]->l2->n == 0) {
      Node* inner = s->l1->d[0];
      return mk_if(C, bool_join(C, 0, s->a, inner->a), inner->l1, nullptr);
    }
    return s;
  }
  if (is_k(s, S_WITH)) {
    if (s->l2->n == 1 && is_k(s->l2->d[0], S_WITH)) {
      Node* inner = s->l2->d[0];
      Node* w = mk(C, S_WITH);
      w->l1 = nv_copy(C, s->l1);
      vextend(C, w->l1, inner->l1);
      w->l2 = inner->l2;
      return w;
    }
    return s;
  }
  return s;
}
HD inline NV* canonicalize_tree(Dc* C, NV* stmts) {
  GUARD(C);
  NV* out = vnew<Node*>(C, stmts ? stmts->n : 0);
  CKR(C, out);
  for (u32 i = 0; stmts && i < stmts->n && !C->err; i++) vpush(C, out, canon_one(C, stmts->d[i]));
  return out;
}

// ------------------------------------------------------------ structurer
struct Structurer {
  Dc* C;
  Code* K;
  Cfg* G;
  Sim sim;
  Vec<TryRegion>* regions;
  Vec<i32>* rbs_idx;   // region indices of kinds except/finally/with, grouped by start, outermost first
  i64 temp_counter;
  Vec<i32>* active_regions;
  u8* active_loops;    // per block id
  u32 end_offset;
  // _lexical_exits index: non-SETUP jumps in offset order, targets, and the max
  // target of each run of 32 (built on first use; C3-shape objects never need it)
  i32 nj;
  u32* joff;
  u32* jtgt;
  u32* jblk;

  HD i64 new_temp() { return temp_counter++; }

  HD const Block* block_at_or_fail(i64 off) {
    i32 b = off >= 0 && off <= 0xFFFFFFFFll ? block_at(G, (u32)off) : -1;
    if (b < 0) {
      fail_struct(C, off, "no block starts here");
      return nullptr;
    }
    return &G->blocks[b];
  }
  HD BlockResult simulate(const Block* b, NV* stack) {
    if (!stack) {
      py_error(C, UPY_ST_PY_TYPE_ERROR, "'NoneType' object is not iterable");
      BlockResult r = {nullptr, nullptr, nullptr, -1};
      return r;
    }
    return sim.simulate(b, stack);
  }
  // first index in rbs_idx (sorted by start, then -end) whose region starts at pos, or n
  HD u32 regions_at(i64 pos) {
    u32 lo = 0, hi = rbs_idx->n;
    while (lo < hi) {
      u32 mid = (lo + hi) >> 1;
      if ((i64)regions->d[rbs_idx->d[mid]].start < pos) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
  HD bool region_starts_at(i64 pos) {
    u32 q = regions_at(pos);
    return q < rbs_idx->n && (i64)regions->d[rbs_idx->d[q]].start == pos;
  }
  HD bool region_active(i32 r) {
    for (u32 q = 0; q < active_regions->n; q++)
      if (active_regions->d[q] == r) return true;
    return false;
  }
  // max(_lexical_exits(lo, hi)) (structurer.py:331-339), -1 if empty.  The exits are
  // the targets >= hi of jumps in [lo, hi), so the answer is the range max of targets
  // when that max is >= hi: answered from 32-wide block maxima instead of a full scan.
  HD i64 lexical_exit_max(i64 lo, i64 hi) {
    if (!joff) {
      i32 n = 0;
      for (i32 i = 0; i < K->n_ins; i++)
        if (ins_is_jump(K->ins[i]) && !is_setup_op(K->ins[i].op)) n++;
      joff = (u32*)ualloc(C, (u64)n * 4 + 4);
      jtgt = (u32*)ualloc(C, (u64)n * 4 + 4);
      jblk = (u32*)zalloc(C, (u64)(n / 32 + 1) * 4);
      CKR(C, -1);
      nj = 0;
      for (i32 i = 0; i < K->n_ins; i++) {
        const Ins& in = K->ins[i];
        if (!ins_is_jump(in) || is_setup_op(in.op)) continue;
        joff[nj] = in.offset;
        jtgt[nj] = jump_target(K, in);
        if (jtgt[nj] > jblk[nj >> 5]) jblk[nj >> 5] = jtgt[nj];
        nj++;
      }
    }
    auto lb = [&](i64 v) {
      i32 a = 0, b = nj;
      while (a < b) {
        i32 mid = (a + b) >> 1;
        if ((i64)joff[mid] < v) a = mid + 1;
        else b = mid;
      }
      return a;
    };
    i32 i0 = lb(lo), i1 = lb(hi);
    i64 m = -1;
    i32 i = i0;
    while (i < i1 && (i & 31)) m = (i64)jtgt[i] > m ? (i64)jtgt[i] : m, i++;
    while (i + 32 <= i1) m = (i64)jblk[i >> 5] > m ? (i64)jblk[i >> 5] : m, i += 32;
    while (i < i1) m = (i64)jtgt[i] > m ? (i64)jtgt[i] : m, i++;
    return m >= hi ? m : -1;
  }
  HD WCtx* ctx_new(i64 c0, i64 c1, i64 brk) {
    WCtx* c = anew<WCtx>(C);
    c->cont0 = c0;
    c->cont1 = c1;
    c->brk = brk;
    c->joins = nullptr;
    c->range_end = (i64)1 << 60;
    return c;
  }
  HD WCtx* ctx_with_join(const WCtx* ctx, i64 off) {
    WCtx* c = anew<WCtx>(C);
    *c = *ctx;
    c->joins = vcopy<i64>(C, ctx->joins);
    vpush(C, c->joins, off);
    return c;
  }
  HD WCtx* ctx_no_joins(const WCtx* ctx) {
    WCtx* c = anew<WCtx>(C);
    *c = *ctx;
    c->joins = nullptr;
    return c;
  }
  HD WCtx* ctx_range(const WCtx* ctx, i64 range_end) {
    WCtx* c = anew<WCtx>(C);
    *c = *ctx;
    c->range_end = range_end;
    return c;
  }

  HD NV* structure() {
    WalkExit ex;
    return walk(seg1(K->ins[0].offset, end_offset), vnew<Node*>(C), ctx_new(-1, -1, -1), &ex);
  }

  HD NV* walk(Segs segs, NV* stack, const WCtx* ctx, WalkExit* ex);
  HD WalkExit consume_block(const Block* b, BlockResult& res, NV* out, NV* stack, const WCtx* ctx);
  HD WalkExit resolve_jump(i64 target, NV* stack, NV* out, const WCtx* ctx);
  HD i64 structure_loop(i32 li, const Block* header, NV* out, NV** stack, const WCtx* ctx);
  HD i64 structure_for(i32 li, const Block* header, BlockResult& hres, NV* out, NV** stack, const WCtx* ctx);
  HD i64 structure_while_true(i32 li, const Block* header, NV* out, NV** stack, const WCtx* ctx, i64 lo, i64 hi);
  HD NV* loop_orelse(i64 after, i64 brk, NV* stack, const WCtx* ctx, i64* cont);
  HD WalkExit structure_conditional(const Block* b, Node* marker, BlockResult& res, NV* out, NV* stack,
                                    const WCtx* ctx);
  HD void collect_chain(Node** fall_cond, i64* target, i64* fall_pos, NV** fall_state);
  HD WalkExit structure_orpop(const Block* b, Node* marker, BlockResult& res, NV* out, NV* stack, const WCtx* ctx);
  HD bool is_chain_fixup(i64 off, bool returning);
  HD i64 structure_region(i32 r, NV* out, NV** stack, const WCtx* ctx);
  HD NV* exc_entry_stack(NV* stack);
  HD i64 structure_with(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx);
  HD i64 after_handler_code(const TryRegion& R);
  HD i64 structure_finally(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx);
  HD i64 structure_finally_38(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx);
  HD i64 structure_except(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx);
  HD NV* parse_handlers(const TryRegion& R, const WCtx* ctx, i64* join);
  HD NV* walk_arm(i64 arm_start, NV* arm_stack, const WCtx* ctx, i64 limit, Str* name, i64* join);
};

#define NO_POS ((i64)-0x7FFFFFFFFFFFFFFFll)

// walk (structurer.py:226-278)
HD NOINL NV* Structurer::walk(Segs segs, NV* stack, const WCtx* ctx, WalkExit* ex) {
  GUARD(C);
  NV* out = vnew<Node*>(C);
  *ex = wx(WX_ENDED);
  CKR(C, out);
  int si = 0;
  i64 pos = segs.s[0];
  while (!C->err) {
    if (pos >= segs.e[si]) {
      si++;
      if (si >= segs.n) {
        *ex = wx(WX_FALL, pos, stack);
        return out;
      }
      pos = segs.s[si];
      continue;
    }
    i32 bid = pos >= 0 && pos <= 0xFFFFFFFFll ? block_at(G, (u32)pos) : -1;
    if (bid < 0) {
      *ex = wx(WX_ENDED);
      return out;
    }
    // first region starting here that is not active (outermost first)
    i32 region = -1;
    for (u32 q = regions_at(pos); q < rbs_idx->n && region < 0; q++) {
      i32 r = rbs_idx->d[q];
      if ((i64)regions->d[r].start != pos) break;
      if (!region_active(r)) region = r;
    }
    if (region >= 0) {
      pos = structure_region(region, out, &stack, ctx);
      if (pos == NO_POS) {
        *ex = wx(WX_ENDED);
        return out;
      }
      continue;
    }
    const Block* block = &G->blocks[bid];
    i32 li = G->loop_of_header[bid];
    if (li >= 0 && !active_loops[bid]) {
      pos = structure_loop(li, block, out, &stack, ctx);
      if (pos == NO_POS) {
        *ex = wx(WX_ENDED);
        return out;
      }
      continue;
    }
    const WCtx* ictx = ctx_range(ctx, segs.e[si]);
    BlockResult res = simulate(block, stack);
    CKR(C, out);
    WalkExit e = consume_block(block, res, out, stack, ictx);
    CKR(C, out);
    if (e.kind == WX_NONE) {
      pos = block->end;
      stack = res.exit_fall;
      continue;
    }
    if (e.kind == WX_NEXT) {
      pos = e.target;
      stack = e.stack;
      continue;
    }
    *ex = e;
    return out;
  }
  return out;
}

// _consume_block (structurer.py:280-310)
HD NOINL WalkExit Structurer::consume_block(const Block* b, BlockResult& res, NV* out, NV* stack,
                                             const WCtx* ctx) {
  if (res.term < 0) {
    vextend(C, out, res.stmts);
    return wx(WX_NONE);
  }
  const Ins& term = K->ins[res.term];
  u8 op = term.op;
  if (op == OP_RETURN_VALUE || op == OP_RAISE_VARARGS || op == OP_RERAISE) {
    vextend(C, out, res.stmts);
    return wx(WX_ENDED);
  }
  if (op == OP_END_FINALLY) {
    vextend(C, out, res.stmts);
    return wx(WX_END_FINALLY, b->end, res.exit_fall);
  }
  if (is_plain_jump(op)) {
    vextend(C, out, res.stmts, 0, res.stmts->n ? res.stmts->n - 1 : 0);
    return resolve_jump(jump_target(K, term), res.exit_jump, out, ctx);
  }
  if (op == OP_FOR_ITER) {
    fail_struct(C, b->id, "FOR_ITER outside a loop header");
    return wx(WX_ENDED);
  }
  vextend(C, out, res.stmts, 0, res.stmts->n ? res.stmts->n - 1 : 0);
  Node* marker = vlast(res.stmts);
  return structure_conditional(b, marker, res, out, stack, ctx);
}

HD inline WalkExit Structurer::resolve_jump(i64 target, NV* stack, NV* out, const WCtx* ctx) {
  if (ctx_is_cont(ctx, target)) {
    vpush(C, out, mk(C, S_CONTINUE));
    return wx(WX_ENDED);
  }
  if (target == ctx->brk) {
    vpush(C, out, mk(C, S_BREAK));
    return wx(WX_ENDED);
  }
  return wx(WX_JUMP, target, stack);
}

// ------------------------------------------------------------ loops
HD NOINL i64 Structurer::structure_loop(i32 li, const Block* header, NV* out, NV** stack, const WCtx* ctx) {
  GUARD(C);
  CKR(C, NO_POS);
  const Loop& L = G->loops->d[li];
  i64 lo = 0x7FFFFFFFFFFFll, hi = -1;
  for (u32 q = 0; q < L.body->n; q++) {
    const Block& B = G->blocks[L.body->d[q]];
    if ((i64)B.start < lo) lo = B.start;
    if ((i64)B.end > hi) hi = B.end;
  }
  active_loops[header->id] = 1;
  i64 r = NO_POS;
  do {
    BlockResult hres = simulate(header, *stack);
    if (C->err) break;
    if (hres.term >= 0 && K->ins[hres.term].op == OP_FOR_ITER) {
      r = structure_for(li, header, hres, out, stack, ctx);
      break;
    }
    if (hres.term >= 0) {
      if (hres.stmts->n == 0) {  // hres.stmts[-1] on an empty list
        py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range");
        break;
      }
      Node* marker = vlast(hres.stmts);
      i64 tgt = is_k(marker, S_CONDJUMP) ? jump_target(K, K->ins[hres.term]) : 0;
      if (hres.stmts->n == 1 && is_k(marker, S_CONDJUMP) && (marker->f & 2) && !(lo <= tgt && tgt < hi)) {
        // while with leading test (3.8/3.9 layout)
        Node* cond = (marker->f & 1) ? negate(C, marker->a) : marker->a;
        i64 after = tgt;
        i64 lx = lexical_exit_max(header->end, after);
        i64 brk = lx > after ? lx : after;
        const WCtx* bctx = ctx_new(header->start, -1, brk);
        WalkExit ex;
        NV* body = walk(seg1(header->end, after), hres.exit_jump, bctx, &ex);
        if (C->err) break;
        body = or_pass(C, strip_trailing_continue(C, body));
        i64 cont;
        NV* orelse = loop_orelse(after, brk, *stack, ctx, &cont);
        if (C->err) break;
        vpush(C, out, mk_while(C, cond, body, orelse));
        r = cont;
        break;
      }
    }
    r = structure_while_true(li, header, out, stack, ctx, lo, hi);
  } while (0);
  active_loops[header->id] = 0;
  return C->err ? NO_POS : r;
}

HD NOINL i64 Structurer::structure_for(i32 li, const Block* header, BlockResult& hres, NV* out, NV** stack,
                                        const WCtx* ctx) {
  const Ins& term = K->ins[hres.term];
  i64 after = jump_target(K, term);
  NV* st = *stack;
  Node* iter_expr = st->n ? vlast(st) : nullptr;
  if (!iter_expr) {
    fail_struct(C, header->id, "FOR_ITER with empty stack");
    return NO_POS;
  }
  iter_expr->f |= F_LOOP_ITER;
  vextend(C, out, hres.stmts);
  i64 lx = lexical_exit_max(header->end, after);
  i64 brk = lx > after ? lx : after;
  const WCtx* bctx = ctx_new(header->start, -1, brk);
  WalkExit ex;
  NV* body = walk(seg1(header->end, after), hres.exit_fall, bctx, &ex);
  CKR(C, NO_POS);
  // _extract_for_target (structurer.py:1005-1013)
  if (!body->n) {
    fail_struct(C, header->id, "empty for body");
    return NO_POS;
  }
  Node* first = body->d[0];
  if (!(is_k(first, S_ASSIGN) && first->l1->n == 1 && is_k(first->a, E_FORITEM))) {
    fail_struct(C, header->id, "for loop does not store its item");
    return NO_POS;
  }
  Node* target = first->l1->d[0];
  body = vcopy<Node*>(C, body, 1);
  body = or_pass(C, strip_trailing_continue(C, body));
  i64 cont;
  NV* orelse = loop_orelse(after, brk, st, ctx, &cont);
  CKR(C, NO_POS);
  Node* f = mk(C, S_FOR);
  f->a = target;
  f->b = iter_expr;
  f->l1 = body;
  f->l2 = orelse;
  vpush(C, out, f);
  *stack = vcopy<Node*>(C, st, 0, st->n - 1);
  return cont;
}

HD inline bool is_pop_jump(u8 op) {
  switch (op) {
    case OP_POP_JUMP_IF_FALSE: case OP_POP_JUMP_IF_TRUE: case OP_POP_JUMP_FORWARD_IF_FALSE:
    case OP_POP_JUMP_FORWARD_IF_TRUE: case OP_POP_JUMP_BACKWARD_IF_FALSE: case OP_POP_JUMP_BACKWARD_IF_TRUE:
    case OP_POP_JUMP_FORWARD_IF_NONE: case OP_POP_JUMP_FORWARD_IF_NOT_NONE:
    case OP_POP_JUMP_BACKWARD_IF_NONE: case OP_POP_JUMP_BACKWARD_IF_NOT_NONE:
      return true;
  }
  return false;
}

HD NOINL i64 Structurer::structure_while_true(i32 li, const Block* header, NV* out, NV** stack,
                                               const WCtx* ctx, i64 lo, i64 hi) {
  const Loop& L = G->loops->d[li];
  i64 lx = lexical_exit_max(lo, hi);
  i64 after = hi;
  i64 brk = lx > hi ? lx : hi;
  const Block* tail = nullptr;
  for (u32 q = 0; q < L.back_tails->n; q++) {
    const Block& ub = G->blocks[L.back_tails->d[q]];
    if (ub.hi <= ub.lo) {
      py_error(C, UPY_ST_PY_INDEX_ERROR, "list index out of range");
      return NO_POS;
    }
    u8 op = K->ins[ub.hi - 1].op;
    if (is_pop_jump(op) || op == OP_JUMP_IF_TRUE_OR_POP || op == OP_JUMP_IF_FALSE_OR_POP) {
      tail = &ub;
      break;
    }
  }
  const WCtx* bctx = ctx_new(header->start, tail ? (i64)tail->start : -1, brk);
  Segs segs = seg1(header->start, hi);
  if (lo < (i64)header->start) {
    segs.n = 2;
    segs.s[1] = lo;
    segs.e[1] = header->start;
  }
  if (tail && tail->start >= header->start) {
    segs.e[0] = tail->start;
    if (lo < (i64)header->start) {
      fail_struct(C, header->id, "rotated loop with tail re-test");
      return NO_POS;
    }
  }
  WalkExit ex;
  NV* body = walk(segs, *stack, bctx, &ex);
  CKR(C, NO_POS);
  Node* cond = mk_const(C, CID_TRUE_SYN);
  Node* tail_cond = nullptr;
  if (tail) {
    BlockResult tres = simulate(tail, *stack);
    CKR(C, NO_POS);
    Node* marker = tres.stmts->n ? vlast(tres.stmts) : nullptr;
    if (is_k(marker, S_CONDJUMP) && tres.stmts->n == 1 && marker->i == (i32)header->start) {
      tail_cond = (marker->f & 1) ? marker->a : negate(C, marker->a);
    } else {
      WalkExit ex2;
      NV* extra = walk(seg1(tail->start, hi), *stack, bctx, &ex2);
      CKR(C, NO_POS);
      vextend(C, body, extra);
      if (ex2.kind == WX_FALL) vpush(C, body, mk(C, S_BREAK));
    }
  }
  body = or_pass(C, strip_trailing_continue(C, body));
  i64 cont;
  NV* orelse = loop_orelse(after, brk, *stack, ctx, &cont);
  CKR(C, NO_POS);
  Node* w = mk(C, S_WHILESHAPE);
  w->a = cond;
  w->l1 = body;
  w->l2 = orelse;
  w->b = tail_cond;
  vpush(C, out, w);
  return cont;
}

HD inline NV* Structurer::loop_orelse(i64 after, i64 brk, NV* stack, const WCtx* ctx, i64* cont) {
  if (brk > after) {
    WalkExit ex;
    NV* orelse = walk(seg1(after, brk), stack, ctx_with_join(ctx, brk), &ex);
    *cont = brk;
    return orelse;
  }
  *cont = after;
  return vnew<Node*>(C);
}

// ------------------------------------------------------------ conditionals
HD inline bool is_assertion_raise(const Node* s) {  // structurer.py:1031-1037
  const Node* e = s->a;
  if (is_k(e, E_NAME) && s_eqc(e->s, "AssertionError")) return true;
  if (is_k(e, E_CALL) && is_k(e->a, E_NAME) && s_eqc(e->a->s, "AssertionError")) return true;
  return false;
}

HD NOINL WalkExit Structurer::structure_conditional(const Block* block, Node* marker, BlockResult& res,
                                                     NV* out, NV* stack, const WCtx* ctx) {
  GUARD(C);
  CKR(C, wx(WX_ENDED));
  Node* cond = marker->a;
  bool jump_when = marker->f & 1;
  i64 target = marker->i;
  NV* fall_state = res.exit_fall;
  NV* jump_state = res.exit_jump;

  if (target <= (i64)block->start) {
    if (ctx_is_cont(ctx, target)) {
      Node* c = jump_when ? cond : negate(C, cond);
      vpush(C, out, mk_if(C, c, nv1(C, mk(C, S_CONTINUE)), nullptr));
      return wx(WX_NEXT, block->end, fall_state);
    }
    fail_struct(C, block->id, "unexpected backward conditional jump");
    return wx(WX_ENDED);
  }
  if (!(marker->f & 2)) return structure_orpop(block, marker, res, out, stack, ctx);

  Node* ctf = jump_when ? negate(C, cond) : cond;
  i64 fall_pos = block->end;
  collect_chain(&ctf, &target, &fall_pos, &fall_state);
  CKR(C, wx(WX_ENDED));

  if (ctx_is_cont(ctx, target)) {
    vpush(C, out, mk_if(C, negate(C, ctf), nv1(C, mk(C, S_CONTINUE)), nullptr));
    return wx(WX_NEXT, fall_pos, fall_state);
  }
  if (target == ctx->brk && !ctx_in_joins(ctx, target)) {
    vpush(C, out, mk_if(C, negate(C, ctf), nv1(C, mk(C, S_BREAK)), nullptr));
    return wx(WX_NEXT, fall_pos, fall_state);
  }

  const WCtx* then_ctx = ctx_with_join(ctx, target);
  WalkExit tx;
  NV* then_stmts = walk(seg1(fall_pos, target), fall_state, then_ctx, &tx);
  CKR(C, wx(WX_ENDED));

  if (tx.kind == WX_FALL && tx.target > target) {
    vpush(C, out, mk_if(C, ctf, then_stmts, nullptr));
    return wx(WX_NEXT, tx.target, tx.stack ? tx.stack : jump_state);
  }
  if (then_stmts->n == 1 && is_k(then_stmts->d[0], S_RAISE) && is_assertion_raise(then_stmts->d[0]) &&
      tx.kind == WX_ENDED) {
    Node* r = then_stmts->d[0];
    Node* msg = (is_k(r->a, E_CALL) && r->a->l1->n) ? r->a->l1->d[0] : nullptr;
    Node* as = mk2(C, S_ASSERT, negate(C, ctf), msg);
    vpush(C, out, as);
    return wx(WX_NEXT, target, jump_state);
  }
  if (tx.kind == WX_ENDED) {
    vpush(C, out, mk_if(C, ctf, then_stmts, nullptr));
    return wx(WX_NEXT, target, jump_state);
  }
  if (tx.kind == WX_JUMP && tx.target != target) {
    i64 join = tx.target;
    if (join <= target || join > ctx->range_end) {
      WalkExit mx;
      NV* more = walk(seg1(join, end_offset), tx.stack, ctx, &mx);
      CKR(C, wx(WX_ENDED));
      vextend(C, then_stmts, more);
      vpush(C, out, mk_if(C, ctf, then_stmts, nullptr));
      return wx(WX_NEXT, target, jump_state);
    }
    WalkExit ex;
    NV* else_stmts = walk(seg1(target, join), jump_state, ctx_with_join(ctx, join), &ex);
    CKR(C, wx(WX_ENDED));
    NV* then_state = tx.stack;
    NV* else_state = (ex.kind == WX_JUMP || ex.kind == WX_FALL) ? ex.stack : nullptr;
    if (!then_stmts->n && !else_stmts->n && then_state && else_state && fall_state &&
        then_state->n == fall_state->n + 1 && else_state->n == fall_state->n + 1) {
      bool same = true;
      for (u32 q = 0; same && q + 1 < then_state->n; q++)
        same = then_state->d[q] == else_state->d[q] || node_eq(C, then_state->d[q], else_state->d[q]);
      CKR(C, wx(WX_ENDED));
      if (same) {
        NV* merged = vcopy<Node*>(C, then_state, 0, then_state->n - 1);
        Node* t = mk(C, E_TERNARY);
        t->a = ctf;
        t->b = vlast(then_state);
        t->c = vlast(else_state);
        vpush(C, merged, t);
        return wx(WX_NEXT, join, merged);
      }
    }
    if (then_state && else_state) {
      if (then_state->n != else_state->n) {
        fail_depth(C, block->id, then_state->n, else_state->n, true);
        return wx(WX_ENDED);
      }
      bool same = nv_eq(C, then_state, else_state);
      CKR(C, wx(WX_ENDED));
      if (same) {
        vpush(C, out, mk_if(C, ctf, then_stmts, else_stmts));
        return wx(WX_NEXT, join, then_state);
      }
      // merge_stack_states (symexec.py:1027-1051)
      NV* merged = vnew<Node*>(C, then_state->n);
      for (u32 q = 0; q < then_state->n && !C->err; q++) {
        Node* a = then_state->d[q];
        Node* b = else_state->d[q];
        if (a == b || node_eq(C, b, a)) {
          vpush(C, merged, a);
          continue;
        }
        i64 k = new_temp();
        vpush(C, then_stmts, mk_assign(C, nv1(C, mk_name_syn(C, "__stack_", k, SC_FAST)), a));
        vpush(C, else_stmts, mk_assign(C, nv1(C, mk_name_syn(C, "__stack_", k, SC_FAST)), b));
        vpush(C, merged, mk_name_syn(C, "__stack_", k, SC_FAST));
      }
      vpush(C, out, mk_if(C, ctf, then_stmts, else_stmts));
      return wx(WX_NEXT, join, merged);
    }
    vpush(C, out, mk_if(C, ctf, then_stmts, else_stmts));
    return wx(WX_NEXT, join, then_state ? then_state : else_state);
  }
  // then-range fell to the target (or jumped to it): plain if
  NV* then_state = tx.stack;
  if (then_state && then_state->n != jump_state->n) {
    fail_struct(C, block->id, "branch leaves a value on one path");
    return wx(WX_ENDED);
  }
  if (then_state) {
    bool same = nv_eq(C, then_state, jump_state);
    CKR(C, wx(WX_ENDED));
    if (!same) {
      NV* merged = vnew<Node*>(C, then_state->n);
      NV* pre = vnew<Node*>(C);
      for (u32 q = 0; q < then_state->n && !C->err; q++) {
        Node* a = then_state->d[q];
        Node* b = jump_state->d[q];
        if (a == b || node_eq(C, b, a)) {
          vpush(C, merged, a);
          continue;
        }
        i64 k = new_temp();
        vpush(C, then_stmts, mk_assign(C, nv1(C, mk_name_syn(C, "__stack_", k, SC_FAST)), a));
        vpush(C, pre, mk_assign(C, nv1(C, mk_name_syn(C, "__stack_", k, SC_FAST)), b));
        vpush(C, merged, mk_name_syn(C, "__stack_", k, SC_FAST));
      }
      vextend(C, out, pre);
      vpush(C, out, mk_if(C, ctf, then_stmts, nullptr));
      return wx(WX_NEXT, target, merged);
    }
  }
  vpush(C, out, mk_if(C, ctf, then_stmts, nullptr));
  return wx(WX_NEXT, target, then_state ? then_state : jump_state);
}

// _collect_chain (structurer.py:619-655)
HD NOINL void Structurer::collect_chain(Node** fall_cond, i64* target, i64* fall_pos, NV** fall_state) {
  while (!C->err) {
    i32 nb = *fall_pos >= 0 && *fall_pos <= 0xFFFFFFFFll ? block_at(G, (u32)*fall_pos) : -1;
    if (nb < 0) break;
    const Block* nxt = &G->blocks[nb];
    if (G->loop_of_header[nb] >= 0 || region_starts_at(nxt->start)) break;
    BlockResult res = simulate(nxt, *fall_state);
    if (C->err) return;
    Node* m2 = res.stmts->n ? vlast(res.stmts) : nullptr;
    if (res.term < 0 || !res.stmts->n || !is_k(m2, S_CONDJUMP) || res.stmts->n != 1 || !(m2->f & 2) ||
        m2->i <= (i64)nxt->start)
      break;
    Node* p2 = (m2->f & 1) ? negate(C, m2->a) : m2->a;
    if (m2->i == *target) {
      *fall_cond = bool_join(C, 0, *fall_cond, p2);
    } else if (*target == (i64)nxt->end) {
      *fall_cond = bool_join(C, 1, negate(C, *fall_cond), p2);
      *target = m2->i;
    } else {
      break;
    }
    *fall_pos = nxt->end;
    *fall_state = res.exit_fall;
  }
}

// _structure_orpop (structurer.py:657-719)
HD NOINL WalkExit Structurer::structure_orpop(const Block* block, Node* marker, BlockResult& res, NV* out,
                                               NV* stack, const WCtx* ctx) {
  u8 op = (marker->f & 1) ? 1 : 0;  // or : and
  i64 join = marker->i;
  NV* ej = res.exit_jump;
  Node* kept = vlast(ej);
  bool chained = op == 0 && is_k(kept, E_COMPARE) && ej->n >= 2 && ej->d[ej->n - 2] == vlast(kept->l2);
  WalkExit rx;
  NV* rhs_stmts = walk(seg1(block->end, join), res.exit_fall, ctx_with_join(ctx, join), &rx);
  CKR(C, wx(WX_ENDED));
  if (chained && !rhs_stmts->n && (rx.kind == WX_JUMP || rx.kind == WX_FALL)) {
    NV* st2 = rx.stack;
    if (st2 && st2->n == res.exit_fall->n && is_k(vlast(st2), E_COMPARE) && vlast(st2)->a == vlast(kept->l2)) {
      Node* rhs = vlast(st2);
      Node* fused = mk(C, E_COMPARE);
      fused->a = kept->a;
      fused->l1 = nv_copy(C, kept->l1);
      vextend(C, fused->l1, rhs->l1);
      fused->l2 = nv_copy(C, kept->l2);
      vextend(C, fused->l2, rhs->l2);
      if (is_chain_fixup(join, false)) {
        NV* merged = vcopy<Node*>(C, st2, 0, st2->n - 1);
        vpush(C, merged, fused);
        return wx(WX_NEXT, rx.target, merged);
      }
    }
  }
  if (chained && rx.kind == WX_ENDED && rhs_stmts->n == 1 && is_k(rhs_stmts->d[0], S_RETURN) &&
      is_k(rhs_stmts->d[0]->a, E_COMPARE) && rhs_stmts->d[0]->a->a == vlast(kept->l2) && is_chain_fixup(join, true)) {
    Node* rhs = rhs_stmts->d[0]->a;
    Node* fused = mk(C, E_COMPARE);
    fused->a = kept->a;
    fused->l1 = nv_copy(C, kept->l1);
    vextend(C, fused->l1, rhs->l1);
    fused->l2 = nv_copy(C, kept->l2);
    vextend(C, fused->l2, rhs->l2);
    vpush(C, out, mk1(C, S_RETURN, fused));
    return wx(WX_ENDED);
  }
  if (rhs_stmts->n || rx.kind == WX_ENDED || !rx.stack || rx.stack->n != ej->n) {
    fail_struct(C, block->id, "unstructured short-circuit value");
    return wx(WX_ENDED);
  }
  Node* rhs = vlast(rx.stack);
  NV* merged = vcopy<Node*>(C, ej, 0, ej->n - 1);
  vpush(C, merged, bool_join(C, op, kept, rhs));
  return wx(WX_NEXT, join, merged);
}

HD inline bool Structurer::is_chain_fixup(i64 off, bool returning) {  // structurer.py:721-735
  i32 b = off >= 0 && off <= 0xFFFFFFFFll ? block_at(G, (u32)off) : -1;
  if (b < 0) return false;
  const Block& B = G->blocks[b];
  i32 n = B.hi - B.lo;
  const Ins* I = K->ins + B.lo;
  if (returning) {
    return n == 3 && (I[0].op == OP_ROT_TWO || I[0].op == OP_SWAP) && I[1].op == OP_POP_TOP &&
           I[2].op == OP_RETURN_VALUE;
  }
  return n == 2 && (I[0].op == OP_ROT_TWO || I[0].op == OP_SWAP) && I[1].op == OP_POP_TOP;
}

// ------------------------------------------------------------ regions
HD NOINL i64 Structurer::structure_region(i32 r, NV* out, NV** stack, const WCtx* ctx) {
  GUARD(C);
  CKR(C, NO_POS);
  vpush(C, active_regions, r);
  TryRegion R = regions->d[r];
  i64 res;
  if (R.kind == RK_WITH) res = structure_with(R, out, stack, ctx);
  else if (R.kind == RK_FINALLY) res = structure_finally(R, out, stack, ctx);
  else res = structure_except(R, out, stack, ctx);
  // remove (first occurrence)
  for (u32 q = 0; q < active_regions->n; q++) {
    if (active_regions->d[q] == r) {
      for (u32 w = q; w + 1 < active_regions->n; w++) active_regions->d[w] = active_regions->d[w + 1];
      active_regions->n--;
      break;
    }
  }
  return C->err ? NO_POS : res;
}

HD inline NV* Structurer::exc_entry_stack(NV* stack) {
  NV* st = nv_copy(C, stack);
  int n = K->minor >= 11 ? 1 : 6;
  for (int q = 0; q < n; q++) {
    Node* ev = mk(C, E_EXCVALUE);
    ev->i = K->minor >= 11 ? 0 : q;
    vpush(C, st, ev);
  }
  return st;
}

HD NOINL i64 Structurer::structure_with(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx) {
  NV* st = *stack;
  Node* ctx_expr = nullptr;
  bool found = false;
  for (i32 q = (i32)st->n - 1; q >= 0; q--) {
    if (is_k(st->d[q], E_WITHEXIT)) {
      ctx_expr = st->d[q]->a;
      found = true;
      break;
    }
  }
  if (!found) {
    i32 b = block_at(G, R.start);
    fail_struct(C, b, "with region without context on stack");
    return NO_POS;
  }
  Node* target = nullptr;
  bool has_target = false;
  if (out->n && is_k(vlast(out), S_ASSIGN) && is_k(vlast(out)->a, E_WITHENTER) && vlast(out)->a->a == ctx_expr) {
    target = vlast(out)->l1->d[0];
    has_target = true;
    out->n--;
  }
  WalkExit bx;
  NV* body = walk(seg1(R.start, R.handler), st, ctx, &bx);
  CKR(C, NO_POS);
  if (!has_target && body->n) {
    Node* first = body->d[0];
    if (is_k(first, S_ASSIGN) && is_k(first->a, E_WITHENTER) && first->a->a == ctx_expr) {
      target = first->l1->d[0];
      body = vcopy<Node*>(C, body, 1);
    }
  }
  NV* ns = vnew<Node*>(C, st->n);
  for (u32 q = 0; q < st->n; q++) {
    Node* e = st->d[q];
    if ((is_k(e, E_WITHEXIT) || is_k(e, E_WITHENTER)) && e->a == ctx_expr) continue;
    vpush(C, ns, e);
  }
  if (K->minor == 8 && bx.kind == WX_FALL) {
    WalkExit x2;
    NV* extra = walk(seg1(R.handler, end_offset), bx.stack, ctx_no_joins(ctx), &x2);
    CKR(C, NO_POS);
    vextend(C, body, extra);
    if (x2.kind == WX_END_FINALLY || x2.kind == WX_JUMP || x2.kind == WX_FALL) bx = wx(WX_JUMP, x2.target, ns);
    else bx = wx(WX_ENDED);
  }
  Node* item = mk2(C, X_WITHITEM, ctx_expr, target);
  Node* w = mk(C, S_WITH);
  w->l1 = nv1(C, item);
  w->l2 = or_pass(C, body);
  vpush(C, out, w);
  *stack = ns;
  if (bx.kind == WX_JUMP) return bx.target;
  if (bx.kind == WX_FALL && bx.target < (i64)R.handler) return bx.target;
  return NO_POS;
}

HD inline i64 Structurer::after_handler_code(const TryRegion& R) {  // structurer.py:813-826
  i32 idx = index_of(C, K, R.handler);
  CKR(C, NO_POS);
  int depth = 0;
  while (idx < K->n_ins) {
    u8 op = K->ins[idx].op;
    if ((op == OP_RERAISE || op == OP_END_FINALLY) && depth == 0) return ins_end(K->ins[idx]);
    if (op == OP_SETUP_FINALLY || op == OP_SETUP_WITH) depth++;
    if (op == OP_POP_BLOCK && depth) depth--;
    idx++;
  }
  return end_offset;
}

HD NOINL i64 Structurer::structure_finally(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx) {
  if (K->minor == 8) return structure_finally_38(R, out, stack, ctx);
  WalkExit fx;
  NV* final = walk(seg1(R.handler, end_offset), exc_entry_stack(vnew<Node*>(C)), ctx_no_joins(ctx), &fx);
  CKR(C, NO_POS);
  const WCtx* bctx = ctx_with_join(ctx, R.handler);
  WalkExit bx;
  NV* body = walk(seg1(R.start, R.end), *stack, bctx, &bx);
  CKR(C, NO_POS);
  WalkExit tx;
  NV* tail;
  if (bx.kind == WX_ENDED) {
    tail = vnew<Node*>(C);
    tx = bx;
  } else {
    i64 tail_from = (i64)R.end > bx.target ? (i64)R.end : bx.target;
    tail = walk(seg1(tail_from, R.handler), bx.stack, bctx, &tx);
    CKR(C, NO_POS);
  }
  vextend(C, body, tail);
  body = strip_finally_copies(C, body, final);
  CKR(C, NO_POS);
  Node* t = mk(C, S_TRY);
  t->l1 = or_pass(C, body);
  t->l2 = vnew<Node*>(C);
  t->l3 = vnew<Node*>(C);
  t->l4 = or_pass(C, final);
  vpush(C, out, t);
  if (tx.kind == WX_JUMP) return tx.target;
  if (tx.kind == WX_FALL && tx.target > (i64)R.handler) return tx.target;
  if (tx.kind == WX_ENDED) return NO_POS;
  return after_handler_code(R);
}

HD NOINL i64 Structurer::structure_finally_38(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx) {
  NV* sent = nv_copy(C, *stack);
  vpush(C, sent, mk(C, E_FINSENT));
  WalkExit fx;
  NV* final = walk(seg1(R.handler, end_offset), sent, ctx_no_joins(ctx), &fx);
  CKR(C, NO_POS);
  const WCtx* bctx = ctx_with_join(ctx, R.handler);
  WalkExit bx;
  NV* body = walk(seg1(R.start, R.end), *stack, bctx, &bx);
  CKR(C, NO_POS);
  if (bx.kind != WX_ENDED) {
    i64 tail_from = (i64)R.end > bx.target ? (i64)R.end : bx.target;
    WalkExit tx;
    NV* tail = walk(seg1(tail_from, R.handler), bx.stack, bctx, &tx);
    CKR(C, NO_POS);
    vextend(C, body, tail);
  }
  Node* t = mk(C, S_TRY);
  t->l1 = or_pass(C, body);
  t->l2 = vnew<Node*>(C);
  t->l3 = vnew<Node*>(C);
  t->l4 = or_pass(C, final);
  vpush(C, out, t);
  if (fx.kind == WX_END_FINALLY) return fx.target;
  i32 idx = index_of(C, K, R.handler);
  CKR(C, NO_POS);
  while (idx < K->n_ins && K->ins[idx].op != OP_END_FINALLY) idx++;
  return idx < K->n_ins ? (i64)ins_end(K->ins[idx]) : (i64)end_offset;
}

HD NOINL i64 Structurer::structure_except(const TryRegion& R, NV* out, NV** stack, const WCtx* ctx) {
  const WCtx* bctx = ctx_with_join(ctx, R.handler);
  WalkExit bx;
  NV* body = walk(seg1(R.start, R.end), *stack, bctx, &bx);
  CKR(C, NO_POS);
  i64 body_join = -1;
  if (bx.kind == WX_JUMP && bx.target >= (i64)R.handler) {
    body_join = bx.target;
  } else if (bx.kind != WX_ENDED) {
    i64 tail_from = (i64)R.end > bx.target ? (i64)R.end : bx.target;
    WalkExit tx;
    NV* tail = walk(seg1(tail_from, R.handler), bx.stack, bctx, &tx);
    CKR(C, NO_POS);
    vextend(C, body, tail);
    if (tx.kind == WX_JUMP) body_join = tx.target;
    else if (tx.kind == WX_FALL && tx.target > (i64)R.handler) body_join = tx.target;
  }
  i64 handler_join;
  NV* handlers = parse_handlers(R, ctx, &handler_join);
  CKR(C, NO_POS);
  NV* orelse = vnew<Node*>(C);
  i64 join = body_join > handler_join ? body_join : handler_join;
  if (body_join != -1 && handler_join != -1 && body_join < handler_join) {
    WalkExit ox;
    orelse = walk(seg1(body_join, handler_join), *stack, ctx_with_join(ctx, handler_join), &ox);
    CKR(C, NO_POS);
    join = handler_join;
  }
  Node* t = mk(C, S_TRY);
  t->l1 = or_pass(C, body);
  t->l2 = handlers;
  t->l3 = orelse;
  t->l4 = vnew<Node*>(C);
  vpush(C, out, t);
  if (join == -1) return NO_POS;
  return join;
}

HD NOINL NV* Structurer::parse_handlers(const TryRegion& R, const WCtx* ctx, i64* join_out) {
  NV* handlers = vnew<Node*>(C);
  i64 best = -1;
  bool any = false;
  i64 h = R.handler;
  bool has_h = true;
  int guard = 0;
  while (has_h && guard < 64 && !C->err) {
    guard++;
    const Block* block = block_at_or_fail(h);
    CKR(C, handlers);
    NV* entry = exc_entry_stack(vnew<Node*>(C));
    BlockResult res = simulate(block, entry);
    CKR(C, handlers);
    Node* marker = (res.stmts->n && is_k(vlast(res.stmts), S_CONDJUMP)) ? vlast(res.stmts) : nullptr;
    Node* type_expr = nullptr;
    i64 next_h = 0;
    bool has_next = false;
    i64 arm_start;
    NV* arm_stack;
    if (marker && is_k(marker->a, E_COMPARE) && marker->a->l1->n == 1 && marker->a->l1->d[0]->op == CO_EXCMATCH) {
      type_expr = marker->a->l2->d[0];
      next_h = marker->i;
      has_next = true;
      arm_start = block->end;
      arm_stack = res.exit_fall;
    } else if (res.term >= 0 && (K->ins[res.term].op == OP_RERAISE || K->ins[res.term].op == OP_END_FINALLY) &&
               !res.stmts->n) {
      break;
    } else {
      arm_start = h;
      arm_stack = entry;
    }
    Str name;
    i64 arm_join;
    NV* arm_body = walk_arm(arm_start, arm_stack, ctx, has_next ? next_h : -1, &name, &arm_join);
    CKR(C, handlers);
    Node* hd = mk(C, X_HANDLER);
    hd->a = type_expr;
    hd->s = name;
    hd->l1 = or_pass(C, arm_body);
    vpush(C, handlers, hd);
    if (arm_join != -1) {
      if (!any || arm_join > best) best = arm_join;
      any = true;
    }
    h = next_h;
    has_h = has_next;
    if (!type_expr) break;
  }
  *join_out = any ? best : -1;
  return handlers;
}

HD NOINL NV* Structurer::walk_arm(i64 arm_start, NV* arm_stack, const WCtx* ctx, i64 limit, Str* name,
                                   i64* join) {
  i64 end = limit >= 0 ? limit : (i64)end_offset;
  WalkExit ex;
  NV* body = walk(seg1(arm_start, end), arm_stack, ctx_no_joins(ctx), &ex);
  *name = Snone();
  *join = -1;
  CKR(C, body);
  if (body->n && is_k(body->d[0], S_ASSIGN) && is_k(body->d[0]->a, E_EXCVALUE)) {
    Node* tgt = body->d[0]->l1->d[0];
    if (is_k(tgt, E_NAME)) {
      *name = tgt->s;
      body = vcopy<Node*>(C, body, 1);
    }
  }
  body = strip_as_cleanup(C, body, *name);
  CKR(C, body);
  if (ex.kind == WX_JUMP) *join = ex.target;
  else if (ex.kind == WX_FALL && ex.target > end) *join = ex.target;
  return body;
}

HD NOINL Structurer* make_structurer(Dc* C, Code* K, Cfg* G) {
  Structurer* S_ = anew<Structurer>(C);
  CKR(C, S_);
  S_->C = C;
  S_->K = K;
  S_->G = G;
  S_->sim.C = C;
  S_->sim.K = K;
  S_->regions = match_try_regions(C, K, G->entries);
  CKR(C, S_);
  // regions_by_start: kinds except/finally/with; per start sorted by -end (stable)
  S_->rbs_idx = vnew<i32>(C, S_->regions->n);
  for (u32 r = 0; r < S_->regions->n; r++)
    if (S_->regions->d[r].kind != RK_AS_CLEANUP) vpush(C, S_->rbs_idx, (i32)r);
  // stable insertion sort by (start, -end): lookups filter by start, so only the
  // order inside one start group matters and it must be the stable -end order
  Vec<i32>* v = S_->rbs_idx;
  for (u32 i = 1; i < v->n; i++) {
    i32 x = v->d[i];
    u32 j = i;
    while (j > 0) {
      const TryRegion& a = S_->regions->d[v->d[j - 1]];
      const TryRegion& b = S_->regions->d[x];
      if (a.start > b.start || (a.start == b.start && a.end < b.end)) {
        v->d[j] = v->d[j - 1];
        j--;
      } else {
        break;
      }
    }
    v->d[j] = x;
  }
  S_->temp_counter = 0;
  S_->active_regions = vnew<i32>(C, 4);
  S_->active_loops = (u8*)zalloc(C, (u64)G->n_blocks);
  S_->end_offset = ins_end(K->ins[K->n_ins - 1]);
  return S_;
}
