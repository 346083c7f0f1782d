// cfg.h -- control-flow facts per code object (cfg.py:61-328, pipeline.py:17-87,
// disasm.py:175-214, structurer.py:62-173).
//
// Blocks are built in O(N) from the sorted leader set (the reference rescans all
// instructions per block, cfg.py:94); block ids follow ascending leader offsets
// exactly as the reference's.  Dominators / loops use the reference's
// DFS orders (successor order preserved) so every derived fact matches.
#pragma once
#include "symexec.h"

struct ExcEntry {
  u32 start, end, target, depth;
  bool lasti;
};
struct TryRegion {  // structurer.py:34-40
  u32 start, end, handler;
  u8 kind;          // 0 except, 1 finally, 2 with, 3 as_cleanup
  i64 setup_offset;
};
enum { RK_EXCEPT = 0, RK_FINALLY = 1, RK_WITH = 2, RK_AS_CLEANUP = 3 };

struct Loop {
  i32 header;
  Vec<i32>* body;       // sorted block ids
  Vec<i32>* back_tails; // back edge sources in discovery order
};

struct Cfg {
  Block* blocks;        // indexed by id (dead blocks have alive=false)
  i32 n_blocks;
  i32 entry;
  u32 end_of_code;
  Vec<ExcEntry>* entries;
  Vec<Loop>* loops;     // keyed by header (unique)
  i32* loop_of_header;  // [n_blocks] index into loops or -1
};

// block_at: start offset -> block id (alive only); binary search over sorted starts
HD inline i32 block_at(const Cfg* G, u32 off) {
  i32 lo = 0, hi = G->n_blocks;
  while (lo < hi) {
    i32 mid = (lo + hi) >> 1;
    if (G->blocks[mid].start < off) lo = mid + 1;
    else hi = mid;
  }
  // several leaders cannot share an offset (leaders is a set), so this is unique
  if (lo < G->n_blocks && G->blocks[lo].start == off && G->blocks[lo].alive) return lo;
  return -1;
}

HD inline i32 ins_index_of(const Code* K, u32 off) {  // first instr with offset >= off
  i32 lo = 0, hi = K->n_ins;
  while (lo < hi) {
    i32 mid = (lo + hi) >> 1;
    if (K->ins[mid].offset < off) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// _index_of (structurer.py:163-173)
HD inline i32 index_of(Dc* C, const Code* K, u32 off) {
  i32 lo = ins_index_of(K, off);
  if (lo == K->n_ins || K->ins[lo].offset != off) {
    fail_struct(C, off, "offset is not an instruction boundary");
    return -1;
  }
  return lo;
}

// ------------------------------------------------------------ instructions
// Materialize the object's instruction list from the decode kernel's records
// and surface the decode status (decode_instructions, disasm.py:71-172).
HD NOINL bool load_instructions(Dc* C, Code* K, u32 oi) {
  K->oi = oi;
  K->o = obj_at(C, oi);
  K->minor = (int)K->o->minor;
  K->has_kwnames = false;
  K->kwnames = nullptr;
  const upy_decoded& d = C->dec_all[oi];
  if (d.status != UPY_ST_OK) {
    // message formatting of the decode errors (errors.py:45-66)
    Text t;
    if (fail_begin(C, d.status, d.aux0, d.aux1, &t)) {
      switch (d.status) {
        case UPY_ST_UNKNOWN_OPCODE:
          m_puts(C, &t, "unknown opcode "); m_i64(C, &t, d.aux0);
          m_puts(C, &t, " at offset "); m_i64(C, &t, d.aux1);
          break;
        case UPY_ST_BAD_JUMP_TARGET:
          m_puts(C, &t, "jump at offset "); m_i64(C, &t, d.aux0);
          m_puts(C, &t, " targets "); m_i64(C, &t, d.aux1);
          m_puts(C, &t, ", not an instruction boundary");
          break;
        case UPY_ST_TRUNCATED_CODE:
          // aux0: 1 empty, 2 odd, 3 inside EXTENDED_ARG run at aux1, 4 inside cache of opcode at aux1, 5 none
          if (d.aux0 == 1) m_puts(C, &t, "empty code object");
          else if (d.aux0 == 2) m_puts(C, &t, "odd code length");
          else if (d.aux0 == 3) { m_puts(C, &t, "code ends inside EXTENDED_ARG run at "); m_i64(C, &t, d.aux1); }
          else if (d.aux0 == 4) {
            const upy_obj* o = K->o;
            u32 opb = C->bytes[o->code_off + (d.aux1 - 2)];
            m_puts(C, &t, "code ends inside inline cache of ");
            m_puts(C, &t, opname_of(UPY_ENT_OP(optab(K->minor, opb))));
            m_puts(C, &t, " at "); m_i64(C, &t, d.aux1);
          } else m_puts(C, &t, "code holds no instruction");
          C->aux0 = C->aux1 = 0;
          break;
        default:
          m_puts(C, &t, "decode failed");
      }
      fail_end(C, &t);
    }
    return false;
  }
  i32 n = d.n_instrs;
  K->n_ins = n;
  K->ins = (Ins*)ualloc(C, (u64)n * sizeof(Ins));  // every field is written below
  CKR(C, false);
  const upy_ins* src = C->ins_all + (K->o->code_off >> 1);
  Ins* const dst = K->ins;      // loop invariants in registers (the stores below
  const int minor = K->minor;   // could alias *K as far as the compiler knows)
  for (i32 i = 0; i < n; i++) {
    const upy_ins& r = src[i];
    u32 e = optab_div(minor, r.opcode);
    Ins& x = dst[i];
    x.offset = r.offset;
    x.arg = r.arg;
    x.op = UPY_ENT_OP(e);
    x.kind = (u8)UPY_ENT_KIND(e);
    x.nprefix = r.n_prefixes;
    x.flags = r.flags & 3;
    x.cache = r.cache_units;
  }
  return true;
}

// rewrite_yield_from (pipeline.py:57-87)
HD NOINL void rewrite_yield_from(Dc* C, Code* K) {
  bool any = false;
  for (i32 i = 0; i < K->n_ins; i++)
    if (K->ins[i].op == OP_SEND) any = true;
  if (!any) return;
  Ins* out = (Ins*)zalloc(C, (u64)K->n_ins * sizeof(Ins));
  CK(C);
  i32 n = 0, i = 0;
  while (i < K->n_ins) {
    const Ins& in = K->ins[i];
    if (in.op == OP_SEND) {
      u8 w0 = i + 1 < K->n_ins ? K->ins[i + 1].op : 0;
      u8 w1 = i + 2 < K->n_ins ? K->ins[i + 2].op : 0;
      u8 w2 = i + 3 < K->n_ins ? K->ins[i + 3].op : 0;
      int skip = 0;
      if (w0 == OP_YIELD_VALUE && w1 == OP_JUMP_BACKWARD_NO_INTERRUPT) skip = 3;
      else if (w0 == OP_YIELD_VALUE && w1 == OP_RESUME && w2 == OP_JUMP_BACKWARD_NO_INTERRUPT) skip = 4;
      if (skip && jump_target(K, K->ins[i + skip - 1]) == in.offset) {
        const Ins& last = K->ins[i + skip - 1];
        Ins y;
        y.offset = in.offset;
        y.arg = 0;
        y.op = OP_YIELD_FROM_311;
        y.kind = K_NONE;
        y.nprefix = 0;
        y.flags = 0;
        y.cache = (ins_end(last) - in.offset) / 2 - 1;
        out[n++] = y;
        i += skip;
        continue;
      }
    }
    out[n++] = in;
    i++;
  }
  K->ins = out;
  K->n_ins = n;
}

// decode_exception_table (disasm.py:175-214)
HD NOINL Vec<ExcEntry>* decode_exception_table(Dc* C, const Code* K) {
  Vec<ExcEntry>* v = vnew<ExcEntry>(C);
  const u8* data = C->bytes + K->o->exc_off;
  u32 len = K->o->exc_len, pos = 0;
  auto bad = [&](const char* what, u32 at) {
    Text t;
    if (fail_begin(C, UPY_ST_MALFORMED_EXCTABLE, 0, 0, &t)) {
      m_puts(C, &t, what);
      m_puts(C, &t, " at byte ");
      m_i64(C, &t, at);
      fail_end(C, &t);
    }
  };
  auto varint = [&](bool first) -> u64 {
    if (pos >= len) { bad("truncated varint", pos); return 0; }
    u8 b = data[pos];
    if (first && !(b & 0x80)) { bad("missing entry marker", pos); return 0; }
    pos++;
    u64 val = b & 0x3F;
    while (b & 0x40) {
      if (pos >= len) { bad("truncated varint", pos); return 0; }
      b = data[pos];
      if (b & 0x80) { bad("entry marker inside varint", pos); return 0; }
      pos++;
      val = (val << 6) | (b & 0x3F);
    }
    return val;
  };
  while (pos < len) {
    u64 start = varint(true) * 2;
    CKR(C, v);
    u64 length = varint(false) * 2;
    CKR(C, v);
    u64 target = varint(false) * 2;
    CKR(C, v);
    u64 dl = varint(false);
    CKR(C, v);
    ExcEntry e;
    e.start = (u32)start;
    e.end = (u32)(start + length);
    e.target = (u32)target;
    e.depth = (u32)(dl >> 1);
    e.lasti = dl & 1;
    if (length == 0) {
      Text t;
      if (fail_begin(C, UPY_ST_MALFORMED_EXCTABLE, 0, 0, &t)) {
        m_puts(C, &t, "empty range in entry at byte ");
        m_i64(C, &t, pos);
        fail_end(C, &t);
      }
      return v;
    }
    vpush(C, v, e);
  }
  return v;
}

// ------------------------------------------------------------ try regions
HD inline u8 classify_handler(Dc* C, const Code* K, u32 handler) {  // structurer.py:91-103
  i32 idx = index_of(C, K, handler);
  CKR(C, RK_FINALLY);
  const Ins* I = K->ins;
  if (I[idx].op == OP_DUP_TOP) return RK_EXCEPT;
  if (I[idx].op == OP_POP_TOP && idx + 2 < K->n_ins && I[idx + 1].op == OP_POP_TOP && I[idx + 2].op == OP_POP_TOP)
    return RK_EXCEPT;
  return RK_FINALLY;
}
HD inline bool is_as_cleanup(const Code* K, i32 idx) {  // structurer.py:154-160
  if (idx + 3 > K->n_ins) return false;
  const Ins* I = K->ins + idx;
  return (I[0].op == OP_LOAD_CONST && I[1].op == OP_STORE_FAST && I[2].op == OP_DELETE_FAST) ||
         (I[0].op == OP_LOAD_CONST && I[1].op == OP_STORE_NAME && I[2].op == OP_DELETE_NAME);
}
HD NOINL Vec<TryRegion>* match_try_regions(Dc* C, const Code* K, const Vec<ExcEntry>* exc) {
  Vec<TryRegion>* out = vnew<TryRegion>(C);
  const Ins* I = K->ins;
  const i32 n_ins = K->n_ins;
  if (K->minor <= 10) {  // _regions_legacy (structurer.py:69-88)
    for (i32 i = 0; i < n_ins; i++) {
      if (I[i].op != OP_SETUP_FINALLY && I[i].op != OP_SETUP_WITH) continue;
      TryRegion r;
      r.start = ins_end(I[i]);
      r.end = jump_target(K, I[i]);
      r.handler = r.end;
      r.kind = I[i].op == OP_SETUP_WITH ? RK_WITH : classify_handler(C, K, r.handler);
      CKR(C, out);
      r.setup_offset = I[i].offset;
      vpush(C, out, r);
    }
    return out;
  }
  // _regions_311 (structurer.py:106-151)
  for (u32 e = 0; exc && e < exc->n; e++) {
    const ExcEntry& en = exc->d[e];
    i32 ti = ins_index_of(K, en.target);
    if (ti >= K->n_ins || I[ti].offset != en.target || I[ti].op != OP_PUSH_EXC_INFO) continue;
    i32 idx = ti;
    u8 kind = RK_FINALLY;
    i32 j = idx + 1;
    if (j < K->n_ins && I[j].op == OP_WITH_EXCEPT_START) {
      kind = RK_WITH;
    } else {
      i32 k = j;
      while (k < K->n_ins && k < j + 24) {
        u8 op = I[k].op;
        if (op == OP_CHECK_EXC_MATCH) { kind = RK_EXCEPT; break; }
        if (op == OP_POP_TOP && k == j) { kind = RK_EXCEPT; break; }
        if (op == OP_LOAD_GLOBAL || op == OP_LOAD_NAME || op == OP_LOAD_FAST || op == OP_LOAD_CONST ||
            op == OP_LOAD_ATTR || op == OP_BUILD_TUPLE || op == OP_EXTENDED_ARG) {
          k++;
          continue;
        }
        break;
      }
      if (kind != RK_EXCEPT && is_as_cleanup(K, idx + 1)) kind = RK_AS_CLEANUP;
    }
    // merge fragments protecting the same handler (dict keyed by handler, insertion order)
    bool merged = false;
    for (u32 q = 0; q < out->n; q++) {
      if (out->d[q].handler == en.target) {
        if (en.start < out->d[q].start) out->d[q].start = en.start;
        if (en.end > out->d[q].end) out->d[q].end = en.end;
        merged = true;
        break;
      }
    }
    if (!merged) {
      TryRegion r;
      r.start = en.start;
      r.end = en.end;
      r.handler = en.target;
      r.kind = kind;
      r.setup_offset = -1;
      vpush(C, out, r);
    }
  }
  return out;
}

// ------------------------------------------------------------ basic blocks
HD inline void link(Dc* C, Cfg* G, i32 src, u32 dst_off, u8 kind) {
  i32 dst = block_at(G, dst_off);
  if (dst < 0) {
    py_key_error(C, dst_off);  // cfg.py:100 block_at[dst_offset]
    return;
  }
  vpush(C, G->blocks[src].succ, dst);
  vpush(C, G->blocks[src].succ_kind, kind);
  vpush(C, G->blocks[dst].pred, src);
}

HD inline bool is_cond_for_cfg(u8 op) {  // cfg.py:122-127
  switch (op) {
    case OP_POP_JUMP_IF_FALSE: case OP_POP_JUMP_IF_TRUE: case OP_POP_JUMP_FORWARD_IF_FALSE:
    case OP_POP_JUMP_FORWARD_IF_TRUE: case OP_POP_JUMP_BACKWARD_IF_FALSE: case OP_POP_JUMP_BACKWARD_IF_TRUE:
    case OP_POP_JUMP_FORWARD_IF_NONE: case OP_POP_JUMP_FORWARD_IF_NOT_NONE:
    case OP_POP_JUMP_BACKWARD_IF_NONE: case OP_POP_JUMP_BACKWARD_IF_NOT_NONE:
    case OP_JUMP_IF_FALSE_OR_POP: case OP_JUMP_IF_TRUE_OR_POP: case OP_JUMP_IF_NOT_EXC_MATCH:
    case OP_CALL_FINALLY:
      return true;
  }
  return false;
}
HD inline bool is_setup_op(u8 op) {
  return op == OP_SETUP_FINALLY || op == OP_SETUP_WITH || op == OP_SETUP_ASYNC_WITH;
}

HD inline void sort_u32(u32* a, i32 n) {  // heap sort (no recursion, no std)
  auto sift = [&](i32 i, i32 m) {
    while (true) {
      i32 l = 2 * i + 1, r = l + 1, g = i;
      if (l < m && a[l] > a[g]) g = l;
      if (r < m && a[r] > a[g]) g = r;
      if (g == i) return;
      u32 t = a[i]; a[i] = a[g]; a[g] = t;
      i = g;
    }
  };
  for (i32 i = n / 2 - 1; i >= 0; i--) sift(i, n);
  for (i32 m = n - 1; m > 0; m--) {
    u32 t = a[0]; a[0] = a[m]; a[m] = t;
    sift(0, m);
  }
}

// build_basic_blocks (cfg.py:72-141)
HD NOINL Cfg* build_basic_blocks(Dc* C, const Code* K, const Vec<ExcEntry>* entries) {
  Cfg* G = anew<Cfg>(C);
  CKR(C, G);
  const Ins* I = K->ins;
  i32 n = K->n_ins;
  u32 end_of_code = ins_end(I[n - 1]);
  G->end_of_code = end_of_code;
  // leaders on the scratch stack (released when analyze() returns)
  u32 ne = entries ? entries->n : 0;
  u32* Ld = sarr<u32>(C, 1 + 2 * (u64)n + 3 * (u64)ne, false);
  CKR(C, G);
  u32 nl = 0;
  Ld[nl++] = I[0].offset;
  for (i32 i = 0; i < n; i++)
    if (ins_is_jump(I[i])) Ld[nl++] = jump_target(K, I[i]);
  for (i32 i = 0; i < n; i++) {
    u8 op = I[i].op;
    bool ender = op == OP_RETURN_VALUE || op == OP_RAISE_VARARGS || op == OP_RERAISE || op == OP_END_FINALLY ||
                 (ins_is_jump(I[i]) && !is_setup_op(op));
    if (ender && ins_end(I[i]) < end_of_code) Ld[nl++] = ins_end(I[i]);
  }
  for (u32 e = 0; e < ne; e++) {
    Ld[nl++] = entries->d[e].target;
    Ld[nl++] = entries->d[e].start;
    if (entries->d[e].end < end_of_code) Ld[nl++] = entries->d[e].end;
  }
  sort_u32(Ld, (i32)nl);
  u32 nu = 0;
  for (u32 i = 0; i < nl; i++)
    if (nu == 0 || Ld[nu - 1] != Ld[i]) Ld[nu++] = Ld[i];
  G->n_blocks = (i32)nu;
  G->blocks = (Block*)zalloc(C, (u64)nu * sizeof(Block));
  CKR(C, G);
  i32 cursor = 0;
  for (u32 b = 0; b < nu; b++) {
    Block& B = G->blocks[b];
    B.id = (i32)b;
    B.start = Ld[b];
    B.end = b + 1 < nu ? Ld[b + 1] : end_of_code;
    while (cursor < n && I[cursor].offset < B.start) cursor++;
    i32 lo = ins_index_of(K, B.start);
    i32 hi = lo;
    while (hi < n && I[hi].offset < B.end) hi++;
    if (B.end <= B.start) hi = lo;
    B.lo = lo;
    B.hi = hi;
    B.succ = vnew<i32>(C, 2);
    B.succ_kind = vnew<u8>(C, 2);
    B.pred = vnew<i32>(C, 2);
    B.alive = true;
  }
  G->entry = block_at(G, I[0].offset);
  for (u32 b = 0; b < nu; b++) {
    CKR(C, G);
    Block& B = G->blocks[b];
    if (B.hi <= B.lo) continue;
    const Ins& last = I[B.hi - 1];
    u8 op = last.op;
    bool falls = true;
    if (op == OP_RETURN_VALUE || op == OP_RAISE_VARARGS || op == OP_RERAISE) {
      falls = false;
    } else if (op == OP_FOR_ITER) {
      link(C, G, (i32)b, jump_target(K, last), EK_TAKEN);
      link(C, G, (i32)b, ins_end(last), EK_NOT_TAKEN);
      falls = false;
    } else if (ins_is_jump(last) && !is_setup_op(op)) {
      link(C, G, (i32)b, jump_target(K, last), EK_TAKEN);
      if (is_cond_for_cfg(op)) link(C, G, (i32)b, ins_end(last), EK_NOT_TAKEN);
      falls = false;
    }
    if (falls && B.end < end_of_code) link(C, G, (i32)b, B.end, EK_FALL);
  }
  for (u32 e = 0; entries && e < entries->n; e++) {
    CKR(C, G);
    const ExcEntry& en = entries->d[e];
    i32 target = block_at(G, en.target);
    // blocks overlapping [start, end): block ends are the next block's start, so
    // they form one contiguous id range starting at the block holding en.start
    u32 first = 0, hi_ = nu;
    while (first < hi_) {
      u32 mid = (first + hi_) >> 1;
      if (G->blocks[mid].start < en.start) first = mid + 1;
      else hi_ = mid;
    }
    if (first > 0) first--;
    for (u32 b = first; b < nu && G->blocks[b].start < en.end; b++) {
      Block& B = G->blocks[b];
      if (B.start < en.end && B.end > en.start) {
        bool has = false;
        for (u32 q = 0; q < B.succ->n && !has; q++)
          has = B.succ->d[q] == target && B.succ_kind->d[q] == EK_EXC;
        if (!has && (i32)b != target) {
          vpush(C, B.succ, target);
          vpush(C, B.succ_kind, (u8)EK_EXC);
          vpush(C, G->blocks[target].pred, (i32)b);
        }
      }
    }
  }
  G->entries = (Vec<ExcEntry>*)entries;
  return G;
}

HD inline u32 total_edges(const Cfg* G) {
  u32 e = 0;
  for (i32 b = 0; b < G->n_blocks; b++) e += G->blocks[b].succ->n;
  return e;
}

// reachable_from (cfg.py:144-157) into a scratch bitmap
HD inline u8* reachable_from(Dc* C, const Cfg* G, i32 root, bool include_exc) {
  u8* seen = sarr<u8>(C, (u64)G->n_blocks);
  i32* work = sarr<i32>(C, (u64)total_edges(G) + 1, false);
  CKR(C, seen);
  u32 sp = 0;
  work[sp++] = root;
  while (sp) {
    i32 b = work[--sp];
    if (seen[b]) continue;
    seen[b] = 1;
    const Block& B = G->blocks[b];
    for (u32 q = 0; q < B.succ->n; q++) {
      if (B.succ_kind->d[q] == EK_EXC && !include_exc) continue;
      if (!seen[B.succ->d[q]]) work[sp++] = B.succ->d[q];
    }
  }
  return seen;
}

// prune_unreachable (cfg.py:316-328)
HD inline void prune_unreachable(Dc* C, Cfg* G) {
  u8* keep = reachable_from(C, G, G->entry, true);
  CK(C);
  for (i32 b = 0; b < G->n_blocks; b++) {
    Block& B = G->blocks[b];
    if (!keep[b]) {
      B.alive = false;
      continue;
    }
    u32 w = 0;
    for (u32 q = 0; q < B.succ->n; q++)
      if (keep[B.succ->d[q]]) {
        B.succ->d[w] = B.succ->d[q];
        B.succ_kind->d[w] = B.succ_kind->d[q];
        w++;
      }
    B.succ->n = w;
    B.succ_kind->n = w;
    w = 0;
    for (u32 q = 0; q < B.pred->n; q++)
      if (keep[B.pred->d[q]]) B.pred->d[w++] = B.pred->d[q];
    B.pred->n = w;
  }
}

HD inline bool has_normal_edge(const Block& P, i32 to) {
  for (u32 q = 0; q < P.succ->n; q++)
    if (P.succ->d[q] == to && P.succ_kind->d[q] != EK_EXC) return true;
  return false;
}

// Scratch shared by the dominator / loop passes of one analyze() call.  Block sets
// are (stamp array, epoch) pairs plus a member list, so each per-handler
// sub-analysis (pipeline.py:37-53) costs O(its own blocks + edges) instead of
// O(all blocks) -- C4-shape objects run ~100 of them over ~2K blocks.
struct BSet {
  const i32* st;
  i32 ep;
  const i32* ls;
  i32 n;
  HD bool has(i32 b) const { return st[b] == ep; }
};

struct AnaWs {
  i32 nb;
  u32 E;
  i32 ep;
  i32* uni_st;   // universe membership
  i32* seen_st;  // dominator DFS seen == set(idom)
  i32* vis_st;   // loop DFS visited
  i32* body_st;  // natural-loop body
  u8* onstack;   // all-zero between DFS runs
  i32* idom;
  i32* rpo_index;
  i32* uni_ls;
  i32* order;
  i32* stk_b;
  u32* stk_q;
  i32* ru;
  i32* rv;
  i32* work;
  i32* hdrs;
  Vec<i32>** tails;
  i32* blist;
};

HD inline bool ana_ws_init(Dc* C, AnaWs* W, const Cfg* G) {
  i32 nb = G->n_blocks;
  W->nb = nb;
  W->E = total_edges(G) + 1;
  W->ep = 0;
  W->uni_st = sarr<i32>(C, (u64)nb);
  W->seen_st = sarr<i32>(C, (u64)nb);
  W->vis_st = sarr<i32>(C, (u64)nb);
  W->body_st = sarr<i32>(C, (u64)nb);
  W->onstack = sarr<u8>(C, (u64)nb);
  W->idom = sarr<i32>(C, (u64)nb, false);
  W->rpo_index = sarr<i32>(C, (u64)nb, false);
  W->uni_ls = sarr<i32>(C, (u64)nb, false);
  W->order = sarr<i32>(C, (u64)nb, false);
  W->stk_b = sarr<i32>(C, (u64)nb, false);
  W->stk_q = sarr<u32>(C, (u64)nb, false);
  W->ru = sarr<i32>(C, W->E, false);
  W->rv = sarr<i32>(C, W->E, false);
  W->work = sarr<i32>(C, (u64)W->E + nb, false);
  W->hdrs = sarr<i32>(C, (u64)nb + 1, false);
  W->tails = sarr<Vec<i32>*>(C, (u64)nb + 1, false);
  W->blist = sarr<i32>(C, (u64)nb + 1, false);
  CKR(C, false);
  for (i32 b = 0; b < nb; b++) W->idom[b] = -1;
  return true;
}

// reachable_from(root, include_exc=False) (cfg.py:144-157) into W's universe, not
// entering blocks in `stop` (analyze() passes the covered set, which is closed
// under normal successors, so stopping there removes exactly the covered blocks
// the reference filters out afterwards)
HD inline BSet collect_reach(AnaWs* W, const Cfg* G, i32 root, const u8* stop) {
  i32 ep = ++W->ep;
  i32 n = 0;
  u32 sp = 0;
  W->work[sp++] = root;
  while (sp) {
    i32 b = W->work[--sp];
    if (W->uni_st[b] == ep) continue;
    W->uni_st[b] = ep;
    W->uni_ls[n++] = b;
    const Block& B = G->blocks[b];
    for (u32 q = 0; q < B.succ->n; q++) {
      i32 s = B.succ->d[q];
      if (B.succ_kind->d[q] == EK_EXC || W->uni_st[s] == ep || (stop && stop[s])) continue;
      W->work[sp++] = s;
    }
  }
  return BSet{W->uni_st, ep, W->uni_ls, n};
}

// compute_dominators (cfg.py:160-220) over universe U; W->idom[b] = -1 when b has
// no entry.  Returns set(idom) (the blocks the DFS reached, in postorder).
HD NOINL BSet compute_dominators(Dc* C, AnaWs* W, const Cfg* G, i32 root, BSet U) {
  i32* idom = W->idom;
  i32* rpo_index = W->rpo_index;
  i32* order = W->order;
  for (i32 i = 0; i < U.n; i++) idom[U.ls[i]] = -1;
  i32 ep = ++W->ep;
  // iterative DFS mirroring the recursive one (postorder)
  i32 no = 0, sp = 0;
  W->seen_st[root] = ep;
  W->stk_b[sp] = root;
  W->stk_q[sp] = 0;
  sp++;
  while (sp) {
    i32 b = W->stk_b[sp - 1];
    const Block& B = G->blocks[b];
    u32& q = W->stk_q[sp - 1];
    bool pushed = false;
    while (q < B.succ->n) {
      i32 s = B.succ->d[q];
      u8 k = B.succ_kind->d[q];
      q++;
      if (k != EK_EXC && U.has(s) && W->seen_st[s] != ep) {
        W->seen_st[s] = ep;
        W->stk_b[sp] = s;
        W->stk_q[sp] = 0;
        sp++;
        pushed = true;
        break;
      }
    }
    if (!pushed) {
      order[no++] = b;
      sp--;
    }
  }
  // rpo = reversed(order)
  for (i32 i = 0; i < no; i++) rpo_index[order[no - 1 - i]] = i;
  idom[root] = root;
  bool changed = true;
  while (changed && !C->err) {
    changed = false;
    for (i32 r = 0; r < no; r++) {
      i32 b = order[no - 1 - r];
      if (b == root) continue;
      const Block& B = G->blocks[b];
      i32 nw = -1;
      for (u32 q = 0; q < B.pred->n; q++) {
        i32 p = B.pred->d[q];
        if (!U.has(p) || idom[p] < 0 || !has_normal_edge(G->blocks[p], b)) continue;
        if (nw < 0) {
          nw = p;
          continue;
        }
        i32 a = nw, c = p;
        while (a != c) {
          while (rpo_index[a] > rpo_index[c]) a = idom[a];
          while (rpo_index[c] > rpo_index[a]) c = idom[c];
        }
        nw = a;
      }
      if (nw < 0) continue;
      if (idom[b] != nw) {
        idom[b] = nw;
        changed = true;
      }
    }
  }
  return BSet{W->seen_st, ep, order, no};
}

HD inline bool dominates(const i32* idom, i32 a, i32 b) {  // cfg.py:223-231
  while (true) {
    if (a == b) return true;
    i32 parent = idom[b];
    if (parent < 0 || parent == b) return a == b;
    b = parent;
  }
}

// analyze_loops (cfg.py:241-313) over universe U with dominator tree W->idom;
// appends loops whose header is new to G->loops (persistent).  Returns false when
// irreducible.
HD NOINL bool analyze_loops(Dc* C, AnaWs* W, Cfg* G, BSet U) {
  const i32* idom = W->idom;
  // roots: universe blocks with no predecessor in the universe (any edge kind)
  i32 root = -1;
  i32 first_root = -1, min_u = -1;
  for (i32 i = 0; i < U.n; i++) {
    i32 b = U.ls[i];
    if (min_u < 0 || b < min_u) min_u = b;
    bool has = false;
    const Block& B = G->blocks[b];
    for (u32 q = 0; q < B.pred->n && !has; q++) has = U.has(B.pred->d[q]);
    if (!has && (first_root < 0 || b < first_root)) first_root = b;
  }
  // roots has at most one element (every other universe block was reached from
  // the dominator root through a predecessor in the universe), so its order is moot
  if (first_root >= 0) root = first_root;
  else root = U.has(G->entry) ? G->entry : min_u;
  if (root < 0) return true;
  i32 vep = ++W->ep;
  i32* stk_b = W->stk_b;
  u32* stk_q = W->stk_q;
  u32 nr = 0;
  i32 sp = 0;
  W->vis_st[root] = vep;
  W->onstack[root] = 1;
  stk_b[0] = root;
  stk_q[0] = 0;
  sp = 1;
  while (sp && !C->err) {
    i32 u = stk_b[sp - 1];
    const Block& B = G->blocks[u];
    u32& q = stk_q[sp - 1];
    bool pushed = false;
    while (q < B.succ->n) {
      i32 v = B.succ->d[q];
      u8 k = B.succ_kind->d[q];
      q++;
      if (k == EK_EXC || !U.has(v)) continue;
      if (W->vis_st[v] != vep) {
        W->vis_st[v] = vep;
        W->onstack[v] = 1;
        stk_b[sp] = v;
        stk_q[sp] = 0;
        sp++;
        pushed = true;
        break;
      } else if (W->onstack[v]) {
        W->ru[nr] = u;
        W->rv[nr] = v;
        nr++;
      }
    }
    if (!pushed) {
      W->onstack[u] = 0;
      sp--;
    }
  }
  bool reducible = true;
  // back edges grouped by header in first-seen order; tails are persistent
  u32 nh = 0;
  for (u32 e = 0; e < nr; e++) {
    i32 u = W->ru[e], v = W->rv[e];
    if (dominates(idom, v, u)) {
      u32 h = 0;
      while (h < nh && W->hdrs[h] != v) h++;
      if (h == nh) {
        W->hdrs[nh] = v;
        W->tails[nh] = vnew<i32>(C, 2);
        nh++;
      }
      CKR(C, true);
      vpush(C, W->tails[h], u);
    } else {
      reducible = false;
    }
  }
  CKR(C, reducible);
  for (u32 h = 0; h < nh && !C->err; h++) {
    i32 header = W->hdrs[h];
    if (G->loop_of_header[header] >= 0) continue;  // only new headers are added
    i32 bep = ++W->ep;
    u32 wn = 0, cnt = 0;
    W->body_st[header] = bep;
    W->blist[cnt++] = header;
    for (u32 t = 0; t < W->tails[h]->n; t++) W->work[wn++] = W->tails[h]->d[t];
    while (wn) {
      i32 nn = W->work[--wn];
      if (W->body_st[nn] == bep) continue;
      W->body_st[nn] = bep;
      W->blist[cnt++] = nn;
      const Block& N = G->blocks[nn];
      for (u32 q = 0; q < N.pred->n; q++) {
        i32 p = N.pred->d[q];
        if (U.has(p) && has_normal_edge(G->blocks[p], nn)) W->work[wn++] = p;
      }
    }
    sort_u32((u32*)W->blist, (i32)cnt);  // body in block-id order, as the reference's
    Loop L;
    L.header = header;
    L.body = vnew<i32>(C, cnt);
    CKR(C, reducible);
    for (u32 i = 0; i < cnt; i++) vpush(C, L.body, W->blist[i]);
    L.back_tails = W->tails[h];
    G->loop_of_header[header] = (i32)G->loops->n;
    vpush(C, G->loops, L);
  }
  return reducible;
}

// analyze (pipeline.py:17-54).  All analysis temporaries live on the scratch
// stack and are released before returning (the Cfg, loops and entries persist).
HD NOINL Cfg* analyze(Dc* C, Code* K) {
  u64 mark = C->top;
  Cfg* G = nullptr;
  do {
    Vec<ExcEntry>* entries = vnew<ExcEntry>(C);
    if (K->minor >= 11) {
      rewrite_yield_from(C, K);
      if (C->err) break;
      Vec<ExcEntry>* raw = decode_exception_table(C, K);
      if (C->err) break;
      for (u32 e = 0; e < raw->n; e++) {
        i32 ti = ins_index_of(K, raw->d[e].target);
        if (ti < K->n_ins && K->ins[ti].offset == raw->d[e].target) vpush(C, entries, raw->d[e]);
      }
    } else {
      Vec<TryRegion>* rs = match_try_regions(C, K, nullptr);
      if (C->err) break;
      for (u32 r = 0; r < rs->n; r++) {
        ExcEntry e;
        e.start = rs->d[r].start;
        e.end = rs->d[r].end;
        e.target = rs->d[r].handler;
        e.depth = 0;
        e.lasti = false;
        vpush(C, entries, e);
      }
    }
    if (C->err) break;
    G = build_basic_blocks(C, K, entries);
    if (C->err) break;
    prune_unreachable(C, G);
    if (C->err) break;
    i32 nb = G->n_blocks;
    G->loops = vnew<Loop>(C, 4);
    G->loop_of_header = (i32*)ualloc(C, (u64)nb * sizeof(i32));
    if (C->err) break;
    for (i32 b = 0; b < nb; b++) G->loop_of_header[b] = -1;
    AnaWs W;
    u8* covered = sarr<u8>(C, (u64)nb);  // universe of analyze_loops = set(idom), then grows
    if (!ana_ws_init(C, &W, G)) break;
    BSet uni = collect_reach(&W, G, G->entry, nullptr);
    BSet dom = compute_dominators(C, &W, G, G->entry, uni);
    if (C->err) break;
    for (i32 i = 0; i < dom.n; i++) covered[dom.ls[i]] = 1;
    if (!analyze_loops(C, &W, G, dom)) {
      if (C->err) break;
      fail_struct(C, G->entry, "irreducible control flow");
      break;
    }
    if (C->err) break;
    for (u32 e = 0; e < entries->n && !C->err; e++) {
      i32 root = block_at(G, entries->d[e].target);
      if (root < 0 || covered[root]) continue;
      // universe = reachable(root) - covered, plus root (never empty: root is in it)
      BSet uni2 = collect_reach(&W, G, root, covered);
      BSet sub = compute_dominators(C, &W, G, root, uni2);
      if (C->err) break;
      if (!analyze_loops(C, &W, G, sub)) {
        if (C->err) break;
        fail_struct(C, root, "irreducible control flow in handler");
        break;
      }
      if (C->err) break;
      for (i32 i = 0; i < sub.n; i++) covered[sub.ls[i]] = 1;
    }
  } while (0);
  if (!C->err) C->top = mark;
  return C->err ? nullptr : G;
}
