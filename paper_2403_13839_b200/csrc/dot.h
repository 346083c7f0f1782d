// dot.h -- the CFG export of `unpyre disasm --cfg --dot` (cli.py:103-105):
// to_dot(analyze(code)[2]) (cfg.py:331-344, pipeline.py:17-54) written by the
// device from the same analysis the decompiler runs (cfg.h), no validation.
//
// Node order is ascending block start (= block id); edge order is block id, then
// the block's successor order.  analyze_loops re-tags back edges for the export
// (cfg.py:304-310): a successor (s, k) of a back-edge tail u with s == header and
// k in {jump_taken, fallthrough} prints as "loop_back".
#pragma once
#include "pipeline.h"

// The instruction's arg as the reference's Python int: the records saturate at
// 2^32-1 (flags bit1), so wide args are re-folded from the code bytes.
HD inline u64 dot_full_arg(Dc* C, const Code* K, const Ins& in) {
  if (!(in.flags & 2)) return in.arg;
  const u8* b = C->bytes + K->o->code_off + in.offset;
  u64 a = 0;
  for (u32 p = 0; p < in.nprefix; p++) a = (a | b[2 * p + 1]) << 8;
  return a | b[2 * in.nprefix + 1];
}

HD inline void dot_u64(Dc* C, Text* t, u64 v) {
  char buf[24];
  int n = 0;
  do {
    buf[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  t_grow(C, t, t->n + n);
  if (C->err) return;
  while (n) t->d[t->n++] = buf[--n];
}

// Is u -> s a loop back edge (u one of the tails of the loop headed by s)?
HD inline bool dot_is_back(const Cfg* G, i32 u, i32 s) {
  i32 li = G->loop_of_header[s];
  if (li < 0) return false;
  const Vec<i32>* tails = G->loops->d[li].back_tails;
  for (u32 q = 0; q < tails->n; q++)
    if (tails->d[q] == u) return true;
  return false;
}

HD NOINL void cfg_dot(Dc* C, u32 oi, Text* out) {
  BodyJob J;
  J.oi = oi;
  if (!body_analyze(C, &J)) return;
  const Code* K = J.K;
  const Cfg* G = J.G;
  t_grow(C, out, 48 * (u32)K->n_ins + 64 * (u32)G->n_blocks + 64);
  t_puts(C, out, "digraph cfg {\n  node [shape=box fontname=monospace];\n");
  for (i32 b = 0; b < G->n_blocks && !C->err; b++) {
    const Block& B = G->blocks[b];
    if (!B.alive) continue;
    t_puts(C, out, "  b");
    t_i64(C, out, B.id);
    t_puts(C, out, " [label=\"B");
    t_i64(C, out, B.id);
    t_puts(C, out, " [");
    t_i64(C, out, B.start);
    t_put(C, out, ',');
    t_i64(C, out, B.end);
    t_puts(C, out, ")\\l");
    for (i32 i = B.lo; i < B.hi; i++) {
      const Ins& in = K->ins[i];
      t_i64(C, out, ins_op_offset(in));
      t_put(C, out, ' ');
      t_puts(C, out, opname_of(in.op));
      if (ins_has_arg(in)) {
        t_put(C, out, ' ');
        dot_u64(C, out, dot_full_arg(C, K, in));
      }
      t_puts(C, out, "\\l");
    }
    t_puts(C, out, "\"];\n");
  }
  for (i32 b = 0; b < G->n_blocks && !C->err; b++) {
    const Block& B = G->blocks[b];
    if (!B.alive) continue;
    for (u32 q = 0; q < B.succ->n; q++) {
      i32 s = B.succ->d[q];
      u8 k = B.succ_kind->d[q];
      t_puts(C, out, "  b");
      t_i64(C, out, B.id);
      t_puts(C, out, " -> b");
      t_i64(C, out, s);
      t_puts(C, out, " [label=\"");
      if ((k == EK_TAKEN || k == EK_FALL) && dot_is_back(G, B.id, s)) t_puts(C, out, "loop_back");
      else t_puts(C, out, k == EK_TAKEN ? "jump_taken" : k == EK_NOT_TAKEN ? "jump_not_taken"
                          : k == EK_FALL ? "fallthrough" : "exception");
      t_put(C, out, '"');
      if (k == EK_EXC) t_puts(C, out, " style=dashed");
      t_puts(C, out, "];\n");
    }
  }
  t_puts(C, out, "}\n");
}
