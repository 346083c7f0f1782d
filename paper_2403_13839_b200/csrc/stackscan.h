// stackscan.h -- stack-depth analysis as a segmented prefix scan (north star (3),
// SURVEY Appendix A), shared by the sm_100a kernel (stackscan_kernel.cu) and the
// host build (tools/hostcheck.cpp).
//
// The reference has no stand-alone depth pass: depth is len(st) inside the
// symbolic simulation (symexec.py:138-210, transfer functions :239-944, the depth
// guard :208-209).  Here every decoded instruction gets its net effect on the
// symbolic stack along the fall-through edge (Appendix A, from the handlers), and
// an inclusive scan segmented at the instruction-rule block leaders (cfg.py:72-86:
// the first instruction, jump targets, the instruction after a block ender) gives
// depth_after(i) relative to the entry of i's segment.  Every reference block
// (cfg.py:89-97: those leaders plus exception-table ones) lies inside one segment,
// so a block entered with depth E reaches E + S(i) - S(lo - 1) after instruction i
// (S(lo - 1) = 0 when lo starts a segment).  Effects that depend on the stack's
// contents (END_FINALLY's sentinel, POP_FINALLY / WITH_CLEANUP_*, POP_EXCEPT's
// clamp, 3.11 CALL_FUNCTION_EX's NULL, SEND) or that the reference does not lift
// make the depth unknown from there to the end of the segment (flag bit1).
//
// Checked against depths recorded from the reference's own simulation
// (tests/golden/stack.jsonl, make_stack_golden.py).
#pragma once
#include "common.h"

enum { SS_SEG_START = 1, SS_UNKNOWN = 2, SS_ENDER = 4 };

// Net fall-through effect of one instruction; *known = false for shape-dependent
// or unlifted ops (Appendix A).
HD inline int stack_effect(int minor, u8 op, u32 arg, bool* known) {
  *known = true;
  const int n = (int)(arg > 0x7FFF ? 0x7FFF : arg);
  switch (op) {
    // pushes (symexec.py:239-268, 524-531, 715-718, 834-835, 854-855, 862-863, 880-894, 923-924)
    case OP_LOAD_CONST: case OP_LOAD_FAST: case OP_LOAD_NAME: case OP_LOAD_DEREF: case OP_LOAD_CLASSDEREF:
    case OP_LOAD_CLOSURE: case OP_LOAD_ASSERTION_ERROR: case OP_LOAD_BUILD_CLASS: case OP_PUSH_NULL:
    case OP_COPY: case OP_DUP_TOP: case OP_LOAD_METHOD: case OP_IMPORT_FROM: case OP_RETURN_GENERATOR:
    case OP_BEGIN_FINALLY: case OP_PUSH_EXC_INFO: case OP_SETUP_WITH: case OP_BEFORE_WITH: case OP_GET_LEN:
      return 1;
    case OP_LOAD_GLOBAL: return minor >= 11 && (arg & 1) ? 2 : 1;
    case OP_DUP_TOP_TWO: return 2;
    // stores / deletes (:272-451)
    case OP_STORE_FAST: case OP_STORE_NAME: case OP_STORE_GLOBAL: case OP_STORE_DEREF: return -1;
    case OP_STORE_ATTR: return -2;
    case OP_STORE_SUBSCR: return -3;
    case OP_UNPACK_SEQUENCE: return n - 1;
    case OP_UNPACK_EX: return (int)(arg & 0xFF) + (int)((arg >> 8) & 0xFFFF) + 1 - 1;
    case OP_DELETE_FAST: case OP_DELETE_NAME: case OP_DELETE_GLOBAL: case OP_DELETE_DEREF: return 0;
    case OP_DELETE_ATTR: return -1;
    case OP_DELETE_SUBSCR: return -2;
    // binary / unary / stack shuffles (:455-546, 927-944)
    case OP_BINARY_ADD: case OP_BINARY_AND: case OP_BINARY_FLOOR_DIVIDE: case OP_BINARY_LSHIFT:
    case OP_BINARY_MATRIX_MULTIPLY: case OP_BINARY_MODULO: case OP_BINARY_MULTIPLY: case OP_BINARY_OP:
    case OP_BINARY_OR: case OP_BINARY_POWER: case OP_BINARY_RSHIFT: case OP_BINARY_SUBSCR:
    case OP_BINARY_SUBTRACT: case OP_BINARY_TRUE_DIVIDE: case OP_BINARY_XOR: case OP_INPLACE_ADD:
    case OP_INPLACE_AND: case OP_INPLACE_FLOOR_DIVIDE: case OP_INPLACE_LSHIFT: case OP_INPLACE_MATRIX_MULTIPLY:
    case OP_INPLACE_MODULO: case OP_INPLACE_MULTIPLY: case OP_INPLACE_OR: case OP_INPLACE_POWER:
    case OP_INPLACE_RSHIFT: case OP_INPLACE_SUBTRACT: case OP_INPLACE_TRUE_DIVIDE: case OP_INPLACE_XOR:
    case OP_COMPARE_OP: case OP_IS_OP: case OP_CONTAINS_OP: case OP_POP_TOP:
      return -1;
    case OP_UNARY_INVERT: case OP_UNARY_NEGATIVE: case OP_UNARY_NOT: case OP_UNARY_POSITIVE:
    case OP_ROT_TWO: case OP_ROT_THREE: case OP_ROT_FOUR: case OP_ROT_N: case OP_SWAP:
      return 0;
    // displays (:550-708)
    case OP_BUILD_TUPLE: case OP_BUILD_LIST: case OP_BUILD_SET: case OP_BUILD_SLICE: case OP_BUILD_STRING:
    case OP_BUILD_TUPLE_UNPACK: case OP_BUILD_LIST_UNPACK: case OP_BUILD_SET_UNPACK: case OP_BUILD_MAP_UNPACK:
    case OP_BUILD_TUPLE_UNPACK_WITH_CALL: case OP_BUILD_MAP_UNPACK_WITH_CALL:
      return 1 - n;
    case OP_BUILD_MAP: return 1 - 2 * n;
    case OP_BUILD_CONST_KEY_MAP: return -n;
    case OP_FORMAT_VALUE: return (arg & 4) ? -1 : 0;
    case OP_LIST_APPEND: case OP_SET_ADD: case OP_LIST_EXTEND: case OP_SET_UPDATE: case OP_DICT_UPDATE:
    case OP_DICT_MERGE:
      return -1;
    case OP_MAP_ADD: return -2;
    case OP_LIST_TO_TUPLE: return 0;
    // calls, functions, imports (:745-839)
    case OP_CALL_FUNCTION: return -n;
    case OP_CALL_FUNCTION_KW: case OP_CALL_METHOD: case OP_CALL: return -n - 1;
    case OP_CALL_FUNCTION_EX:
      if (minor >= 11) *known = false;  // a further pop when a NULL sits below
      return -1 - (int)(arg & 1);
    case OP_MAKE_FUNCTION: return -__builtin_popcount(arg & 0xF) - (minor <= 10 ? 1 : 0);
    case OP_IMPORT_NAME: case OP_IMPORT_STAR: return -1;
    // generators, exceptions (:843-914)
    case OP_YIELD_VALUE: return 0;
    case OP_YIELD_FROM: case OP_YIELD_FROM_311: return -1;
    // control (:153-201); conditional jumps: the fall-through edge
    case OP_RETURN_VALUE: return -1;
    case OP_RAISE_VARARGS: return -n;
    case OP_POP_JUMP_IF_FALSE: case OP_POP_JUMP_IF_TRUE: case OP_POP_JUMP_FORWARD_IF_FALSE:
    case OP_POP_JUMP_FORWARD_IF_TRUE: case OP_POP_JUMP_BACKWARD_IF_FALSE: case OP_POP_JUMP_BACKWARD_IF_TRUE:
    case OP_POP_JUMP_FORWARD_IF_NONE: case OP_POP_JUMP_FORWARD_IF_NOT_NONE: case OP_POP_JUMP_BACKWARD_IF_NONE:
    case OP_POP_JUMP_BACKWARD_IF_NOT_NONE:
      return -1;
    case OP_JUMP_IF_FALSE_OR_POP: case OP_JUMP_IF_TRUE_OR_POP: return -1;
    case OP_JUMP_IF_NOT_EXC_MATCH: return -2;
    case OP_FOR_ITER: return 1;
    // no effect (_NOPS, :41-45; SETUP_FINALLY :859-860; KW_NAMES :722-723; LOAD_ATTR :712-713;
    // CHECK_EXC_MATCH :885-887; unconditional jumps)
    case OP_NOP: case OP_RESUME: case OP_PRECALL: case OP_MAKE_CELL: case OP_COPY_FREE_VARS: case OP_GEN_START:
    case OP_SETUP_ANNOTATIONS: case OP_POP_BLOCK: case OP_GET_ITER: case OP_GET_YIELD_FROM_ITER:
    case OP_CALL_FINALLY: case OP_SETUP_FINALLY: case OP_KW_NAMES: case OP_LOAD_ATTR: case OP_CHECK_EXC_MATCH:
    case OP_JUMP_FORWARD: case OP_JUMP_ABSOLUTE: case OP_JUMP_BACKWARD: case OP_JUMP_BACKWARD_NO_INTERRUPT:
    case OP_RERAISE:
      return 0;
    default:  // END_FINALLY, POP_FINALLY, WITH_CLEANUP_*, POP_EXCEPT, SEND, async / match ops, ...
      *known = false;
      return 0;
  }
}

// block enders (cfg.py:57-66 _block_enders): the next instruction leads a block
HD inline bool stack_block_ender(u8 op, u8 kind) {
  const bool jump = kind == K_JUMP_REL || kind == K_JUMP_ABS || kind == K_JUMP_BACK;
  return op == OP_RETURN_VALUE || op == OP_RAISE_VARARGS || op == OP_RERAISE || op == OP_END_FINALLY ||
         (jump && op != OP_SETUP_FINALLY && op != OP_SETUP_WITH && op != OP_SETUP_ASYNC_WITH);
}

// Per-instruction scan element: (segment start, unknown, effect).
struct StackElem {
  int seg;   // 1: this instruction starts a segment
  int unk;   // 1: an unknown effect at or before this instruction in the segment
  int sum;   // inclusive effect sum since the segment start
};
// Segmented combine, `a` earlier than `b`.
HD inline StackElem stack_combine(StackElem a, StackElem b) {
  if (b.seg) return b;
  return StackElem{a.seg, a.unk | b.unk, a.sum + b.sum};
}

// Reference-order scalar scan of one decoded object (host build; the kernel's
// per-lane sequential part runs the same element function).
HD inline void stack_elem_of(int minor, const upy_ins& r, u32 ent, bool prev_ender, bool first, StackElem* e,
                             bool* ender) {
  bool known;
  const u8 op = UPY_ENT_OP(ent);
  e->sum = stack_effect(minor, op, r.arg, &known);
  e->unk = known ? 0 : 1;
  e->seg = (first || prev_ender || (r.flags & 4)) ? 1 : 0;
  *ender = stack_block_ender(op, (u8)UPY_ENT_KIND(ent));
}

HD inline void stackscan_scalar(const upy_ins* rec, i32 n, int minor, upy_stackrec* out, upy_stackinfo* info) {
  StackElem acc{1, 0, 0};
  bool prev_ender = false;
  info->n_segments = 0;
  info->max_depth = 0;
  info->min_depth = 0;
  info->n_pushes = 0;
  info->n_unknown = 0;
  for (i32 i = 0; i < n; i++) {
    const u32 ent = optab(minor, rec[i].opcode);
    StackElem e;
    bool ender;
    stack_elem_of(minor, rec[i], ent, prev_ender, i == 0, &e, &ender);
    acc = i == 0 ? e : stack_combine(acc, e);
    info->n_segments += e.seg;
    info->n_unknown += e.unk;
    info->n_pushes += (!e.unk && e.sum > 0) ? e.sum : 0;
    if (!acc.unk) {
      if (acc.sum > info->max_depth) info->max_depth = acc.sum;
      if (acc.sum < info->min_depth) info->min_depth = acc.sum;
    }
    out[i].depth = (int16_t)(acc.sum > 32767 ? 32767 : acc.sum < -32768 ? -32768 : acc.sum);
    out[i].flags = (u8)((e.seg ? SS_SEG_START : 0) | (acc.unk ? SS_UNKNOWN : 0) | (ender ? SS_ENDER : 0));
    out[i].pad = 0;
    prev_ender = ender;
  }
}

// ---------------------------------------------------------------- table form
// The kernel evaluates effects from a per-(version, opcode) descriptor in shared
// memory instead of the switch above (branch-free per instruction):
//   bits 0-7 base (int8), bits 8-10 arg term, bits 11-14 multiplier (int4),
//   bit 15 unknown, bit 16 block ender;
//   effect = base + mul * term(arg), term: 0 none, 1 n = min(arg, 0x7FFF),
//   2 popcount(arg & 0xF), 3 arg & 1, 4 (arg & 4) != 0, 5 (arg & 0xFF) + (arg >> 8 & 0xFFFF).
// stack_desc is derived from stack_effect by probing it, and the host test
// checks desc-form == switch-form for every (version, opcode) over all 16-bit args.
enum { SD_NONE = 0, SD_N = 1, SD_POP4 = 2, SD_BIT0 = 3, SD_BIT2 = 4, SD_UNPACK_EX = 5 };
HD inline u32 stack_desc_make(int base, int term, int mul, bool unknown, bool ender) {
  return (u32)(base & 0xFF) | ((u32)term << 8) | ((u32)(mul & 0xF) << 11) | (unknown ? 1u << 15 : 0u) |
         (ender ? 1u << 16 : 0u);
}
HD inline int stack_desc_term(u32 d, u32 arg) {  // branch-free selection of the arg term
  const u32 k = (d >> 8) & 7;
  const int n = (int)(arg > 0x7FFF ? 0x7FFF : arg);
  const int pop = __builtin_popcount(arg & 0xF);
  const int ux = (int)(arg & 0xFF) + (int)((arg >> 8) & 0xFFFF);
  int t = k == SD_N ? n : 0;
  t = k == SD_POP4 ? pop : t;
  t = k == SD_BIT0 ? (int)(arg & 1) : t;
  t = k == SD_BIT2 ? (int)((arg >> 2) & 1) : t;
  t = k == SD_UNPACK_EX ? ux : t;
  return t;
}
HD inline int stack_desc_effect(u32 d, u32 arg) {
  const int base = (int)(int8_t)(d & 0xFF);
  const int mul = (int)((d >> 11) & 0xF) - (((d >> 11) & 0x8) ? 16 : 0);
  return base + mul * stack_desc_term(d, arg);
}
// Descriptor of one (version, table entry): the term is identified by probing
// stack_effect with args that separate the candidate terms.
HD inline u32 stack_desc(int minor, u32 ent) {
  if (!ent) return stack_desc_make(0, SD_NONE, 0, true, false);
  const u8 op = UPY_ENT_OP(ent);
  bool k0, k;
  const int e0 = stack_effect(minor, op, 0, &k0);
  const bool ender = stack_block_ender(op, (u8)UPY_ENT_KIND(ent));
  const u32 probes[6] = {1, 2, 4, 0x100, 0xF, 0x7FFF0};
  for (int t = SD_NONE; t <= SD_UNPACK_EX; t++) {
    int mul = 0;
    if (t != SD_NONE) {
      mul = stack_effect(minor, op, t == SD_BIT2 ? 4u : 1u, &k) - e0;  // the term is 1 at this arg
      if (mul == 0 || mul < -8 || mul > 7) continue;
    }
    if (e0 < -128 || e0 > 127) break;
    const u32 d = stack_desc_make(e0, t, mul, !k0, ender);
    bool ok = true;
    for (int p = 0; p < 6 && ok; p++) ok = stack_effect(minor, op, probes[p], &k) == stack_desc_effect(d, probes[p]);
    if (ok) return d;
  }
  return stack_desc_make(0, SD_NONE, 0, true, ender);  // no descriptor fits: unknown
}

// Host check: the descriptor form equals the switch form for every table entry and
// every arg in [0, n_args) (plus a few wide ones); returns the number of mismatches.
HD inline u64 stack_desc_selfcheck(u32 n_args) {
  u64 bad = 0;
  for (int minor = 8; minor <= 11; minor++)
    for (u32 opc = 0; opc < 256; opc++) {
      const u32 ent = optab(minor, opc);
      if (!ent) continue;
      const u32 d = stack_desc(minor, ent);
      for (u32 a = 0; a < n_args + 4; a++) {
        const u32 arg = a < n_args ? a : (a == n_args ? 0xFFFFFFFFu : a == n_args + 1 ? 0x12345678u
                                                        : a == n_args + 2 ? 0x7FFFu : 0x10000u);
        bool k;
        const int e = stack_effect(minor, UPY_ENT_OP(ent), arg, &k);
        if (k == (((d >> 15) & 1) != 0) || (k && e != stack_desc_effect(d, arg))) bad++;
      }
    }
  return bad;
}
