// common.h -- per-thread decompile context: bump arena, growable vectors,
// strings, error state and the frozen tables (opcodes, cmp_op, printable).
//
// Everything here compiles for sm_100a device code (one thread owns one root
// code object and its arena slot) and, for the test-only host harness, as
// plain C++.  Python-level failure semantics are modelled by a sticky status
// in Dc: the first failure wins, every loop/recursive step checks `C->err`.
#pragma once
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include "../../include/upy.h"
#include "optables.h"
#include "unicode_tables.h"

#ifdef __CUDACC__
#define HD __host__ __device__
#define DI __device__ __forceinline__
#define NOINL __noinline__
#define FORCEINL __forceinline__
#else
#define HD
#define DI inline
#define NOINL __attribute__((noinline))
#define FORCEINL inline __attribute__((always_inline))
#endif

typedef uint8_t u8;
typedef uint16_t u16;
typedef uint32_t u32;
typedef uint64_t u64;
typedef int32_t i32;
typedef int64_t i64;

// ------------------------------------------------------------------ tables
#ifdef __CUDACC__
__constant__ uint32_t UPY_OPTABLE_DEV[4][256] = UPY_OPTABLE_INIT;
__constant__ uint32_t UPY_PRINTABLE_DEV[UPY_N_PRINTABLE_RANGES][2] = UPY_PRINTABLE_INIT;
__constant__ int UPY_NCMP_DEV[4] = UPY_NCMP_INIT;
__device__ const char* const UPY_OPNAMES_DEV[OP__COUNT] = UPY_OPNAMES_INIT;
__device__ const char* const UPY_CMPOP_DEV[UPY_NCMP_ALL] = UPY_CMPOP_INIT;
#endif
static const uint32_t UPY_OPTABLE_HOST[4][256] = UPY_OPTABLE_INIT;
static const uint32_t UPY_PRINTABLE_HOST[UPY_N_PRINTABLE_RANGES][2] = UPY_PRINTABLE_INIT;
static const int UPY_NCMP_HOST[4] = UPY_NCMP_INIT;
static const char* const UPY_OPNAMES_HOST[OP__COUNT] = UPY_OPNAMES_INIT;
static const char* const UPY_CMPOP_HOST[UPY_NCMP_ALL] = UPY_CMPOP_INIT;

#if defined(__CUDA_ARCH__)
#define T_OPTABLE UPY_OPTABLE_DEV
#define T_PRINTABLE UPY_PRINTABLE_DEV
#define T_NCMP UPY_NCMP_DEV
#define T_OPNAMES UPY_OPNAMES_DEV
#define T_CMPOP UPY_CMPOP_DEV
#else
#define T_OPTABLE UPY_OPTABLE_HOST
#define T_PRINTABLE UPY_PRINTABLE_HOST
#define T_NCMP UPY_NCMP_HOST
#define T_OPNAMES UPY_OPNAMES_HOST
#define T_CMPOP UPY_CMPOP_HOST
#endif

HD inline u32 optab(int minor, u32 opcode) { return T_OPTABLE[minor - 8][opcode & 0xFF]; }
#ifdef __CUDACC__
// Global-memory copy of the opcode tables for lookups that diverge across a warp
// (one object per thread): divergent __constant__ reads serialize, while __ldg
// reads of this 4 KB table stay L1-resident.  (A shared-memory copy cost more L1
// capacity than it saved: 62.5 -> 64.9 ms per 262K C3 objects.)
__device__ const uint32_t UPY_OPTABLE_GLB[4][256] = UPY_OPTABLE_INIT;
#endif
HD inline u32 optab_div(int minor, u32 opcode) {
#ifdef __CUDA_ARCH__
  return __ldg(&UPY_OPTABLE_GLB[minor - 8][opcode & 0xFF]);
#else
  return optab(minor, opcode);
#endif
}
HD inline const char* opname_of(int op) { return T_OPNAMES[op]; }

HD inline size_t cstrlen(const char* s) {
  size_t n = 0;
  while (s[n]) n++;
  return n;
}

// ------------------------------------------------------------------ strings
// UTF-8 (surrogatepass) byte string; p == nullptr means Python None.
struct Str {
  const char* p;
  u32 n;
};
HD inline Str S(const char* lit) { return Str{lit, (u32)cstrlen(lit)}; }
HD inline Str Snone() { return Str{nullptr, 0}; }
HD inline bool s_is_none(Str a) { return a.p == nullptr; }
HD inline bool s_eq(Str a, Str b) {
  if (a.p == nullptr || b.p == nullptr) return a.p == b.p;
  if (a.n != b.n) return false;
  if (a.p == b.p) return true;
  for (u32 i = 0; i < a.n; i++)
    if (a.p[i] != b.p[i]) return false;
  return true;
}
HD inline bool s_eqc(Str a, const char* lit) {
  if (a.p == nullptr) return false;
  u32 i = 0;
  for (; i < a.n; i++)
    if (lit[i] == 0 || lit[i] != a.p[i]) return false;
  return lit[i] == 0;
}
HD inline bool s_has(Str a, char ch) {
  for (u32 i = 0; i < a.n; i++)
    if (a.p[i] == ch) return true;
  return false;
}

// ------------------------------------------------------------------ context
struct NodeT;
struct Dc;

// Decoded instruction as the structurer sees it (disasm.py:28-52).
struct Ins {
  u32 offset;     // extent start
  u32 arg;        // saturated arg
  u8 op;          // canonical op id (optables.h)
  u8 kind;        // UpyKind
  u8 nprefix;
  u8 flags;       // bit0 has_arg, bit1 arg saturated
  u32 cache;      // cache units (3.11 yield-from collapse can exceed 255)
};
HD inline u32 ins_op_offset(const Ins& i) { return i.offset + 2 * i.nprefix; }
HD inline u32 ins_end(const Ins& i) { return i.offset + 2 * (1 + i.nprefix + i.cache); }
HD inline bool ins_is_jump(const Ins& i) {
  return i.kind == K_JUMP_REL || i.kind == K_JUMP_ABS || i.kind == K_JUMP_BACK;
}
HD inline bool ins_has_arg(const Ins& i) { return i.flags & 1; }

struct Dc {
  // arena
  u8* base;
  u64 cap;
  u64 used;
  u64 top;         // scratch stack boundary (== cap when empty); bump region is [0, used)
  u64 low_top;     // lowest `top` seen (scratch high-water mark, for slot sizing)
  u8* sink;        // scratch returned after an overflow (zeroed), SINK_BYTES long
  // status (first failure wins)
  int err;
  i64 aux0, aux1;
  // message of the failure (device-formatted)
  char* msg;
  u32 msg_len, msg_cap;
  // inputs
  const upy_arena* A;
  // the arena's section bases copied out of *A: one dependent load less on every
  // string / const / ref lookup (A points at the kernel-parameter copy)
  const upy_obj* objs;
  const upy_const* consts;
  const upy_str* strs;
  const uint32_t* refs;
  const uint32_t* limbs;
  const uint8_t* bytes;
  const upy_ins* ins_all;
  const upy_decoded* dec_all;
  // recursion guard
  int depth;
  int max_depth;
  // FuncExpr / BuildClass nodes created so far (recovery is an identity
  // transform on trees that contain neither, see recover.h decompile_body)
  u32 n_defs;
};

#define SINK_BYTES (64u * 1024u)

// 16-byte-granular zero / copy for 16-aligned arena blocks (device memset /
// memcpy on generic pointers compile to byte loops).
#ifndef UPY_ZERO_HOOK
#define UPY_ZERO_HOOK(bytes)
#endif
HD inline void zero16(void* p, u64 bytes) {
  UPY_ZERO_HOOK(bytes);
#ifdef __CUDA_ARCH__
  uint4* q = (uint4*)p;
  const uint4 z = make_uint4(0, 0, 0, 0);
  // not unrolled: inlined at ~2000 call sites, unrolled copies were 29% of the
  // kernel's SASS and the instruction-cache misses they caused its top stall
#pragma unroll 1
  for (u64 i = 0, n = bytes >> 4; i < n; i++) q[i] = z;
#else
  memset(p, 0, bytes);
#endif
}
HD inline void copy16(void* dst, const void* src, u64 bytes) {  // both 16-aligned; copies ceil16(bytes)
#ifdef __CUDA_ARCH__
  uint4* d = (uint4*)dst;
  const uint4* s = (const uint4*)src;
#pragma unroll 1
  for (u64 i = 0, n = (bytes + 15) >> 4; i < n; i++) d[i] = s[i];
#else
  memcpy(dst, src, bytes);
#endif
}

// Bump allocation; zeroed unless `zero` is false (buffers written before read).
#ifndef UPY_ALLOC_HOOK
#define UPY_ALLOC_HOOK(bytes)
#endif
#if !defined(UPY_INLINE_SLOW) && defined(__CUDA_ARCH__)
// Cold paths live out of line: every helper below is inlined at thousands of
// call sites, and their rarely taken branches (overflow handling, vector growth,
// message formatting) were most of the decompile kernel's 8 MB of SASS.
#define SLOWPATH NOINL inline
#else
#define SLOWPATH inline
#endif
HD SLOWPATH void* alloc_overflow(Dc* C, u64 bytes) {
  if (!C->err) {
    C->err = UPY_ST_ARENA_OVERFLOW;
    C->aux0 = (i64)C->used;
    C->aux1 = (i64)bytes;
  }
  u64 z = bytes < SINK_BYTES ? bytes : SINK_BYTES;
  zero16(C->sink, z);
  return C->sink;
}
#if defined(UPY_ALLOC_NOINL) && defined(__CUDA_ARCH__)
#define ALLOCFN NOINL inline  // variant: one out-of-line copy of the allocator / node constructor
#else
#define ALLOCFN inline
#endif
HD ALLOCFN void* alloc_raw(Dc* C, u64 bytes, bool zero) {
  bytes = (bytes + 15) & ~(u64)15;
  UPY_ALLOC_HOOK(bytes);
  const u64 u = C->used;
  if (u + bytes > C->top) return alloc_overflow(C, bytes);
  void* p = C->base + u;
  C->used = u + bytes;
  if (zero) zero16(p, bytes);
  return p;
}
HD inline void* zalloc(Dc* C, u64 bytes) { return alloc_raw(C, bytes, true); }
HD inline void* ualloc(Dc* C, u64 bytes) { return alloc_raw(C, bytes, false); }

// Scratch stack growing down from the top of the slot: temporaries of one
// analysis phase, released together (`C->top = mark`).  Never grown in place.
HD inline void* salloc(Dc* C, u64 bytes, bool zero = true) {
  bytes = (bytes + 15) & ~(u64)15;
  if (C->used + bytes > C->top) return alloc_raw(C, C->top - C->used + 16, false);  // records the overflow
  C->top -= bytes;
  if (C->top < C->low_top) C->low_top = C->top;
  void* p = C->base + C->top;
  if (zero) zero16(p, bytes);
  return p;
}
template <class T>
HD inline T* sarr(Dc* C, u64 n, bool zero = true) {
  return (T*)salloc(C, n * sizeof(T) + 16, zero);
}
// Clear of a compile-time-sized block: straight-line 16-B stores (no loop) up to
// 256 bytes -- vector headers and the other small records take one to a few stores.
template <u64 R>
HD FORCEINL void zero_const(void* p) {
#ifdef __CUDA_ARCH__
  if (R <= 256) {
    uint4* q = (uint4*)p;
    const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (u64 i = 0; i < R / 16; i++) q[i] = z;
  } else {
    zero16(p, R);
  }
#else
  memset(p, 0, R);
#endif
}
template <class T>
HD inline T* anew(Dc* C) {
#ifndef UPY_ANEW_LOOP
  constexpr u64 r = (sizeof(T) + 15) & ~(u64)15;
  T* p = (T*)alloc_raw(C, r, false);
  zero_const<r>(p);
  return p;
#else
  return (T*)zalloc(C, sizeof(T));
#endif
}

// ------------------------------------------------------------------ vectors
template <class T>
struct Vec {
  T* d;
  u32 n, cap;
};
template <class T>
HD inline Vec<T>* vnew(Dc* C, u32 cap = 0) {
  Vec<T>* v = anew<Vec<T>>(C);
  if (cap && !C->err) {
    u64 b = (u64)cap * sizeof(T);
    if (b > SINK_BYTES && C->used + b > C->top) {
      zalloc(C, b);  // records the overflow
      return v;
    }
    v->d = (T*)ualloc(C, b);
    v->cap = C->err ? 0 : cap;
  }
  return v;
}
template <class T>
HD SLOWPATH bool vgrow(Dc* C, Vec<T>* v, u32 need) {
  if (need <= v->cap) return true;
  if (C->err) return false;
  u32 nc = v->cap ? v->cap * 2 : 4;
  while (nc < need) nc *= 2;
  T* nd = (T*)ualloc(C, (u64)nc * sizeof(T));
  if (C->err) return false;
  if (v->n) copy16(nd, v->d, (u64)v->n * sizeof(T));
  v->d = nd;
  v->cap = nc;
  return true;
}
template <class T>
HD inline void vpush(Dc* C, Vec<T>* v, T x) {
  if (v->n >= v->cap && !vgrow(C, v, v->n + 1)) return;
  v->d[v->n++] = x;
}
template <class T>
HD inline Vec<T>* vcopy(Dc* C, const Vec<T>* src, u32 lo = 0, u32 hi = 0xFFFFFFFFu) {
  u32 n = src ? src->n : 0;
  if (hi > n) hi = n;
  if (lo > hi) lo = hi;
  Vec<T>* v = vnew<T>(C, hi - lo);
  if (C->err) return v;
  if (lo == 0 && hi) {
    copy16(v->d, src->d, (u64)hi * sizeof(T));
  } else {
#pragma unroll 1
    for (u32 i = lo; i < hi; i++) v->d[i - lo] = src->d[i];
  }
  v->n = hi - lo;
  return v;
}
template <class T>
HD inline void vextend(Dc* C, Vec<T>* dst, const Vec<T>* src, u32 lo = 0, u32 hi = 0xFFFFFFFFu) {
  if (!src) return;
  if (hi > src->n) hi = src->n;
  if (lo >= hi) return;
  if (dst->n + (hi - lo) > dst->cap && !vgrow(C, dst, dst->n + (hi - lo))) return;
#pragma unroll 1
  for (u32 i = lo; i < hi; i++) dst->d[dst->n++] = src->d[i];
}
template <class T>
HD inline T vlast(const Vec<T>* v) { return v->d[v->n - 1]; }

// ------------------------------------------------------------------ text
struct Text {
  char* d;
  u32 n, cap;
};
HD SLOWPATH bool t_grow_slow(Dc* C, Text* t, u32 need);
HD inline bool t_grow(Dc* C, Text* t, u32 need) {
  if (need <= t->cap) return true;
  return t_grow_slow(C, t, need);
}
HD SLOWPATH bool t_grow_slow(Dc* C, Text* t, u32 need) {
  if (C->err) return false;
  u32 nc = t->cap ? t->cap * 2 : 256;
  while (nc < need) nc *= 2;
  char* nd = (char*)ualloc(C, nc);
  if (C->err) return false;
  if (t->n) copy16(nd, t->d, t->n);
  t->d = nd;
  t->cap = nc;
  return true;
}
// Inlined: out of line these were 12% less SASS but 1.7% slower on C3 (same-session
// A/B, 255.5 vs 251.3 ms) -- they sit on the emitter's hot path.
#ifdef UPY_TEXT_OOL
#define TEXTFN SLOWPATH
#else
#define TEXTFN inline
#endif
HD TEXTFN void t_putn(Dc* C, Text* t, const char* p, u32 n) {
  if (!n) return;
  if (!t_grow(C, t, t->n + n)) return;
  char* d = t->d + t->n;
#pragma unroll 1
  for (u32 i = 0; i < n; i++) d[i] = p[i];
  t->n += n;
}
HD inline void t_put(Dc* C, Text* t, char ch) {
  if (t->n >= t->cap && !t_grow(C, t, t->n + 1)) return;
  t->d[t->n++] = ch;
}
HD TEXTFN void t_puts(Dc* C, Text* t, const char* s) { t_putn(C, t, s, (u32)cstrlen(s)); }
HD inline void t_str(Dc* C, Text* t, Str s) { t_putn(C, t, s.p, s.n); }
HD inline void t_u32(Dc* C, Text* t, u32 v) {
  char buf[10];
  int k = 0;
  do {
    buf[k++] = (char)('0' + (v % 10));
    v /= 10;
  } while (v);
  if (!t_grow(C, t, t->n + (u32)k)) return;
  while (k) t->d[t->n++] = buf[--k];
}
HD inline void t_i64(Dc* C, Text* t, i64 v) {
  char buf[24];
  int k = 0;
  u64 m = v < 0 ? (u64)(-(v + 1)) + 1 : (u64)v;
  do {
    buf[k++] = (char)('0' + (m % 10));
    m /= 10;
  } while (m);
  if (v < 0) t_put(C, t, '-');
  while (k) t_put(C, t, buf[--k]);
}
HD inline Str t_as_str(const Text* t) { return Str{t->d, t->n}; }

// ------------------------------------------------------------------ errors
// Failure with a device-formatted message: fail_begin() returns the message
// buffer (or nullptr when a failure is already recorded).
struct MsgBuf {
  Dc* C;
  Text t;
};
HD inline bool fail_begin(Dc* C, int status, i64 a0, i64 a1, Text* out) {
  if (C->err) return false;
  C->err = status;
  C->aux0 = a0;
  C->aux1 = a1;
  out->d = C->msg;
  out->n = 0;
  out->cap = C->msg_cap;
  return true;
}
HD inline void fail_end(Dc* C, Text* t) {
  // message buffer is fixed (never grows: t_grow refuses once err is set)
  C->msg_len = t->n;
}
// Message appenders that work after err is set (fixed buffer, truncating).
HD SLOWPATH void m_putn(Dc* C, Text* t, const char* p, u32 n) {
#pragma unroll 1
  for (u32 i = 0; i < n && t->n < t->cap; i++) t->d[t->n++] = p[i];
}
HD SLOWPATH void m_puts(Dc* C, Text* t, const char* s) { m_putn(C, t, s, (u32)cstrlen(s)); }
HD inline void m_str(Dc* C, Text* t, Str s) { m_putn(C, t, s.p, s.n); }
HD SLOWPATH void m_i64(Dc* C, Text* t, i64 v) {
  char buf[24];
  int k = 0;
  u64 m = v < 0 ? (u64)(-(v + 1)) + 1 : (u64)v;
  do {
    buf[k++] = (char)('0' + (m % 10));
    m /= 10;
  } while (m);
  if (v < 0) m_putn(C, t, "-", 1);
  while (k) {
    char ch = buf[--k];
    m_putn(C, t, &ch, 1);
  }
}

// Plain-message failures.
HD inline void fail_msg(Dc* C, int status, const char* m, i64 a0 = 0, i64 a1 = 0) {
  Text t;
  if (!fail_begin(C, status, a0, a1, &t)) return;
  m_puts(C, &t, m);
  fail_end(C, &t);
}
HD inline void py_error(Dc* C, int status, const char* what) { fail_msg(C, status, what); }
// KeyError on an int-keyed dict: str(KeyError(k)) is repr(k)
HD inline void py_key_error(Dc* C, i64 key) {
  Text t;
  if (!fail_begin(C, UPY_ST_PY_KEY_ERROR, 0, 0, &t)) return;
  m_i64(C, &t, key);
  fail_end(C, &t);
}

// StackUnderflow(offset, opname)  errors.py:69-72
HD inline void fail_underflow(Dc* C, const Ins* ins) {
  Text t;
  if (!fail_begin(C, UPY_ST_STACK_UNDERFLOW, ins->offset, 0, &t)) return;
  m_puts(C, &t, "evaluation stack underflow at offset ");
  m_i64(C, &t, ins->offset);
  m_puts(C, &t, " (");
  m_puts(C, &t, opname_of(ins->op));
  m_puts(C, &t, ")");
  fail_end(C, &t);
}
// UnsupportedOpcode(opname, offset)  errors.py:75-81
HD inline void fail_unsupported(Dc* C, const char* opname, i64 offset) {
  Text t;
  if (!fail_begin(C, UPY_ST_UNSUPPORTED_OPCODE, offset, 0, &t)) return;
  m_puts(C, &t, "no lifting rule for ");
  m_puts(C, &t, opname);
  m_puts(C, &t, " at offset ");
  m_i64(C, &t, offset);
  fail_end(C, &t);
}
// StructuringFailed(block_id, reason)  errors.py:92-96
HD inline void fail_struct(Dc* C, i64 block_id, const char* reason) {
  Text t;
  if (!fail_begin(C, UPY_ST_STRUCTURING_FAILED, block_id, 0, &t)) return;
  m_puts(C, &t, "cannot structure region at block ");
  m_i64(C, &t, block_id);
  m_puts(C, &t, ": ");
  m_puts(C, &t, reason);
  fail_end(C, &t);
}
// StackDepthMismatch(block_id, depths)  errors.py:84-89; depths an int or a 2-list
HD inline void fail_depth(Dc* C, i64 block_id, i64 d0, i64 d1, bool is_list) {
  Text t;
  if (!fail_begin(C, UPY_ST_STACK_DEPTH_MISMATCH, block_id, 0, &t)) return;
  m_puts(C, &t, "predecessors of block ");
  m_i64(C, &t, block_id);
  m_puts(C, &t, " disagree on stack depth: ");
  if (is_list) {
    m_puts(C, &t, "[");
    m_i64(C, &t, d0);
    m_puts(C, &t, ", ");
    m_i64(C, &t, d1);
    m_puts(C, &t, "]");
  } else {
    m_i64(C, &t, d0);
  }
  fail_end(C, &t);
}

// recursion guard (the reference runs under Python's default limit of 1000)
struct DepthGuard {
  Dc* C;
  HD DepthGuard(Dc* c) : C(c) {
    if (++C->depth > C->max_depth && !C->err) {
      fail_msg(C, UPY_ST_DEPTH_LIMIT, "device recursion guard");
    }
  }
  HD ~DepthGuard() { --C->depth; }
};
#define GUARD(C) DepthGuard _g_(C)
#define CK(C) \
  if ((C)->err) return
#define CKR(C, v) \
  if ((C)->err) return (v)
