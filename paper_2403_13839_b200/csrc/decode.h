// decode.h -- wordcode decoding (disasm.py:71-172) into upy_ins records.
//
// decode_scalar: one thread walks the object in reference order (used for
//   3.11 objects, whose cache-unit skipping makes instruction starts a serial
//   chain, and by the host harness).
// decode_chunk:  one warp per object for 3.8-3.10 (no caches: every unit is an
//   instruction unit), one 256-unit chunk per call (the kernel streams chunks
//   into shared memory with TMA bulk copies, decode_kernel.cu).  Lanes own 8 consecutive units (one 128-bit load each),
//   EXTENDED_ARG runs are folded with a warp shuffle scan over (all-prefix,
//   run length, run value) summaries, record slots come from a popc scan, and
//   jump targets are validated inline: in <=3.10 an offset is an extent start
//   iff it is in range and the previous unit is not EXTENDED_ARG.
#pragma once
#include "common.h"

#define EXT_OP 144
// extra bits of the opcode-table entries the decode kernel stages in shared memory
#define ENT_JUMP_BIT 31
#define ENT_EXT_BIT 30
#define ENT_PAD (1u << 29)

// error aux conventions (consumed by cfg.h load_instructions):
//   UNKNOWN_OPCODE: aux0 opcode, aux1 offset
//   TRUNCATED_CODE: aux0 reason (1 empty, 2 odd, 3 ext run, 4 cache, 5 none), aux1 position
//   BAD_JUMP_TARGET: aux0 offset, aux1 target
HD inline i64 jump_target_u64(int minor, u32 kind, u64 op_offset, u64 arg, bool* ok) {
  *ok = true;
  if (kind == K_JUMP_ABS) return (i64)(minor == 10 ? arg * 2 : arg);
  if (kind == K_JUMP_BACK) return (i64)(op_offset + 2) - (i64)(2 * arg);
  return (i64)(op_offset + 2 + (minor >= 10 ? arg * 2 : arg));
}

HD inline void decode_scalar(const u8* code, u32 len, int minor, upy_ins* rec, upy_decoded* res) {
  res->status = UPY_ST_OK;
  res->n_instrs = 0;
  res->aux0 = res->aux1 = 0;
  if (!len) {
    res->status = UPY_ST_TRUNCATED_CODE;
    res->aux0 = 1;
    return;
  }
  if (len & 1) {
    res->status = UPY_ST_TRUNCATED_CODE;
    res->aux0 = 2;
    return;
  }
  u32 i = 0, n = 0, nprefix = 0, extent = 0;
  u64 ext = 0;
  bool sat = false;
  while (i < len) {
    u32 op = code[i];
    u32 e = optab(minor, op);
    if (!e) {
      res->status = UPY_ST_UNKNOWN_OPCODE;
      res->aux0 = op;
      res->aux1 = i;
      return;
    }
    if (op == EXT_OP) {
      if (nprefix >= 7) sat = true;
      ext = (ext | code[i + 1]) << 8;
      nprefix++;
      i += 2;
      if (i >= len) {
        res->status = UPY_ST_TRUNCATED_CODE;
        res->aux0 = 3;
        res->aux1 = i;
        return;
      }
      continue;
    }
    u64 arg = UPY_ENT_HASARG(e) ? (code[i + 1] | ext) : 0;
    upy_ins& r = rec[n];
    r.offset = extent;
    r.opcode = (u8)op;
    r.n_prefixes = (u8)(nprefix > 255 ? 255 : nprefix);
    u32 cache = UPY_ENT_CACHE(e);
    r.cache_units = (u8)cache;
    bool big = UPY_ENT_HASARG(e) && (sat || (arg >> 32));
    r.arg = big ? 0xFFFFFFFFu : (u32)arg;
    r.flags = (u8)(UPY_ENT_HASARG(e) | (big ? 2 : 0));
    i += 2;
    if (cache) {
      u32 end = i + 2 * cache;
      if (end > len) {
        res->status = UPY_ST_TRUNCATED_CODE;
        res->aux0 = 4;
        res->aux1 = i;
        return;
      }
      i = end;
    }
    n++;
    ext = 0;
    sat = false;
    nprefix = 0;
    extent = i;
  }
  if (!n) {
    res->status = UPY_ST_TRUNCATED_CODE;
    res->aux0 = 5;
    return;
  }
  res->n_instrs = (i32)n;
  // resolve_jump_targets: first jump (in order) whose target is not an extent start
  for (u32 k = 0; k < n; k++) {
    u32 e = optab(minor, rec[k].opcode);
    u32 kind = UPY_ENT_KIND(e);
    if (kind != K_JUMP_REL && kind != K_JUMP_ABS && kind != K_JUMP_BACK) continue;
    u64 arg = rec[k].arg;
    bool ok;
    i64 t = jump_target_u64(minor, kind, rec[k].offset + 2ull * rec[k].n_prefixes, arg, &ok);
    bool valid = false;
    if (!(rec[k].flags & 2) && t >= 0 && t <= 0xFFFFFFFFll) {
      u32 lo = 0, hi = n;
      while (lo < hi) {
        u32 mid = (lo + hi) >> 1;
        if ((i64)rec[mid].offset < t) lo = mid + 1;
        else hi = mid;
      }
      valid = lo < n && (i64)rec[lo].offset == t;
      if (valid) rec[lo].flags |= 4;  // is_jump_target (disasm.py:168-171)
    }
    if (!valid) {
      res->status = UPY_ST_BAD_JUMP_TARGET;
      res->aux0 = rec[k].offset;
      res->aux1 = t;
      return;
    }
  }
}

#ifdef __CUDACC__
// Summary of a span of units w.r.t. the pending EXTENDED_ARG run at its end.
struct ExtRun {
  u32 all;   // 1 if every unit of the span is EXTENDED_ARG (empty span: identity)
  u32 len;   // trailing EXTENDED_ARG run length
  u64 val;   // trailing run bytes concatenated (exact while len <= 7)
};
__device__ __forceinline__ ExtRun ext_combine(ExtRun a, ExtRun b) {  // a then b
  if (!b.all) return b;
  ExtRun r;
  r.all = a.all;
  r.len = a.len + b.len;
  u32 sh = 8 * b.len;
  r.val = sh >= 64 ? b.val : ((a.val << sh) | b.val);
  return r;
}
__device__ __forceinline__ ExtRun shfl_up_run(ExtRun x, int d) {
  ExtRun r;
  r.all = __shfl_up_sync(0xffffffffu, x.all, d);
  r.len = __shfl_up_sync(0xffffffffu, x.len, d);
  r.val = __shfl_up_sync(0xffffffffu, x.val, d);
  return r;
}
__device__ __forceinline__ ExtRun shfl_run(ExtRun x, int src) {
  ExtRun r;
  r.all = __shfl_sync(0xffffffffu, x.all, src);
  r.len = __shfl_sync(0xffffffffu, x.len, src);
  r.val = __shfl_sync(0xffffffffu, x.val, src);
  return r;
}

// Per-object state carried across the 256-unit chunks of one <=3.10 object.
struct ChunkState {
  ExtRun carry;   // EXTENDED_ARG run pending at the end of the previous chunk
  u32 n_before;   // records emitted by earlier chunks
  i64 bad_ins;    // first bad jump (instruction index) so far, -1 if none
  i64 bad_off, bad_tgt;
  u32 has_jump;   // some chunk so far holds a jump (is_jump_target marking needed)
};
__device__ __forceinline__ void chunk_state_init(ChunkState& st) {
  st.carry = ExtRun{0, 0, 0};
  st.n_before = 0;
  st.bad_ins = -1;
  st.bad_off = st.bad_tgt = 0;
  st.has_jump = 0;
}

// One warp decodes chunk [base, base+256) units of a <=3.10 object.  Must be
// called by all 32 lanes.  w: this lane's 16 code bytes (units base+8*lane ..
// +8); code: the object's bytes in global memory (only read for jump-target
// checks of objects with EXTENDED_ARG or more than one chunk); tab: this
// version's opcode table in shared memory; stage: 256 records of shared
// memory the chunk's records are written to (the caller stores them out).
// Returns the number of records, or -1 after an UnknownOpcode (res written).
// 3.11 (decode_kernel.cu): `skip` marks this lane's units that lie inside an
// instruction's inline-cache span (neither instructions nor EXTENDED_ARG), and
// `xs` is the object's extent-start bitmap for jump validation (nullptr: the
// <=3.10 rule "in range and the previous unit is not EXTENDED_ARG").
__device__ __forceinline__ int decode_chunk(const u8* __restrict__ code, u32 len, int minor, u32 base,
                                            const u32* __restrict__ tab, upy_ins* stage, uint4 w,
                                            ChunkState& st, upy_decoded* res, u32 skip = 0,
                                            const u32* __restrict__ xs = nullptr) {
  const int lane = threadIdx.x & 31;
  const u32 units = len >> 1;
  const u32 u0 = base + 8 * lane;
  u32 nu = 0;
  if (u0 < units) nu = units - u0 < 8 ? units - u0 : 8;
  const u32 words[4] = {w.x, w.y, w.z, w.w};
#define UNIT_OP(q) ((words[(q) >> 1] >> (16 * ((q) & 1))) & 0xFFu)
#define UNIT_ARG(q) ((words[(q) >> 1] >> (16 * ((q) & 1) + 8)) & 0xFFu)
  // staged entries carry two extra bits (decode_kernel.cu): ENT_JUMP (jump kinds)
  // and ENT_EXT (EXTENDED_ARG); ENT_PAD marks units past the end (defined, inert)
  u32 ent[8];
#pragma unroll
  for (int q = 0; q < 8; q++) ent[q] = (u32)q < nu ? tab[UNIT_OP(q)] : ENT_PAD;
  u32 ext_mask = 0, unknown_mask = 0, jump_mask = 0;
#pragma unroll
  for (int q = 0; q < 8; q++) {
    unknown_mask |= (ent[q] == 0 ? 1u : 0u) << q;
    ext_mask |= ((ent[q] >> ENT_EXT_BIT) & 1u) << q;
    jump_mask |= (ent[q] >> ENT_JUMP_BIT) << q;
  }
  unknown_mask &= ~skip;
  ext_mask &= ~skip;
  jump_mask &= ~skip;
  if (__ballot_sync(0xffffffffu, jump_mask != 0)) st.has_jump = 1;
  // first unknown opcode of the chunk (reference order) stops the object
  u32 has_unknown = __ballot_sync(0xffffffffu, unknown_mask != 0);
  if (has_unknown) {
    int first_lane = __ffs(has_unknown) - 1;
    if (lane == first_lane) {
      int q = __ffs(unknown_mask) - 1;
      res->status = UPY_ST_UNKNOWN_OPCODE;
      res->n_instrs = 0;
      res->aux0 = UNIT_OP(q);
      res->aux1 = 2 * (u0 + q);
    }
    return -1;
  }
  // Fast path (warp-uniform): no EXTENDED_ARG in the chunk and none pending, so
  // every unit is one instruction, lane L's records start at 8*L and need no
  // scans; a single-chunk object with no EXTENDED_ARG also has every even
  // in-range offset as an extent start.
  // (the fast path stores 8 records per lane -- also past the end of the object --
  // as whole uint4 groups: only into a shared-memory staging area, xs == nullptr)
  const bool fast = xs == nullptr && __ballot_sync(0xffffffffu, (ext_mask | skip) != 0) == 0 &&
                    st.carry.len == 0;
  u32 total;
  i64 my_bad = -1, my_bad_off = 0, my_bad_tgt = 0;
  ExtRun inc = {0, 0, 0};
  if (fast) {
    total = units - base < 256 ? units - base : 256;
    uint4* st4 = reinterpret_cast<uint4*>(stage) + 6 * lane;
#pragma unroll
    for (int g = 0; g < 2; g++) {  // 4 records = 12 words = 3 uint4 per group
      u32 wr[12];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int q = 4 * g + r;
        const u32 has_arg = UPY_ENT_HASARG(ent[q]);
        wr[3 * r] = 2 * (u0 + q);
        wr[3 * r + 1] = has_arg ? UNIT_ARG(q) : 0u;
        wr[3 * r + 2] = UNIT_OP(q) | (UPY_ENT_CACHE(ent[q]) << 16) | (has_arg << 24);
      }
#pragma unroll
      for (int k = 0; k < 3; k++) st4[3 * g + k] = make_uint4(wr[4 * k], wr[4 * k + 1], wr[4 * k + 2], wr[4 * k + 3]);
    }
    if (jump_mask) {  // straight-line code skips the jump checks entirely
      const bool no_ext_obj = units <= 256;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        if (((jump_mask >> q) & 1) && my_bad < 0) {
          const u32 u = u0 + q;
          const u32 arg = UPY_ENT_HASARG(ent[q]) ? UNIT_ARG(q) : 0u;
          bool okk;
          i64 t = jump_target_u64(minor, UPY_ENT_KIND(ent[q]), 2ull * u, arg, &okk);
          bool valid = t >= 0 && t < (i64)len && !(t & 1) &&
                       (xs ? ((xs[t >> 6] >> ((t >> 1) & 31)) & 1u) != 0
                           : (no_ext_obj || t == 0 || code[t - 2] != EXT_OP));
          if (!valid) {
            my_bad = st.n_before + 8 * lane + q;
            my_bad_off = 2 * u;
            my_bad_tgt = t;
          }
        }
      }
    }
  } else {
    // no EXTENDED_ARG anywhere in the chunk and none pending (the usual 3.11 case,
    // where only the inline-cache skips keep it off the fast path): no run scan
    const bool noext = __ballot_sync(0xffffffffu, ext_mask != 0) == 0 && st.carry.len == 0;
    ExtRun excl = {0, 0, 0};
    if (!noext) {
    // lane summary of its 8 units
    ExtRun mine;
    {
      u32 valid_mask = nu >= 8 ? 0xFF : ((1u << nu) - 1);
      mine.all = (nu > 0 && (ext_mask & valid_mask) == valid_mask) ? 1 : (nu == 0 ? 1 : 0);
      u32 len_ = 0;
      u64 val = 0;
      bool in_run = true;
#pragma unroll
      for (int q = 7; q >= 0; q--) {
        if ((u32)q >= nu) continue;
        in_run = in_run && ((ext_mask >> q) & 1);
        if (in_run) len_++;
      }
#pragma unroll
      for (int q = 0; q < 8; q++)
        if ((u32)q < nu && (u32)q >= nu - len_) val = (val << 8) | UNIT_ARG(q);
      mine.len = len_;
      mine.val = val;
    }
    // inclusive scan over lanes, then exclusive = shifted
    inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      ExtRun o = shfl_up_run(inc, d);
      if (lane >= d) inc = ext_combine(o, inc);
    }
    excl = shfl_up_run(inc, 1);
    if (lane == 0) excl = ExtRun{1, 0, 0};
    excl = ext_combine(st.carry, excl);
    } else {
      inc = ExtRun{0, 0, 0};
    }
    // instruction slots: non-EXT units before this lane
    u32 my_ins = (u32)__popc((~(ext_mask | skip)) & (nu >= 8 ? 0xFF : ((1u << nu) - 1)));
    u32 pre = my_ins;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u32 o = __shfl_up_sync(0xffffffffu, pre, d);
      if (lane >= d) pre += o;
    }
    total = __shfl_sync(0xffffffffu, pre, 31);
    u32 idx = st.n_before + pre - my_ins;
    u32 run_len = excl.len;  // trailing EXTENDED_ARG run entering my span
    u64 run_val = excl.val;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if ((u32)q >= nu) continue;
      u32 u = u0 + q;
      if ((skip >> q) & 1) continue;  // inline cache unit (3.11)
      if ((ext_mask >> q) & 1) {
        run_val = (run_val << 8) | UNIT_ARG(q);
        run_len++;
        continue;
      }
      u32 e = ent[q];
      bool has_arg = UPY_ENT_HASARG(e);
      u64 ext = run_len ? (run_len >= 8 ? 0 : (run_val << 8)) : 0;
      bool sat = run_len >= 8;
      u64 arg = has_arg ? (UNIT_ARG(q) | ext) : 0;
      bool big = has_arg && (sat || (arg >> 32));
      u32* sw = reinterpret_cast<u32*>(stage) + 3 * (idx - st.n_before);
      u32 off = 2 * (u - run_len);
      sw[0] = off;
      sw[1] = big ? 0xFFFFFFFFu : (u32)arg;
      sw[2] = UNIT_OP(q) | ((run_len > 255 ? 255u : run_len) << 8) | (UPY_ENT_CACHE(e) << 16) |
              (((has_arg ? 1u : 0u) | (big ? 2u : 0u)) << 24);
      u32 kind = UPY_ENT_KIND(e);
      if (my_bad < 0 && (kind == K_JUMP_REL || kind == K_JUMP_ABS || kind == K_JUMP_BACK)) {
        bool okk;
        i64 t = jump_target_u64(minor, kind, 2ull * u, arg, &okk);
        bool valid = !big && t >= 0 && t < (i64)len && !(t & 1) &&
                     (xs ? ((xs[t >> 6] >> ((t >> 1) & 31)) & 1u) != 0 : (t == 0 || code[t - 2] != EXT_OP));
        if (!valid) {
          my_bad = idx;
          my_bad_off = off;
          my_bad_tgt = t;
        }
      }
      idx++;
      run_len = 0;
      run_val = 0;
    }
  }
  // first bad jump of the chunk (lowest instruction index)
  u32 badm = __ballot_sync(0xffffffffu, my_bad >= 0);
  if (badm && st.bad_ins < 0) {
    int bl = __ffs(badm) - 1;
    st.bad_ins = __shfl_sync(0xffffffffu, my_bad, bl);
    st.bad_off = __shfl_sync(0xffffffffu, my_bad_off, bl);
    st.bad_tgt = __shfl_sync(0xffffffffu, my_bad_tgt, bl);
  }
  // carry into the next chunk (a chunk without EXTENDED_ARG leaves no pending run)
  if (fast) st.carry = ExtRun{0, 0, 0};
  else st.carry = ext_combine(st.carry, shfl_run(inc, 31));
#undef UNIT_OP
#undef UNIT_ARG
  return (int)total;
}

// is_jump_target (resolve_jump_targets, disasm.py:166-171): bit2 of every record
// whose extent start is some jump's target.  Warp-cooperative over n records at
// `rec` (shared staging or global memory): pass 1 sets bit (t/2 - unit_lo) of the
// bitmap `bm` (nbits bits, shared memory, cleared here) for every jump target t,
// pass 2 ORs the flag into the records whose offset is marked.  Targets outside
// the bitmap's unit range are ignored (the caller sizes it to the object).  Must
// be called by all 32 lanes after the records are visible to the warp.
__device__ __forceinline__ void mark_jump_targets(upy_ins* rec, u32 n, u32 unit_lo, u32 nbits, int minor,
                                                  const u32* __restrict__ tab, u32* bm) {
  // Both passes load MJ_U records per lane before using any of them, so a warp has
  // 32 * MJ_U record loads in flight instead of 32 (the records of a long object are
  // in global memory: one load round trip per 32 records made C4 decode latency-bound).
  constexpr int MJ_U = 8;
  const int lane = threadIdx.x & 31;
  const u32 nw = (nbits + 31) >> 5;
  for (u32 k = lane; k < nw; k += 32) bm[k] = 0;
  __syncwarp();
  for (u32 base = 0; base < n; base += 32 * MJ_U) {
    u32 w0[MJ_U], w1[MJ_U], w2[MJ_U];
#pragma unroll
    for (int j = 0; j < MJ_U; j++) {
      const u32 k = base + 32 * j + lane;
      const u32* w = reinterpret_cast<const u32*>(rec + (k < n ? k : 0));
      w0[j] = w[0];
      w1[j] = w[1];
      w2[j] = k < n ? w[2] : 0u;
    }
#pragma unroll
    for (int j = 0; j < MJ_U; j++) {
      const u32 e = tab[w2[j] & 0xFFu];
      if (!w2[j] || !((e >> ENT_JUMP_BIT) & 1u) || ((w2[j] >> 24) & 2u)) continue;
      bool ok;
      const i64 t = jump_target_u64(minor, UPY_ENT_KIND(e), (u64)w0[j] + 2ull * ((w2[j] >> 8) & 0xFFu), w1[j], &ok);
      if (t < 0 || (t & 1)) continue;
      const u64 u = (u64)(t >> 1) - unit_lo;
      if ((t >> 1) >= (i64)unit_lo && u < nbits) atomicOr(&bm[u >> 5], 1u << (u & 31));
    }
  }
  __syncwarp();
  for (u32 base = 0; base < n; base += 32 * MJ_U) {
    u32 w0[MJ_U];
#pragma unroll
    for (int j = 0; j < MJ_U; j++) {
      const u32 k = base + 32 * j + lane;
      w0[j] = k < n ? reinterpret_cast<const u32*>(rec + k)[0] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int j = 0; j < MJ_U; j++) {
      if (w0[j] == 0xFFFFFFFFu) continue;
      const u32 u = (w0[j] >> 1) - unit_lo;
      if ((w0[j] >> 1) >= unit_lo && u < nbits && ((bm[u >> 5] >> (u & 31)) & 1u))
        atomicOr(reinterpret_cast<u32*>(rec + base + 32 * j + lane) + 2, 4u << 24);  // RED: no round trip
    }
  }
  __syncwarp();
}

// Same, for objects whose unit range exceeds every shared bitmap: each jump's
// target record is found by binary search over the (offset-sorted) records.
__device__ __forceinline__ void mark_jump_targets_search(upy_ins* rec, u32 n, int minor, const u32* __restrict__ tab) {
  const int lane = threadIdx.x & 31;
  for (u32 k = lane; k < n; k += 32) {
    const u32* w = reinterpret_cast<const u32*>(rec + k);
    const u32 w2 = w[2];
    const u32 e = tab[w2 & 0xFFu];
    if (!((e >> ENT_JUMP_BIT) & 1u) || ((w2 >> 24) & 2u)) continue;
    bool ok;
    const i64 t = jump_target_u64(minor, UPY_ENT_KIND(e), (u64)w[0] + 2ull * ((w2 >> 8) & 0xFFu), w[1], &ok);
    u32 lo = 0, hi = n;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if ((i64)rec[mid].offset < t) lo = mid + 1;
      else hi = mid;
    }
    if (lo < n && (i64)rec[lo].offset == t) atomicOr(reinterpret_cast<u32*>(rec + lo) + 2, 4u << 24);
  }
  __syncwarp();
}

// Final status of a <=3.10 object after its last chunk (reference error order:
// UnknownOpcode / TruncatedCode pre-empt BadJumpTarget).
__device__ __forceinline__ void chunk_finish(u32 len, const ChunkState& st, upy_decoded* res) {
  if (st.carry.len) {  // code ends inside an EXTENDED_ARG run
    res->status = UPY_ST_TRUNCATED_CODE;
    res->n_instrs = 0;
    res->aux0 = 3;
    res->aux1 = len;
  } else if (st.bad_ins >= 0) {
    res->status = UPY_ST_BAD_JUMP_TARGET;
    res->n_instrs = 0;
    res->aux0 = st.bad_off;
    res->aux1 = st.bad_tgt;
  } else {
    res->status = UPY_ST_OK;
    res->n_instrs = (i32)st.n_before;
    res->aux0 = res->aux1 = 0;
  }
}

#endif
