// decode_kernel.cu -- the sm_100a decode kernel (disasm.py:71-172) and its
// launcher, compiled as its own object so it can be tuned without rebuilding
// the decompile kernel (upy.cu).
//
// HBM-bound streaming design.  Every warp is an independent pipeline over
// groups of 32 consecutive objects (group g = warp, warp + nwarps, ...):
//   * the 32 object headers of the current and the next group sit one per lane
//     (two coalesced header loads per 32 objects), broadcast by shuffles;
//   * code bytes move global -> shared in 512-B chunks (256 units) by TMA bulk
//     copies (cp.async.bulk ... mbarrier::complete_tx) into a DSTAGES-deep ring
//     with one mbarrier per stage; lane 0 keeps the ring DSTAGES chunks ahead of
//     the decoder across object and group boundaries, so several KB per warp
//     are in flight with no registers held for them;
//   * each chunk's records are built in a shared staging buffer (double
//     buffered) and leave as ONE bulk shared -> global copy (cp.async.bulk
//     .global.shared::cta.bulk_group) when the destination is 16-B aligned,
//     else as coalesced 16-B / 4-B stores.
// 3.11 objects (inline caches make instruction starts a serial chain) of up to
// 2 KB come through the same ring whole and are decoded by decode311_body from
// the gathered copy; larger ones are copied synchronously (decode311_warp), and
// anything the warp passes reject goes to the scalar decoder (decode_scalar).
#include <cuda_runtime.h>
#include "decode.h"
#include "tma.h"
#include <atomic>
extern std::atomic<unsigned long long> g_upy_launches;  // upy.cu: upy_launch_count

#define DSTAGES 4
#define DWARPS 4  // warps per block

#define X11_UNITS 3072  // 3.11 objects up to 6 KB of code take the warp path

struct __align__(128) DecWarpSmem {
  uint4 in[DSTAGES][32];    // DSTAGES x 512 B of code
  upy_ins out[2][256];      // 2 x 3 KB of records (3.11: the object's code copy)
  u32 cov[X11_UNITS / 32];  // 3.11: units inside an inline-cache span
  u32 xs[X11_UNITS / 32];   // 3.11: extent starts (jump targets)
  u32 tgt[8];               // jump targets of a one-chunk object (is_jump_target)
  unsigned long long bar[DSTAGES];
};


// chunks an object streams through the ring (0: handled elsewhere).  3.8-3.10:
// any size, decoded chunk by chunk; 3.11 objects go to the lane kernel below or,
// when it rejects them, to decode311_warp.
__device__ __forceinline__ u32 n_chunks(u32 len, u32 minor) {
  if (len == 0 || (len & 1)) return 0;
  if (minor == 11) return 0;  // lane kernel (upy_decode311_lane_kernel) or decode311_warp
  if (minor < 8 || minor > 10) return 0;
  return ((len >> 1) + 255) >> 8;
}

#ifndef DEC_MINB
#define DEC_MINB 5  // 5 x 4 warps per SM at <= 96 registers (no spills): 0.712 ms vs 0.735 ms at 6
#endif
// 3.11: inline caches make instruction starts a serial chain.  The warp copies the
// code into shared memory (coalesced), marks cache-covered units and extent starts
// in two bitmaps with a speculative warp prefix-max scan over cache-span ends
// (pass 1), then decodes the object 256 units at a time with decode_chunk,
// skipping covered units, folding EXTENDED_ARG with the scans and validating jumps
// against the extent-start bitmap; records go straight to global memory.  Any
// decode error or failed speculation sends the object to the scalar
// reference-order decoder (same shared-memory copy), so error semantics are
// decode_scalar's.
// The object's code is in S.out (decode311_warp copies it there from global
// memory; ring objects are gathered from the TMA stages by the kernel).
__device__ __noinline__ void decode311_body(u32 len, upy_ins* __restrict__ rec, upy_decoded* res,
                                            const u32* __restrict__ tab, DecWarpSmem& S) {
  const int lane = threadIdx.x & 31;
  const u32 units = len >> 1;
  uint4* buf = reinterpret_cast<uint4*>(&S.out[0][0]);
  const u32 nwords = (units + 31) / 32;
  for (u32 k = lane; k < nwords; k += 32) S.cov[k] = S.xs[k] = 0;
  __syncwarp();
  const u8* code = reinterpret_cast<const u8*>(buf);
  // Pass 1 (warp-parallel, speculative): every unit's span end = u + cache(op(u));
  // a unit is covered iff an earlier unit's span reaches it (warp prefix-max scan,
  // carried across chunks).  Exact when no covered unit has caches of its own
  // (real cache slots hold CACHE = 0); anything else -- such a conflict, an
  // unknown opcode, caches or an EXTENDED_ARG run past the end -- goes to the
  // scalar decoder, which reports errors in reference order.
  int ok = 1;
  int cmax = -1;          // max span end of earlier chunks
  u32 prev_ext = 0;       // last unit of the previous chunk is an uncovered EXTENDED_ARG
  // Lean path: while no chunk so far has an EXTENDED_ARG or a jump, every uncovered
  // unit is one instruction with a 1-byte arg, so the records are written right here
  // (slots by a warp scan of per-lane counts, staged in S.out[1], copied out as
  // coalesced words) and pass 2 is skipped.  Code up to 3 KB sits in S.out[0].
  bool lean = len <= 3072u;
  u32 n_lean = 0;
  for (u32 base = 0; base < units; base += 256) {
    const u32 u0 = base + 8 * lane;
    u32 nu = 0;
    if (u0 < units) nu = units - u0 < 8 ? units - u0 : 8;
    const uint4 w = u0 < units ? buf[u0 >> 3] : make_uint4(0, 0, 0, 0);
    const u32 words[4] = {w.x, w.y, w.z, w.w};
    int se[8];
    u32 ent[8];
    int lane_max = -1;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const u32 op = (words[q >> 1] >> (16 * (q & 1))) & 0xFFu;
      ent[q] = (u32)q < nu ? tab[op] : ENT_PAD;
      se[q] = (u32)q < nu ? (int)(u0 + q + UPY_ENT_CACHE(ent[q])) : -1;
      lane_max = se[q] > lane_max ? se[q] : lane_max;
    }
    int inc = lane_max;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc = o > inc ? o : inc;
    }
    int run = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) run = -1;
    run = run > cmax ? run : cmax;
    u32 cov_bits = 0, xs_bits = 0, bad = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if ((u32)q >= nu) continue;
      const int u = (int)(u0 + q);
      const bool covered = run >= u;
      if (covered) {
        cov_bits |= 1u << q;
        if (se[q] > u) bad = 1;                              // a cache slot with caches
      } else {
        if (!ent[q]) bad = 1;                                // unknown opcode
        if (se[q] >= (int)units) bad = 1;                    // caches past the end
      }
      run = se[q] > run ? se[q] : run;
    }
    // extent starts: uncovered units not preceded by an uncovered EXTENDED_ARG
    const u32 ext_bits = [&] {
      u32 m = 0;
#pragma unroll
      for (int q = 0; q < 8; q++)
        if ((u32)q < nu && !((cov_bits >> q) & 1u) && ((ent[q] >> ENT_EXT_BIT) & 1u)) m |= 1u << q;
      return m;
    }();
    u32 prev_last = __shfl_up_sync(0xffffffffu, (ext_bits >> 7) & 1u, 1);
    if (lane == 0) prev_last = prev_ext;
    const u32 prev_of = ((ext_bits << 1) | prev_last) & 0xFFu;  // bit q: unit q-1 is an uncovered EXT
    xs_bits = ~cov_bits & ~prev_of & (nu >= 8 ? 0xFFu : ((1u << nu) - 1));
    if (u0 < units) {
      reinterpret_cast<u8*>(S.cov)[u0 >> 3] = (u8)cov_bits;
      reinterpret_cast<u8*>(S.xs)[u0 >> 3] = (u8)xs_bits;
    }
    if (__ballot_sync(0xffffffffu, bad)) {
      ok = 0;
      break;
    }
    if (lean) {
      const u32 inst = ~cov_bits & (nu >= 8 ? 0xFFu : ((1u << nu) - 1));
      u32 jmp = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) jmp |= ((inst >> q) & (ent[q] >> ENT_JUMP_BIT) & 1u) << q;
      if (__ballot_sync(0xffffffffu, ext_bits | jmp) != 0) {
        lean = false;  // pass 2 redoes the object from its first record
      } else {
        const u32 cnt = (u32)__popc(inst);
        u32 incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += o;
        }
        const u32 total = __shfl_sync(0xffffffffu, incl, 31);
        u32* sw = reinterpret_cast<u32*>(&S.out[1][0]) + 3 * (incl - cnt);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if (!((inst >> q) & 1u)) continue;
          const u32 unit = (words[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
          const u32 has_arg = UPY_ENT_HASARG(ent[q]);
          sw[0] = 2 * (u0 + q);
          sw[1] = has_arg ? (unit >> 8) : 0u;
          sw[2] = (unit & 0xFFu) | (UPY_ENT_CACHE(ent[q]) << 16) | (has_arg << 24);
          sw += 3;
        }
        __syncwarp();
        const u32* src = reinterpret_cast<const u32*>(&S.out[1][0]);
        u32* dst = reinterpret_cast<u32*>(rec + n_lean);
        for (u32 k = lane; k < 3 * total; k += 32) dst[k] = src[k];
        __syncwarp();
        n_lean += total;
      }
    }
    cmax = __shfl_sync(0xffffffffu, inc, 31);
    prev_ext = __shfl_sync(0xffffffffu, (ext_bits >> 7) & 1u, 31);
  }
  if (ok && lean) {  // no EXTENDED_ARG, so no run can reach the end; no jumps to mark
    if (lane == 0) {
      res->status = UPY_ST_OK;
      res->n_instrs = (i32)n_lean;
      res->aux0 = res->aux1 = 0;
    }
    __syncwarp();
    return;
  }
  // an EXTENDED_ARG run reaching the end of the code: the scalar decoder's error
  __syncwarp();
  if (ok) {
    const u32 last = units - 1;
    const bool end_ext = !((S.cov[last >> 5] >> (last & 31)) & 1u) && code[2 * last] == EXT_OP;
    if (end_ext) ok = 0;
  }
  __syncwarp();
  if (!ok) {
    if (lane == 0) decode_scalar(code, len, 11, rec, res);
    __syncwarp();
    return;
  }
  ChunkState st;
  chunk_state_init(st);
  for (u32 base = 0; base < units; base += 256) {
    const u32 u0 = base + 8 * lane;
    uint4 w = make_uint4(0, 0, 0, 0);
    u32 skip = 0;
    if (u0 < units) {
      w = buf[u0 >> 3];
      skip = (S.cov[u0 >> 5] >> (u0 & 31)) & 0xFFu;
    }
    const int total = decode_chunk(code, len, 11, base, tab, rec + st.n_before, w, st, res, skip, S.xs);
    if (total < 0) {  // cannot happen after pass 1 (unknown opcodes are caught there)
      if (lane == 0) decode_scalar(code, len, 11, rec, res);
      __syncwarp();
      return;
    }
    st.n_before += (u32)total;
  }
  // is_jump_target: the cache-cover bitmap is dead now and spans the object
  if (st.has_jump && st.carry.len == 0 && st.bad_ins < 0) {
    __syncwarp();
    mark_jump_targets(rec, st.n_before, 0, units, 11, tab, S.cov);
  }
  if (lane == 0) chunk_finish(len, st, res);
  __syncwarp();
}

// 3.11 objects too large for the ring (up to X11_UNITS units): a coalesced
// synchronous copy into S.out, then the same passes.
__device__ __noinline__ void decode311_warp(const u8* __restrict__ gcode, u32 len, upy_ins* __restrict__ rec,
                                            upy_decoded* res, const u32* __restrict__ tab, DecWarpSmem& S) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) bulk_wait_all();  // the staging buffers are about to hold the code
  __syncwarp();
  uint4* buf = reinterpret_cast<uint4*>(&S.out[0][0]);
  const uint4* src = reinterpret_cast<const uint4*>(gcode);
  for (u32 k = lane; k < (len + 15) / 16; k += 32) buf[k] = src[k];
  __syncwarp();
  decode311_body(len, rec, res, tab, S);
}


// ---------------------------------------------------------------------------
// 3.11, lane-serial (upy_decode311_lane_kernel, launched before the main kernel).
// In 3.11 the instruction starts are a serial chain (each instruction skips its
// inline-cache units), so the cheapest exact decoder is the reference's own walk
// (disasm.py:71-122) run by ONE LANE PER OBJECT.  Lanes are independent: lane L
// of warp w walks objects 32*g + L for the warp's groups g = w, w + nw, ...,
// eight units (one 16-B load, prefetched two steps ahead) per step, and takes
// its next object as soon as one ends, so the warp never waits for its longest
// object.  Records are packed one word each into the lane's shared row
// (unit index 11 b | code unit 16 b | cache count 4 b | has_arg 1 b -- objects
// of at most 2048 units); rows that are nearly full, or whose object ended, are
// expanded and copied out by the whole warp (one lane's row at a time, lane t
// writing record t: coalesced).
// The walk covers the common case only -- no EXTENDED_ARG, no jumps, every
// opcode known, no cache run past the end.  A lane that meets anything else marks
// its object L11_REDO and the main kernel, which runs next, decodes it from
// scratch with decode311_warp (error reporting in decode_scalar's reference
// order).  For the objects it keeps, the records are exactly decode_scalar's:
// offset = 2u, arg = the arg byte when the opcode has an argument, n_prefixes 0,
// cache_units, flags = has_arg (no jump targets: there are no jumps).
#define L11_MAX 4096u   // bytes of code (2048 units: the packed row word's 11-bit unit index)
#ifndef L11_ROUND
#define L11_ROUND 8     // instructions per lane per round (refill, flush check once per round)
#endif
#ifndef L11_FLUSH
#define L11_FLUSH 32u   // records per row flush while an object runs (one full store round; 16: 1.47 ms vs 1.20)
#endif
#define L11_R (L11_FLUSH + L11_ROUND) // records per lane row: one flush + one round (row stride L11_R + 1)
#define L11_RING 128u   // code units per lane ring (a power of two)
#define L11_CHUNK 16u   // units per ring refill (one cp.async group)
#define L11_AHEAD 112u  // units kept buffered ahead of the walk: L11_RING - L11_CHUNK
#define L11_PRE 8u      // 16-B pieces of the next object held in registers (its first 64 units)
#define L11_WARPS 2     // warps per block
#define L11_REDO 0x7ffffff0  // dec status: the main kernel decodes the object
#ifndef L11_MINB
#define L11_MINB 8      // blocks per SM (~28 KB of shared memory each; 64-unit ring: 2.06 ms, 256: 1.97 ms, 128: 1.55 ms)
#endif
// opcode entry of the walk: bits 0-3 cache count, bit 4 reject (unknown opcode,
// EXTENDED_ARG, jump), bits 27-30 cache count and bit 31 has_arg (the packed
// record's fields, in place)
#define L11_REJECT (1u << 4)

// the lane kernel takes a 3.11 object iff this holds
__device__ __forceinline__ bool l11_eligible(u32 len, const upy_ins* rec) {
  return len && !(len & 1) && len <= L11_MAX && (reinterpret_cast<uintptr_t>(rec) & 15) == 0;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, u32 src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait3() { asm volatile("cp.async.wait_group 3;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait2() { asm volatile("cp.async.wait_group 2;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void sts_if(bool p, u32* a, u32 v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.shared.u32 [%1], %2;\n}\n" ::"r"((u32)p),
               "r"(smem_addr(a)), "r"(v)
               : "memory");
}

__global__ void __launch_bounds__(L11_WARPS * 32, L11_MINB) upy_decode311_lane_kernel(upy_arena A,
                                                                                      upy_ins* __restrict__ ins,
                                                                                      upy_decoded* __restrict__ dec) {
  __shared__ u32 tab[256];
  __shared__ u32 rows_all[L11_WARPS][32][L11_R + 1];  // odd stride: lane L's word k in bank (L + k) % 32
  __shared__ __align__(16) u8 ring_all[L11_WARPS][32][L11_RING * 2];  // per-lane code ring
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const u32 e = UPY_OPTABLE_DEV[3][i];
    const u32 k = UPY_ENT_KIND(e);
    const u32 cache = UPY_ENT_CACHE(e);
    const bool reject = !e || i == EXT_OP || k == K_JUMP_REL || k == K_JUMP_ABS || k == K_JUMP_BACK;
    tab[i] = cache | (reject ? L11_REJECT : 0u) | (cache << 27) | ((u32)UPY_ENT_HASARG(e) << 31);
  }
  __syncthreads();
  u32* const row = rows_all[wid][lane];
  u8* const ring = ring_all[wid][lane];
  const i64 nw = (i64)gridDim.x * L11_WARPS;
  const i64 n_groups = (A.n_objs + 31) >> 5;
  i64 g = (i64)blockIdx.x * L11_WARPS + wid;  // the lane's next group
  // A warp whose groups hold no 3.11 object leaves at once: one coalesced minor read
  // per lane per group, four groups per round trip (a 3.8-3.10 batch costs the kernel
  // a few microseconds instead of a dependent header walk per lane).
  {
    bool any = false;
    for (i64 g0 = g; g0 < n_groups && !any; g0 += 4 * nw) {
      u32 m[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const i64 c = (g0 + j * nw) * 32 + lane;
        m[j] = (g0 + j * nw < n_groups && c < A.n_objs) ? A.objs[c].minor : 0u;
      }
      any = __any_sync(0xffffffffu, m[0] == 11 || m[1] == 11 || m[2] == 11 || m[3] == 11);
    }
    if (!any) return;
  }
  // Objects move through two prefetch stages so that no load is waited on when a
  // lane switches objects: the header of the lane's next candidate (h*) and the
  // next eligible object with its first 128 code bytes (n*), both loaded one whole
  // object walk before they are needed.
  i64 hc = -1;
  u64 hoff = 0;
  u32 hlen = 0, hmin = 0;
  auto load_hdr = [&]() {
    hc = -1;
    while (g < n_groups) {
      const i64 c = g * 32 + lane;
      g += nw;
      if (c < A.n_objs) {
        const upy_obj* ob = &A.objs[c];
        hc = c;
        hoff = ob->code_off;
        hlen = ob->code_len;
        hmin = ob->minor;
        break;
      }
    }
  };
  i64 no = -1;
  u64 noff = 0;
  u32 nunits = 0;
  uint4 nx[L11_PRE];  // the next object's first L11_PRE * 8 code units
  auto advance_next = [&]() {
    no = -1;
    while (hc >= 0) {
      const i64 c = hc;
      const u64 off = hoff;
      const u32 len = hlen, mn = hmin;
      load_hdr();
      if (mn == 11 && l11_eligible(len, ins + (off >> 1))) {
        no = c;
        noff = off;
        nunits = len >> 1;
        const uint4* cp = reinterpret_cast<const uint4*>(A.bytes + off);
#pragma unroll
        for (int k = 0; k < (int)L11_PRE; k++)
          if (8u * k < nunits) nx[k] = cp[k];
        break;
      }
    }
  };
  load_hdr();
  advance_next();

  // the lane's current object; its code units [F - L11_RING, F) sit in the ring at
  // index u % L11_RING, the newest chunks possibly still in flight (cp.async)
  i64 o = -1;
  const u8* code = nullptr;
  upy_ins* rec = nullptr;
  u32 units = 0, u = 0, cnt = 0, nout = 0, F = 0, lim = 0;
  bool ok = false;
  // refill: the next chunk of code units behind F (zero-filled past the object's
  // readable 16-B-rounded end)
  auto refill = [&]() {
#pragma unroll
    for (int k = 0; k < L11_CHUNK / 8; k++) {
      const u32 p = 2u * (F + 8u * k);
      cp_async16(ring + 2u * ((F + 8u * k) & (L11_RING - 1)), code + (p < lim ? p : 0u), p < lim ? 16u : 0u);
    }
    cp_async_commit();
    F += L11_CHUNK;
  };
  for (;;) {
    if (o < 0 && no >= 0) {
      cp_async_wait0();  // the previous object's ring writes
      o = no;
      code = A.bytes + noff;
      rec = ins + (noff >> 1);
      units = nunits;
      lim = (2u * units + 15u) & ~15u;
      uint4* rq = reinterpret_cast<uint4*>(ring);
#pragma unroll
      for (int k = 0; k < (int)L11_PRE; k++) rq[k] = nx[k];
      F = 8 * L11_PRE;
      u = cnt = nout = 0;
      ok = true;
      advance_next();
    }
    if (!__any_sync(0xffffffffu, o >= 0)) break;
    // Ring refill, once per round: keep L11_AHEAD units behind the walk issued, then
    // wait only for the chunk holding unit u (the walk reads the opcode unit of each
    // instruction, never its cache units); newer chunks stay in flight (<= 3) and
    // an instruction whose opcode unit is not in shared memory yet (u >= V) waits
    // for the next round.
    u32 V = 0;
    if (o >= 0 && ok && u < units) {
      while (F < u + L11_AHEAD && F < units) refill();
      const u32 pend = min((F - u - 1) / L11_CHUNK, 3u);
      if (pend == 3) cp_async_wait3();
      else if (pend == 2) cp_async_wait2();
      else if (pend == 1) cp_async_wait1();
      else cp_async_wait0();
      V = F - L11_CHUNK * pend;
    }
    // L11_ROUND instructions per lane: read the unit at u, look its opcode up, append
    // the packed record, jump over the instruction's cache units
#pragma unroll
    for (int k = 0; k < L11_ROUND; k++) {
      const bool live = o >= 0 && ok && u < units && u < V;
      const u32 unit = *reinterpret_cast<const unsigned short*>(ring + 2u * (u & (L11_RING - 1)));
      const u32 e = tab[unit & 0xFFu];
      const u32 cache = e & 15u;
      const bool bad = (e & L11_REJECT) || u + 1 + cache > units;
      const bool emit = live && !bad;
      sts_if(emit, row + cnt, u | (unit << 11) | (e & 0xF8000000u));
      cnt += emit;
      u += live ? 1 + cache : 0u;
      ok = ok && !(live && bad);
    }
    const bool done = o >= 0 && (!ok || u >= units);
    // rows holding L11_FLUSH records, or whose object ended, go out, expanded to upy_ins
    // records: 32 at a time (one full store round per row) while the object runs,
    // everything at its end
    const u32 fc = done ? cnt : L11_FLUSH;
    u32 who = __ballot_sync(0xffffffffu, ok && cnt && (done || cnt >= L11_FLUSH));
    if (who) {
      __syncwarp();
      const u32 mine = who;
      while (who) {
        const int L = __ffs(who) - 1;
        who &= who - 1;
        const u32 c = __shfl_sync(0xffffffffu, fc, L);
        const u32 base = __shfl_sync(0xffffffffu, nout, L);
        upy_ins* dst = reinterpret_cast<upy_ins*>(__shfl_sync(0xffffffffu, reinterpret_cast<u64>(rec), L)) + base;
        const u32* src = rows_all[wid][L];
        for (u32 t = lane; t < c; t += 32) {
          const u32 p = src[t];
          const u32 has = p >> 31;
          u32* d = reinterpret_cast<u32*>(dst + t);
          d[0] = 2u * (p & 0x7FFu);
          d[1] = has ? (p >> 19) & 0xFFu : 0u;
          d[2] = ((p >> 11) & 0xFFu) | (((p >> 27) & 15u) << 16) | (has << 24);
        }
      }
      __syncwarp();
      if ((mine >> lane) & 1u) {
        for (u32 k = fc; k < cnt; k++) row[k - fc] = row[k];  // the records past the flushed ones
        nout += fc;
        cnt -= fc;
      }
    }
    if (done) {
      upy_decoded* r = &dec[o];
      r->status = ok ? UPY_ST_OK : L11_REDO;
      r->n_instrs = ok ? (i32)nout : 0;
      r->aux0 = r->aux1 = 0;
      o = -1;
    }
  }
}

__global__ void __launch_bounds__(DWARPS * 32, DEC_MINB) upy_decode_kernel(upy_arena A, upy_ins* __restrict__ ins,
                                                                    upy_decoded* __restrict__ dec) {
  __shared__ u32 tab[4][256];  // 3.8-3.11 opcode tables
  __shared__ DecWarpSmem wsm[DWARPS];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  DecWarpSmem& S = wsm[wid];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
    u32 e = UPY_OPTABLE_DEV[i >> 8][i & 255];
    if (e) {
      const u32 k = UPY_ENT_KIND(e);
      if (k == K_JUMP_REL || k == K_JUMP_ABS || k == K_JUMP_BACK) e |= 1u << ENT_JUMP_BIT;
      if ((i & 255) == EXT_OP) e |= 1u << ENT_EXT_BIT;
    }
    tab[i >> 8][i & 255] = e;
  }
  if (lane == 0) {
    for (int s = 0; s < DSTAGES; s++) mbar_init(&S.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const i64 nw = (i64)gridDim.x * DWARPS;
  const i64 n_groups = (A.n_objs + 31) >> 5;
  i64 g = (i64)blockIdx.x * DWARPS + wid;
  if (g >= n_groups) return;

  // headers: lane j holds object 32*group + j of the current (c) and next (n) group
  auto load_hdr = [&](i64 grp, u64& off, u32& len, u32& minor) {
    i64 o = grp * 32 + lane;
    if (grp < n_groups && o < A.n_objs) {
      const upy_obj* ob = &A.objs[o];
      off = ob->code_off;
      len = ob->code_len;
      minor = ob->minor;
    } else {
      off = 0;
      len = 0;
      minor = 0;
    }
  };
  u64 c_off, n_off;
  u32 c_len, c_min, n_len, n_min;
  load_hdr(g, c_off, c_len, c_min);
  load_hdr(g + nw, n_off, n_len, n_min);

  // producer cursor (warp-uniform): group selector (0 current, 1 next, 2 none),
  // object within the group, chunk within the object
  u32 psel = 0, pj = 0, pc = 0;
  u32 prod = 0, cons = 0;  // chunks issued / consumed
  auto pump = [&]() {
    while (prod < cons + DSTAGES && psel < 2) {
      const i64 grp = g + (i64)psel * nw;
      const i64 o = grp * 32 + pj;
      if (grp >= n_groups || o >= A.n_objs) {
        psel = 2;
        break;
      }
      const u64 off = __shfl_sync(0xffffffffu, psel ? n_off : c_off, pj);
      const u32 len = __shfl_sync(0xffffffffu, psel ? n_len : c_len, pj);
      const u32 minor = __shfl_sync(0xffffffffu, psel ? n_min : c_min, pj);
      const u32 nch = n_chunks(len, minor);
      if (pc < nch) {
        const u32 s = prod % DSTAGES;
        const u32 start = pc * 512u;
        u32 bytes = len - start < 512u ? len - start : 512u;
        bytes = (bytes + 15u) & ~15u;  // code is readable to the next 16-B boundary (upy.h)
        if (lane == 0) {
          fence_async_smem();
          mbar_expect_tx(&S.bar[s], bytes);
          bulk_g2s(&S.in[s][0], A.bytes + off + start, bytes, &S.bar[s]);
        }
        prod++;
        pc++;
      }
      if (pc >= nch) {
        pc = 0;
        if (++pj == 32) {
          pj = 0;
          psel++;
        }
      }
    }
  };

  u32 ob = 0;  // output staging buffer toggle
  for (; g < n_groups; g += nw) {
    // objects of this group the lane kernel already decoded (one coalesced status read)
    const i64 ol = g * 32 + lane;
    const bool l11_done = ol < A.n_objs && c_min == 11 && l11_eligible(c_len, ins + (c_off >> 1)) &&
                          dec[ol].status != L11_REDO;
    const u32 todo = ~__ballot_sync(0xffffffffu, l11_done);
    for (u32 j = 0; j < 32; j++) {
      const i64 o = g * 32 + j;
      if (o >= A.n_objs) break;
      if (!((todo >> j) & 1u)) continue;
      const u64 off = __shfl_sync(0xffffffffu, c_off, j);
      const u32 len = __shfl_sync(0xffffffffu, c_len, j);
      const u32 minor = __shfl_sync(0xffffffffu, c_min, j);
      const u32 nch = n_chunks(len, minor);
      upy_ins* rec = ins + (off >> 1);
      if (nch == 0) {
        if (minor == 11 && len && !(len & 1) && len <= 2 * X11_UNITS) {
          decode311_warp(A.bytes + off, len, rec, &dec[o], tab[3], S);
          continue;
        }
        if (lane == 0) {
          if (minor == 11 || ((minor >= 8 && minor <= 10) && (len == 0 || (len & 1)))) {
            decode_scalar(A.bytes + off, len, (int)minor, rec, &dec[o]);
          } else {
            dec[o].status = UPY_ST_INTERNAL;
            dec[o].n_instrs = 0;
            dec[o].aux0 = dec[o].aux1 = 0;
          }
        }
        continue;
      }
      ChunkState st;
      chunk_state_init(st);
      bool stopped = false;
      for (u32 c = 0; c < nch; c++) {
        pump();
        const u32 s = cons % DSTAGES;
        mbar_wait(&S.bar[s], (cons / DSTAGES) & 1);
        if (!stopped) {
          const uint4 w = S.in[s][lane];
          // the staging buffer was last stored out two chunks ago: its bulk read must be done
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
          upy_ins* stage = S.out[ob];
          const int total = decode_chunk(A.bytes + off, len, (int)minor, c * 256u, tab[minor - 8], stage, w, st, &dec[o]);
          if (total < 0) {
            stopped = true;
          } else {
            __syncwarp();
            // is_jump_target of a one-chunk object: marked in the staging area
            if (nch == 1 && st.has_jump && st.bad_ins < 0)
              mark_jump_targets(stage, (u32)total, 0, 256, (int)minor, tab[minor - 8], S.tgt);
            upy_ins* dst = rec + st.n_before;
            // bulk store: 16-B aligned destination, size rounded up to 16 B -- only on
            // the object's last chunk (the overshoot, < 16 B, stays inside this object's
            // record slots, which extend to 6 * round16(len) bytes) or when exact, so an
            // async store never overlaps a later chunk's records
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (c + 1 == nch || (total & 3) == 0)) {
              if (lane == 0) {
                fence_async_smem();
                bulk_s2g(dst, stage, ((u32)total * 12u + 15u) & ~15u);
              }
              ob ^= 1;
            } else {
              const u32 nwd = 3u * (u32)total;
              u32* d = reinterpret_cast<u32*>(dst);
              const u32* sw = reinterpret_cast<const u32*>(stage);
              for (u32 k = lane; k < nwd; k += 32) d[k] = sw[k];
              __syncwarp();
            }
            st.n_before += (u32)total;
          }
        }
        __syncwarp();
        cons++;
      }
      if (!stopped && nch > 1 && st.has_jump && st.carry.len == 0 && st.bad_ins < 0) {
        // is_jump_target of a multi-chunk object: targets may lie in chunks already
        // stored out, so mark once the object's records are all in global memory
        // (the staging buffers, idle now, hold the object's target bitmap)
        if (lane == 0) {
          bulk_wait_all();
          fence_async_global();
        }
        __syncwarp();
        const u32 units = len >> 1;
        if (units <= (u32)sizeof(S.out) * 8)
          mark_jump_targets(rec, st.n_before, 0, units, (int)minor, tab[minor - 8],
                            reinterpret_cast<u32*>(&S.out[0][0]));
        else
          mark_jump_targets_search(rec, st.n_before, (int)minor, tab[minor - 8]);
      }
      if (!stopped && lane == 0) chunk_finish(len, st, &dec[o]);
    }
    // shift the header window; the producer cursor moves down one group
    c_off = n_off, c_len = n_len, c_min = n_min;
    load_hdr(g + 2 * nw, n_off, n_len, n_min);
    if (psel > 0) psel--;
  }
  if (lane == 0) bulk_wait_all();
}

// Launcher used by upy_decode_batch (upy.cu); returns the launch error.
// Grid: at most 6 resident blocks of 4 warps per SM, one warp per 32-object group.
cudaError_t upy_decode_launch(const upy_arena* arena, upy_ins* ins, upy_decoded* dec, cudaStream_t s, int sms) {
  const i64 groups = (arena->n_objs + 31) / 32;
  // 3.11 objects first (a batch without any costs one pass over the object headers);
  // the main kernel then decodes everything else, including the objects the lane
  // walk handed back (L11_REDO)
  i64 lblocks = (groups + L11_WARPS - 1) / L11_WARPS;
  const i64 lmax = (i64)sms * L11_MINB;
  if (lblocks > lmax) lblocks = lmax;
  upy_decode311_lane_kernel<<<(unsigned)lblocks, L11_WARPS * 32, 0, s>>>(*arena, ins, dec);
  g_upy_launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  i64 blocks = (groups + DWARPS - 1) / DWARPS;
  const i64 max_blocks = (i64)sms * DEC_MINB;
  if (blocks > max_blocks) blocks = max_blocks;
  upy_decode_kernel<<<(unsigned)blocks, DWARPS * 32, 0, s>>>(*arena, ins, dec);
  g_upy_launches += 1;
  return cudaGetLastError();
}
