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


// chunks an object streams through the ring (0: handled from global memory).
// 3.8-3.10: any size, decoded chunk by chunk.  3.11: objects of at most
// DSTAGES chunks, which the consumer gathers whole (the inline-cache passes need
// every unit) -- their code is prefetched by TMA while earlier objects decode.
#define X11_RING_BYTES (DSTAGES * 512u)
__device__ __forceinline__ u32 n_chunks(u32 len, u32 minor) {
  if (len == 0 || (len & 1)) return 0;
  if (minor == 11) return len <= X11_RING_BYTES ? (len + 511u) >> 9 : 0;
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
    for (u32 j = 0; j < 32; j++) {
      const i64 o = g * 32 + j;
      if (o >= A.n_objs) break;
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
      if (minor == 11) {
        // all of the object's chunks are (or will be) in the ring: wait for them,
        // gather them into S.out, release the stages and refill the ring before
        // decoding, so the next objects' code is in flight meanwhile
        for (u32 c = 0; c < nch; c++) {
          pump();
          mbar_wait(&S.bar[(cons + c) % DSTAGES], ((cons + c) / DSTAGES) & 1);
        }
        if (lane == 0) bulk_wait_all();  // S.out may still be read by a bulk store
        __syncwarp();
        uint4* buf = reinterpret_cast<uint4*>(&S.out[0][0]);
        for (u32 k = lane; k < nch * 32u; k += 32) buf[k] = S.in[(cons + (k >> 5)) % DSTAGES][k & 31];
        __syncwarp();
        cons += nch;
        pump();
        decode311_body(len, rec, &dec[o], tab[3], S);
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
  i64 blocks = (groups + DWARPS - 1) / DWARPS;
  const i64 max_blocks = (i64)sms * DEC_MINB;
  if (blocks > max_blocks) blocks = max_blocks;
  upy_decode_kernel<<<(unsigned)blocks, DWARPS * 32, 0, s>>>(*arena, ins, dec);
  g_upy_launches += 1;
  return cudaGetLastError();
}
