// stackscan_kernel.cu -- the stack-depth scan (stackscan.h; SURVEY Appendix A;
// north-star subsystem 3) on sm_100a.
//
// HBM-bound streaming kernel over the decode kernel's records: one warp per
// group of 32 consecutive objects (headers loaded one per lane, summaries stored
// one per lane), one object at a time, 256 instructions per warp step,
// 8 consecutive instructions per lane.  A lane loads its 8 records (96 B) as six
// 16-B streaming loads (record runs start 96-B aligned: code_off is 16-B aligned
// and the records of unit u live at code_off/2 + u), evaluates each effect from a
// per-(version, opcode) descriptor table in shared memory (branch-free; the
// descriptors are derived from the reference-order switch, stackscan.h), scans
// its 8 values in registers with segment resets, and the warp combines the 32
// lane aggregates with a segmented shuffle scan carried across steps.  Each lane
// writes its 8 upy_stackrec (32 B) as two 16-B streaming stores.  An object's
// first 256 records arrive in a per-warp shared-memory stage by one TMA bulk copy
// (cp.async.bulk + mbarrier) issued while the previous object is scanned, so the
// load latency of short objects (C3: ~200 records) is hidden.  Segment starts
// need "the previous instruction ends a block": from lane - 1 by shuffle, or from
// the previous step.
//
// Algorithmic bytes per object: 12 B x N_instr read + 4 B x N_instr written
// + the object's decode result (24 B) and summary (24 B) + its code_off (8 B).
#include <cuda_runtime.h>
#include "stackscan.h"
#include "tma.h"
#include <atomic>
extern std::atomic<unsigned long long> g_upy_launches;  // upy.cu: upy_launch_count

#define SS_WARPS 8  // 8 x 3 KB record stages + 4 KB descriptor table per block
#ifndef SS_MINB
#define SS_MINB 4  // 4 x 8 warps per SM at <= 64 registers
#endif

__global__ void __launch_bounds__(SS_WARPS * 32, SS_MINB)
    upy_stackscan_kernel(upy_arena A, const upy_ins* __restrict__ ins, const upy_decoded* __restrict__ dec,
                         upy_stackrec* __restrict__ out, upy_stackinfo* __restrict__ info, int gshift) {
  __shared__ u32 tab[4][256];
  // per warp: one 256-record stage the next object's first step lands in by TMA
  // while the current object is scanned from registers
  __shared__ __align__(128) upy_ins stage[SS_WARPS][256];
  __shared__ unsigned long long bar[SS_WARPS];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
    tab[i >> 8][i & 255] = stack_desc(8 + (i >> 8), UPY_OPTABLE_DEV[i >> 8][i & 255]);
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  if (lane == 0) {
    mbar_init(&bar[wid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  u32 phase = 0;
  auto prefetch = [&](u64 rbase, u32 n) {  // lane 0: the object's first <= 256 records
    if (lane == 0) {
      const u32 bytes = ((n < 256 ? n : 256) * 12u + 15u) & ~15u;
      fence_async_smem();
      mbar_expect_tx(&bar[wid], bytes);
      bulk_g2s(&stage[wid][0], ins + rbase, bytes, &bar[wid]);
    }
  };
  const i64 nw = (i64)gridDim.x * SS_WARPS;
  const int gsize = 1 << gshift;  // objects per group (32 for short objects, fewer for long)
  const i64 n_groups = (A.n_objs + gsize - 1) >> gshift;
  // groups of 32 consecutive objects per warp: lane j loads object j's decode
  // result and code offset (one round of loads per 32 objects), the warp scans the
  // objects one after another, and lane j keeps object j's summary for one
  // coalesced store at the end of the group
  for (i64 g = (i64)blockIdx.x * SS_WARPS + (threadIdx.x >> 5); g < n_groups; g += nw) {
    const i64 my_o = g * gsize + lane;
    int h_status = UPY_ST_INTERNAL, h_n = 0;
    u64 h_base = 0;
    u32 h_minor = 8;
    if (lane < gsize && my_o < A.n_objs) {
      const upy_decoded d = dec[my_o];
      h_status = d.status;
      h_n = d.n_instrs;
      h_base = A.objs[my_o].code_off >> 1;
      h_minor = A.objs[my_o].minor;
    }
    upy_stackinfo mine;
    mine.status = h_status;
    mine.n_segments = mine.max_depth = mine.min_depth = mine.n_pushes = mine.n_unknown = 0;
    // objects of the group with records, and the first one's prefetch
    u32 todo = __ballot_sync(0xffffffffu, h_status == UPY_ST_OK && h_n > 0);
    if (todo) {
      const int f = __ffs((int)todo) - 1;
      prefetch(__shfl_sync(0xffffffffu, h_base, f), (u32)__shfl_sync(0xffffffffu, h_n, f));
    }
    while (todo) {
      const int j = __ffs((int)todo) - 1;
      todo &= todo - 1;
      const u32 n = (u32)__shfl_sync(0xffffffffu, h_n, j);
      const u64 base = __shfl_sync(0xffffffffu, h_base, j);
      const u32* tb = tab[(__shfl_sync(0xffffffffu, h_minor, j) - 8) & 3];
      const upy_ins* rec = ins + base;
      upy_stackrec* dst = out + base;
      // carry from the previous step: inclusive (sum, unknown) at its last
      // instruction, and whether that instruction ends a block
      int c_sum = 0, c_unk = 0, c_end = 0;
      int segs = 0, unks = 0, pushes = 0, mx = 0, mn = 0;
      for (u32 t0 = 0; t0 < n; t0 += 256) {
        const u32 i0 = t0 + 8 * (u32)lane;
        const u32 cnt = i0 < n ? (n - i0 < 8 ? n - i0 : 8) : 0;
        u32 w[24];  // 8 records x (offset, arg, opcode | prefixes | caches | flags)
        if (t0 == 0) {
          // first step: from the TMA stage; then the stage takes the next object's
          mbar_wait(&bar[wid], phase);
          phase ^= 1;
          const u32* sp = reinterpret_cast<const u32*>(&stage[wid][8 * lane]);
          if (cnt == 8) {
            const uint4* p4 = reinterpret_cast<const uint4*>(sp);
#pragma unroll
            for (int k = 0; k < 6; k++) {
              const uint4 v = p4[k];
              w[4 * k] = v.x, w[4 * k + 1] = v.y, w[4 * k + 2] = v.z, w[4 * k + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 24; k++) w[k] = (u32)(k / 3) < cnt ? sp[k] : 0u;
          }
          __syncwarp();
          if (todo) {
            const int nx = __ffs((int)todo) - 1;
            prefetch(__shfl_sync(0xffffffffu, h_base, nx), (u32)__shfl_sync(0xffffffffu, h_n, nx));
          }
        } else if (cnt == 8) {
          const uint4* p = reinterpret_cast<const uint4*>(rec + i0);
#pragma unroll
          for (int k = 0; k < 6; k++) {
            const uint4 v = __ldcs(p + k);
            w[4 * k] = v.x, w[4 * k + 1] = v.y, w[4 * k + 2] = v.z, w[4 * k + 3] = v.w;
          }
        } else {
          const u32* p = reinterpret_cast<const u32*>(rec + i0);
#pragma unroll
          for (int k = 0; k < 24; k++) w[k] = (u32)(k / 3) < cnt ? p[k] : 0u;
        }
        int sums[8];
        u32 segm = 0, unkm = 0, endm = 0;
        u32 descs[8];
        u32 rare = 0;  // arg terms other than none / n (popcount, bit tests, UNPACK_EX)
#pragma unroll
        for (int q = 0; q < 8; q++) {
          descs[q] = tb[w[3 * q + 2] & 0xFF];
          rare |= ((descs[q] >> 8) & 7u) > SD_N;
        }
        const bool common = !__any_sync(0xffffffffu, rare);  // warp-uniform
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const u32 arg = w[3 * q + 1], meta = w[3 * q + 2];
          const u32 desc = descs[q];
          const bool valid = (u32)q < cnt;
          int eff;
          if (common) {  // base + mul * min(arg, 0x7FFF) (mul is 0 for term "none")
            const int mul = (int)((desc >> 11) & 0xF) - (((desc >> 11) & 0x8) ? 16 : 0);
            eff = (int)(int8_t)(desc & 0xFF) + mul * (int)(arg > 0x7FFF ? 0x7FFF : arg);
          } else {
            eff = stack_desc_effect(desc, arg);
          }
          eff = valid ? eff : 0;
          const u32 unk = valid ? (desc >> 15) & 1u : 0u;
          sums[q] = eff;
          pushes += (!unk && eff > 0) ? eff : 0;
          unkm |= unk << q;
          endm |= (valid ? (desc >> 16) & 1u : 0u) << q;
          segm |= (valid ? (meta >> 26) & 1u : 0u) << q;  // is_jump_target (flags bit2)
        }
        // "the previous instruction ends a block" (or this is the object's first)
        const u32 up = __shfl_up_sync(0xffffffffu, endm, 1);
        const u32 prev_end = lane ? (up >> 7) & 1u : (u32)(c_end | (t0 == 0));
        segm |= ((endm << 1) | prev_end) & (cnt >= 8 ? 0xFFu : ((1u << cnt) - 1u));
        // in-lane inclusive scan with resets; unknown propagates to the segment's end
        u32 unk_inc = 0, ru = 0;
        int run = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if ((segm >> q) & 1u) run = 0, ru = 0;
          run += sums[q];
          ru |= (unkm >> q) & 1u;
          sums[q] = run;
          unk_inc |= ru << q;
        }
        // warp segmented scan of the lane aggregates, packed in one word per lane:
        // bit31 segment seen, bit30 unknown, bits 0-29 the sum (30-bit two's
        // complement; a step's sums stay far inside that range)
        u32 agg = (segm ? 0x80000000u : 0u) | (((unk_inc >> 7) & 1u) << 30) | ((u32)sums[7] & 0x3FFFFFFFu);
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const u32 o = __shfl_up_sync(0xffffffffu, agg, dd);
          if (lane >= dd && !(agg >> 31))
            agg = (o & 0x80000000u) | ((o | agg) & 0x40000000u) | ((o + agg) & 0x3FFFFFFFu);
        }
        // this lane's incoming prefix (exclusive), seeded with the carry
        u32 ex = __shfl_up_sync(0xffffffffu, agg, 1);
        if (lane == 0) ex = 0;
        int e_sum = (int)(ex << 2) >> 2, e_unk = (int)((ex >> 30) & 1u);
        if (!(ex >> 31)) e_sum += c_sum, e_unk |= c_unk;
        // positions before the lane's first segment start continue the incoming prefix
        const u32 first_seg = segm ? (u32)(__ffs((int)segm) - 1) : 8u;
        u32 words[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          int v = sums[q];
          u32 unk = (unk_inc >> q) & 1u;
          if ((u32)q < first_seg) {
            v += e_sum;
            unk |= (u32)e_unk;
          }
          if ((u32)q < cnt && !unk) {
            mx = v > mx ? v : mx;
            mn = v < mn ? v : mn;
          }
          const int cl = v > 32767 ? 32767 : v < -32768 ? -32768 : v;
          words[q] = ((u32)cl & 0xFFFFu) |
                     ((((segm >> q) & 1u) * SS_SEG_START | unk * SS_UNKNOWN | ((endm >> q) & 1u) * SS_ENDER) << 16);
          sums[q] = v;
        }
        segs += __popc(segm);
        unks += __popc(unkm);
        if (cnt == 8) {
          uint4* p = reinterpret_cast<uint4*>(dst + i0);
          __stcs(p, make_uint4(words[0], words[1], words[2], words[3]));
          __stcs(p + 1, make_uint4(words[4], words[5], words[6], words[7]));
        } else {
          u32* p = reinterpret_cast<u32*>(dst + i0);
#pragma unroll
          for (int q = 0; q < 8; q++)
            if ((u32)q < cnt) p[q] = words[q];
        }
        if (t0 + 256 < n) {  // carry: the step's last instruction (lane 31, q = 7)
          c_sum = __shfl_sync(0xffffffffu, sums[7], 31);
          c_unk = __shfl_sync(0xffffffffu, (int)((words[7] >> 17) & 1u), 31);
          c_end = __shfl_sync(0xffffffffu, (int)((endm >> 7) & 1u), 31);
        }
      }
      segs = (int)__reduce_add_sync(0xffffffffu, (u32)segs);
      unks = (int)__reduce_add_sync(0xffffffffu, (u32)unks);
      pushes = (int)__reduce_add_sync(0xffffffffu, (u32)pushes);
      mx = __reduce_max_sync(0xffffffffu, mx);
      mn = __reduce_min_sync(0xffffffffu, mn);
      if (lane == j) {
        mine.n_segments = segs;
        mine.n_unknown = unks;
        mine.n_pushes = pushes;
        mine.max_depth = mx;
        mine.min_depth = mn;
      }
    }
    if (lane < gsize && my_o < A.n_objs) info[my_o] = mine;
  }
}

extern "C" int upy_stackscan_batch(const upy_arena* arena, const upy_ins* ins, const upy_decoded* dec,
                                   upy_stackrec* stack, upy_stackinfo* info, void* stream) {
  if (!arena || !ins || !dec || !stack || !info) return 1;
  if (arena->n_objs == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one warp per group of consecutive objects: 32 objects for short ones (headers and
  // summaries move one per lane), down to 1 for long ones (each warp gets work)
  const double avg = (double)arena->total_code_units / (double)arena->n_objs;
  int gshift = 5;
  while (gshift > 0 && avg * (double)(1 << gshift) > 8192.0) gshift--;
  const i64 groups = (arena->n_objs + (1 << gshift) - 1) >> gshift;
  i64 blocks = (groups + SS_WARPS - 1) / SS_WARPS;
  const i64 cap = (i64)sms * SS_MINB;
  if (blocks > cap) blocks = cap;
  upy_stackscan_kernel<<<(unsigned)blocks, SS_WARPS * 32, 0, (cudaStream_t)stream>>>(*arena, ins, dec, stack, info, gshift);
  g_upy_launches += 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
