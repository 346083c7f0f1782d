// upy.cu -- sm_100a kernels and the C ABI of include/upy.h.
//
//   upy_decode_kernel      (decode_kernel.cu) one warp per code object (roots and nested): HBM-bound
//                          decode of co_code into 12-byte instruction records
//                          (disasm.py:71-172).
//   upy_decompile_kernel   persistent, one thread per root object at a time:
//                          validate -> analyze -> structure -> recover -> emit
//                          (pipeline.py:143-160) inside a per-thread arena slot,
//                          then the text is appended to the flat output buffer.
#include <cuda_runtime.h>
#include <stdio.h>
#include <atomic>
#include <mutex>
#include "pipeline.h"
#include "dot.h"

// decode_kernel.cu
cudaError_t upy_decode_launch(const upy_arena* arena, upy_ins* ins, upy_decoded* dec, cudaStream_t s, int sms);

#define MSG_BYTES 4096u
#define SLOT_HEADER (MSG_BYTES + SINK_BYTES)

static __thread char g_last_error[512];
std::atomic<unsigned long long> g_upy_launches{0};  // upy_launch_count (decode_kernel.cu, stackscan_kernel.cu too)
static constexpr int kMaxDevices = 64;
static std::mutex g_dev_cfg_mu;
static bool g_dev_cfg_done[kMaxDevices];
static void set_err(const char* fmt, const char* a = "") {
  snprintf(g_last_error, sizeof g_last_error, fmt, a);
}

struct KParams {
  upy_arena A;
  const upy_ins* ins;
  const upy_decoded* dec;
  upy_out out;
  u8* slots_base;
  u64 slot_bytes;
  u32* next_root;
  int header;
  int max_depth;
  u64 indent_len, tool_len;
  const char* indent_ptr;  // style strings: `indent` / `tool` below when <= 64 bytes,
  const char* tool_ptr;    // else a workspace copy
  char indent[64];
  char tool[64];
  int lane_stride;  // 1: every thread takes roots; 32: one root-taking thread per warp
  int schedule;     // upy_options.schedule: 0 each thread takes the next root, 1 warp-synchronous
  int function_tree;
  int output;       // upy_options.output: 0 source text, 1 CFG dot export
  const int32_t* order;  // upy_options.order: processing order of root positions (or null)
  // schedule 3 (split): positions [k_begin, k_end) of the order; arena slot = k - k_begin
  struct SplitState* state;  // one per arena slot: the built tree and its context
  u8* scratch_base;          // per-thread message buffer + overflow sink (SLOT_HEADER each)
  u32 k_begin, k_end;
};

#ifndef UPY_MINB
#define UPY_MINB 8  // <= 64 registers: 32 resident warps per SM (measured +43% vs unbounded)
#endif
#ifndef UPY_TREE_MINB  // split schedule: resident 128-thread blocks per SM of each kernel
#define UPY_TREE_MINB UPY_MINB
#endif
#ifndef UPY_EMIT_MINB
#define UPY_EMIT_MINB UPY_MINB
#endif
// Per-thread state reset for a new root object: message buffer + sink at `scratch`,
// the bump/scratch arena [arena, arena + cap).
__device__ __forceinline__ void dc_reset_at(Dc& C, const KParams& P, u8* scratch, u8* arena, u64 cap) {
  C.msg = (char*)scratch;
  C.msg_len = 0;
  C.msg_cap = MSG_BYTES;
  C.sink = scratch + MSG_BYTES;
  C.base = arena;
  C.cap = cap;
  C.used = 0;
  C.top = C.cap;
  C.low_top = C.cap;
  C.err = 0;
  C.aux0 = C.aux1 = 0;
  C.A = &P.A;
  C.objs = P.A.objs;
  C.consts = P.A.consts;
  C.strs = P.A.strs;
  C.refs = P.A.refs;
  C.limbs = P.A.limbs;
  C.bytes = P.A.bytes;
  C.ins_all = P.ins;
  C.dec_all = P.dec;
  C.depth = 0;
  C.max_depth = P.max_depth;
  C.n_defs = 0;
}
// one slot = [message | sink | arena]
__device__ __forceinline__ void dc_reset(Dc& C, const KParams& P, u8* base) {
  dc_reset_at(C, P, base, base + SLOT_HEADER, P.slot_bytes - SLOT_HEADER);
}

// Text (or the error message) of root r into the flat output buffer.
__device__ __forceinline__ void emit_result(const KParams& P, Dc& C, u32 r, const Text& out) {
  const char* src;
  u32 len;
  if (C.err) {
    src = C.msg;
    len = C.msg_len;
  } else {
    src = out.d;
    len = out.n;
  }
  int status = C.err;
  // reservations are 16-byte granular so the copy-out is whole uint4 stores
  u64 resv = ((u64)len + 15) & ~(u64)15;
  u64 off = atomicAdd((unsigned long long*)P.out.text_used, (unsigned long long)resv);
  if (off + resv > P.out.text_cap) {
    status = UPY_ST_OUTPUT_OVERFLOW;
    len = 0;
  } else if (len) {
    copy16(P.out.text + off, src, len);
  }
  P.out.text_off[r] = off;
  P.out.text_len[r] = len;
  P.out.status[r] = status;
  P.out.aux[2 * (u64)r] = C.aux0;
  P.out.aux[2 * (u64)r + 1] = C.aux1;
}

// ---------------------------------------------------------------- statement-parallel emit
// North-star subsystem (5): a warp emits one object at a time with its statements
// spread over the 32 lanes.  The emitter is stateless across statements apart from
// the indentation depth (emitter.py:112-132), so statement s rendered on its own at
// the right depth is exactly its slice of the sequential text.  Each lane renders
// statements s = lane, lane + 32, ... into its own scratch (its arena above its live
// data, a fresh error state and message buffer), the lengths are summed, the owner
// reserves the object's range of the flat output once, and a per-round exclusive
// scan of the statement lengths places every lane's text.  The first failing
// statement in order decides the error, as in the sequential emitter.  A root that
// is one `def` (every function root: root_tree_of, pipeline.py:121-130) is split
// into its header lines (decorators, the def line; the owner lane) and its body at
// depth 1.
__device__ __forceinline__ void copy_bytes(char* dst, const char* src, u32 n) {
#pragma unroll 1
  for (u32 i = 0; i < n; i++) dst[i] = src[i];
}

// One round: lane k owns object k (ok: tree built, r its root position, oi its
// object).  Every lane first renders its OWN object's header lines in parallel (the
// provenance comment, decorators and the def line of a single-def root, `pass` for
// an empty body); then the warp emits the objects one after another, statements
// spread over the lanes.  One scratch context per lane for the whole round.
__device__ __noinline__ void coemit_round(const KParams& P, Dc& C, const EmitOpts& opt, bool ok, u32 r, u32 oi,
                                          NV* tree) {
  const int lane = threadIdx.x & 31;
  Dc H = C;  // scratch context on this lane's arena, above its live data
  H.err = 0;
  H.aux0 = H.aux1 = 0;
  H.depth = 0;
  H.msg = (char*)ualloc(&H, MSG_BYTES);
  H.msg_len = 0;
  H.msg_cap = H.err ? 0 : MSG_BYTES;
  if (H.err) H.msg = C.msg;
  Emitter EM;
  EM.C = &H;
  EM.indent = opt.indent;
  // own header
  NV* body = nullptr;
  int depth = 0;
  Text head = {nullptr, 0, 0};
  if (ok) {
    const bool split = tree->n == 1 && tree->d[0]->k == S_FUNCDEF;
    body = split ? tree->d[0]->l1 : tree;
    depth = split ? 1 : 0;
    EM.out = &head;
    EM.depth = 0;
    if (opt.header) {
      t_puts(&H, &head, "# decompiled by ");
      t_str(&H, &head, opt.tool);
      t_puts(&H, &head, " from ");
      Str qn = obj_qualname(&H, oi);
      t_str(&H, &head, qn.n ? qn : obj_name(&H, oi));
      t_puts(&H, &head, " (python 3.");
      t_i64(&H, &head, obj_at(&H, oi)->minor);
      t_puts(&H, &head, ")\n");
    }
    if (split) EM.funcdef_head(tree->d[0]);
    if (!body->n) {
      EM.depth = depth;
      EM.simple_line("pass");
    }
    if (H.err) {  // the header failed: that is the object's result
      Text none = {nullptr, 0, 0};
      emit_result(P, H, r, none);
      ok = false;
    }
  }
  const u64 mark = H.used;
  for (u32 todo = __ballot_sync(0xffffffffu, ok); todo; todo &= todo - 1) {
    const int j = __ffs((int)todo) - 1;
    NV* bj = (NV*)__shfl_sync(0xffffffffu, (unsigned long long)body, j);
    const int dj = __shfl_sync(0xffffffffu, depth, j);
    const u32 rj = __shfl_sync(0xffffffffu, r, j);
    const u32 nb = bj->n;
    H.used = mark;
    H.err = 0;
    H.msg_len = 0;
    H.aux0 = H.aux1 = 0;
    // this lane's statements of object j, back to back; ends[] marks where each stops
    Text mine = {nullptr, 0, 0};
    const u32 m = nb > (u32)lane ? (nb - (u32)lane + 31) / 32 : 0;
    u32* ends = m ? (u32*)ualloc(&H, 4ull * m) : nullptr;
    u32 fail = H.err ? (u32)lane : 0xFFFFFFFFu;  // scratch overflow: retryable
    EM.out = &mine;
    EM.depth = dj;
    for (u32 q = 0; q < m && !H.err; q++) {
      EM.stmt(bj->d[(u64)lane + 32ull * q]);
      if (H.err) fail = (u32)lane + 32u * q;
      else ends[q] = mine.n;
    }
    const u32 first_fail = __reduce_min_sync(0xffffffffu, fail);
    if (first_fail != 0xFFFFFFFFu) {  // the first failing statement in order decides
      if (lane == (int)(first_fail & 31u)) {
        Text none = {nullptr, 0, 0};
        emit_result(P, H, rj, none);
      }
      continue;
    }
    const u32 head_len = __shfl_sync(0xffffffffu, head.n, j);
    const u32 total = head_len + __reduce_add_sync(0xffffffffu, mine.n);
    u64 off = 0;
    int status = 0;
    if (lane == j) {
      const u64 resv = ((u64)total + 15) & ~(u64)15;
      off = atomicAdd((unsigned long long*)P.out.text_used, (unsigned long long)resv);
      if (off + resv > P.out.text_cap) status = UPY_ST_OUTPUT_OVERFLOW;
      else if (head.n) copy16(P.out.text + off, head.d, head.n);  // both 16-B aligned; 16-B granular
    }
    off = __shfl_sync(0xffffffffu, off, j);
    status = __shfl_sync(0xffffffffu, status, j);
    if (!status) {
      u64 pos = off + head_len;
      for (u32 q = 0; 32ull * q < nb; q++) {  // round q: statements 32q .. 32q+31
        const bool has = q < m;
        const u32 beg = has ? (q ? ends[q - 1] : 0u) : 0u;
        const u32 len = has ? ends[q] - beg : 0u;
        u32 incl = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += o;
        }
        __syncwarp();  // the header's 16-B stores end before statement bytes land next to them
        if (len) copy_bytes((char*)P.out.text + pos + (incl - len), mine.d + beg, len);
        pos += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == j) {
      P.out.text_off[rj] = off;
      P.out.text_len[rj] = status ? 0 : total;
      P.out.status[rj] = status;
      P.out.aux[2 * (u64)rj] = 0;
      P.out.aux[2 * (u64)rj + 1] = 0;
    }
  }
}

__global__ void __launch_bounds__(128, UPY_MINB) upy_decompile_kernel(KParams P) {
  // Small batches (fewer roots than resident warps) run one root-taking thread per
  // warp: a lone thread issues without divergence serialisation, and the roots
  // spread over all SMs instead of packing into a few blocks -- latency, not
  // throughput, is what a small batch measures.
  if (P.lane_stride > 1 && (threadIdx.x & 31)) return;
  const u64 slot = ((u64)blockIdx.x * blockDim.x + threadIdx.x) / (u64)P.lane_stride;
  u8* base = P.slots_base + slot * P.slot_bytes;
  EmitOpts opt;
  opt.header = P.header != 0;
  opt.function_tree = P.function_tree != 0;
  opt.indent = Str{P.indent_len <= 64 ? P.indent : P.indent_ptr, (u32)P.indent_len};
  opt.tool = Str{P.tool_len <= 64 ? P.tool : P.tool_ptr, (u32)P.tool_len};
#ifndef UPY_DC_SHARED
  // The per-thread context lives on the thread's stack: the shared-memory copy
  // (17 KB per block, 139 KB per SM at 8 blocks) cost more in L1 capacity for the
  // arena than it saved (C3 278.6 -> 261.4 ms with the context in local memory).
  Dc C_local;
  Dc& C = C_local;
#else
  __shared__ Dc dcs[128];
  Dc& C = dcs[threadIdx.x];
#endif
  const u64 n_roots = (u64)P.A.n_roots;
  if (P.schedule == 2 && P.lane_stride == 1) {
    // warp-synchronous + statement-parallel emission: every lane builds its own
    // object's tree (validate .. finish), then the warp emits the 32 trees in turn
    const int lane = threadIdx.x & 31;
    while (true) {
      u32 k0 = 0;
      if (lane == 0) k0 = atomicAdd(P.next_root, 32u);
      k0 = __shfl_sync(0xffffffffu, k0, 0);
      if (k0 >= n_roots) break;
      const u32 k = k0 + (u32)lane;
      const bool has = k < n_roots;
      const u32 r = has ? (P.order ? (u32)P.order[k] : k) : 0u;
      dc_reset(C, P, base);
      SourceJob S;
      S.oi = has ? (u32)P.A.roots[r] : 0u;
      S.opt = &opt;
      S.tree = nullptr;
      Text none = {nullptr, 0, 0};
      S.out = &none;
      if (has) decompile_tree(&C, &S);
      __syncwarp();
      if (has && C.err) emit_result(P, C, r, none);  // failed before emit: its message
#ifndef UPY_SKIP_COEMIT  // timing experiment only: trees built, nothing emitted
      coemit_round(P, C, opt, has && !C.err, r, S.oi, S.tree);
#endif
      __syncwarp();
    }
    return;
  }
  if (P.schedule == 1 && P.lane_stride == 1) {
    // warp-synchronous: a warp takes 32 consecutive positions of the order and its
    // lanes start their objects together (similar neighbours then share code paths)
    const int lane = threadIdx.x & 31;
    while (true) {
      u32 k0 = 0;
      if (lane == 0) k0 = atomicAdd(P.next_root, 32u);
      k0 = __shfl_sync(0xffffffffu, k0, 0);
      if (k0 >= n_roots) break;
      const u32 k = k0 + (u32)lane;
      if (k < n_roots) {
        const u32 r = P.order ? (u32)P.order[k] : k;
        dc_reset(C, P, base);
        Text out = {nullptr, 0, 0};
        decompile_source(&C, (u32)P.A.roots[r], &opt, &out);
        emit_result(P, C, r, out);
      }
      __syncwarp();
    }
    return;
  }
  // each thread takes the next root from the global queue
  while (true) {
    u32 r = atomicAdd(P.next_root, 1u);
    if (r >= n_roots) break;
    if (P.order) r = (u32)P.order[r];
    dc_reset(C, P, base);
    Text out = {nullptr, 0, 0};
    decompile_source(&C, (u32)P.A.roots[r], &opt, &out);
    emit_result(P, C, r, out);
  }
}

// ---------------------------------------------------------------- split schedule
// schedule 3: the pipeline in two launches per chunk of positions.  upy_tree_kernel
// runs validate .. finish for every root of the chunk, each in its own arena slot,
// and leaves the tree with its context in `state`; upy_emit_kernel then renders every
// tree.  Each kernel's hot code is one part of the pipeline: the emitter no longer
// competes with analysis / structuring for the SM instruction cache (the
// decompile kernel's first limit).  The arena slots must hold the
// trees of a whole chunk (one slot per position), so the chunk is the slot count.
struct SplitState {
  Dc C;
  BodyJob body;  // the root body's analysis (schedule 4 hands it from analyze to structure)
  NV* tree;
  u32 oi;
  u32 ok;
};

__device__ __forceinline__ EmitOpts kernel_opts(const KParams& P) {
  EmitOpts opt;
  opt.header = P.header != 0;
  opt.function_tree = P.function_tree != 0;
  opt.indent = Str{P.indent_len <= 64 ? P.indent : P.indent_ptr, (u32)P.indent_len};
  opt.tool = Str{P.tool_len <= 64 ? P.tool : P.tool_ptr, (u32)P.tool_len};
  return opt;
}

// Stages FIRST..LAST of decompile_source for every position of the chunk.  FIRST == 0
// starts the object in its slot; otherwise the state the previous kernel left is
// restored (its arena context on this thread's message buffer and sink).  A failure
// writes the object's message at once; LAST == DS_EMIT writes the text.  `ctr` is the
// kernel's own position counter.
template <int FIRST, int LAST>
__device__ __forceinline__ void stage_range(const KParams& P, u32* ctr) {
  if (P.lane_stride > 1 && (threadIdx.x & 31)) return;
  const u64 t = ((u64)blockIdx.x * blockDim.x + threadIdx.x) / (u64)P.lane_stride;
  u8* scratch = P.scratch_base + t * SLOT_HEADER;
  const EmitOpts opt = kernel_opts(P);
  Dc C;
  while (true) {
    const u32 k = P.k_begin + atomicAdd(ctr, 1u);
    if (k >= P.k_end) break;
    const u64 slot = k - P.k_begin;
    SplitState* sv = P.state + slot;
    if (FIRST > 0 && !sv->ok) continue;
    const u32 r = P.order ? (u32)P.order[k] : k;
    SourceJob S;
    S.opt = &opt;
    Text out = {nullptr, 0, 0};
    S.out = &out;
    if (FIRST == 0) {
      dc_reset_at(C, P, scratch, P.slots_base + slot * P.slot_bytes, P.slot_bytes);
      S.oi = (u32)P.A.roots[r];
      S.tree = nullptr;
    } else {
      C = sv->C;
      C.A = &P.A;
      C.msg = (char*)scratch;
      C.msg_len = 0;
      C.msg_cap = MSG_BYTES;
      C.sink = scratch + MSG_BYTES;
      S.oi = sv->oi;
      S.body = sv->body;
      S.tree = sv->tree;
    }
#pragma unroll 1
    for (int st = FIRST; st <= LAST; st++) ds_stage(&C, &S, st);
    if (LAST == DS_EMIT || C.err) {
      emit_result(P, C, r, out);  // the text, or the message of the failing stage
      sv->ok = 0;
    } else {
      sv->C = C;
      sv->body = S.body;
      sv->tree = S.tree;
      sv->oi = S.oi;
      sv->ok = 1;
    }
  }
}

// schedule 3: build every tree, then emit every tree
__global__ void __launch_bounds__(128, UPY_TREE_MINB) upy_tree_kernel(KParams P) {
  stage_range<DS_VALIDATE, DS_FINISH>(P, P.next_root);
}
__global__ void __launch_bounds__(128, UPY_EMIT_MINB) upy_emit_kernel(KParams P) {
  stage_range<DS_EMIT, DS_EMIT>(P, P.next_root + 1);
}
// schedule 4: validate + analyze, then structure + finish, then emit
__global__ void __launch_bounds__(128, UPY_TREE_MINB) upy_analyze_kernel(KParams P) {
  stage_range<DS_VALIDATE, DS_ANALYZE>(P, P.next_root + 2);
}
__global__ void __launch_bounds__(128, UPY_TREE_MINB) upy_structure_kernel(KParams P) {
  stage_range<DS_STRUCTURE, DS_FINISH>(P, P.next_root);
}

// `unpyre disasm --cfg --dot` (cli.py:103-105): to_dot(analyze(root)) per root
// (dot.h), same schedule and per-thread arena as the decompile kernel.
__global__ void __launch_bounds__(128, UPY_MINB) upy_cfgdot_kernel(KParams P) {
  if (P.lane_stride > 1 && (threadIdx.x & 31)) return;
  const u64 slot = ((u64)blockIdx.x * blockDim.x + threadIdx.x) / (u64)P.lane_stride;
  u8* base = P.slots_base + slot * P.slot_bytes;
  Dc C;
  const u64 n_roots = (u64)P.A.n_roots;
  while (true) {
    u32 r = atomicAdd(P.next_root, 1u);
    if (r >= n_roots) break;
    if (P.order) r = (u32)P.order[r];
    dc_reset(C, P, base);
    Text out = {nullptr, 0, 0};
    cfg_dot(&C, (u32)P.A.roots[r], &out);
    emit_result(P, C, r, out);
  }
}

// ------------------------------------------------------------ C ABI
struct WsLayout {
  u64 ins_off, dec_off, ctr_off, style_off, state_off, scratch_off, slots_off, total;
  u64 slots, slot_bytes;
  u64 threads;  // split schedule: root-taking threads (each with its scratch)
  int lane_stride;
  bool split;
};
static u64 al(u64 x) { return (x + 255) & ~(u64)255; }

static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// threads per block: <= 128 (shared Dc array), whole warps
static int eff_tpb(const upy_options* o) {
  int tpb = o && o->threads_per_block > 0 && o->threads_per_block < 128 ? o->threads_per_block : 128;
  return tpb < 32 ? 32 : tpb & ~31;
}

// schedule 3: [state per slot][scratch per thread][arena slots]; slots = positions per
// chunk, each slot an arena only (no header: messages and sinks are per thread).
static WsLayout layout_split(const upy_arena* a, const upy_options* o, WsLayout L) {
  // measured peaks (tools: hostcheck upyh_arena_peaks): C3 3.10 25 KB mean / 27 KB max at
  // 428 code bytes, 3.11 28 / 34 KB at 1,418; larger objects overflow and are retried
  u64 sb = o->arena_bytes ? o->arena_bytes : (u64)(32u << 10) + (u64)a->max_code_len * 16u;
  sb = (sb + 255) & ~(u64)255;
  L.slot_bytes = sb;
  u64 slots;
  if (o->slots > 0) {
    slots = (u64)o->slots;
  } else {
    u64 cap_bytes = 40ull << 30;
    slots = cap_bytes / (sb + sizeof(SplitState));
  }
  if (slots > (u64)a->n_roots) slots = (u64)a->n_roots;
  if (slots < 1) slots = 1;
  const int mb = UPY_TREE_MINB > UPY_EMIT_MINB ? UPY_TREE_MINB : UPY_EMIT_MINB;
  int tpb = eff_tpb(o);
  const u64 full = (u64)sm_count() * mb * tpb;  // resident threads of the larger grid
  L.lane_stride = 1;
  u64 thr;
  if ((u64)a->n_roots <= (u64)sm_count() * (4 * UPY_MINB)) {
    L.lane_stride = 32;
    const u64 wpb = (u64)tpb / 32;
    thr = (slots + wpb - 1) / wpb * wpb;
    if (thr > (u64)sm_count() * (4 * UPY_MINB)) thr = (u64)sm_count() * (4 * UPY_MINB);
  } else {
    thr = slots < full ? slots : full;
    thr = (thr + tpb - 1) / tpb * tpb;
  }
  L.threads = thr;
  L.slots = slots;
  L.state_off = L.slots_off;
  L.scratch_off = L.state_off + al(slots * sizeof(SplitState));
  L.slots_off = L.scratch_off + al(thr * SLOT_HEADER);
  L.total = L.slots_off + slots * sb;
  if (o->decode_only) L.total = L.ctr_off + 256;
  return L;
}

static WsLayout layout(const upy_arena* a, const upy_options* o) {
  WsLayout L;
  u64 units = a->total_code_units + 1;
  L.ins_off = 0;
  L.dec_off = al(units * sizeof(upy_ins));
  L.ctr_off = L.dec_off + al((u64)a->n_objs * sizeof(upy_decoded));
  L.style_off = L.ctr_off + 256;
  u64 style_bytes = 0;  // EmitStyle strings longer than the kernel-parameter copies
  if (o && o->indent_len > 64) style_bytes += o->indent_len;
  if (o && o->tool_len > 64) style_bytes += o->tool_len;
  L.slots_off = L.style_off + al(style_bytes);
  L.split = o && (o->schedule == 3 || o->schedule == 4) && o->output == 0;
  if (L.split) return layout_split(a, o, L);
  // C3-size objects use ~55 KB; larger ones overflow and are retried by the host with 4x
  // measured peaks: C3 (400 B code) ~25 KB, C4 (19 KB code) ~2.2 MB => ~115 B per code byte
  u64 sb = o && o->arena_bytes ? o->arena_bytes : (u64)(64u << 10) + (u64)a->max_code_len * 160u;
  sb = (sb + SLOT_HEADER + 255) & ~(u64)255;
#ifdef UPY_SLOT_STAGGER
  // slot stride off the power-of-two grid: every thread starts allocating at the
  // same offset of its slot, so a 2^k stride lines the hot lines of all slots up
  // on the same L2 sets / DRAM banks
  sb += UPY_SLOT_STAGGER;
#endif
  L.slot_bytes = sb;
  u64 slots;
  if (o && o->slots > 0) {
    slots = (u64)o->slots;
  } else {
    u64 cap_bytes = 40ull << 30;  // default arena budget (of 180 GB HBM)
    slots = cap_bytes / sb;
    u64 full = (u64)sm_count() * 1024;
    if (slots > full) slots = full;
  }
  if (slots > (u64)a->n_roots) slots = (u64)a->n_roots;
  if (slots < 1) slots = 1;
  int tpb = eff_tpb(o);
  L.lane_stride = 1;
  if (!(o && o->slots > 0) && (u64)a->n_roots <= (u64)sm_count() * (4 * UPY_MINB)) {
    L.lane_stride = 32;  // one root-taking thread per warp (see the kernel)
    const u64 wpb = (u64)tpb / 32;
    slots = (slots + wpb - 1) / wpb * wpb;
  } else {
    slots = (slots + tpb - 1) / tpb * tpb;
  }
  L.slots = slots;
  L.total = L.slots_off + slots * sb;
  if (o && o->decode_only) L.total = L.slots_off;
  return L;
}

extern "C" {

size_t upy_abi_sizeof(int which) {
  switch (which) {
    case 0: return sizeof(upy_obj);
    case 1: return sizeof(upy_const);
    case 2: return sizeof(upy_str);
    case 3: return sizeof(upy_arena);
    case 4: return sizeof(upy_options);
    case 5: return sizeof(upy_out);
    case 6: return sizeof(upy_ins);
    case 7: return sizeof(upy_decoded);
    case 8: return sizeof(upy_stackrec);
    case 9: return sizeof(upy_stackinfo);
  }
  return 0;
}
int upy_abi_version(void) { return UPY_ABI_VERSION; }
const char* upy_last_error(void) { return g_last_error; }
uint64_t upy_launch_count(void) { return g_upy_launches.load(); }

int upy_query_workspace(const upy_arena* arena, const upy_options* opt, size_t* ws_bytes) {
  if (!arena || !ws_bytes) {
    set_err("upy_query_workspace: null argument");
    return 1;
  }
  *ws_bytes = (size_t)layout(arena, opt).total;
  return 0;
}

int upy_decode_batch(const upy_arena* arena, upy_ins* ins, upy_decoded* dec, void* stream) {
  if (!arena || !ins || !dec) {
    set_err("upy_decode_batch: null argument");
    return 1;
  }
  if (arena->n_objs == 0) return 0;
  cudaError_t e = upy_decode_launch(arena, ins, dec, (cudaStream_t)stream, sm_count());
  if (e != cudaSuccess) {
    set_err("decode launch: %s", cudaGetErrorString(e));
    return 2;
  }
  return 0;
}

int upy_decompile_batch(const upy_arena* arena, const upy_options* opt, const upy_out* out, void* workspace,
                        size_t ws_bytes, void* stream) {
  if (!arena || !out || !workspace) {
    set_err("upy_decompile_batch: null argument");
    return 1;
  }
  if (opt && (opt->output < 0 || opt->output > 1)) {
    set_err("upy_decompile_batch: options.output must be 0 (source) or 1 (CFG dot)");
    return 1;
  }
  WsLayout L = layout(arena, opt);
  if (ws_bytes < L.total) {
    set_err("upy_decompile_batch: workspace too small");
    return 1;
  }
  cudaStream_t s = (cudaStream_t)stream;
  u8* ws = (u8*)workspace;
  upy_ins* ins = (upy_ins*)(ws + L.ins_off);
  upy_decoded* dec = (upy_decoded*)(ws + L.dec_off);
  u32* ctr = (u32*)(ws + L.ctr_off);
  if (!(opt && opt->skip_decode)) {
    int rc = upy_decode_batch(arena, ins, dec, stream);
    if (rc) return rc;
  }
  if (opt && opt->decode_only) return 0;
  if (arena->n_roots == 0) return 0;
  {
    // one-time per-device settings (both are per device: the kernel runs on the
    // caller's current device); guarded for concurrent callers
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_dev_cfg_mu);
    if (dev < 0 || dev >= kMaxDevices) {
      set_err("upy_decompile_batch: device ordinal out of range");
      return 1;
    }
    if (!g_dev_cfg_done[dev]) {
      // no shared memory: give the whole L1/shared pool to L1 (arena + stack hit rate)
      cudaFuncSetAttribute(upy_decompile_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute(upy_cfgdot_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute(upy_tree_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute(upy_emit_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute(upy_analyze_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaFuncSetAttribute(upy_structure_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
      cudaError_t e = cudaDeviceSetLimit(cudaLimitStackSize, 48 * 1024);
      if (e != cudaSuccess) {
        set_err("cudaDeviceSetLimit(stack): %s", cudaGetErrorString(e));
        return 2;
      }
      g_dev_cfg_done[dev] = true;
    }
  }
  cudaMemsetAsync(ctr, 0, 256, s);
  KParams P;
  memset(&P, 0, sizeof P);
  P.A = *arena;
  P.ins = ins;
  P.dec = dec;
  P.out = *out;
  P.slots_base = ws + L.slots_off;
  P.slot_bytes = L.slot_bytes;
  P.next_root = ctr;
  P.max_depth = opt && opt->max_depth > 0 ? opt->max_depth : 600;
  static const char kIndent[] = "    ", kTool[] = "unpyre";
  const char* ind = opt && opt->indent ? opt->indent : kIndent;
  const char* tool = opt && opt->tool ? opt->tool : kTool;
  P.indent_len = opt && opt->indent ? opt->indent_len : 4;
  P.tool_len = opt && opt->tool ? opt->tool_len : 6;
  P.header = opt ? opt->header : 0;
  P.function_tree = opt ? opt->function_tree : 0;
  P.output = opt ? opt->output : 0;
  P.order = opt ? opt->order : nullptr;
  P.schedule = opt ? opt->schedule : 0;
  u8* style_ws = ws + L.style_off;
  if (P.indent_len <= 64) {
    memcpy(P.indent, ind, P.indent_len);
  } else {
    cudaMemcpyAsync(style_ws, ind, P.indent_len, cudaMemcpyHostToDevice, s);
    P.indent_ptr = (const char*)style_ws;
    style_ws += P.indent_len;
  }
  if (P.tool_len <= 64) {
    memcpy(P.tool, tool, P.tool_len);
  } else {
    cudaMemcpyAsync(style_ws, tool, P.tool_len, cudaMemcpyHostToDevice, s);
    P.tool_ptr = (const char*)style_ws;
  }
  P.lane_stride = L.lane_stride;
  int tpb = eff_tpb(opt);
  if (L.split) {
    P.state = (SplitState*)(ws + L.state_off);
    P.scratch_base = ws + L.scratch_off;
    // each kernel's grid: the scratch threads, at most its resident blocks per SM
    const u64 blocks_all = L.threads * L.lane_stride / tpb;
    const u64 sms = (u64)sm_count();
    const unsigned tree_blocks = (unsigned)(blocks_all < sms * UPY_TREE_MINB ? blocks_all : sms * UPY_TREE_MINB);
    const unsigned emit_blocks = (unsigned)(blocks_all < sms * UPY_EMIT_MINB ? blocks_all : sms * UPY_EMIT_MINB);
    const u64 n = (u64)arena->n_roots;
    for (u64 k0 = 0; k0 < n; k0 += L.slots) {
      P.k_begin = (u32)k0;
      P.k_end = (u32)(k0 + L.slots < n ? k0 + L.slots : n);
      if (k0) cudaMemsetAsync(ctr, 0, 16, s);
      if (P.schedule == 4) {
        upy_analyze_kernel<<<tree_blocks, tpb, 0, s>>>(P);
        upy_structure_kernel<<<tree_blocks, tpb, 0, s>>>(P);
        g_upy_launches += 1;
      } else {
        upy_tree_kernel<<<tree_blocks, tpb, 0, s>>>(P);
      }
      upy_emit_kernel<<<emit_blocks, tpb, 0, s>>>(P);
      g_upy_launches += 2;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_err("decompile launch: %s", cudaGetErrorString(e));
      return 2;
    }
    return 0;
  }
  unsigned blocks = (unsigned)(L.slots * L.lane_stride / tpb);
  if (P.output == 1) upy_cfgdot_kernel<<<blocks, tpb, 0, s>>>(P);
  else upy_decompile_kernel<<<blocks, tpb, 0, s>>>(P);
  g_upy_launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("decompile launch: %s", cudaGetErrorString(e));
    return 2;
  }
  return 0;
}

#ifdef UPY_PHASE_PROF
int upy_prof_read(unsigned long long* host, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, g_stage_cycles, sizeof(g_stage_cycles));
  if (reset) {
    unsigned long long z[DS_STAGES] = {};
    cudaMemcpyToSymbol(g_stage_cycles, z, sizeof z);
  }
  return DS_STAGES;
}
#endif
}  // extern "C"
