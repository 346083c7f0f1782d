// hostcheck.cpp -- TEST-ONLY host build of the device decompiler sources.
//
// Compiles the same headers the sm_100a kernels use (paper_2403_13839_b200/csrc)
// with g++ so their logic can be diffed against the reference on CPU during
// development (tools/dev_compare.py) and in the CPU test tier.  The product
// never loads this library: the public API only calls libupy_cuda.so.
#include <stdlib.h>
#include <string.h>
#include <vector>
#include "../paper_2403_13839_b200/csrc/pipeline.h"
#include "../paper_2403_13839_b200/csrc/decode.h"
#include "../paper_2403_13839_b200/csrc/dot.h"
#include "../paper_2403_13839_b200/csrc/stackscan.h"

extern "C" int upyh_decompile(const upy_arena* A, int header, const char* indent, int indent_len, const char* tool,
                              int tool_len, uint64_t arena_bytes, uint8_t* text, uint64_t text_cap,
                              uint64_t* text_off, uint32_t* text_len, int32_t* status, int64_t* aux,
                              upy_decoded* dec_out, int function_tree, int output) {
  std::vector<upy_ins> ins(A->total_code_units + 1);
  std::vector<upy_decoded> dec(A->n_objs);
  for (int64_t o = 0; o < A->n_objs; o++) {
    const upy_obj* ob = &A->objs[o];
    decode_scalar(A->bytes + ob->code_off, ob->code_len, (int)ob->minor, ins.data() + (ob->code_off >> 1), &dec[o]);
    if (dec_out) dec_out[o] = dec[o];
  }
  std::vector<uint8_t> slot(arena_bytes);
  std::vector<char> msg(4096);
  std::vector<uint8_t> sink(SINK_BYTES);
  EmitOpts opt;
  opt.header = header != 0;
  opt.function_tree = function_tree != 0;
  opt.indent = Str{indent, (u32)indent_len};
  opt.tool = Str{tool, (u32)tool_len};
  uint64_t used = 0;
  for (int64_t r = 0; r < A->n_roots; r++) {
    Dc C;
    memset(&C, 0, sizeof C);
    C.base = slot.data();
    C.cap = arena_bytes;
    C.top = arena_bytes;
    C.low_top = arena_bytes;
    C.sink = sink.data();
    C.msg = msg.data();
    C.msg_cap = 4096;
    C.A = A;
    C.objs = A->objs;
    C.consts = A->consts;
    C.strs = A->strs;
    C.refs = A->refs;
    C.limbs = A->limbs;
    C.bytes = A->bytes;
    C.ins_all = ins.data();
    C.dec_all = dec.data();
    C.max_depth = 600;
    Text out = {nullptr, 0, 0};
    if (output == 1) cfg_dot(&C, (u32)A->roots[r], &out);
    else decompile_source(&C, (u32)A->roots[r], &opt, &out);
    const char* src = C.err ? C.msg : out.d;
    uint32_t len = C.err ? C.msg_len : out.n;
    int st = C.err;
    if (used + len > text_cap) {
      st = UPY_ST_OUTPUT_OVERFLOW;
      len = 0;
    } else if (len) {
      memcpy(text + used, src, len);
    }
    text_off[r] = used;
    text_len[r] = len;
    status[r] = st;
    aux[2 * r] = C.aux0;
    aux[2 * r + 1] = C.aux1;
    used += len;
  }
  return 0;
}

// decode_instructions only (the reference-order scalar decoder) for every object:
// records at ins_out[code_off/2 + i], statuses in dec_out -- the oracle the
// device decode kernel's records are compared with (tests/test_decode_gpu.py).
extern "C" int upyh_decode(const upy_arena* A, upy_ins* ins_out, upy_decoded* dec_out) {
  for (int64_t o = 0; o < A->n_objs; o++) {
    const upy_obj* ob = &A->objs[o];
    decode_scalar(A->bytes + ob->code_off, ob->code_len, (int)ob->minor, ins_out + (ob->code_off >> 1), &dec_out[o]);
  }
  return 0;
}

// Arena high-water mark per root (bump region + deepest scratch), for slot sizing.
extern "C" int upyh_arena_peaks(const upy_arena* A, uint64_t arena_bytes, uint64_t* peak) {
  std::vector<upy_ins> ins(A->total_code_units + 1);
  std::vector<upy_decoded> dec(A->n_objs);
  for (int64_t o = 0; o < A->n_objs; o++) {
    const upy_obj* ob = &A->objs[o];
    decode_scalar(A->bytes + ob->code_off, ob->code_len, (int)ob->minor, ins.data() + (ob->code_off >> 1), &dec[o]);
  }
  std::vector<uint8_t> slot(arena_bytes);
  std::vector<char> msg(4096);
  std::vector<uint8_t> sink(SINK_BYTES);
  EmitOpts opt;
  opt.header = false;
  opt.function_tree = false;
  opt.indent = Str{"    ", 4};
  opt.tool = Str{"unpyre", 6};
  for (int64_t r = 0; r < A->n_roots; r++) {
    Dc C;
    memset(&C, 0, sizeof C);
    C.base = slot.data();
    C.cap = C.top = C.low_top = arena_bytes;
    C.sink = sink.data();
    C.msg = msg.data();
    C.msg_cap = 4096;
    C.A = A;
    C.objs = A->objs;
    C.consts = A->consts;
    C.strs = A->strs;
    C.refs = A->refs;
    C.limbs = A->limbs;
    C.bytes = A->bytes;
    C.ins_all = ins.data();
    C.dec_all = dec.data();
    C.max_depth = 600;
    Text out = {nullptr, 0, 0};
    decompile_source(&C, (u32)A->roots[r], &opt, &out);
    peak[r] = C.used + (arena_bytes - C.low_top);
  }
  return 0;
}

// Stack-depth scan (csrc/stackscan.h) of every object after the scalar decoder:
// the reference-order oracle of the device's segmented warp scan.
extern "C" int upyh_stackscan(const upy_arena* A, upy_stackrec* out, upy_stackinfo* info) {
  std::vector<upy_ins> ins(A->total_code_units + 1);
  for (int64_t o = 0; o < A->n_objs; o++) {
    const upy_obj* ob = &A->objs[o];
    upy_decoded d;
    upy_ins* rec = ins.data() + (ob->code_off >> 1);
    decode_scalar(A->bytes + ob->code_off, ob->code_len, (int)ob->minor, rec, &d);
    memset(&info[o], 0, sizeof info[o]);
    info[o].status = d.status;
    if (d.status == UPY_ST_OK) stackscan_scalar(rec, d.n_instrs, (int)ob->minor, out + (ob->code_off >> 1), &info[o]);
  }
  return 0;
}

extern "C" uint64_t upyh_stack_desc_selfcheck(uint32_t n_args) { return stack_desc_selfcheck(n_args); }
