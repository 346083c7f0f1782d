/*
 * upy.h -- C ABI of the B200 batched decompiler (libupy_cuda.so).
 *
 * This is the drop-in boundary for the reference's hot path
 *     unpyre.decompile_source(code, style=None) -> str
 *     (/root/reference/pkg/src/unpyre/pipeline.py:143-160, exported at __init__.py:13,23)
 * and, for the decoder stage on its own,
 *     unpyre.disasm.decode_instructions(code) -> list[Instruction]
 *     (/root/reference/pkg/src/unpyre/disasm.py:71-122, 125-172).
 *
 * Inputs are a packed "arena": a struct-of-arrays image of a batch of CodeObject
 * trees (code_model.py:101-123) already resident in device memory.  Every root
 * object (and, recursively, its nested code constants) is decompiled
 * independently; outputs land in one flat UTF-8 buffer plus per-root
 * (offset, length, status, aux) records.  Plain pointers and sizes only; the
 * caller owns every buffer; calls are stream-ordered.
 */
#ifndef UPY_H
#define UPY_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UPY_ABI_VERSION 4

/* Const kinds (code_model.py:56-59). */
enum {
  UPY_C_NONE = 0, UPY_C_BOOL = 1, UPY_C_INT = 2, UPY_C_FLOAT = 3, UPY_C_COMPLEX = 4,
  UPY_C_STR = 5, UPY_C_BYTES = 6, UPY_C_TUPLE = 7, UPY_C_FROZENSET = 8, UPY_C_CODE = 9,
  UPY_C_ELLIPSIS = 10
};

/* One code object (code_model.py:105-123).  Python ints are carried as int64. */
typedef struct {
  int64_t argcount, posonlyargcount, kwonlyargcount, nlocals, stacksize, flags, firstlineno;
  uint64_t code_off, exc_off, lnt_off;      /* byte-pool offsets; code_off 16-B aligned and the
                                               pool readable up to the next 16-B boundary */
  uint32_t code_len, exc_len, lnt_len;
  uint32_t consts_off, n_consts;            /* refs pool: const ids */
  uint32_t names_off, n_names;              /* refs pool: string ids */
  uint32_t varnames_off, n_varnames;
  uint32_t freevars_off, n_freevars;
  uint32_t cellvars_off, n_cellvars;
  uint32_t name, filename, qualname;        /* string ids */
  uint32_t minor;                           /* 8..11 (major is always 3) */
  uint32_t pad;
} upy_obj;

/* One constant-tree node. */
typedef struct {
  uint32_t kind;
  int32_t  ival;   /* bool value; int sign (-1/0/1) */
  uint32_t n;      /* str/bytes: byte length; int: limb count; tuple/frozenset: element count */
  uint32_t pad;
  uint64_t off;    /* str/bytes: byte pool; int: limb pool; tuple/frozenset: refs pool; code: object index */
  double   re, im; /* float: re; complex: re, im */
} upy_const;

typedef struct { uint64_t off; uint32_t len; uint32_t pad; } upy_str;  /* UTF-8 (surrogatepass) */

/* Device-resident arena (all pointers are device pointers). */
typedef struct {
  const upy_obj*   objs;   int64_t n_objs;
  const upy_const* consts; int64_t n_consts;
  const upy_str*   strs;   int64_t n_strs;
  const uint32_t*  refs;   int64_t n_refs;
  const uint32_t*  limbs;  int64_t n_limbs;   /* little-endian base-2^32 magnitudes */
  const uint8_t*   bytes;  int64_t n_bytes;
  const int32_t*   roots;  int64_t n_roots;   /* objects to decompile */
  uint64_t max_code_len;                       /* host-known max(code_len), sizes scratch */
  uint64_t total_code_units;                   /* sum(code_len)/2 upper bound incl. odd */
} upy_arena;

/* EmitStyle (emitter.py:46-50) plus launch knobs.  indent / tool are UTF-8
 * (surrogatepass) of any length, in HOST memory; they are read during the
 * call (copied into the workspace when longer than 64 bytes). */
typedef struct {
  const char* indent;        /* EmitStyle.indent */
  uint64_t indent_len;
  const char* tool;          /* EmitStyle.tool */
  uint64_t tool_len;
  int32_t header;            /* EmitStyle.header */
  int32_t threads_per_block; /* 0 = default */
  int32_t slots;             /* concurrent per-thread arenas; 0 = auto */
  int32_t decode_only;       /* 1: run only the decode kernel */
  uint64_t arena_bytes;      /* bytes per slot arena; 0 = auto from max_code_len */
  int32_t skip_decode;       /* 1: reuse the records of a previous decode_only call on the same workspace */
  int32_t schedule;          /* 0: each thread takes the next root position; 1: warp-synchronous (a warp
                                takes 32 consecutive positions of `order` and its lanes start together);
                                2: warp-synchronous with statement-parallel emission (the warp emits
                                each of its 32 trees with the statements spread over its lanes);
                                3: split -- two launches per chunk of `slots` positions: every tree
                                is built (validate .. finish) into its own arena slot, then every
                                tree is emitted (source output only; `slots` = positions per chunk,
                                `arena_bytes` = bytes per slot); 4: as 3 with validate + analyze and
                                structure + finish in two launches (three per chunk) */
  int32_t max_depth;         /* device recursion guard (UPY_ST_DEPTH_LIMIT); 0 = default 600 */
  int32_t function_tree;     /* 1: emit_module([function_tree(root)]) without validation -- the
                                reference CLI's --function path (cli.py:75-78) -- instead of
                                decompile_source */
  int32_t output;            /* 0: source text (above); 1: the CFG export of `unpyre disasm --cfg --dot`
                                (cli.py:103-105): to_dot(analyze(root)[2]) (cfg.py:331-344,
                                pipeline.py:17-54) per root, no validation */
  int32_t pad0;
  const int32_t* order;      /* device pointer or NULL: the order in which root positions are taken (a
                                permutation of [0, n_roots)); results stay indexed by root position.
                                The host layer passes largest-tree-first (paper_2403_13839_b200
                                .api schedule "cost"), so big objects do not form the batch's tail */
} upy_options;

/* Per-root results (device pointers, caller-allocated). */
typedef struct {
  uint8_t*  text; uint64_t text_cap;  /* flat UTF-8 output; text of root i at text_off[i] */
  uint64_t* text_used;                /* device counter, caller zeroes before the call */
  uint64_t* text_off;                 /* [n_roots] */
  uint32_t* text_len;                 /* [n_roots] */
  int32_t*  status;                   /* [n_roots] UPY_ST_* (decompile text or error message) */
  int64_t*  aux;                      /* [n_roots*2] error attributes */
} upy_out;

/* Decoded instruction record written by the decode kernel (disasm.py:28-43). */
typedef struct {
  uint32_t offset;      /* extent start incl. EXTENDED_ARG prefixes */
  uint32_t arg;         /* folded arg (saturated at 2^32-1, see flags) */
  uint8_t  opcode;
  uint8_t  n_prefixes;
  uint8_t  cache_units;
  uint8_t  flags;       /* bit0 has_arg, bit1 arg saturated, bit2 is_jump_target */
} upy_ins;

/* Per-object decode result. */
typedef struct {
  int32_t status;       /* UPY_ST_OK or a decode error */
  int32_t n_instrs;
  int64_t aux0, aux1;   /* error attributes (opcode/offset, offset/target, position) */
} upy_decoded;

/* Stack-depth scan record, one per decoded instruction (same index as upy_ins):
 * the symbolic stack depth after the instruction along the fall-through edge,
 * relative to the entry of its segment -- the run of instructions from one
 * instruction-rule block leader (first instruction, jump target, instruction
 * after a block ender; cfg.py:72-86) to the next.  Every reference basic block
 * lies inside one segment, so a block entered at depth E has depth
 * E + depth[i] - depth[lo-1] after instruction i (depth[lo-1] = 0 when lo starts
 * a segment).  Effects per symexec.py's transfer functions. */
typedef struct {
  int16_t depth;
  uint8_t flags;        /* bit0 segment start, bit1 depth unknown (a contents-dependent effect
                           earlier in the segment), bit2 block ender */
  uint8_t pad;
} upy_stackrec;
/* Per-object summary of the scan. */
typedef struct {
  int32_t status;       /* the object's decode status (UPY_ST_OK or a decode error: no records) */
  int32_t n_segments;
  int32_t max_depth;    /* max / min relative depth over known positions */
  int32_t min_depth;
  int32_t n_pushes;     /* sum of positive known effects (symbolic values created) */
  int32_t n_unknown;    /* instructions with a contents-dependent effect */
} upy_stackinfo;
enum {
  UPY_ST_OK = 0, UPY_ST_UNPYRE = 1, UPY_ST_UNKNOWN_OPCODE = 2, UPY_ST_TRUNCATED_CODE = 3,
  UPY_ST_BAD_JUMP_TARGET = 4, UPY_ST_MALFORMED_EXCTABLE = 5, UPY_ST_STACK_UNDERFLOW = 6,
  UPY_ST_UNSUPPORTED_OPCODE = 7, UPY_ST_STACK_DEPTH_MISMATCH = 8, UPY_ST_STRUCTURING_FAILED = 9,
  UPY_ST_MARKER_LEAK = 10,
  /* loader errors (upy_pyc_load, include/upy_pyc.h; pyc.py:36-352) */
  UPY_ST_UNKNOWN_MAGIC = 11, UPY_ST_TRUNCATED_HEADER = 12, UPY_ST_MALFORMED_MARSHAL = 13,
  UPY_ST_PY_INDEX_ERROR = 20, UPY_ST_PY_ATTRIBUTE_ERROR = 21, UPY_ST_PY_TYPE_ERROR = 22,
  UPY_ST_PY_KEY_ERROR = 23, UPY_ST_PY_VALUE_ERROR = 24, UPY_ST_PY_RECURSION_ERROR = 25,
  UPY_ST_ARENA_OVERFLOW = 30, UPY_ST_OUTPUT_OVERFLOW = 31, UPY_ST_DEPTH_LIMIT = 32,
  UPY_ST_INTERNAL = 33, UPY_ST_NOT_RUN = 34
};

/* sizeof() of the ABI structs, for binding-side layout checks:
 * which = 0 upy_obj, 1 upy_const, 2 upy_str, 3 upy_arena, 4 upy_options, 5 upy_out,
 *         6 upy_ins, 7 upy_decoded, 8 upy_stackrec, 9 upy_stackinfo.  Returns 0 for unknown. */
size_t upy_abi_sizeof(int which);
int upy_abi_version(void);

/* Workspace bytes needed by upy_decompile_batch for this arena and options
 * (opt may be NULL: default style and knobs). */
int upy_query_workspace(const upy_arena* arena, const upy_options* opt, size_t* ws_bytes);

/* Decompile every root of the arena (≡ decompile_source per root, pipeline.py:143).
 * Returns 0 on success of the launch sequence; per-root failures are in out->status.
 * stream is a cudaStream_t. */
int upy_decompile_batch(const upy_arena* arena, const upy_options* opt, const upy_out* out,
                        void* workspace, size_t ws_bytes, void* stream);

/* Decode every object of the arena (≡ decode_instructions, disasm.py:71-172).
 * ins must hold total_code_units records; record j of object o lives at
 * ins[objs[o].code_off/2 + j].  Returns 0 on launch success. */
int upy_decode_batch(const upy_arena* arena, upy_ins* ins, upy_decoded* dec, void* stream);

/* Stack-depth scan (north-star subsystem 3) over the records of a
 * previous upy_decode_batch on the same ins / dec: one upy_stackrec per record
 * (stack[objs[o].code_off/2 + i]) and one upy_stackinfo per object.  Warp per
 * object, segmented warp scan.  Returns 0 on launch success. */
int upy_stackscan_batch(const upy_arena* arena, const upy_ins* ins, const upy_decoded* dec, upy_stackrec* stack,
                        upy_stackinfo* info, void* stream);
/* Last API-level error message of this thread ("" when none). */
const char* upy_last_error(void);
/* Kernels this library has launched in this process (all devices, all entry points):
 * read before and after a region to count its launches. */
uint64_t upy_launch_count(void);


#ifdef __cplusplus
}
#endif
#endif
