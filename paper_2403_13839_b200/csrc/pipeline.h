// pipeline.h -- decompile_source for one root object (pipeline.py:121-160):
// validate (code_model.py:198-253) -> module/function tree -> emit_module
// (emitter.py:535-547).  The result text (or the error message) is left in
// `out`; the status in C->err.
#pragma once
#include "emitter.h"

struct EmitOpts {
  bool header;
  bool function_tree;  // CLI --function (cli.py:75-78): no validation, always a def
  Str indent;
  Str tool;
};

// ------------------------------------------------------------ validation
struct Validator {
  Dc* C;
  Text rep;        // "; "-joined violation messages
  u32 n_viol;
  u32 path_stack[64];
  int path_n;

  HD void add_begin(Str where) {
    if (n_viol) t_puts(C, &rep, "; ");
    n_viol++;
    t_str(C, &rep, where);
  }
  HD void add(Str where, const char* msg) {
    add_begin(where);
    t_puts(C, &rep, msg);
  }
  HD NOINL void one(u32 oi, Str path) {
    GUARD(C);
    CK(C);
    const upy_obj* o = obj_at(C, oi);
    Text wt = {nullptr, 0, 0};
    if (path.n) {
      t_str(C, &wt, path);
      t_puts(C, &wt, ": ");
    }
    Str where = t_as_str(&wt);
    for (int q = 0; q < path_n; q++) {
      if (path_stack[q] == oi) {
        add(where, "code constant cycle detected");
        return;
      }
    }
    if (path_n >= 64) {
      py_error(C, UPY_ST_PY_RECURSION_ERROR, "maximum recursion depth exceeded");
      return;
    }
    path_stack[path_n++] = oi;
    if (o->code_len % 2) add(where, "code length not word-aligned");
    if (!o->code_len) add(where, "empty code");
    if (o->stacksize < 0) add(where, "negative stacksize");
    if (o->flags < 0) add(where, "negative flags");
    if (o->exc_len && o->minor < 11) add(where, "exception table requires >=3.11");
    if (o->minor <= 10) {
      if (!(o->argcount + o->kwonlyargcount <= o->nlocals && o->nlocals <= (i64)o->n_varnames)) {
        add_begin(where);
        t_puts(C, &rep, "argcount ");
        t_i64(C, &rep, o->argcount);
        t_puts(C, &rep, "+kwonly ");
        t_i64(C, &rep, o->kwonlyargcount);
        t_puts(C, &rep, " vs nlocals ");
        t_i64(C, &rep, o->nlocals);
        t_puts(C, &rep, " vs varnames ");
        t_i64(C, &rep, o->n_varnames);
        t_puts(C, &rep, " inconsistent");
      }
    } else {
      if (o->nlocals != (i64)o->n_varnames) {
        add_begin(where);
        t_puts(C, &rep, "nlocals ");
        t_i64(C, &rep, o->nlocals);
        t_puts(C, &rep, " != len(varnames) ");
        t_i64(C, &rep, o->n_varnames);
      }
      if (o->argcount + o->kwonlyargcount > o->nlocals) add(where, "more arguments than local slots");
    }
    if (o->posonlyargcount > o->argcount) add(where, "posonlyargcount exceeds argcount");
    consts(oi, o->consts_off, o->n_consts, where, 0);
    path_n--;
  }
  HD void consts(u32 owner, u32 off, u32 n, Str where, int depth) {
    GUARD(C);
    CK(C);
    if (depth > 128) {
      add(where, "constant tree too deep");
      return;
    }
    for (u32 q = 0; q < n && !C->err; q++) {
      u32 cid = ref_at(C, (u64)off + q);
      u32 k = ckind(C, cid);
      if (k == UPY_C_CODE) {
        u32 child = (u32)cget(C, cid)->off;
        const upy_obj* co = obj_at(C, child);
        const upy_obj* oo = obj_at(C, owner);
        if (co->minor != oo->minor) {
          add_begin(where);
          t_puts(C, &rep, "nested code ");
          t_str_repr(C, &rep, obj_name(C, child));
          t_puts(C, &rep, " has version 3.");
          t_i64(C, &rep, co->minor);
          t_puts(C, &rep, ", parent has 3.");
          t_i64(C, &rep, oo->minor);
        }
        Text pt = {nullptr, 0, 0};
        t_str(C, &pt, where);
        t_str(C, &pt, obj_name(C, child));
        one(child, t_as_str(&pt));
      } else if (k == UPY_C_TUPLE || k == UPY_C_FROZENSET) {
        consts(owner, (u32)cget(C, cid)->off, cget(C, cid)->n, where, depth + 1);
      }
    }
  }
};

// function_tree / module_tree (pipeline.py:121-140) around a decompiled body
HD NOINL NV* root_tree_of(Dc* C, u32 oi, NV* body, bool function_tree = false) {
  CKR(C, nullptr);
  if (!function_tree && s_eqc(obj_name(C, oi), "<module>")) {
    if (body->n && is_k(body->d[0], S_ASSIGN)) {
      Node* first = body->d[0];
      if (first->l1->n == 1 && is_k(first->l1->d[0], E_NAME) && s_eqc(first->l1->d[0]->s, "__doc__") &&
          is_k(first->a, E_CONST))
        body->d[0] = mk1(C, S_EXPR, first->a);
    }
    return or_pass(C, body);
  }
  if (code_is_str_doc(C, oi)) {
    NV* b2 = nv1(C, mk1(C, S_EXPR, mk_const(C, obj_const_id(C, oi, 0))));
    vextend(C, b2, body);
    body = b2;
  }
  Node* params = params_from_code(C, oi, nullptr, nullptr);
  CKR(C, nullptr);
  Node* fn = mk(C, S_FUNCDEF);
  fn->s = obj_name(C, oi);
  fn->p = params;
  fn->l1 = or_pass(C, body);
  fn->l2 = vnew<Node*>(C);
  return nv1(C, fn);
}

HD inline NV* root_tree(Dc* C, u32 oi) { return root_tree_of(C, oi, decompile_body(C, oi)); }

// decompile_source (pipeline.py:143-160) + emit_module (emitter.py:535-547) as
// stages: validate | analyze | structure | finish + tree | emit.  The kernel
// either runs them back to back per thread or in warp lockstep.
enum { DS_VALIDATE, DS_ANALYZE, DS_STRUCTURE, DS_FINISH, DS_EMIT, DS_STAGES };
struct SourceJob {
  u32 oi;
  BodyJob body;
  NV* tree;
  const EmitOpts* opt;
  Text* out;
};

HD NOINL void ds_validate(Dc* C, SourceJob* S) {
  Validator V;
  V.C = C;
  V.rep = {nullptr, 0, 0};
  V.n_viol = 0;
  V.path_n = 0;
  V.one(S->oi, Str{"", 0});
  if (C->err) return;
  if (V.n_viol) {
    Text m;
    if (fail_begin(C, UPY_ST_UNPYRE, 0, 0, &m)) {
      m_puts(C, &m, "validation failed: ");
      m_putn(C, &m, V.rep.d, V.rep.n);
      fail_end(C, &m);
    }
  }
}

HD NOINL void ds_emit(Dc* C, SourceJob* S) {
  u32 oi = S->oi;
  NV* tree = S->tree;
  Text* out = S->out;
  t_grow(C, out, 3 * obj_at(C, oi)->code_len + 256);  // text is ~1.5-4.5x co_code
  Emitter E;
  E.C = C;
  E.out = out;
  E.depth = 0;
  E.indent = S->opt->indent;
  if (S->opt->header) {
    t_puts(C, out, "# decompiled by ");
    t_str(C, out, S->opt->tool);
    t_puts(C, out, " from ");
    Str qn = obj_qualname(C, oi);
    t_str(C, out, qn.n ? qn : obj_name(C, oi));
    t_puts(C, out, " (python 3.");
    t_i64(C, out, obj_at(C, oi)->minor);
    t_puts(C, out, ")\n");
  }
  if (!tree->n) E.simple_line("pass");
  for (u32 q = 0; q < tree->n && !C->err; q++) E.stmt(tree->d[q]);
}

// one stage of the root object; the root body holds one depth-guard level
// across its stages, like decompile_body's GUARD
HD inline void ds_stage(Dc* C, SourceJob* S, int stage) {
  if (C->err) return;
  switch (stage) {
    case DS_VALIDATE:
      if (!S->opt->function_tree) ds_validate(C, S);
      return;
    case DS_ANALYZE:
      S->body.oi = S->oi;
      if (++C->depth > C->max_depth) fail_msg(C, UPY_ST_DEPTH_LIMIT, "device recursion guard");
      else body_analyze(C, &S->body);
      return;
    case DS_STRUCTURE: body_structure(C, &S->body); return;
    case DS_FINISH:
      if (body_finish(C, &S->body)) {
        C->depth--;
        S->tree = root_tree_of(C, S->oi, S->body.stmts, S->opt->function_tree);
      }
      return;
    case DS_EMIT:
#ifndef UPY_SKIP_EMIT  // timing experiment only: the text stays empty
      ds_emit(C, S);
#endif
      return;
  }
}

#if defined(UPY_PHASE_PROF) && defined(__CUDACC__)
// Profiling variant (tools/build_variant.sh prof -DUPY_PHASE_PROF): thread-cycles
// per stage summed over all roots, read back with upy_prof_read.
__device__ unsigned long long g_stage_cycles[DS_STAGES];
#endif
// Stages validate .. finish of decompile_source: the tree to emit (S->tree), or C->err.
HD inline void decompile_tree(Dc* C, SourceJob* S) {
  for (int st = 0; st < DS_EMIT; st++) ds_stage(C, S, st);
}

HD inline void decompile_source(Dc* C, u32 oi, const EmitOpts* opt, Text* out) {
  SourceJob S;
  S.oi = oi;
  S.opt = opt;
  S.out = out;
  for (int st = 0; st < DS_STAGES; st++) {
#if defined(UPY_PHASE_PROF) && defined(__CUDA_ARCH__)
    long long t0 = clock64();
    ds_stage(C, &S, st);
    atomicAdd(&g_stage_cycles[st], (unsigned long long)(clock64() - t0));
#else
    ds_stage(C, &S, st);
#endif
  }
}
