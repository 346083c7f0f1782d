// model.h -- read-only views of the packed arena (include/upy.h) as the
// reference's CodeObject / Const model (code_model.py:46-180).
#pragma once
#include "common.h"

// Synthetic constants the path creates out of thin air (symexec.py:176,
// structurer.py:451).  Real consts are indices into arena->consts.
#define CID_NONE_SYN 0xFFFFFFF0u
#define CID_TRUE_SYN 0xFFFFFFF1u
#define CID_INVALID 0xFFFFFFFFu   // ConstE(None): argval of an out-of-range LOAD_CONST

struct Obj {
  const upy_obj* o;
  u32 idx;
};

HD inline const upy_obj* obj_at(const Dc* C, u32 i) { return &C->objs[i]; }
HD inline Str str_at(const Dc* C, u32 sid) {
  const upy_str& s = C->strs[sid];
  return Str{(const char*)(C->bytes + s.off), s.len};
}
HD inline u32 ref_at(const Dc* C, u64 i) { return C->refs[i]; }
HD inline Str obj_name(const Dc* C, u32 oi) { return str_at(C, obj_at(C, oi)->name); }
HD inline Str obj_qualname(const Dc* C, u32 oi) { return str_at(C, obj_at(C, oi)->qualname); }
HD inline Str obj_varname(const Dc* C, u32 oi, u32 k) {
  const upy_obj* o = obj_at(C, oi);
  return str_at(C, ref_at(C, (u64)o->varnames_off + k));
}
HD inline Str obj_tab(const Dc* C, u32 off, u32 k) { return str_at(C, ref_at(C, (u64)off + k)); }
HD inline u32 obj_const_id(const Dc* C, u32 oi, u32 k) {
  return ref_at(C, (u64)obj_at(C, oi)->consts_off + k);
}

// const kinds (upy.h UPY_C_*); synthetic ids map to none / bool
HD inline u32 ckind(const Dc* C, u32 cid) {
  if (cid == CID_NONE_SYN) return UPY_C_NONE;
  if (cid == CID_TRUE_SYN) return UPY_C_BOOL;
  return C->consts[cid].kind;
}
HD inline const upy_const* cget(const Dc* C, u32 cid) { return &C->consts[cid]; }
HD inline Str cstr(const Dc* C, u32 cid) {
  const upy_const* k = cget(C, cid);
  return Str{(const char*)(C->bytes + k->off), k->n};
}
HD inline u32 celem(const Dc* C, u32 cid, u32 i) { return ref_at(C, cget(C, cid)->off + i); }
HD inline u32 cnelem(const Dc* C, u32 cid) { return cget(C, cid)->n; }
HD inline int cbool(const Dc* C, u32 cid) { return cid == CID_TRUE_SYN ? 1 : cget(C, cid)->ival; }

// localsplus (code_model.py:129-139): varnames + cells not in varnames + freevars
HD inline Str obj_localsplus(const Dc* C, u32 oi, u32 k, bool* ok) {
  const upy_obj* o = obj_at(C, oi);
  *ok = true;
  if (k < o->n_varnames) return obj_tab(C, o->varnames_off, k);
  u32 r = k - o->n_varnames;
  for (u32 c = 0; c < o->n_cellvars; c++) {
    Str cv = obj_tab(C, o->cellvars_off, c);
    bool in_vars = false;
    for (u32 v = 0; v < o->n_varnames && !in_vars; v++)
      in_vars = s_eq(cv, obj_tab(C, o->varnames_off, v));
    if (in_vars) continue;
    if (r == 0) return cv;
    r--;
  }
  if (r < o->n_freevars) return obj_tab(C, o->freevars_off, r);
  *ok = false;
  return Snone();
}
HD inline u32 obj_n_localsplus(const Dc* C, u32 oi) {
  const upy_obj* o = obj_at(C, oi);
  u32 n = o->n_varnames + o->n_freevars;
  for (u32 c = 0; c < o->n_cellvars; c++) {
    Str cv = obj_tab(C, o->cellvars_off, c);
    bool in_vars = false;
    for (u32 v = 0; v < o->n_varnames && !in_vars; v++)
      in_vars = s_eq(cv, obj_tab(C, o->varnames_off, v));
    if (!in_vars) n++;
  }
  return n;
}
// deref_names (code_model.py:141-145)
HD inline Str obj_deref_name(const Dc* C, u32 oi, u32 k, bool* ok) {
  const upy_obj* o = obj_at(C, oi);
  if (o->minor >= 11) return obj_localsplus(C, oi, k, ok);
  *ok = true;
  if (k < o->n_cellvars) return obj_tab(C, o->cellvars_off, k);
  if (k - o->n_cellvars < o->n_freevars) return obj_tab(C, o->freevars_off, k - o->n_cellvars);
  *ok = false;
  return Snone();
}

// ------------------------------------------------------------ const equality
// Const._key() equality (code_model.py:61-86): bit-pattern floats, bool != int,
// frozenset as a set of keys, code by CodeObject._key().
HD bool const_key_eq(Dc* C, u32 a, u32 b);
HD bool code_key_eq(Dc* C, u32 oa, u32 ob);

HD inline bool limbs_eq(const Dc* C, const upy_const* x, const upy_const* y) {
  // normalized magnitudes (packer strips leading zero limbs except a single zero)
  if (x->ival != y->ival) return false;
  u32 nx = x->n, ny = y->n;
  const u32* lx = C->limbs + x->off;
  const u32* ly = C->limbs + y->off;
  while (nx > 1 && lx[nx - 1] == 0) nx--;
  while (ny > 1 && ly[ny - 1] == 0) ny--;
  if (nx != ny) return false;
  for (u32 i = 0; i < nx; i++)
    if (lx[i] != ly[i]) return false;
  return true;
}
HD inline bool bytes_eq(const Dc* C, u64 oa, u32 na, u64 ob, u32 nb) {
  if (na != nb) return false;
  const u8* p = C->bytes;
  for (u32 i = 0; i < na; i++)
    if (p[oa + i] != p[ob + i]) return false;
  return true;
}
HD inline u64 dbits(double d) {
  u64 u;
  memcpy(&u, &d, 8);
  return u;
}

HD NOINL bool const_key_eq(Dc* C, u32 a, u32 b) {
  GUARD(C);
  CKR(C, false);
  if (a == b) return true;
  u32 ka = ckind(C, a), kb = ckind(C, b);
  if (ka != kb) return false;
  switch (ka) {
    case UPY_C_NONE:
    case UPY_C_ELLIPSIS:
      return true;
    case UPY_C_BOOL:
      return cbool(C, a) == cbool(C, b);
    case UPY_C_INT:
      return limbs_eq(C, cget(C, a), cget(C, b));
    case UPY_C_FLOAT:
      return dbits(cget(C, a)->re) == dbits(cget(C, b)->re);
    case UPY_C_COMPLEX:
      return dbits(cget(C, a)->re) == dbits(cget(C, b)->re) &&
             dbits(cget(C, a)->im) == dbits(cget(C, b)->im);
    case UPY_C_STR:
    case UPY_C_BYTES:
      return bytes_eq(C, cget(C, a)->off, cget(C, a)->n, cget(C, b)->off, cget(C, b)->n);
    case UPY_C_TUPLE: {
      u32 n = cnelem(C, a);
      if (n != cnelem(C, b)) return false;
      for (u32 i = 0; i < n; i++)
        if (!const_key_eq(C, celem(C, a, i), celem(C, b, i))) return false;
      return true;
    }
    case UPY_C_FROZENSET: {
      // set-of-keys equality: every element of each side has an equal on the other
      u32 na = cnelem(C, a), nb = cnelem(C, b);
      for (u32 i = 0; i < na; i++) {
        bool f = false;
        for (u32 j = 0; j < nb && !f; j++) f = const_key_eq(C, celem(C, a, i), celem(C, b, j));
        if (!f) return false;
      }
      for (u32 j = 0; j < nb; j++) {
        bool f = false;
        for (u32 i = 0; i < na && !f; i++) f = const_key_eq(C, celem(C, b, j), celem(C, a, i));
        if (!f) return false;
      }
      return true;
    }
    case UPY_C_CODE:
      return code_key_eq(C, (u32)cget(C, a)->off, (u32)cget(C, b)->off);
  }
  return false;
}

HD inline bool strtab_eq(Dc* C, u32 offa, u32 na, u32 offb, u32 nb) {
  if (na != nb) return false;
  for (u32 i = 0; i < na; i++)
    if (!s_eq(obj_tab(C, offa, i), obj_tab(C, offb, i))) return false;
  return true;
}

// CodeObject._key() (code_model.py:147-164): excludes filename/linetable/exctable/qualname
HD NOINL bool code_key_eq(Dc* C, u32 ia, u32 ib) {
  if (ia == ib) return true;
  const upy_obj* a = obj_at(C, ia);
  const upy_obj* b = obj_at(C, ib);
  if (a->minor != b->minor || a->argcount != b->argcount || a->posonlyargcount != b->posonlyargcount ||
      a->kwonlyargcount != b->kwonlyargcount || a->nlocals != b->nlocals || a->stacksize != b->stacksize ||
      a->flags != b->flags || a->firstlineno != b->firstlineno)
    return false;
  if (!bytes_eq(C, a->code_off, a->code_len, b->code_off, b->code_len)) return false;
  if (a->n_consts != b->n_consts) return false;
  for (u32 i = 0; i < a->n_consts; i++)
    if (!const_key_eq(C, ref_at(C, (u64)a->consts_off + i), ref_at(C, (u64)b->consts_off + i))) return false;
  if (!strtab_eq(C, a->names_off, a->n_names, b->names_off, b->n_names)) return false;
  if (!strtab_eq(C, a->varnames_off, a->n_varnames, b->varnames_off, b->n_varnames)) return false;
  if (!strtab_eq(C, a->freevars_off, a->n_freevars, b->freevars_off, b->n_freevars)) return false;
  if (!strtab_eq(C, a->cellvars_off, a->n_cellvars, b->cellvars_off, b->n_cellvars)) return false;
  return s_eq(str_at(C, a->name), str_at(C, b->name));
}

// Full dataclass equality of CodeObject (FuncExpr.code compare): all 19 fields.
HD inline bool code_full_eq(Dc* C, u32 ia, u32 ib) {
  if (ia == ib) return true;
  if (!code_key_eq(C, ia, ib)) return false;
  const upy_obj* a = obj_at(C, ia);
  const upy_obj* b = obj_at(C, ib);
  return s_eq(str_at(C, a->filename), str_at(C, b->filename)) &&
         bytes_eq(C, a->lnt_off, a->lnt_len, b->lnt_off, b->lnt_len) &&
         bytes_eq(C, a->exc_off, a->exc_len, b->exc_off, b->exc_len) &&
         s_eq(str_at(C, a->qualname), str_at(C, b->qualname));
}
