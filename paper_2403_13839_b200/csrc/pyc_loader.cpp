// pyc_loader.cpp -- native .pyc loader: PEP 552 header + marshal stream of
// 3.8-3.11 code objects straight into the device arena layout (include/upy.h),
// with the reference's exact acceptance rules and error messages.
//
// Reference: /root/reference/pkg/src/unpyre/pyc.py
//   parse_pyc_header / load_pyc   :36-52   (TruncatedHeader, UnknownMagic)
//   _Reader.read_object           :78-152  (FLAG_REF slots, 'r' back-references,
//                                           nesting limit 256, unsupported types)
//   _read_* handlers              :155-233
//   _expect / _expect_str_tuple   :236-244
//   _read_code                    :247-321 (3.8-3.10 and 3.11 field layouts,
//                                           localsplus reconstruction check)
//   parse_marshal                 :346-352
// and the CodeObject defaults of code_model.py:101-127 (qualname = name when
// empty; 3.11 nlocals = len(varnames)).
//
// Files are parsed independently (one worker thread per slice of files) into
// per-file section vectors, then concatenated into one 256-B-aligned image:
// every file's co_code segments first (16-B aligned, so decoded record i of an
// object lives at code_off/2 + i), then exception/line tables and payloads.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <stddef.h>
#include <stdint.h>

// The device headers define their out-of-line (__noinline__) helpers without
// `inline`; upy.cu defines the same symbols, so this host-side copy (used for
// Python str repr in error messages) gets its own namespace.
namespace pyc_host {
#include "numfmt.h"
#include "../../include/upy_pyc.h"
}  // namespace pyc_host
using namespace pyc_host;

namespace {

enum { S_OBJS, S_CONSTS, S_STRS, S_REFS, S_LIMBS, S_BYTES, S_ROOTS, S_N };

struct Fail {};  // unwinds a file's parse; the message is in Parser::msg

// Output of one worker thread: the sections of its (contiguous) slice of files,
// indices local to the thread; merged into the image by rebasing.
struct ThreadOut {
  std::vector<upy_obj> objs;
  std::vector<upy_const> consts;
  std::vector<upy_str> strs;
  std::vector<u32> refs;
  std::vector<u8> ref_is_str;  // rebase refs by the const or the str base
  std::vector<u32> limbs;
  std::vector<u8> code;        // co_code segments, 16-B aligned
  std::vector<u8> rest;        // exception/line tables, str/bytes payloads
  u64 max_code = 0;
  void mark(u64* m) const {
    m[0] = objs.size(), m[1] = consts.size(), m[2] = strs.size(), m[3] = refs.size();
    m[4] = limbs.size(), m[5] = code.size(), m[6] = rest.size();
  }
  void rollback(const u64* m) {
    objs.resize(m[0]), consts.resize(m[1]), strs.resize(m[2]), refs.resize(m[3]);
    ref_is_str.resize(m[3]), limbs.resize(m[4]), code.resize(m[5]), rest.resize(m[6]);
  }
};

struct FileRes {
  i32 status = UPY_ST_OK;
  i32 root = -1;  // thread-local object index
  i64 aux = 0;
  std::string msg;
};

const char* kind_name(u8 k) {
  switch (k) {
    case UPY_C_NONE: return "none";
    case UPY_C_BOOL: return "bool";
    case UPY_C_INT: return "int";
    case UPY_C_FLOAT: return "float";
    case UPY_C_COMPLEX: return "complex";
    case UPY_C_STR: return "str";
    case UPY_C_BYTES: return "bytes";
    case UPY_C_TUPLE: return "tuple";
    case UPY_C_FROZENSET: return "frozenset";
    case UPY_C_CODE: return "code";
    default: return "ellipsis";
  }
}

// UTF-8 with lone surrogates allowed (decode("utf-8", "surrogatepass")).
bool utf8_surrogatepass_ok(const u8* p, u64 n) {
  u64 i = 0;
  while (i < n) {
    u8 c = p[i];
    if (c < 0x80) {
      i++;
      continue;
    }
    u32 need, cp;
    if (c >= 0xC2 && c <= 0xDF) need = 1, cp = c & 0x1F;
    else if (c >= 0xE0 && c <= 0xEF) need = 2, cp = c & 0x0F;
    else if (c >= 0xF0 && c <= 0xF4) need = 3, cp = c & 0x07;
    else return false;
    if (i + need >= n) return false;  // truncated sequence
    for (u32 k = 1; k <= need; k++) {
      u8 d = p[i + k];
      if ((d & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (d & 0x3F);
    }
    if (need == 2 && cp < 0x800) return false;
    if (need == 3 && (cp < 0x10000 || cp > 0x10FFFF)) return false;
    i += need + 1;
  }
  return true;
}

// float(ascii_text) acceptance (Python's float() on a str: surrounding
// whitespace, optional sign, decimal literal with single underscores between
// digits, or inf/infinity/nan in any case).  Returns false when Python raises.
bool py_float_from_ascii(const u8* p, u64 n, double* out) {
  u64 a = 0, b = n;
  auto ws = [](u8 c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r' ||
                              c == 0x1c || c == 0x1d || c == 0x1e || c == 0x1f; };
  while (a < b && ws(p[a])) a++;
  while (b > a && ws(p[b - 1])) b--;
  if (a == b) return false;
  std::string s;
  u64 i = a;
  bool neg = false;
  if (p[i] == '+' || p[i] == '-') neg = p[i++] == '-';
  std::string rest;
  for (u64 k = i; k < b; k++) rest.push_back((char)(p[k] >= 'A' && p[k] <= 'Z' ? p[k] + 32 : p[k]));
  if (rest == "inf" || rest == "infinity") {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (rest == "nan") {
    *out = neg ? -NAN : NAN;
    return true;
  }
  // digits [. digits] [e [sign] digits], underscores only between two digits
  auto digit = [](u8 c) { return c >= '0' && c <= '9'; };
  s.push_back(neg ? '-' : '+');
  u64 k = i;
  auto run = [&](bool& any) {
    any = false;
    while (k < b) {
      if (digit(p[k])) {
        s.push_back((char)p[k++]);
        any = true;
      } else if (p[k] == '_' && any && k + 1 < b && digit(p[k + 1])) {
        k++;
      } else {
        break;
      }
    }
  };
  bool int_digits, frac_digits = false;
  run(int_digits);
  if (k < b && p[k] == '.') {
    s.push_back('.');
    k++;
    run(frac_digits);
  }
  if (!int_digits && !frac_digits) return false;
  if (k < b && (p[k] == 'e' || p[k] == 'E')) {
    s.push_back('e');
    k++;
    if (k < b && (p[k] == '+' || p[k] == '-')) s.push_back((char)p[k++]);
    bool exp_digits;
    run(exp_digits);
    if (!exp_digits) return false;
  }
  if (k != b) return false;
  *out = strtod(s.c_str(), nullptr);
  return true;
}

// One parsed marshal value (the reference's Const).  Const rows and str-table
// rows are created lazily, only when the value is used as a constant
// (co_consts) or as a name: most strings of a file are names only.
struct Val {
  u8 kind;
  u8 in_code;  // bytes moved into the code region (a co_code payload)
  i32 cid;   // const row (-1 until used as a constant)
  i32 sid;   // str row (-1 until used as a name)
  i32 ival;  // bool value / int sign
  u32 n;     // str/bytes length; int limb count; tuple element count
  u64 off;   // str/bytes: rest offset; int: limb offset; tuple: kids offset; code: object index
  double re, im;
};

struct Parser {
  const u8* d;
  u64 n;
  u64 pos;
  int minor;
  int depth;
  std::vector<i32> refs;  // marshal ref table: index into vals, -1 = reserved (incomplete)
  std::vector<Val> vals;
  std::vector<i32> kids;  // tuple elements (value indices)
  ThreadOut* T;
  std::string msg;
  u64 fail_off;

  [[noreturn]] void fail(const std::string& m, i64 off = -1) {
    msg = m;
    fail_off = off < 0 ? pos : (u64)off;
    throw Fail{};
  }
  [[noreturn]] void fail_take(u64 k) {
    fail("need " + std::to_string(k) + " bytes, " + std::to_string(n - pos) + " left");
  }
  const u8* take(u64 k) {
    if (k > n - pos) fail_take(k);
    const u8* p = d + pos;
    pos += k;
    return p;
  }
  u32 u8_() {
    if (pos >= n) fail_take(1);
    return d[pos++];
  }
  i32 i32_() {
    const u8* p = take(4);
    return (i32)((u32)p[0] | ((u32)p[1] << 8) | ((u32)p[2] << 16) | ((u32)p[3] << 24));
  }
  static double f64_(const u8* p) {
    double v;
    memcpy(&v, p, 8);
    return v;
  }

  i32 new_val(u8 kind) {
    Val v;
    memset(&v, 0, sizeof v);
    v.kind = kind;
    v.cid = v.sid = -1;
    vals.push_back(v);
    return (i32)vals.size() - 1;
  }
  u64 put_rest(const u8* p, u64 k) {
    u64 off = T->rest.size();
    T->rest.insert(T->rest.end(), p, p + k);
    return off;
  }
  i32 str_val(u64 off, u64 k) {
    i32 v = new_val(UPY_C_STR);
    vals[v].off = off;
    vals[v].n = (u32)k;
    return v;
  }
  i32 latin1_val(const u8* p, u64 k) {
    u64 off = T->rest.size();
    u64 hi = 0;
    for (u64 i = 0; i < k; i++) hi += p[i] >> 7;
    if (!hi) {
      T->rest.insert(T->rest.end(), p, p + k);
    } else {
      T->rest.reserve(T->rest.size() + k + hi);
      for (u64 i = 0; i < k; i++) {
        if (p[i] < 0x80) {
          T->rest.push_back(p[i]);
        } else {
          T->rest.push_back((u8)(0xC0 | (p[i] >> 6)));
          T->rest.push_back((u8)(0x80 | (p[i] & 0x3F)));
        }
      }
    }
    return str_val(off, k + hi);
  }
  i32 sid_of(i32 v) {  // str-table row of a str value
    if (vals[v].sid < 0) {
      upy_str s;
      s.off = vals[v].off;
      s.len = vals[v].n;
      s.pad = 0;
      T->strs.push_back(s);
      vals[v].sid = (i32)T->strs.size() - 1;
    }
    return vals[v].sid;
  }
  i32 cid_of(i32 v) {  // const row of a value (tuples: elements first)
    if (vals[v].cid >= 0) return vals[v].cid;
    upy_const c;
    memset(&c, 0, sizeof c);
    c.kind = vals[v].kind;
    c.ival = vals[v].ival;
    c.n = vals[v].n;
    c.off = vals[v].off;
    c.re = vals[v].re;
    c.im = vals[v].im;
    if (c.kind == UPY_C_TUPLE || c.kind == UPY_C_FROZENSET) {
      u64 k0 = vals[v].off;
      u32 cnt = vals[v].n;
      std::vector<u32> ids(cnt);
      for (u32 i = 0; i < cnt; i++) ids[i] = (u32)cid_of(kids[k0 + i]);
      c.off = T->refs.size();
      T->refs.insert(T->refs.end(), ids.begin(), ids.end());
      T->ref_is_str.insert(T->ref_is_str.end(), cnt, (u8)0);
    }
    c.pad = vals[v].in_code;  // merge-time marker: rebase by the code region, then cleared
    T->consts.push_back(c);
    vals[v].cid = (i32)T->consts.size() - 1;
    return vals[v].cid;
  }

  // pyc.py:105-152
  i32 read_object() {
    u64 start = pos;
    if (depth >= 256) fail("marshal nesting too deep", (i64)start);
    u32 tbyte = u8_();
    bool flag_ref = (tbyte & 0x80) != 0;
    u32 t = tbyte & 0x7F;
    if (t == 'r') {
      i32 idx = i32_();
      if (idx < 0 || (u64)idx >= refs.size()) fail("reference " + std::to_string(idx) + " out of range", (i64)start);
      if (refs[idx] < 0) fail("reference " + std::to_string(idx) + " to incomplete object", (i64)start);
      return refs[idx];
    }
    if (t == 'N' || t == 'T' || t == 'F' || t == '.') {
      i32 v = new_val(t == 'N' ? UPY_C_NONE : t == '.' ? UPY_C_ELLIPSIS : UPY_C_BOOL);
      vals[v].ival = t == 'T';
      if (flag_ref) refs.push_back(v);
      return v;
    }
    const char* unsup = t == '[' ? "list" : t == '{' ? "dict" : t == '<' ? "set" : t == 'S' ? "StopIteration"
                        : t == '0' ? "NULL" : t == '?' ? "unknown" : nullptr;
    if (unsup) fail(std::string("marshal type '") + unsup + "' not produced by compile", (i64)start);
    if (t == 0 || !strchr("ilgfysutaAzZ()>c", (int)t)) {
      char b[64];
      snprintf(b, sizeof b, "bad marshal type byte 0x%02x", t);  // Python f"{t:#04x}"
      fail(b, (i64)start);
    }
    bool container = t == '(' || t == ')' || t == '>' || t == 'c';
    i64 slot = -1;
    if (flag_ref && container) {
      slot = (i64)refs.size();
      refs.push_back(-1);
    }
    depth++;
    i32 v = handler(t);
    depth--;
    if (slot >= 0) refs[slot] = v;
    else if (flag_ref) refs.push_back(v);
    return v;
  }

  i32 handler(u32 t) {
    switch (t) {
      case 'i': {  // pyc.py:155-156
        i32 x = i32_();
        i32 v = new_val(UPY_C_INT);
        vals[v].ival = x > 0 ? 1 : x < 0 ? -1 : 0;
        vals[v].n = 1;
        vals[v].off = T->limbs.size();
        T->limbs.push_back(x < 0 ? (u32)(-(i64)x) : (u32)x);
        return v;
      }
      case 'l': {  // pyc.py:159-168: 15-bit digits, little-endian
        i32 nd = i32_();
        u64 ndigits = nd < 0 ? (u64)(-(i64)nd) : (u64)nd;
        u64 base = T->limbs.size();
        u64 bit = 0;
        for (u64 i = 0; i < ndigits; i++) {
          const u8* p = take(2);
          u32 dg = (u32)p[0] | ((u32)p[1] << 8);
          if (dg >= (1u << 15)) fail("long digit out of range");
          u64 w = bit >> 5, sh = bit & 31;
          while (T->limbs.size() < base + w + 2) T->limbs.push_back(0);
          T->limbs[base + w] |= dg << sh;
          if (sh > 17) T->limbs[base + w + 1] |= dg >> (32 - sh);
          bit += 15;
        }
        while (T->limbs.size() > base + 1 && T->limbs.back() == 0) T->limbs.pop_back();
        if (T->limbs.size() == base) T->limbs.push_back(0);
        u32 cnt = (u32)(T->limbs.size() - base);
        bool zero = cnt == 1 && T->limbs[base] == 0;
        i32 v = new_val(UPY_C_INT);
        vals[v].ival = zero ? 0 : (nd < 0 ? -1 : 1);
        vals[v].n = cnt;
        vals[v].off = base;
        return v;
      }
      case 'g': {  // pyc.py:171-172
        double x = f64_(take(8));
        i32 v = new_val(UPY_C_FLOAT);
        vals[v].re = x;
        return v;
      }
      case 'f': {  // pyc.py:175-180
        u32 k = u8_();
        const u8* p = take(k);
        double x;
        bool ascii = true;
        for (u32 i = 0; i < k; i++) ascii = ascii && p[i] < 0x80;
        if (!ascii || !py_float_from_ascii(p, k, &x)) fail("bad text float");
        i32 v = new_val(UPY_C_FLOAT);
        vals[v].re = x;
        return v;
      }
      case 'y': {  // pyc.py:183-185
        const u8* p = take(16);
        i32 v = new_val(UPY_C_COMPLEX);
        vals[v].re = f64_(p);
        vals[v].im = f64_(p + 8);
        return v;
      }
      case 's': {  // pyc.py:188-192
        i32 k = i32_();
        if (k < 0) fail("negative bytes length");
        const u8* p = take((u64)k);
        i32 v = new_val(UPY_C_BYTES);
        vals[v].off = put_rest(p, (u64)k);
        vals[v].n = (u32)k;
        return v;
      }
      case 'u':
      case 't': {  // pyc.py:195-202
        i32 k = i32_();
        if (k < 0) fail("negative string length");
        const u8* p = take((u64)k);
        if (!utf8_surrogatepass_ok(p, (u64)k)) fail("undecodable unicode payload");
        return str_val(put_rest(p, (u64)k), (u64)k);
      }
      case 'a':
      case 'A': {  // pyc.py:205-209
        i32 k = i32_();
        if (k < 0) fail("negative string length");
        const u8* p = take((u64)k);
        return latin1_val(p, (u64)k);
      }
      case 'z':
      case 'Z': {  // pyc.py:212-214
        u32 k = u8_();
        const u8* p = take(k);
        return latin1_val(p, k);
      }
      case '(':
      case ')':
      case '>': {  // pyc.py:217-233
        i64 k;
        if (t == ')') {
          k = u8_();
        } else {
          k = i32_();
          if (k < 0) fail(t == '>' ? "negative frozenset length" : "negative tuple length");
        }
        // elements are read first (they may be tuples themselves), then copied
        // contiguously into kids
        std::vector<i32> el;
        el.reserve(k < 64 ? (size_t)k : 64);
        for (i64 i = 0; i < k; i++) el.push_back(read_object());
        i32 v = new_val(t == '>' ? UPY_C_FROZENSET : UPY_C_TUPLE);
        vals[v].n = (u32)k;
        vals[v].off = kids.size();
        kids.insert(kids.end(), el.begin(), el.end());
        return v;
      }
      case 'c':
        return read_code();
    }
    fail("internal");
  }

  i32 expect(i32 v, u8 what) {  // pyc.py:236-239
    if (vals[v].kind != what)
      fail(std::string("expected ") + kind_name(what) + " in code object, got " + kind_name(vals[v].kind));
    return v;
  }
  void expect_str_tuple(i32 v, std::vector<i32>* out) {  // pyc.py:242-244
    expect(v, UPY_C_TUPLE);
    out->clear();
    for (u32 i = 0; i < vals[v].n; i++) out->push_back(expect(kids[vals[v].off + i], UPY_C_STR));
  }
  bool s_same(i32 a, i32 b) {
    const Val& x = vals[a];
    const Val& y = vals[b];
    return x.n == y.n && (x.n == 0 || memcmp(&T->rest[x.off], &T->rest[y.off], x.n) == 0);
  }
  void str_list(const std::vector<i32>& items, u32* off, u32* cnt) {
    *off = (u32)T->refs.size();
    *cnt = (u32)items.size();
    for (i32 x : items) {
      T->refs.push_back((u32)sid_of(x));
      T->ref_is_str.push_back(1);
    }
  }

  const u8* bytes_ptr(i32 v) { return (vals[v].in_code ? T->code.data() : T->rest.data()) + vals[v].off; }
  // co_code payloads live in the code region (16-B aligned segments at the front
  // of the bytes section).  A payload this read just appended to rest moves
  // instead of being copied; a back-reference to an earlier bytes object (a
  // constant, a line table, ... whose rest offset is already recorded) is
  // copied, and one to an earlier co_code is shared.  `fresh` = the first value
  // index created by the read that produced v.
  i32 to_code_region(i32 v, i32 fresh) {
    Val& x = vals[v];
    if (x.in_code) return v;
    u64 off = T->code.size();
    T->code.insert(T->code.end(), T->rest.begin() + x.off, T->rest.begin() + x.off + x.n);
    T->code.resize((T->code.size() + 15) & ~(size_t)15, 0);
    if (v >= fresh && x.off + x.n == T->rest.size()) {
      T->rest.resize(x.off);
      x.in_code = 1;
      x.off = off;
      return v;
    }
    i32 c = new_val(UPY_C_BYTES);
    vals[c].in_code = 1;
    vals[c].off = off;
    vals[c].n = vals[v].n;
    return c;
  }
  i32 in_rest(i32 v) {  // line/exception tables are addressed in the rest region
    if (!vals[v].in_code) return v;
    i32 c = new_val(UPY_C_BYTES);
    vals[c].n = vals[v].n;
    vals[c].off = put_rest(bytes_ptr(v), vals[v].n);
    return c;
  }

  // pyc.py:247-321
  i32 read_code() {
    upy_obj o;
    memset(&o, 0, sizeof o);
    o.minor = (u32)minor;
    o.argcount = i32_();
    o.posonlyargcount = i32_();
    o.kwonlyargcount = i32_();
    if (minor <= 10) o.nlocals = i32_();
    o.stacksize = i32_();
    o.flags = i32_();
    const i32 fresh = (i32)vals.size();
    i32 code = to_code_region(expect(read_object(), UPY_C_BYTES), fresh);
    i32 consts = expect(read_object(), UPY_C_TUPLE);
    std::vector<i32> names, varnames, freevars, cellvars, lp;
    expect_str_tuple(read_object(), &names);
    i32 filename, name, qualname, linetable, exctable = -1;
    if (minor <= 10) {
      expect_str_tuple(read_object(), &varnames);
      expect_str_tuple(read_object(), &freevars);
      expect_str_tuple(read_object(), &cellvars);
      filename = expect(read_object(), UPY_C_STR);
      name = expect(read_object(), UPY_C_STR);
      qualname = name;
      o.firstlineno = i32_();
      linetable = expect(read_object(), UPY_C_BYTES);
    } else {
      expect_str_tuple(read_object(), &lp);
      i32 kinds = expect(read_object(), UPY_C_BYTES);
      if (vals[kinds].n != lp.size()) fail("localsplus kinds/names length mismatch");
      const u8* kp = bytes_ptr(kinds);
      for (size_t i = 0; i < lp.size(); i++)
        if (kp[i] & 0x20) varnames.push_back(lp[i]);
      for (size_t i = 0; i < lp.size(); i++)
        if (kp[i] & 0x40) cellvars.push_back(lp[i]);
      for (size_t i = 0; i < lp.size(); i++)
        if (kp[i] & 0x80) freevars.push_back(lp[i]);
      o.nlocals = (i64)varnames.size();
      filename = expect(read_object(), UPY_C_STR);
      name = expect(read_object(), UPY_C_STR);
      qualname = expect(read_object(), UPY_C_STR);
      o.firstlineno = i32_();
      linetable = expect(read_object(), UPY_C_BYTES);
      exctable = expect(read_object(), UPY_C_BYTES);
      // CodeObject.localsplus (code_model.py:129-139) must reproduce the layout
      std::vector<i32> derived = varnames;
      for (i32 c : cellvars) {
        bool in = false;
        for (i32 v : varnames) in = in || s_same(c, v);
        if (!in) derived.push_back(c);
      }
      derived.insert(derived.end(), freevars.begin(), freevars.end());
      bool same = derived.size() == lp.size();
      for (size_t i = 0; same && i < lp.size(); i++) same = s_same(derived[i], lp[i]);
      if (!same) fail("localsplus layout " + repr_str_tuple(lp) + " not reproducible from varnames/cellvars/freevars");
    }
    if (vals[qualname].n == 0) qualname = name;  // CodeObject.__post_init__
    o.code_len = vals[code].n;
    o.code_off = vals[code].off;
    if (o.code_len > T->max_code) T->max_code = o.code_len;
    i32 lt = in_rest(linetable);
    o.lnt_off = vals[lt].off;
    o.lnt_len = vals[lt].n;
    if (exctable >= 0) {
      i32 et = in_rest(exctable);
      o.exc_off = vals[et].off;
      o.exc_len = vals[et].n;
    }
    std::vector<u32> cids(vals[consts].n);
    for (u32 i = 0; i < vals[consts].n; i++) cids[i] = (u32)cid_of(kids[vals[consts].off + i]);
    o.consts_off = (u32)T->refs.size();
    o.n_consts = (u32)cids.size();
    T->refs.insert(T->refs.end(), cids.begin(), cids.end());
    T->ref_is_str.insert(T->ref_is_str.end(), cids.size(), (u8)0);
    str_list(names, &o.names_off, &o.n_names);
    str_list(varnames, &o.varnames_off, &o.n_varnames);
    str_list(freevars, &o.freevars_off, &o.n_freevars);
    str_list(cellvars, &o.cellvars_off, &o.n_cellvars);
    o.name = (u32)sid_of(name);
    o.filename = (u32)sid_of(filename);
    o.qualname = (u32)sid_of(qualname);
    i32 idx = (i32)T->objs.size();
    T->objs.push_back(o);
    i32 v = new_val(UPY_C_CODE);
    vals[v].off = (u64)idx;
    return v;
  }

  std::string repr_str_tuple(const std::vector<i32>& items) {
    std::vector<u8> slot(1 << 20);
    std::vector<char> m(4096);
    std::vector<u8> sink(SINK_BYTES);
    Dc C;
    memset(&C, 0, sizeof C);
    C.base = slot.data();
    C.cap = C.top = C.low_top = slot.size();
    C.sink = sink.data();
    C.msg = m.data();
    C.msg_cap = (u32)m.size();
    Text t = {nullptr, 0, 0};
    t_put(&C, &t, '(');
    for (size_t i = 0; i < items.size(); i++) {
      if (i) t_puts(&C, &t, ", ");
      t_str_repr(&C, &t, Str{(const char*)&T->rest[vals[items[i]].off], vals[items[i]].n});
    }
    if (items.size() == 1) t_put(&C, &t, ',');
    t_put(&C, &t, ')');
    return C.err ? std::string("(...)") : std::string(t.d, t.n);
  }
};

std::string magic_msg(u32 magic) {
  char b[128];
  snprintf(b, sizeof b, "unknown pyc magic 0x%04x (unsupported interpreter version)", magic);  // {magic:#06x}
  return b;
}

// load_pyc (pyc.py:50-52) of one file into the thread's sections
void load_one(const u8* data, u64 size, Parser* P, FileRes* R) {
  // parse_pyc_header (pyc.py:36-47)
  if (size < 16) {
    R->status = UPY_ST_TRUNCATED_HEADER;
    R->msg = "pyc header needs 16 bytes, got " + std::to_string(size);
    return;
  }
  if (data[2] != '\r' || data[3] != '\n') {
    u32 magic = (u32)data[0] | ((u32)data[1] << 8) | ((u32)data[2] << 16) | ((u32)data[3] << 24);
    R->status = UPY_ST_UNKNOWN_MAGIC;
    R->aux = magic;
    R->msg = magic_msg(magic);
    return;
  }
  u32 magic = (u32)data[0] | ((u32)data[1] << 8);
  int minor = magic == 3413 ? 8 : magic == 3425 ? 9 : magic == 3439 ? 10 : magic == 3495 ? 11 : -1;
  if (minor < 0) {
    R->status = UPY_ST_UNKNOWN_MAGIC;
    R->aux = magic;
    R->msg = magic_msg(magic);
    return;
  }
  ThreadOut* T = P->T;
  u64 m[7];
  T->mark(m);
  u64 max_code = T->max_code;
  P->d = data + 16;
  P->n = size - 16;
  P->pos = 0;
  P->minor = minor;
  P->depth = 0;
  P->refs.clear();
  P->vals.clear();
  P->kids.clear();
  try {
    i32 v = P->read_object();
    if (P->vals[v].kind != UPY_C_CODE) P->fail("top-level marshal object is not a code object", 0);
    R->root = (i32)P->vals[v].off;
  } catch (Fail&) {
    R->status = UPY_ST_MALFORMED_MARSHAL;
    R->aux = (i64)P->fail_off;
    R->msg = P->msg + " (at byte offset " + std::to_string(P->fail_off) + ")";
    T->rollback(m);
    T->max_code = max_code;
  }
}

u64 al(u64 x, u64 a) { return (x + a - 1) / a * a; }

}  // namespace

struct upy_pyc_batch_impl {
  upy_pyc_batch pub;  // first member: the public handle points here
  u8* image = nullptr;  // owned when materialised by upy_pyc_load
  int n_threads = 0;
  std::vector<ThreadOut> outs;
  std::vector<u64> b_obj, b_const, b_str, b_ref, b_limb, b_code, b_rest;
  u64 code_end = 0, offs[S_N] = {}, ends[S_N] = {}, total = 0;
  std::vector<i32> status, root, pos;  // root: object index; pos: position in the roots section
  std::vector<i64> aux;
  std::vector<u64> msg_off;
  std::vector<u32> msg_len;
  std::string messages;
  ~upy_pyc_batch_impl() { free(image); }
  void write(u8* img) const;
};

// Concatenate the workers' sections into img (total bytes), rebasing every index.
void upy_pyc_batch_impl::write(u8* img) const {
  for (int s = 0; s < S_N; s++) memset(img + ends[s], 0, (s + 1 < S_N ? offs[s + 1] : total) - ends[s]);
  upy_obj* objs = (upy_obj*)(img + offs[S_OBJS]);
  upy_const* consts = (upy_const*)(img + offs[S_CONSTS]);
  upy_str* strs = (upy_str*)(img + offs[S_STRS]);
  u32* refs = (u32*)(img + offs[S_REFS]);
  u32* limbs = (u32*)(img + offs[S_LIMBS]);
  u8* bytes = img + offs[S_BYTES];
  i32* roots = (i32*)(img + offs[S_ROOTS]);
  for (i64 f = 0, r = 0; f < pub.n_files; f++)
    if (status[f] == UPY_ST_OK) roots[r++] = root[f];
  std::vector<std::thread> pool;
  for (int t = 0; t < n_threads; t++)
    pool.emplace_back([&, t] {
      const ThreadOut& T = outs[t];
      u64 rest_base = code_end + b_rest[t];
      for (size_t i = 0; i < T.objs.size(); i++) {
        upy_obj o = T.objs[i];
        o.code_off += b_code[t];
        o.exc_off = o.exc_len ? o.exc_off + rest_base : 0;  // empty table: no address
        o.lnt_off += rest_base;
        o.consts_off += (u32)b_ref[t];
        o.names_off += (u32)b_ref[t];
        o.varnames_off += (u32)b_ref[t];
        o.freevars_off += (u32)b_ref[t];
        o.cellvars_off += (u32)b_ref[t];
        o.name += (u32)b_str[t];
        o.filename += (u32)b_str[t];
        o.qualname += (u32)b_str[t];
        objs[b_obj[t] + i] = o;
      }
      for (size_t i = 0; i < T.consts.size(); i++) {
        upy_const c = T.consts[i];
        switch (c.kind) {
          case UPY_C_STR: case UPY_C_BYTES: c.off += c.pad ? b_code[t] : rest_base; c.pad = 0; break;
          case UPY_C_INT: c.off += b_limb[t]; break;
          case UPY_C_TUPLE: case UPY_C_FROZENSET: c.off += b_ref[t]; break;
          case UPY_C_CODE: c.off += b_obj[t]; break;
          default: break;
        }
        consts[b_const[t] + i] = c;
      }
      for (size_t i = 0; i < T.strs.size(); i++) {
        upy_str s = T.strs[i];
        s.off += rest_base;
        strs[b_str[t] + i] = s;
      }
      const u32 cb = (u32)b_const[t], sb = (u32)b_str[t];
      for (size_t i = 0; i < T.refs.size(); i++) refs[b_ref[t] + i] = T.refs[i] + (T.ref_is_str[i] ? sb : cb);
      if (!T.limbs.empty()) memcpy(limbs + b_limb[t], T.limbs.data(), T.limbs.size() * 4);
      if (!T.code.empty()) memcpy(bytes + b_code[t], T.code.data(), T.code.size());
      if (!T.rest.empty()) memcpy(bytes + rest_base, T.rest.data(), T.rest.size());
    });
  for (auto& th : pool) th.join();
}

extern "C" int upy_pyc_load(const uint8_t* const* data, const uint64_t* sizes, int64_t n_files, int n_threads,
                            int flags, upy_pyc_batch** out) {
  if (!out || n_files < 0 || (n_files && (!data || !sizes))) return 1;
  if (n_threads <= 0) {
    unsigned hc = std::thread::hardware_concurrency();
    n_threads = hc ? (int)hc : 1;
  }
  if ((i64)n_threads > n_files) n_threads = (int)(n_files ? n_files : 1);
  upy_pyc_batch_impl* B = new upy_pyc_batch_impl();
  B->n_threads = n_threads;
  B->pub.n_files = n_files;
  // contiguous slices of files per worker (file order is kept inside a slice)
  std::vector<i64> lo(n_threads + 1);
  for (int t = 0; t <= n_threads; t++) lo[t] = n_files * t / n_threads;
  B->outs.resize((size_t)n_threads);
  std::vector<FileRes> res((size_t)n_files);
  {
    std::vector<std::thread> pool;
    for (int t = 0; t < n_threads; t++)
      pool.emplace_back([&, t] {
        ThreadOut& T = B->outs[t];
        u64 in_bytes = 0;
        for (i64 f = lo[t]; f < lo[t + 1]; f++) in_bytes += sizes[f];
        T.rest.reserve(in_bytes);
        T.code.reserve(in_bytes / 2);
        Parser P;
        P.T = &T;
        for (i64 f = lo[t]; f < lo[t + 1]; f++) load_one(data[f], sizes[f], &P, &res[(size_t)f]);
      });
    for (auto& th : pool) th.join();
  }
  // section sizes and per-thread bases
  for (auto* v : {&B->b_obj, &B->b_const, &B->b_str, &B->b_ref, &B->b_limb, &B->b_code, &B->b_rest})
    v->assign(n_threads + 1, 0);
  u64 max_code = 0;
  for (int t = 0; t < n_threads; t++) {
    const ThreadOut& T = B->outs[t];
    B->b_obj[t + 1] = B->b_obj[t] + T.objs.size();
    B->b_const[t + 1] = B->b_const[t] + T.consts.size();
    B->b_str[t + 1] = B->b_str[t] + T.strs.size();
    B->b_ref[t + 1] = B->b_ref[t] + T.refs.size();
    B->b_limb[t + 1] = B->b_limb[t] + T.limbs.size();
    B->b_code[t + 1] = B->b_code[t] + T.code.size();
    B->b_rest[t + 1] = B->b_rest[t] + T.rest.size();
    if (T.max_code > max_code) max_code = T.max_code;
  }
  B->code_end = B->b_code[n_threads];
  B->status.resize(n_files);
  B->root.resize(n_files);
  B->pos.resize(n_files);
  B->aux.resize(n_files);
  B->msg_off.resize(n_files);
  B->msg_len.resize(n_files);
  u64 r = 0;
  std::vector<i32> root_obj((size_t)n_files, -1);
  for (int t = 0; t < n_threads; t++)
    for (i64 f = lo[t]; f < lo[t + 1]; f++) {
      const FileRes& R = res[(size_t)f];
      B->status[f] = R.status;
      B->aux[f] = R.aux;
      B->msg_off[f] = B->messages.size();
      B->msg_len[f] = (u32)R.msg.size();
      B->messages += R.msg;
      if (R.status == UPY_ST_OK) {
        B->root[f] = (i32)(B->b_obj[t] + R.root);
        B->pos[f] = (i32)r++;
      } else {
        B->root[f] = B->pos[f] = -1;
      }
    }
  u64 counts[S_N] = {B->b_obj[n_threads], B->b_const[n_threads], B->b_str[n_threads], B->b_ref[n_threads],
                     B->b_limb[n_threads], B->code_end + B->b_rest[n_threads], r};
  const u64 esz[S_N] = {sizeof(upy_obj), sizeof(upy_const), sizeof(upy_str), 4, 4, 1, 4};
  u64 total = 0;
  for (int s = 0; s < S_N; s++) {
    B->offs[s] = total;
    B->ends[s] = total + counts[s] * esz[s];
    total = al(B->ends[s], 256);
  }
  B->total = total < 256 ? 256 : total;
  upy_pyc_batch& P = B->pub;
  memset(&P, 0, sizeof P);
  P.image_bytes = B->total;
  for (int s = 0; s < S_N; s++) {
    P.section_off[s] = B->offs[s];
    P.section_count[s] = (int64_t)counts[s];
  }
  P.max_code_len = max_code;
  P.total_code_units = (B->code_end + 1) / 2;
  P.n_files = n_files;
  P.file_status = B->status.data();
  P.file_aux = B->aux.data();
  P.messages = B->messages.data();
  P.msg_off = B->msg_off.data();
  P.msg_len = B->msg_len.data();
  P.file_root = B->pos.data();
  if (!(flags & UPY_PYC_DEFER_IMAGE)) {
    B->image = (u8*)malloc(B->total);
    if (!B->image) {
      delete B;
      return 2;
    }
    B->write(B->image);
    P.image = B->image;
  }
  *out = &B->pub;
  return 0;
}

extern "C" int upy_pyc_write_image(upy_pyc_batch* b, uint8_t* dst, uint64_t dst_bytes) {
  if (!b || !dst) return 1;
  upy_pyc_batch_impl* B = reinterpret_cast<upy_pyc_batch_impl*>(b);
  if (dst_bytes < B->total) return 1;
  B->write(dst);
  return 0;
}

extern "C" void upy_pyc_free(upy_pyc_batch* b) {
  if (b) delete reinterpret_cast<upy_pyc_batch_impl*>(b);
}
