// packer.cpp -- native arena packer (CPython extension `_packer`): walks
// CodeObject trees (this package's model classes or the reference's own
// `unpyre.CodeObject` / `Const`, code_model.py:27-180 -- attributes only) and
// writes the arena image the device reads (include/upy.h).
//
// It restates arena.py's `_Packer` + `pack` exactly (same object / const / ref /
// string order, the same 16-B code alignment and 256-B sections, the same int
// clamping), so its output is byte-identical to the Python packer
// (tests/test_packer.py) -- at ~0.3M C3 objects/s instead of ~24K/s, which is what
// keeps `decompile_many(codes)` from being host-bound (the
// flattening of nested code trees into the arena happens here, in one pass).
//
// Build: paper_2403_13839_b200/build.py (g++ -O2 -shared against Python.h).
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <unordered_map>
#include <vector>

namespace {

constexpr int64_t kLim = int64_t(1) << 62;
constexpr uint64_t kAlign = 256;
enum { K_NONE, K_BOOL, K_INT, K_FLOAT, K_COMPLEX, K_STR, K_BYTES, K_TUPLE, K_FROZENSET, K_CODE, K_ELLIPSIS };

#pragma pack(push, 1)
struct Obj {  // upy_obj
  int64_t argcount, posonly, kwonly, nlocals, stacksize, flags, firstlineno;
  uint64_t code_off, exc_off, lnt_off;
  uint32_t code_len, exc_len, lnt_len;
  uint32_t consts_off, n_consts, names_off, n_names, varnames_off, n_varnames;
  uint32_t freevars_off, n_freevars, cellvars_off, n_cellvars;
  uint32_t name, filename, qualname, minor, pad;
};
struct ConstRow {  // upy_const
  uint32_t kind;
  int32_t ival;
  uint32_t n, pad;
  uint64_t off;
  double re, im;
};
struct StrRow {
  uint64_t off;
  uint32_t len, pad;
};
#pragma pack(pop)
static_assert(sizeof(Obj) == 152 && sizeof(ConstRow) == 40 && sizeof(StrRow) == 16, "ABI");

struct Names {  // interned attribute names
  PyObject *code, *exceptiontable, *linetable, *consts, *names, *varnames, *freevars, *cellvars, *name,
      *filename, *qualname, *version, *minor, *kind, *value, *argcount, *posonlyargcount, *kwonlyargcount,
      *nlocals, *stacksize, *flags, *firstlineno, *real, *imag;
  PyObject* kinds[11];
  bool init() {
#define I(x) if (!(x = PyUnicode_InternFromString(#x))) return false
    I(code); I(exceptiontable); I(linetable); I(consts); I(names); I(varnames); I(freevars); I(cellvars);
    I(name); I(filename); I(qualname); I(version); I(minor); I(kind); I(value); I(argcount);
    I(posonlyargcount); I(kwonlyargcount); I(nlocals); I(stacksize); I(flags); I(firstlineno); I(real); I(imag);
#undef I
    const char* kn[11] = {"none", "bool", "int", "float", "complex", "str", "bytes", "tuple", "frozenset", "code",
                          "ellipsis"};
    for (int i = 0; i < 11; i++)
      if (!(kinds[i] = PyUnicode_InternFromString(kn[i]))) return false;
    return true;
  }
};
Names N;

struct Ref {  // owned reference
  PyObject* p;
  explicit Ref(PyObject* x = nullptr) : p(x) {}
  ~Ref() { Py_XDECREF(p); }
  Ref(const Ref&) = delete;
  Ref& operator=(const Ref&) = delete;
  operator PyObject*() const { return p; }
};

struct Packer {
  std::vector<Obj> objs;
  std::unordered_map<PyObject*, uint32_t> obj_index;  // id(code) -> index (objects kept alive by the caller)
  std::vector<ConstRow> consts;
  std::vector<uint8_t> payload_of;  // per const: 1 when off is a payload offset
  PyObject* str_index = nullptr;    // dict str -> index
  std::vector<std::string> strs;
  std::vector<uint32_t> refs;
  std::vector<uint32_t> limbs;
  // code / exception / line tables: a pointer into the caller's bytes object (kept
  // alive by a reference) or, for other buffer types, an owned copy
  struct Bytes {
    PyObject* ref;
    const char* p;
    size_t n;
    std::string own;
    size_t size() const { return n; }
    const char* data() const { return p; }
  };
  std::vector<Bytes> codes, excs, lnts;
  std::string payload;
  bool err = false;

  ~Packer() {
    Py_XDECREF(str_index);
    for (auto* v : {&codes, &excs, &lnts})
      for (auto& b : *v) Py_XDECREF(b.ref);
  }
  static bool take_bytes(PyObject* v, std::vector<Bytes>* out) {  // bytes(v or b"")
    out->emplace_back();
    Bytes& b = out->back();
    b.ref = nullptr;
    b.p = "";
    b.n = 0;
    if (v == Py_None) return true;
    if (PyBytes_CheckExact(v)) {
      Py_INCREF(v);
      b.ref = v;
      b.p = PyBytes_AS_STRING(v);
      b.n = (size_t)PyBytes_GET_SIZE(v);
      return true;
    }
    if (!as_bytes(v, &b.own)) return false;
    b.p = b.own.data();
    b.n = b.own.size();
    return true;
  }

  static bool utf8(PyObject* s, std::string* out) {
    Ref b(PyUnicode_AsEncodedString(s, "utf-8", "surrogatepass"));
    if (!b) return false;
    out->assign(PyBytes_AS_STRING(b.p), PyBytes_GET_SIZE(b.p));
    return true;
  }
  static bool as_bytes(PyObject* v, std::string* out) {  // bytes(v) (None -> b"")
    if (v == Py_None) {
      out->clear();
      return true;
    }
    if (PyBytes_Check(v)) {
      out->assign(PyBytes_AS_STRING(v), PyBytes_GET_SIZE(v));
      return true;
    }
    Ref b(PyBytes_FromObject(v));
    if (!b) return false;
    out->assign(PyBytes_AS_STRING(b.p), PyBytes_GET_SIZE(b.p));
    return true;
  }

  int64_t sid(PyObject* s) {  // _Packer.sid
    Ref tmp;
    if (!PyUnicode_Check(s)) {
      tmp.p = PyObject_Str(s);
      if (!tmp.p) return -1;
      s = tmp.p;
    }
    PyObject* hit = PyDict_GetItemWithError(str_index, s);
    if (hit) return PyLong_AsLongLong(hit);
    if (PyErr_Occurred()) return -1;
    std::string b;
    if (!utf8(s, &b)) return -1;
    int64_t i = (int64_t)strs.size();
    Ref iv(PyLong_FromLongLong(i));
    if (!iv || PyDict_SetItem(str_index, s, iv) < 0) return -1;
    strs.push_back(std::move(b));
    return i;
  }

  // int(getattr(co, f)) clamped to +-2**62 (arena.py _clamp)
  bool clamp_attr(PyObject* co, PyObject* attr, int64_t* out) {
    Ref v(PyObject_GetAttr(co, attr));
    if (!v) return false;
    Ref iv(PyNumber_Index(v));
    if (!iv) {  // int(x) semantics for non-index numbers
      PyErr_Clear();
      iv.p = PyNumber_Long(v);
      if (!iv) return false;
    }
    int ovf = 0;
    long long x = PyLong_AsLongLongAndOverflow(iv, &ovf);
    if (ovf) x = ovf > 0 ? kLim : -kLim;
    else if (x == -1 && PyErr_Occurred()) return false;
    *out = x > kLim ? kLim : x < -kLim ? -kLim : x;
    return true;
  }
  // arena.py _flags62: low 62 bits, sign kept
  bool flags_attr(PyObject* co, int64_t* out) {
    Ref v(PyObject_GetAttr(co, N.flags));
    if (!v) return false;
    if (PyLong_Check(v)) {  // fits int64: two's complement & equals Python's & here
      int ovf = 0;
      const long long x = PyLong_AsLongLongAndOverflow(v, &ovf);
      if (!ovf && !(x == -1 && PyErr_Occurred())) {
        const long long lo = x & (kLim - 1);
        *out = x < 0 ? lo - kLim : lo;
        return true;
      }
      PyErr_Clear();
    }
    Ref iv(PyNumber_Long(v));
    if (!iv) return false;
    Ref mask(PyLong_FromLongLong(kLim - 1));
    Ref low(PyNumber_And(iv, mask));
    if (!low) return false;
    long long lo = PyLong_AsLongLong(low);
    if (lo == -1 && PyErr_Occurred()) return false;
    Ref zero(PyLong_FromLong(0));
    int neg = PyObject_RichCompareBool(iv, zero, Py_LT);
    if (neg < 0) return false;
    *out = neg ? lo - kLim : lo;
    return true;
  }

  bool strlist(PyObject* co, PyObject* attr, uint32_t* off, uint32_t* n) {
    Ref seq(PyObject_GetAttr(co, attr));
    if (!seq) return false;
    Ref fast(PySequence_Fast(seq, "expected a sequence of names"));
    if (!fast) return false;
    Py_ssize_t k = PySequence_Fast_GET_SIZE(fast.p);
    PyObject** items = PySequence_Fast_ITEMS(fast.p);
    std::vector<uint32_t> ids((size_t)k);
    for (Py_ssize_t i = 0; i < k; i++) {
      int64_t s = sid(items[i]);
      if (s < 0) return false;
      ids[(size_t)i] = (uint32_t)s;
    }
    *off = (uint32_t)refs.size();
    *n = (uint32_t)k;
    refs.insert(refs.end(), ids.begin(), ids.end());
    return true;
  }

  int kind_of(PyObject* k) {
    for (int i = 0; i < 11; i++)
      if (k == N.kinds[i]) return i;
    for (int i = 0; i < 11; i++) {
      int eq = PyObject_RichCompareBool(k, N.kinds[i], Py_EQ);
      if (eq < 0) return -1;
      if (eq) return i;
    }
    PyErr_Format(PyExc_ValueError, "bad const kind %R", k);
    return -1;
  }

  // int(v) of any size: sign and 32-bit limbs of the magnitude (arena.py _Packer.const)
  bool int_slow(PyObject* v, ConstRow* row) {
    Ref iv(PyNumber_Long(v));
    if (!iv) return false;
    row->ival = _PyLong_Sign(iv.p);
    Ref mag(PyNumber_Absolute(iv));
    if (!mag) return false;
    int64_t bits = (int64_t)_PyLong_NumBits(mag.p);
    if (bits < 0) return false;
    uint32_t nb = bits ? (uint32_t)((bits + 31) / 32) : 1u;
    std::vector<uint8_t> buf((size_t)nb * 4);
    if (_PyLong_AsByteArray((PyLongObject*)mag.p, buf.data(), buf.size(), 1, 0) < 0) return false;
    row->n = nb;
    row->off = limbs.size();
    for (uint32_t i = 0; i < nb; i++) {
      uint32_t w;
      memcpy(&w, buf.data() + 4 * i, 4);
      limbs.push_back(w);
    }
    return true;
  }
  int64_t push_row(const ConstRow& row, uint8_t is_payload) {
    consts.push_back(row);
    payload_of.push_back(is_payload);
    return (int64_t)consts.size() - 1;
  }

  int64_t cnst(PyObject* c) {  // _Packer.const
    Ref kobj(PyObject_GetAttr(c, N.kind));
    if (!kobj) return -1;
    int k = kind_of(kobj);
    if (k < 0) return -1;
    Ref v(PyObject_GetAttr(c, N.value));
    if (!v) return -1;
    ConstRow row;
    memset(&row, 0, sizeof row);
    row.kind = (uint32_t)k;
    uint8_t is_payload = 0;
    if (k == K_BOOL) {
      int t = PyObject_IsTrue(v);
      if (t < 0) return -1;
      row.ival = t ? 1 : 0;
    } else if (k == K_INT && PyLong_Check(v) && !PyBool_Check(v)) {
      int ovf = 0;
      const long long x = PyLong_AsLongLongAndOverflow(v, &ovf);
      if (x == -1 && PyErr_Occurred()) return -1;
      if (ovf) return int_slow(v, &row) ? push_row(row, 0) : -1;
      row.ival = (x > 0) - (x < 0);
      const unsigned long long mag = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
      row.n = (mag >> 32) ? 2u : 1u;
      row.off = limbs.size();
      limbs.push_back((uint32_t)mag);
      if (row.n == 2) limbs.push_back((uint32_t)(mag >> 32));
    } else if (k == K_INT) {
      if (!int_slow(v, &row)) return -1;
    } else if (k == K_FLOAT) {
      row.re = PyFloat_AsDouble(v);
      if (row.re == -1.0 && PyErr_Occurred()) return -1;
    } else if (k == K_COMPLEX) {
      Ref re(PyObject_GetAttr(v, N.real)), im(PyObject_GetAttr(v, N.imag));
      if (!re || !im) return -1;
      row.re = PyFloat_AsDouble(re);
      row.im = PyFloat_AsDouble(im);
      if (PyErr_Occurred()) return -1;
    } else if (k == K_STR || k == K_BYTES) {
      std::string b;
      if (k == K_STR) {
        if (!PyUnicode_Check(v)) {
          PyErr_SetString(PyExc_TypeError, "str const value is not a str");
          return -1;
        }
        if (!utf8(v, &b)) return -1;
      } else if (!as_bytes(v, &b)) {
        return -1;
      }
      row.n = (uint32_t)b.size();
      row.off = payload.size();
      is_payload = 1;
      payload += b;
    } else if (k == K_TUPLE || k == K_FROZENSET) {
      Ref fast(PySequence_Fast(v, "tuple const value is not a sequence"));
      if (!fast) return -1;
      Py_ssize_t n = PySequence_Fast_GET_SIZE(fast.p);
      std::vector<uint32_t> ids((size_t)n);
      for (Py_ssize_t i = 0; i < n; i++) {
        int64_t id = cnst(PySequence_Fast_GET_ITEM(fast.p, i));
        if (id < 0) return -1;
        ids[(size_t)i] = (uint32_t)id;
      }
      row.n = (uint32_t)n;
      row.off = refs.size();
      refs.insert(refs.end(), ids.begin(), ids.end());
    } else if (k == K_CODE) {
      int64_t oi = code(v);
      if (oi < 0) return -1;
      row.off = (uint64_t)oi;
    }
    consts.push_back(row);
    payload_of.push_back(is_payload);
    return (int64_t)consts.size() - 1;
  }

  int64_t code(PyObject* co) {  // _Packer.code
    auto it = obj_index.find(co);
    if (it != obj_index.end()) return it->second;
    uint32_t idx = (uint32_t)objs.size();
    obj_index.emplace(co, idx);
    objs.emplace_back();
    memset(&objs.back(), 0, sizeof(Obj));
    {
      Ref v(PyObject_GetAttr(co, N.code));
      if (!v || !take_bytes(v, &codes)) return -1;
    }
    {
      Ref v(PyObject_GetAttr(co, N.exceptiontable));
      if (!v || !take_bytes(v, &excs)) return -1;
    }
    {
      Ref v(PyObject_GetAttr(co, N.linetable));
      if (!v || !take_bytes(v, &lnts)) return -1;
    }
    Obj o;
    memset(&o, 0, sizeof o);
    if (!clamp_attr(co, N.argcount, &o.argcount) || !clamp_attr(co, N.posonlyargcount, &o.posonly) ||
        !clamp_attr(co, N.kwonlyargcount, &o.kwonly) || !clamp_attr(co, N.nlocals, &o.nlocals) ||
        !clamp_attr(co, N.stacksize, &o.stacksize) || !clamp_attr(co, N.firstlineno, &o.firstlineno) ||
        !flags_attr(co, &o.flags))
      return -1;
    {
      Ref ver(PyObject_GetAttr(co, N.version));
      if (!ver) return -1;
      Ref mi(PyObject_GetAttr(ver, N.minor));
      if (!mi) return -1;
      long m = PyLong_AsLong(mi);
      if (m == -1 && PyErr_Occurred()) return -1;
      o.minor = (uint32_t)m;
    }
    {
      Ref cs(PyObject_GetAttr(co, N.consts));
      if (!cs) return -1;
      Ref fast(PySequence_Fast(cs, "consts is not a sequence"));
      if (!fast) return -1;
      Py_ssize_t n = PySequence_Fast_GET_SIZE(fast.p);
      std::vector<uint32_t> ids((size_t)n);
      for (Py_ssize_t i = 0; i < n; i++) {
        int64_t id = cnst(PySequence_Fast_GET_ITEM(fast.p, i));
        if (id < 0) return -1;
        ids[(size_t)i] = (uint32_t)id;
      }
      o.consts_off = (uint32_t)refs.size();
      o.n_consts = (uint32_t)n;
      refs.insert(refs.end(), ids.begin(), ids.end());
    }
    if (!strlist(co, N.names, &o.names_off, &o.n_names) ||
        !strlist(co, N.varnames, &o.varnames_off, &o.n_varnames) ||
        !strlist(co, N.freevars, &o.freevars_off, &o.n_freevars) ||
        !strlist(co, N.cellvars, &o.cellvars_off, &o.n_cellvars))
      return -1;
    Ref name(PyObject_GetAttr(co, N.name));
    Ref filename(PyObject_GetAttr(co, N.filename));
    Ref qualname(PyObject_GetAttr(co, N.qualname));
    if (!name || !filename || !qualname) return -1;
    int q = PyObject_IsTrue(qualname);
    if (q < 0) return -1;
    int64_t s1 = sid(name), s2 = sid(filename), s3 = sid(q ? qualname.p : name.p);
    if (s1 < 0 || s2 < 0 || s3 < 0) return -1;
    o.name = (uint32_t)s1;
    o.filename = (uint32_t)s2;
    o.qualname = (uint32_t)s3;
    objs[idx] = o;
    return idx;
  }
};

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

PyObject* py_pack(PyObject*, PyObject* args) {
  PyObject* roots_in;
  if (!PyArg_ParseTuple(args, "O", &roots_in)) return nullptr;
  Ref fast(PySequence_Fast(roots_in, "roots must be a sequence"));
  if (!fast) return nullptr;
  Packer P;
  P.str_index = PyDict_New();
  if (!P.str_index) return nullptr;
  Py_ssize_t n_roots = PySequence_Fast_GET_SIZE(fast.p);
  std::vector<int32_t> roots((size_t)n_roots);
  for (Py_ssize_t i = 0; i < n_roots; i++) {
    int64_t r = P.code(PySequence_Fast_GET_ITEM(fast.p, i));
    if (r < 0) return nullptr;
    roots[(size_t)i] = (int32_t)r;
  }
  // byte pool: code segments (16-aligned), exception tables, line tables, strings, payloads
  size_t n_obj = P.objs.size();
  uint64_t pos = 0, max_code = 0;
  for (size_t i = 0; i < n_obj; i++) {
    P.objs[i].code_off = pos;
    P.objs[i].code_len = (uint32_t)P.codes[i].size();
    if (P.codes[i].size() > max_code) max_code = P.codes[i].size();
    pos = align_up(pos + P.codes[i].size(), 16);
  }
  uint64_t code_end = pos;
  for (size_t i = 0; i < n_obj; i++) {
    P.objs[i].exc_off = pos;
    P.objs[i].exc_len = (uint32_t)P.excs[i].size();
    pos += P.excs[i].size();
  }
  for (size_t i = 0; i < n_obj; i++) {
    P.objs[i].lnt_off = pos;
    P.objs[i].lnt_len = (uint32_t)P.lnts[i].size();
    pos += P.lnts[i].size();
  }
  std::vector<uint64_t> str_off(P.strs.size());
  for (size_t i = 0; i < P.strs.size(); i++) {
    str_off[i] = pos;
    pos += P.strs[i].size();
  }
  uint64_t payload_base = pos;
  pos += P.payload.size();
  uint64_t n_bytes = pos;
  const char* names[7] = {"objs", "consts", "strs", "refs", "limbs", "bytes", "roots"};
  uint64_t counts[7] = {n_obj, P.consts.size(), P.strs.size(), P.refs.size(), P.limbs.size(), n_bytes,
                        (uint64_t)n_roots};
  uint64_t sizes[7] = {sizeof(Obj), sizeof(ConstRow), sizeof(StrRow), 4, 4, 1, 4};
  uint64_t offs[7], total = 0;
  for (int s = 0; s < 7; s++) {
    offs[s] = total;
    total = align_up(total + counts[s] * sizes[s], kAlign);
  }
  if (total < kAlign) total = kAlign;
  Ref blob(PyByteArray_FromStringAndSize(nullptr, (Py_ssize_t)total));
  if (!blob) return nullptr;
  uint8_t* B = (uint8_t*)PyByteArray_AS_STRING(blob.p);
  memset(B, 0, total);
  if (n_obj) memcpy(B + offs[0], P.objs.data(), n_obj * sizeof(Obj));
  for (size_t i = 0; i < P.consts.size(); i++) {
    ConstRow r = P.consts[i];
    if (P.payload_of[i]) r.off += payload_base;
    memcpy(B + offs[1] + i * sizeof(ConstRow), &r, sizeof r);
  }
  for (size_t i = 0; i < P.strs.size(); i++) {
    StrRow r{str_off[i], (uint32_t)P.strs[i].size(), 0};
    memcpy(B + offs[2] + i * sizeof(StrRow), &r, sizeof r);
  }
  if (!P.refs.empty()) memcpy(B + offs[3], P.refs.data(), P.refs.size() * 4);
  if (!P.limbs.empty()) memcpy(B + offs[4], P.limbs.data(), P.limbs.size() * 4);
  uint8_t* by = B + offs[5];
  for (size_t i = 0; i < n_obj; i++) {
    memcpy(by + P.objs[i].code_off, P.codes[i].data(), P.codes[i].size());
    memcpy(by + P.objs[i].exc_off, P.excs[i].data(), P.excs[i].size());
    memcpy(by + P.objs[i].lnt_off, P.lnts[i].data(), P.lnts[i].size());
  }
  for (size_t i = 0; i < P.strs.size(); i++) memcpy(by + str_off[i], P.strs[i].data(), P.strs[i].size());
  if (!P.payload.empty()) memcpy(by + payload_base, P.payload.data(), P.payload.size());
  if (n_roots) memcpy(B + offs[6], roots.data(), roots.size() * 4);
  Ref off_d(PyDict_New()), cnt_d(PyDict_New());
  if (!off_d || !cnt_d) return nullptr;
  for (int s = 0; s < 7; s++) {
    Ref o(PyLong_FromUnsignedLongLong(offs[s])), c(PyLong_FromUnsignedLongLong(counts[s]));
    if (!o || !c || PyDict_SetItemString(off_d, names[s], o) < 0 || PyDict_SetItemString(cnt_d, names[s], c) < 0)
      return nullptr;
  }
  return Py_BuildValue("(OOOKK)", blob.p, off_d.p, cnt_d.p, (unsigned long long)max_code,
                       (unsigned long long)((code_end + 1) / 2));
}

PyMethodDef kMethods[] = {
    {"pack", py_pack, METH_VARARGS,
     "pack(roots) -> (bytearray blob, offsets, counts, max_code_len, total_code_units); "
     "byte-identical to arena.pack_py"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_packer", "Native arena packer (arena.py _Packer restated).", -1,
                       kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__packer(void) {
  if (!N.init()) return nullptr;
  return PyModule_Create(&kModule);
}
