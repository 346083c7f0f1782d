// c3gen.cpp -- native generator of the C3 corpus (1M straight-line
// objects, seed_i = splitmix64(0xC3 ^ i)).  BENCHMARK INPUT GENERATION, not the
// product: it restates synth/corpus.py's `c3(seed, minor)` (_Gen.simple /
// finish, Rng, splitmix64) and synth/asm.py's `assemble` for the straight-line
// ops C3 uses (no labels, every arg < 256, inline caches zero-filled), so that
// seeds map to byte-identical co_code and constant pools -- checked against the
// Python generator in tests/test_synth_c3.py.  synth/c3fast.py lays the results
// out exactly like arena.pack() would.
//
//   g++ -O2 -std=c++17 -shared -fPIC -pthread -o build/libc3gen.so c3gen.cpp
#include <stdint.h>
#include <string.h>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Rng {  // corpus.py Rng
  uint64_t s;
  uint64_t next() {
    s += kGolden;
    return splitmix64(s);
  }
  uint64_t below(uint64_t n) { return next() % n; }
};

// op ids into the caller's table (synth/c3fast.py OPS)
enum {
  LOAD_FAST, LOAD_CONST, BINARY_MULTIPLY, BINARY_ADD, BINARY_SUBTRACT, BINARY_OP, STORE_FAST,
  LOAD_GLOBAL, LOAD_ATTR, PRECALL, CALL, CALL_FUNCTION, LOAD_METHOD, CALL_METHOD, BINARY_SUBSCR,
  STORE_ATTR, RETURN_VALUE, RESUME, N_OPS
};

struct Emit {
  const int32_t* tab;  // [N_OPS][3]: opcode, has_arg, cache units
  uint8_t* out;
  uint32_t n;
  void op(int id, uint32_t arg = 0) {
    const int32_t* t = tab + 3 * id;
    out[n++] = (uint8_t)t[0];
    out[n++] = t[1] ? (uint8_t)arg : 0;
    for (int c = 0; c < t[2]; c++) {
      out[n++] = 0;
      out[n++] = 0;
    }
  }
};

struct Gen {  // corpus.py _Gen, C3 subset
  int minor;
  Rng r;
  Emit e;
  uint8_t consts[8];  // pool values in first-use order: 0 = None, k = int k
  uint32_t n_consts;
  uint32_t lv() { return (uint32_t)r.below(6); }
  uint32_t nm() { return (uint32_t)r.below(6); }
  uint32_t konst(uint8_t v) {  // Asm.const: dedup by value
    for (uint32_t i = 0; i < n_consts; i++)
      if (consts[i] == v) return i;
    consts[n_consts] = v;
    return n_consts++;
  }
  void binop(int v310, uint32_t nb) {
    if (minor >= 11) e.op(BINARY_OP, nb);
    else e.op(v310);
  }
  void simple() {
    uint64_t t = r.below(4);
    if (t == 0) {  // x = a + b * K
      uint32_t a = lv();
      e.op(LOAD_FAST, a);
      uint32_t b = lv();
      e.op(LOAD_FAST, b);
      e.op(LOAD_CONST, konst((uint8_t)(1 + r.below(3))));
      binop(BINARY_MULTIPLY, 5);
      binop(BINARY_ADD, 0);
      e.op(STORE_FAST, lv());
    } else if (t == 1) {  // x = g(a, b.attr)
      if (minor >= 11) e.op(LOAD_GLOBAL, (nm() << 1) | 1);
      else e.op(LOAD_GLOBAL, nm());
      uint32_t a = lv();
      e.op(LOAD_FAST, a);
      uint32_t b = lv();
      e.op(LOAD_FAST, b);
      e.op(LOAD_ATTR, nm());
      if (minor >= 11) {
        e.op(PRECALL, 2);
        e.op(CALL, 2);
      } else {
        e.op(CALL_FUNCTION, 2);
      }
      e.op(STORE_FAST, lv());
    } else if (t == 2) {  // x = a.m(b)[c]
      uint32_t a = lv();
      e.op(LOAD_FAST, a);
      e.op(LOAD_METHOD, nm());
      e.op(LOAD_FAST, lv());
      if (minor >= 11) {
        e.op(PRECALL, 1);
        e.op(CALL, 1);
      } else {
        e.op(CALL_METHOD, 1);
      }
      e.op(LOAD_FAST, lv());
      e.op(BINARY_SUBSCR);
      e.op(STORE_FAST, lv());
    } else {  // a.attr = b - c
      uint32_t a = lv();
      e.op(LOAD_FAST, a);
      uint32_t b = lv();
      e.op(LOAD_FAST, b);
      binop(BINARY_SUBTRACT, 10);
      e.op(LOAD_FAST, lv());
      e.op(STORE_ATTR, nm());
    }
  }
};

void gen_range(int minor, uint64_t first, int64_t lo, int64_t hi, int n_stmts, const int32_t* tab, uint8_t* base,
               const uint64_t* code_off, uint32_t* code_len, uint8_t* consts, uint8_t* n_consts) {
  std::vector<uint8_t> scratch(64 * (size_t)(n_stmts + 1));
  for (int64_t i = lo; i < hi; i++) {
    Gen g;
    g.minor = minor;
    g.r.s = splitmix64(0xC3ull ^ (first + (uint64_t)i));
    g.e = Emit{tab, base ? base + code_off[i] : scratch.data(), 0};
    g.n_consts = 0;
    g.konst(0);  // a.const(None)
    if (minor >= 11) g.e.op(RESUME, 0);
    for (int s = 0; s < n_stmts; s++) g.simple();
    g.e.op(LOAD_CONST, 0);  // finish(): return None
    g.e.op(RETURN_VALUE);
    code_len[i] = g.e.n;
    memcpy(consts + 4 * i, g.consts, 4);
    n_consts[i] = (uint8_t)g.n_consts;
  }
}

void name_range(uint64_t first, int64_t lo, int64_t hi, uint8_t* base, const uint64_t* off) {
  for (int64_t i = lo; i < hi; i++) {
    uint8_t* p = base + off[i];
    p[0] = 'c', p[1] = '3', p[2] = '_';
    char d[24];
    int k = 0;
    uint64_t v = first + (uint64_t)i;
    do {
      d[k++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    for (int j = 0; j < k; j++) p[3 + j] = (uint8_t)d[k - 1 - j];
  }
}

template <class F>
void parallel(int64_t n, int threads, F f) {
  if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; t++) pool.emplace_back(f, n * t / threads, n * (t + 1) / threads);
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// Objects seed = first + i, i < n: code lengths, constant pools (values in pool
// order, 0 = None) and their sizes; with `base` non-null the code bytes are also
// written at base + code_off[i] (a first call without `base` sizes the layout).
int c3gen(int minor, uint64_t first, int64_t n, int n_stmts, const int32_t* optab, uint8_t* base,
          const uint64_t* code_off, uint32_t* code_len, uint8_t* consts, uint8_t* n_consts, int threads) {
  parallel(n, threads, [=](int64_t lo, int64_t hi) {
    gen_range(minor, first, lo, hi, n_stmts, optab, base, code_off, code_len, consts, n_consts);
  });
  return 0;
}

// The objects' names "c3_<seed>" at base + off[i].
int c3names(uint64_t first, int64_t n, uint8_t* base, const uint64_t* off, int threads) {
  parallel(n, threads, [=](int64_t lo, int64_t hi) { name_range(first, lo, hi, base, off); });
  return 0;
}
}
