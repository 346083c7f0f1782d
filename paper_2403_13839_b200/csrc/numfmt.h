// numfmt.h -- CPython 3.12 literal rendering on device: repr(int) with the
// 4300-digit limit, repr(float) (shortest round-trip, 'r' format), repr(complex),
// repr(str) / repr(bytes) with the Unicode 15.0 printable table
// (emitter.py:53-109 delegates all of these to CPython's repr).
#pragma once
#include "common.h"

// ------------------------------------------------------------ bignum (fixed)
#define BN_LIMBS 80  // 2560 bits: enough for 2^1077 * 10^326 scaled values
struct Big {
  u32 n;
  u32 d[BN_LIMBS];
};
HD inline void bn_set(Big* a, u64 v) {
  a->n = 0;
  while (v) {
    a->d[a->n++] = (u32)v;
    v >>= 32;
  }
}
HD inline void bn_mul_small(Big* a, u32 m) {
  u64 carry = 0;
  for (u32 i = 0; i < a->n; i++) {
    u64 t = (u64)a->d[i] * m + carry;
    a->d[i] = (u32)t;
    carry = t >> 32;
  }
  if (carry && a->n < BN_LIMBS) a->d[a->n++] = (u32)carry;
}
HD inline void bn_shl(Big* a, u32 k) {
  if (!a->n) return;
  u32 w = k / 32, b = k % 32;
  if (b) {
    u32 carry = 0;
    for (u32 i = 0; i < a->n; i++) {
      u32 x = a->d[i];
      a->d[i] = (x << b) | carry;
      carry = x >> (32 - b);
    }
    if (carry && a->n < BN_LIMBS) a->d[a->n++] = carry;
  }
  if (w) {
    u32 nn = a->n + w > BN_LIMBS ? BN_LIMBS : a->n + w;
    for (i32 i = (i32)nn - 1; i >= (i32)w; i--) a->d[i] = a->d[i - w];
    for (u32 i = 0; i < w && i < nn; i++) a->d[i] = 0;
    a->n = nn;
  }
}
HD inline int bn_cmp(const Big* a, const Big* b) {
  if (a->n != b->n) return a->n < b->n ? -1 : 1;
  for (i32 i = (i32)a->n - 1; i >= 0; i--)
    if (a->d[i] != b->d[i]) return a->d[i] < b->d[i] ? -1 : 1;
  return 0;
}
HD inline void bn_add(Big* r, const Big* a, const Big* b) {  // r may alias a
  u32 n = a->n > b->n ? a->n : b->n;
  u64 carry = 0;
  for (u32 i = 0; i < n; i++) {
    u64 t = carry + (i < a->n ? a->d[i] : 0) + (i < b->n ? b->d[i] : 0);
    r->d[i] = (u32)t;
    carry = t >> 32;
  }
  r->n = n;
  if (carry && r->n < BN_LIMBS) r->d[r->n++] = (u32)carry;
}
HD inline void bn_sub(Big* a, const Big* b) {  // a -= b, a >= b
  i64 borrow = 0;
  for (u32 i = 0; i < a->n; i++) {
    i64 t = (i64)a->d[i] - (i < b->n ? b->d[i] : 0) - borrow;
    borrow = t < 0;
    a->d[i] = (u32)(t + (borrow << 32));
  }
  while (a->n && a->d[a->n - 1] == 0) a->n--;
}
HD inline void bn_pow10(Big* a, u32 k) {
  while (k >= 9) {
    bn_mul_small(a, 1000000000u);
    k -= 9;
  }
  u32 m = 1;
  while (k--) m *= 10;
  if (m > 1) bn_mul_small(a, m);
}

// ------------------------------------------------------------ float repr
// Shortest round-trip digits (Burger & Dybvig free-format, with closest-digit
// fix-up), matching CPython's dtoa mode 0.  digits[] gets ASCII, returns count;
// *decpt = position of the decimal point (value = 0.DIGITS * 10^decpt).
HD NOINL int shortest_digits(double v, char* digits, int* decpt) {
  u64 bits;
  memcpy(&bits, &v, 8);
  u64 frac = bits & ((1ull << 52) - 1);
  int bexp = (int)((bits >> 52) & 0x7FF);
  u64 f;
  int e;
  if (bexp == 0) {
    f = frac;
    e = -1074;
  } else {
    f = frac | (1ull << 52);
    e = bexp - 1075;
  }
  bool even = (f & 1) == 0;
  Big r, s, mp, mm;
  bool unequal = (frac == 0 && bexp > 1);
  if (e >= 0) {
    bn_set(&r, f);
    bn_shl(&r, e + (unequal ? 2 : 1));
    bn_set(&s, unequal ? 4 : 2);
    bn_set(&mp, 1);
    bn_shl(&mp, e + (unequal ? 1 : 0));
    bn_set(&mm, 1);
    bn_shl(&mm, e);
  } else {
    bn_set(&r, f);
    bn_shl(&r, unequal ? 2 : 1);
    bn_set(&s, 1);
    bn_shl(&s, (unequal ? 1 : 0) - e + 1);
    bn_set(&mp, unequal ? 2 : 1);
    bn_set(&mm, 1);
  }
  // k estimate: ceil(log10(v))
  double lg = 0.0;
  {
    // log10 via exponent: v = f * 2^e
    int nb = 63;
    while (nb > 0 && !((f >> nb) & 1)) nb--;
    double approx = (nb + e) * 0.30102999566398119521;  // log10(2)
    lg = approx;
  }
  int k = (int)(lg >= 0 ? lg + 1 : lg) ;  // rough; fixed below
  if (k >= 0) bn_pow10(&s, (u32)k);
  else {
    bn_pow10(&r, (u32)(-k));
    bn_pow10(&mp, (u32)(-k));
    bn_pow10(&mm, (u32)(-k));
  }
  // fix-up so that (r + m+) / s lies in (0.1, 1] (or [.., 1) when !even)
  Big t;
  for (int it = 0; it < 400; it++) {
    bn_add(&t, &r, &mp);
    int c = bn_cmp(&t, &s);
    if (even ? c >= 0 : c > 0) {
      bn_mul_small(&s, 10);
      k++;
      continue;
    }
    // too small?  (r + m+) * 10 vs s
    Big t10 = t;
    bn_mul_small(&t10, 10);
    int c2 = bn_cmp(&t10, &s);
    if (even ? c2 < 0 : c2 <= 0) {
      bn_mul_small(&r, 10);
      bn_mul_small(&mp, 10);
      bn_mul_small(&mm, 10);
      k--;
      continue;
    }
    break;
  }
  *decpt = k;
  int nd = 0;
  while (nd < 40) {
    bn_mul_small(&r, 10);
    bn_mul_small(&mp, 10);
    bn_mul_small(&mm, 10);
    int dgt = 0;
    while (bn_cmp(&r, &s) >= 0) {
      bn_sub(&r, &s);
      dgt++;
    }
    int c1 = bn_cmp(&r, &mm);
    bool tc1 = even ? c1 <= 0 : c1 < 0;
    bn_add(&t, &r, &mp);
    int c2 = bn_cmp(&t, &s);
    bool tc2 = even ? c2 >= 0 : c2 > 0;
    if (!tc1 && !tc2) {
      digits[nd++] = (char)('0' + dgt);
      continue;
    }
    if (tc1 && !tc2) {
      digits[nd++] = (char)('0' + dgt);
    } else if (!tc1 && tc2) {
      digits[nd++] = (char)('0' + dgt + 1);
    } else {
      Big r2 = r;
      bn_shl(&r2, 1);
      int c3 = bn_cmp(&r2, &s);
      if (c3 < 0 || (c3 == 0 && (dgt & 1) == 0)) digits[nd++] = (char)('0' + dgt);
      else digits[nd++] = (char)('0' + dgt + 1);
    }
    break;
  }
  // a round-up can carry ('9' + 1)
  for (int q = nd - 1; q > 0; q--) {
    if (digits[q] > '9') {
      digits[q] = '0';
      digits[q - 1]++;
    }
  }
  if (digits[0] > '9') {
    digits[0] = '1';
    for (int q = 1; q < nd; q++) digits[q] = '0';
    (*decpt)++;
  }
  while (nd > 1 && digits[nd - 1] == '0') nd--;
  return nd;
}

// repr(float): finite non-special values in CPython's 'r' style
HD inline void t_float_repr(Dc* C, Text* t, double v) {
  u64 bits;
  memcpy(&bits, &v, 8);
  bool neg = bits >> 63;
  u64 mag = bits & ~(1ull << 63);
  if (mag > 0x7FF0000000000000ull) {
    t_puts(C, t, "nan");
    return;
  }
  if (mag == 0x7FF0000000000000ull) {
    t_puts(C, t, neg ? "-inf" : "inf");
    return;
  }
  if (neg) t_put(C, t, '-');
  if (mag == 0) {
    t_puts(C, t, "0.0");
    return;
  }
  double a;
  memcpy(&a, &mag, 8);
  char dg[48];
  int decpt;
  int nd = shortest_digits(a, dg, &decpt);
  if (decpt <= -4 || decpt > 16) {
    t_put(C, t, dg[0]);
    if (nd > 1) {
      t_put(C, t, '.');
      t_putn(C, t, dg + 1, nd - 1);
    }
    t_put(C, t, 'e');
    int x = decpt - 1;
    t_put(C, t, x < 0 ? '-' : '+');
    if (x < 0) x = -x;
    if (x < 10) t_put(C, t, '0');
    t_i64(C, t, x);
  } else if (decpt <= 0) {
    t_puts(C, t, "0.");
    for (int q = 0; q < -decpt; q++) t_put(C, t, '0');
    t_putn(C, t, dg, nd);
  } else if (decpt >= nd) {
    t_putn(C, t, dg, nd);
    for (int q = nd; q < decpt; q++) t_put(C, t, '0');
    t_puts(C, t, ".0");
  } else {
    t_putn(C, t, dg, decpt);
    t_put(C, t, '.');
    t_putn(C, t, dg + decpt, nd - decpt);
  }
}

HD inline bool d_isnan(double v) {
  u64 b;
  memcpy(&b, &v, 8);
  return (b & ~(1ull << 63)) > 0x7FF0000000000000ull;
}
HD inline bool d_isinf(double v) {
  u64 b;
  memcpy(&b, &v, 8);
  return (b & ~(1ull << 63)) == 0x7FF0000000000000ull;
}
HD inline bool d_signbit(double v) {
  u64 b;
  memcpy(&b, &v, 8);
  return b >> 63;
}

// repr(float) in 'r' format without the trailing ".0" (complex_repr parts)
HD inline void t_float_r_nodot(Dc* C, Text* t, double x) {
  Text tmp = {nullptr, 0, 0};
  t_float_repr(C, &tmp, x);
  u32 n = tmp.n;
  if (n >= 2 && tmp.d[n - 2] == '.' && tmp.d[n - 1] == '0') {
    bool has_e = false;
    for (u32 q = 0; q < n; q++) has_e |= tmp.d[q] == 'e';
    if (!has_e) n -= 2;
  }
  t_putn(C, t, tmp.d, n);
}
// repr(complex) (CPython 3.12 complex_repr)
HD inline void t_complex_repr(Dc* C, Text* t, double re, double im) {
  if (re == 0.0 && !d_signbit(re)) {
    t_float_r_nodot(C, t, im);
    t_put(C, t, 'j');
    return;
  }
  t_put(C, t, '(');
  t_float_r_nodot(C, t, re);
  if (d_isnan(im) || !d_signbit(im)) t_put(C, t, '+');
  t_float_r_nodot(C, t, im);
  t_puts(C, t, "j)");
}

// ------------------------------------------------------------ int repr
// repr of a sign/magnitude bigint from the arena (ValueError above 4300 digits)
HD NOINL bool t_int_repr(Dc* C, Text* t, int sign, const u32* limbs, u32 n) {
  while (n > 0 && limbs[n - 1] == 0) n--;
  if (n == 0) {
    t_put(C, t, '0');
    return true;
  }
  if (n <= 2) {
    u64 v = limbs[0] | (n == 2 ? (u64)limbs[1] << 32 : 0);
    if (sign < 0) t_put(C, t, '-');
    char buf[24];
    int k = 0;
    do {
      buf[k++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    while (k) t_put(C, t, buf[--k]);
    return true;
  }
  // general: repeated division by 1e9 into a scratch copy
  u32* w = (u32*)zalloc(C, (u64)n * 4);
  u32* chunks = (u32*)zalloc(C, ((u64)n * 32 / 29 + 2) * 4);
  if (C->err) return false;
  for (u32 i = 0; i < n; i++) w[i] = limbs[i];
  u32 nc = 0, wn = n;
  while (wn) {
    u64 rem = 0;
    for (i32 i = (i32)wn - 1; i >= 0; i--) {
      u64 cur = (rem << 32) | w[i];
      w[i] = (u32)(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    chunks[nc++] = (u32)rem;
    while (wn && w[wn - 1] == 0) wn--;
  }
  // digit count check (sys.int_info.default_max_str_digits = 4300)
  u32 top = chunks[nc - 1];
  u32 topd = 1;
  while (top >= 10) {
    top /= 10;
    topd++;
  }
  u64 ndig = (u64)(nc - 1) * 9 + topd;
  if (ndig > 4300) {
    py_error(C, UPY_ST_PY_VALUE_ERROR,
             "Exceeds the limit (4300 digits) for integer string conversion; use sys.set_int_max_str_digits() to increase the limit");
    return false;
  }
  if (sign < 0) t_put(C, t, '-');
  t_i64(C, t, chunks[nc - 1]);
  for (i32 i = (i32)nc - 2; i >= 0; i--) {
    char buf[9];
    u32 v = chunks[i];
    for (int q = 8; q >= 0; q--) {
      buf[q] = (char)('0' + v % 10);
      v /= 10;
    }
    t_putn(C, t, buf, 9);
  }
  return true;
}

// ------------------------------------------------------------ str / bytes repr
HD inline bool is_printable_cp(u32 cp) {
  i32 lo = 0, hi = UPY_N_PRINTABLE_RANGES - 1;
  while (lo <= hi) {
    i32 mid = (lo + hi) >> 1;
    if (cp < T_PRINTABLE[mid][0]) hi = mid - 1;
    else if (cp > T_PRINTABLE[mid][1]) lo = mid + 1;
    else return true;
  }
  return false;
}
// decode one UTF-8 (surrogatepass) code point; returns bytes consumed
HD inline u32 utf8_next(const char* p, u32 n, u32* cp) {
  u8 b0 = (u8)p[0];
  if (b0 < 0x80 || n < 2) {
    *cp = b0;
    return 1;
  }
  if ((b0 & 0xE0) == 0xC0) {
    *cp = ((b0 & 0x1F) << 6) | ((u8)p[1] & 0x3F);
    return 2;
  }
  if ((b0 & 0xF0) == 0xE0 && n >= 3) {
    *cp = ((b0 & 0x0F) << 12) | (((u8)p[1] & 0x3F) << 6) | ((u8)p[2] & 0x3F);
    return 3;
  }
  if (n >= 4) {
    *cp = ((b0 & 0x07) << 18) | (((u8)p[1] & 0x3F) << 12) | (((u8)p[2] & 0x3F) << 6) | ((u8)p[3] & 0x3F);
    return 4;
  }
  *cp = b0;
  return 1;
}
HD inline void t_hex(Dc* C, Text* t, u32 v, int width) {
  const char* hx = "0123456789abcdef";
  for (int q = width - 1; q >= 0; q--) t_put(C, t, hx[(v >> (4 * q)) & 0xF]);
}
HD NOINL void t_str_repr(Dc* C, Text* t, Str s) {  // unicode_repr (CPython 3.12)
  bool sq = false, dq = false;
  for (u32 i = 0; i < s.n; i++) {
    if (s.p[i] == '\'') sq = true;
    if (s.p[i] == '"') dq = true;
  }
  char quote = (sq && !dq) ? '"' : '\'';
  t_put(C, t, quote);
  u32 i = 0;
  while (i < s.n && !C->err) {
    u32 cp;
    u32 k = utf8_next(s.p + i, s.n - i, &cp);
    if (cp == (u32)quote || cp == '\\') {
      t_put(C, t, '\\');
      t_put(C, t, (char)cp);
    } else if (cp == '\t') {
      t_puts(C, t, "\\t");
    } else if (cp == '\n') {
      t_puts(C, t, "\\n");
    } else if (cp == '\r') {
      t_puts(C, t, "\\r");
    } else if (cp < ' ' || cp == 0x7F) {
      t_puts(C, t, "\\x");
      t_hex(C, t, cp, 2);
    } else if (cp < 0x7F) {
      t_put(C, t, (char)cp);
    } else if (is_printable_cp(cp)) {
      t_putn(C, t, s.p + i, k);
    } else if (cp <= 0xFF) {
      t_puts(C, t, "\\x");
      t_hex(C, t, cp, 2);
    } else if (cp <= 0xFFFF) {
      t_puts(C, t, "\\u");
      t_hex(C, t, cp, 4);
    } else {
      t_puts(C, t, "\\U");
      t_hex(C, t, cp, 8);
    }
    i += k;
  }
  t_put(C, t, quote);
}
HD inline void t_bytes_repr(Dc* C, Text* t, const u8* p, u32 n) {  // bytes_repr
  bool sq = false, dq = false;
  for (u32 i = 0; i < n; i++) {
    if (p[i] == '\'') sq = true;
    if (p[i] == '"') dq = true;
  }
  char quote = (sq && !dq) ? '"' : '\'';
  t_put(C, t, 'b');
  t_put(C, t, quote);
  for (u32 i = 0; i < n && !C->err; i++) {
    u8 c = p[i];
    if (c == (u8)quote || c == '\\') {
      t_put(C, t, '\\');
      t_put(C, t, (char)c);
    } else if (c == '\t') {
      t_puts(C, t, "\\t");
    } else if (c == '\n') {
      t_puts(C, t, "\\n");
    } else if (c == '\r') {
      t_puts(C, t, "\\r");
    } else if (c < ' ' || c >= 0x7F) {
      t_puts(C, t, "\\x");
      t_hex(C, t, c, 2);
    } else {
      t_put(C, t, (char)c);
    }
  }
  t_put(C, t, quote);
}
