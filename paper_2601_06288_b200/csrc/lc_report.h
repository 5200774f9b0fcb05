// Host-side report writer: the "rows" / "frontier"
// lists of SearchReport.to_json() (search.py:224-264; json.dumps(sort_keys=True,
// indent=2)) written from column arrays, byte-identical to the Python writer in
// fastreport.py.  Floats use CPython's repr: the shortest round-trip digits
// (std::to_chars, same tie rule as David Gay's mode 0), fixed notation when the
// decimal exponent is in [-4, 16), else d.ddde+XX.
#pragma once
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>

namespace lcr {

struct Out {
  char* p;
  int64_t n, cap;
  void put(const char* s, size_t k) {
    if (n + (int64_t)k <= cap) memcpy(p + n, s, k);
    n += (int64_t)k;
  }
  template <size_t N>
  void put(const char (&s)[N]) { put(s, N - 1); }  // string literals: length known at compile time
  void puts(const char* s) { put(s, strlen(s)); }
  void put(const std::string& s) { put(s.data(), s.size()); }
  void pad(int depth) {
    static const char sp[] = "                                ";  // 16 levels
    put(sp, (size_t)(2 * depth));
  }
  void i64(int64_t v) {
    char b[24];
    auto r = std::to_chars(b, b + sizeof(b), v);
    put(b, (size_t)(r.ptr - b));
  }
};

// CPython float repr (Python/pystrtod.c, format_float_short with mode 'r')
inline int py_repr(double v, char* out) {
  char b[64];
  auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::scientific);
  *r.ptr = 0;
  char* q = b;
  int k = 0;
  if (*q == '-') { out[k++] = '-'; ++q; }
  char digits[40];
  int nd = 0;
  for (; *q && *q != 'e'; ++q)
    if (*q != '.') digits[nd++] = *q;
  const int exp10 = atoi(q + 1);
  const int decpt = exp10 + 1;
  if (decpt <= -4 || decpt > 16) {
    out[k++] = digits[0];
    if (nd > 1) {
      out[k++] = '.';
      for (int i = 1; i < nd; ++i) out[k++] = digits[i];
    }
    out[k++] = 'e';
    int e = decpt - 1;
    out[k++] = e < 0 ? '-' : '+';
    if (e < 0) e = -e;
    char eb[8];
    int ne = 0;
    do { eb[ne++] = (char)('0' + e % 10); e /= 10; } while (e);
    if (ne < 2) eb[ne++] = '0';
    while (ne) out[k++] = eb[--ne];
  } else if (decpt <= 0) {
    out[k++] = '0';
    out[k++] = '.';
    for (int i = 0; i < -decpt; ++i) out[k++] = '0';
    for (int i = 0; i < nd; ++i) out[k++] = digits[i];
  } else if (decpt >= nd) {
    for (int i = 0; i < nd; ++i) out[k++] = digits[i];
    for (int i = nd; i < decpt; ++i) out[k++] = '0';
    out[k++] = '.';
    out[k++] = '0';
  } else {
    for (int i = 0; i < decpt; ++i) out[k++] = digits[i];
    out[k++] = '.';
    for (int i = decpt; i < nd; ++i) out[k++] = digits[i];
  }
  out[k] = 0;
  return k;
}

}  // namespace lcr
