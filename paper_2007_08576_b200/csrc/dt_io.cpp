// dt_io.cpp -- native text codecs of the file formats (the reference's
// deformtrack/fileio.py:23-259 writes them from Python).
//
// The reference's writers are deterministic because every real is printed as Python's
// repr(): the SHORTEST decimal string that reads back to the same double, laid out in
// fixed notation for decimal exponents -4 < e <= 16 and in scientific notation otherwise
// (at least two exponent digits, no ".0" in the exponent form). dt_format_reals produces
// exactly those bytes natively (std::to_chars gives the shortest round-trip digits; the
// layout is Python's), so an ascii PLY written here is byte-identical to the
// reference's, and dt_parse_reals reads decimal text back with correctly rounded
// std::from_chars (the same doubles as Python's float()).

#include <charconv>
#include <cstdint>
#include <cstring>
#include <system_error>
#include <thread>
#include <vector>
#include <algorithm>

#include "../../include/deformtrack_b200.h"

namespace {

// Python repr of one double into p (needs <= 32 bytes); returns the end pointer.
char* repr_double(double x, char* p) {
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  *r.ptr = '\0';
  const char* s = sci;
  if (*s == '-') {
    *p++ = '-';
    ++s;
  }
  if (std::strcmp(s, "inf") == 0 || std::strcmp(s, "nan") == 0 || std::strncmp(s, "nan", 3) == 0) {
    const char* word = s[0] == 'i' ? "inf" : "nan";
    std::memcpy(p, word, 3);
    return p + 3;
  }
  // s = D[.DDD]e(+|-)XX
  char digits[24];
  int nd = 0;
  const char* q = s;
  for (; *q && *q != 'e'; ++q)
    if (*q != '.') digits[nd++] = *q;
  int e10 = 0;
  std::from_chars(q + 1 + (q[1] == '+' ? 1 : 0), r.ptr, e10);
  const int decpt = e10 + 1;  // value = 0.d1d2... x 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *p++ = digits[0];
    if (nd > 1) {
      *p++ = '.';
      std::memcpy(p, digits + 1, nd - 1);
      p += nd - 1;
    }
    *p++ = 'e';
    int ex = decpt - 1;
    *p++ = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    if (ex < 10) *p++ = '0';
    const auto er = std::to_chars(p, p + 4, ex);
    return er.ptr;
  }
  if (decpt <= 0) {
    *p++ = '0';
    *p++ = '.';
    for (int i = 0; i < -decpt; ++i) *p++ = '0';
    std::memcpy(p, digits, nd);
    return p + nd;
  }
  if (decpt >= nd) {
    std::memcpy(p, digits, nd);
    p += nd;
    for (int i = nd; i < decpt; ++i) *p++ = '0';
    *p++ = '.';
    *p++ = '0';
    return p;
  }
  std::memcpy(p, digits, decpt);
  p += decpt;
  *p++ = '.';
  std::memcpy(p, digits + decpt, nd - decpt);
  return p + (nd - decpt);
}

}  // namespace

extern "C" {

int64_t dt_format_reals(const double* values, int64_t rows, int64_t cols, char* out, int64_t capacity) {
  if (rows < 0 || cols <= 0 || (rows > 0 && values == nullptr)) return -1;
  // worst case per value: 24 characters + a separator
  const int64_t need = rows * cols * 25 + 1;
  if (out == nullptr || capacity < need) return -need;
  // rows [r0, r1) into out + worst-case offset of r0; returns the end
  auto fmt = [&](int64_t r0, int64_t r1) {
    char* p = out + r0 * cols * 25;
    for (int64_t i = r0; i < r1; ++i) {
      for (int64_t j = 0; j < cols; ++j) {
        if (j) *p++ = ' ';
        p = repr_double(values[i * cols + j], p);
      }
      *p++ = '\n';
    }
    return p;
  };
  // a streamed frame's PLY body is ~120 k values (~190 ns each): row blocks on host
  // threads, then the blocks are moved together in order (same bytes as one pass)
  const unsigned hw = std::thread::hardware_concurrency();
  const int64_t nb = rows * cols < 16384 ? 1 : std::min<int64_t>(std::max(1u, hw), 16);
  if (nb <= 1) return (int64_t)(fmt(0, rows) - out);
  std::vector<char*> ends(nb);
  std::vector<std::thread> pool;
  for (int64_t b = 0; b < nb; ++b)
    pool.emplace_back([&, b] { ends[b] = fmt(rows * b / nb, rows * (b + 1) / nb); });
  for (auto& th : pool) th.join();
  char* p = ends[0];
  for (int64_t b = 1; b < nb; ++b) {
    const char* src = out + (rows * b / nb) * cols * 25;
    const int64_t len = ends[b] - src;
    std::memmove(p, src, (size_t)len);
    p += len;
  }
  return (int64_t)(p - out);
}

int64_t dt_parse_reals(const char* text, int64_t length, double* out, int64_t capacity) {
  if (length < 0 || (length > 0 && text == nullptr) || capacity < 0) return -1;
  const char* p = text;
  const char* end = text + length;
  int64_t n = 0;
  while (true) {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    if (p >= end || n >= capacity) break;
    double v = 0.0;
    const char* q = p + (*p == '+' ? 1 : 0);  // Python's float() accepts a leading '+'
    const auto r = std::from_chars(q, end, v);
    if (r.ec != std::errc() || (r.ptr < end && !(*r.ptr == ' ' || *r.ptr == '\n' || *r.ptr == '\r' ||
                                                 *r.ptr == '\t')))
      return -2 - n;  // malformed token n
    out[n++] = v;
    p = r.ptr;
  }
  return n;
}

}  // extern "C"
