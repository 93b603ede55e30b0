// Text formats either side of the hot path (reference
// io.py): a multithreaded row formatter that writes floats exactly as
// Python's repr(float) does (shortest round-trip digits, io.py:42-47) and
// integers in decimal, so the writers in paper_2005_02704_b200/io.py produce
// the reference's bytes at native speed.
//
// repr rules (CPython format_float_short, mode 'r'): shortest digits d1..dn
// and decimal exponent E (value = d1.d2..dn x 10^E); fixed notation when
// -4 <= E < 16 (a ".0" is appended to integral values), otherwise
// d1[.d2..dn]e(+|-)XX with at least two exponent digits; "nan", "inf",
// "-inf"; "-0.0".

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lidarseg_b200.h"

namespace {

// Writes repr(x) at p, returns the end pointer (at most 32 bytes).
char* repr_double(double x, char* p) {
  if (std::isnan(x)) { std::memcpy(p, "nan", 3); return p + 3; }
  if (std::isinf(x)) {
    if (x < 0) *p++ = '-';
    std::memcpy(p, "inf", 3);
    return p + 3;
  }
  if (x == 0.0) {
    if (std::signbit(x)) *p++ = '-';
    std::memcpy(p, "0.0", 3);
    return p + 3;
  }
  char buf[40];
  auto res = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  // buf = [-]d[.ddd]e(+|-)XX[X]
  char* e = std::find(buf, res.ptr, 'e');
  const char* m = buf;
  if (*m == '-') { *p++ = '-'; ++m; }
  char digits[24];
  int nd = 0;
  for (const char* q = m; q < e; ++q)
    if (*q != '.') digits[nd++] = *q;
  int E = 0;
  std::from_chars(e + 1 + (e[1] == '+' ? 1 : 0), res.ptr, E);
  if (E >= -4 && E < 16) {
    if (E >= 0) {
      const int ip = E + 1;  // integer digits
      for (int i = 0; i < ip; ++i) *p++ = i < nd ? digits[i] : '0';
      *p++ = '.';
      if (nd > ip) {
        for (int i = ip; i < nd; ++i) *p++ = digits[i];
      } else {
        *p++ = '0';
      }
    } else {
      *p++ = '0';
      *p++ = '.';
      for (int i = 0; i < -E - 1; ++i) *p++ = '0';
      for (int i = 0; i < nd; ++i) *p++ = digits[i];
    }
    return p;
  }
  *p++ = digits[0];
  if (nd > 1) {
    *p++ = '.';
    for (int i = 1; i < nd; ++i) *p++ = digits[i];
  }
  *p++ = 'e';
  *p++ = E < 0 ? '-' : '+';
  const int a = E < 0 ? -E : E;
  if (a < 10) *p++ = '0';
  auto r = std::to_chars(p, p + 8, a);
  return r.ptr;
}

char* int_text(double v, char* p) {
  auto r = std::to_chars(p, p + 24, (long long)v);
  return r.ptr;
}

constexpr size_t kMaxCell = 34;  // longest repr / int64 text + separator

}  // namespace

extern "C" {

int64_t lseg_format_rows(int64_t n_rows, int32_t n_cols, const double* values, const uint8_t* col_kind,
                         char* out, int64_t capacity, int32_t threads) {
  if (n_rows < 0 || n_cols < 1 || !values || !col_kind) return -1;
  if (n_rows == 0) return 0;
  const int64_t worst = n_rows * (int64_t)n_cols * (int64_t)kMaxCell;
  if (!out) return worst;  // size query
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if ((int64_t)nt > n_rows / 256 + 1) nt = (int)(n_rows / 256 + 1);
  // each thread formats a contiguous block of rows into its own buffer
  std::vector<std::string> parts(nt);
  auto work = [&](int t) {
    const int64_t r0 = n_rows * t / nt, r1 = n_rows * (t + 1) / nt;
    std::string& s = parts[t];
    s.resize((size_t)((r1 - r0) * n_cols * kMaxCell));
    char* p = s.data();
    for (int64_t r = r0; r < r1; ++r) {
      const double* row = values + r * n_cols;
      for (int c = 0; c < n_cols; ++c) {
        p = col_kind[c] ? int_text(row[c], p) : repr_double(row[c], p);
        *p++ = (c + 1 == n_cols) ? '\n' : ' ';
      }
    }
    s.resize((size_t)(p - s.data()));
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t total = 0;
  for (auto& s : parts) total += (int64_t)s.size();
  if (total > capacity) return -2;
  char* p = out;
  for (auto& s : parts) {
    std::memcpy(p, s.data(), s.size());
    p += s.size();
  }
  return total;
}

}  // extern "C"
