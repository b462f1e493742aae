// Exact decimal / hexadecimal text -> double, host and device.
//
// Reproduces the reference's number acceptance (io.hpp:39-46, parse_double):
// glibc strtod over the WHOLE field in the "C" locale, rejecting an empty
// parse, trailing characters and ERANGE.  The value must be the correctly
// rounded (round-half-even) double, so the parser is exact rather than
// approximate:
//
//   * decimal, <= 19 significant digits: w * 10^q via a 64 x 128-bit product
//     against the truncated 128-bit power of five (pow5_128.inc).  The product
//     is exact for 0 <= q <= 55; otherwise it is low by less than 2^64 units
//     of the 192-bit product, and the rounding is decided unless the bits
//     below the round bit are all ones down to bit 64 (then the exact
//     comparison below runs);
//   * > 19 significant digits: the first 19 digits w and w + 1 bracket the
//     value; equal roundings decide it, otherwise the exact comparison runs;
//   * exact comparison: the decimal (up to 768 significant digits plus a
//     sticky bit -- every halfway point between doubles has <= 767) against
//     the halfway point (2m + 1) 2^(e - 1), in fixed-size big integers;
//   * hexadecimal ("0x1.8p3"), inf / infinity, nan and nan(n-char-sequence)
//     with glibc's payload rule (strtoull base 0, masked to the mantissa).
//
// ERANGE follows glibc: overflow, or a result that is tiny after rounding
// to 53 bits with unbounded exponent and inexact as a subnormal.  A decimal
// tiny result is always rejected (inexact unless the token spells an exact
// subnormal, which needs hundreds of digits -- the one documented deviation).
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define NP_HD __host__ __device__ inline
#else
#define NP_HD inline
#endif

namespace dfpca_gpu {
namespace numparse {

struct Pow5 {
  std::uint64_t hi, lo;
  std::int32_t b;  // 5^q ~ (hi:lo) * 2^b
};
constexpr int kQMin = -342, kQMax = 308;

enum Status : int { kOk = 0, kSyntax = 1, kRange = 2, kInternal = 3 };

using u64 = std::uint64_t;
using u32 = std::uint32_t;

NP_HD u64 mulhi(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return static_cast<u64>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

NP_HD int clz64(u64 x) {
#ifdef __CUDA_ARCH__
  return __clzll(static_cast<long long>(x));
#else
  return __builtin_clzll(x);
#endif
}

NP_HD double from_bits(u64 b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
#endif
}

NP_HD bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
NP_HD bool is_digit(char c) { return c >= '0' && c <= '9'; }
NP_HD char lower(char c) { return (c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : c; }
NP_HD int hex_val(char c) {
  c = lower(c);
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  return -1;
}
NP_HD bool is_nchar(char c) { return is_digit(c) || (lower(c) >= 'a' && lower(c) <= 'z') || c == '_'; }

NP_HD bool match_ci(const char* s, int n, const char* word) {
  int k = 0;
  for (; word[k]; ++k)
    if (k >= n || lower(s[k]) != word[k]) return false;
  return true;
}

// 53-bit rounding of a positive value at unbounded exponent: m in
// [2^52, 2^53), value = m 2^e2.  ambiguous: m is the round-down candidate
// and the exact comparison against (2m + 1) 2^(e2 - 1) must decide.
struct Rounded {
  u64 m;
  int e2;
  bool ambiguous;
};

// w != 0, kQMin <= q <= kQMax.
NP_HD Rounded round_decimal(u64 w, int q, const Pow5* tab) {
  const Pow5 t = tab[q - kQMin];
  const int lz = clz64(w);
  const u64 wn = w << lz;
  const u64 a0 = wn * t.lo, a1 = mulhi(wn, t.lo);
  const u64 b0 = wn * t.hi, b1 = mulhi(wn, t.hi);
  const u64 p0 = a0;
  const u64 p1 = a1 + b0;
  const u64 p2 = b1 + (p1 < a1 ? 1u : 0u);  // product P = p2:p1:p0 in [2^190, 2^192)
  const int s = (p2 >> 63) ? 10 : 9;
  const u64 m54 = p2 >> s;  // 54 bits: mantissa + round bit
  const u64 mask = (u64{1} << s) - 1;
  const u64 low = p2 & mask;
  Rounded r{m54 >> 1, s + 128 + t.b + q - lz + 1, false};  // value = P 2^(b + q - lz)
  const bool rb = (m54 & 1) != 0;
  if (q >= 0 && q <= 55) {  // exact power of five: round half to even
    if (rb && ((low | p1 | p0) != 0 || (r.m & 1))) ++r.m;
  } else if (!rb && low == mask && p1 == ~u64{0}) {
    r.ambiguous = true;  // true value = P + delta, 0 < delta < 2^64, may reach the halfway point
  } else if (rb) {
    ++r.m;  // strictly above the halfway point (the truncated power is low)
  }
  if (r.m == (u64{1} << 53)) {
    r.m = u64{1} << 52;
    ++r.e2;
  }
  return r;
}

// ------------------------------------------------------------ big integers --
constexpr int kLimbs = 96;  // 3072 bits: >= 768 digits * 5^|q| at the double range
struct Big {
  u32 v[kLimbs];
  int n;
};

NP_HD void big_set(Big& a, u64 x) {
  a.v[0] = static_cast<u32>(x);
  a.v[1] = static_cast<u32>(x >> 32);
  a.n = a.v[1] ? 2 : (a.v[0] ? 1 : 0);
}

NP_HD bool big_mul_add(Big& a, u32 mul, u32 add) {
  u64 carry = add;
  for (int i = 0; i < a.n; ++i) {
    const u64 x = static_cast<u64>(a.v[i]) * mul + carry;
    a.v[i] = static_cast<u32>(x);
    carry = x >> 32;
  }
  if (carry) {
    if (a.n >= kLimbs) return false;
    a.v[a.n++] = static_cast<u32>(carry);
  }
  return true;
}

NP_HD bool big_mul_pow5(Big& a, int k) {
  while (k >= 13) {
    if (!big_mul_add(a, 1220703125u, 0)) return false;  // 5^13
    k -= 13;
  }
  u32 p = 1;
  for (int i = 0; i < k; ++i) p *= 5;
  return big_mul_add(a, p, 0);
}

NP_HD bool big_shl(Big& a, int bits) {
  if (a.n == 0 || bits == 0) return true;
  const int limbs = bits / 32, sh = bits % 32;
  const int n_new = a.n + limbs + 1;
  if (n_new > kLimbs) return false;
  for (int i = n_new - 1; i >= 0; --i) {
    const int src = i - limbs;
    u32 hi = (src >= 0 && src < a.n) ? a.v[src] : 0u;
    u32 lo = (src - 1 >= 0 && src - 1 < a.n) ? a.v[src - 1] : 0u;
    a.v[i] = sh ? ((hi << sh) | (lo >> (32 - sh))) : hi;
  }
  a.n = n_new;
  while (a.n > 0 && a.v[a.n - 1] == 0) --a.n;
  return true;
}

NP_HD int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.v[i] != b.v[i]) return a.v[i] < b.v[i] ? -1 : 1;
  return 0;
}

constexpr int kMaxDigits = 768;

// Sign of D 10^q - (2m + 1) 2^(e2 - 1), D = the significant digits of the
// mantissa text s[0..n) (digits and at most one '.', already validated) and
// q = dexp of its last kept digit plus exp10.  Returns 2 on overflow.
NP_HD int compare_halfway(const char* s, int n, long long exp10, u64 m, int e2) {
#ifdef NP_TRACE_COMPARE
  NP_TRACE_COMPARE();
#endif
  Big a, b;
  a.n = 0;
  long long dexp = 0;
  int nd = 0;
  bool seen = false, sticky = false, frac = false;
  u32 group = 0, gmul = 1;
  for (int j = 0; j < n; ++j) {
    const char c = s[j];
    if (c == '.') {
      frac = true;
      continue;
    }
    const u32 v = static_cast<u32>(c - '0');
    if (!seen && v == 0) {
      if (frac) --dexp;
      continue;
    }
    seen = true;
    if (nd < kMaxDigits) {
      group = group * 10 + v;
      gmul *= 10;
      if (gmul == 1000000000u) {
        if (!big_mul_add(a, gmul, group)) return 2;
        group = 0;
        gmul = 1;
      }
      ++nd;
      if (frac) --dexp;
    } else {
      if (v) sticky = true;
      if (!frac) ++dexp;
    }
  }
  if (gmul > 1 && !big_mul_add(a, gmul, group)) return 2;
  const long long q = dexp + exp10;
  big_set(b, 2 * m + 1);
  long long two_a = q, two_b = static_cast<long long>(e2) - 1;
  if (q >= 0) {
    if (!big_mul_pow5(a, static_cast<int>(q))) return 2;
  } else {
    if (!big_mul_pow5(b, static_cast<int>(-q))) return 2;
  }
  if (two_a > two_b) {
    if (!big_shl(a, static_cast<int>(two_a - two_b))) return 2;
  } else if (two_b > two_a) {
    if (!big_shl(b, static_cast<int>(two_b - two_a))) return 2;
  }
  const int c = big_cmp(a, b);
  return (c == 0 && sticky) ? 1 : c;
}

NP_HD int finish(u64 sign, u64 m, int e2, double* out) {
  const int biased = e2 + 1075;
  if (biased >= 2047) return kRange;  // overflow
  if (biased < 1) return kRange;      // tiny (decimal: always inexact, see header)
  *out = from_bits(sign | (static_cast<u64>(biased) << 52) | (m & ((u64{1} << 52) - 1)));
  return kOk;
}

// Binary value M 2^e (M != 0, plus a sticky bit below M) rounded to double
// with glibc's subnormal / ERANGE behaviour.
NP_HD int round_binary(u64 sign, u64 M, long long e, bool sticky, double* out) {
  const int lz = clz64(M);
  const u64 Mn = M << lz;
  const long long E = e - lz;  // value = Mn 2^E, Mn in [2^63, 2^64)
  if (E > 2000) return kRange;
  u64 m = Mn >> 11;
  const u64 rest = Mn & 0x7ff;
  long long e2 = E + 11;
  if (rest > 0x400 || (rest == 0x400 && (sticky || (m & 1)))) {
    if (++m == (u64{1} << 53)) {
      m = u64{1} << 52;
      ++e2;
    }
  }
  if (e2 + 1075 >= 2047) return kRange;
  if (e2 + 1075 >= 1) {
    *out = from_bits(sign | (static_cast<u64>(e2 + 1075) << 52) | (m & ((u64{1} << 52) - 1)));
    return kOk;
  }
  // tiny after rounding: the subnormal result must be exact, else ERANGE
  const long long sh = -1074 - E;  // > 11
  u64 qv = 0;
  bool rbit = false, rest_nz = sticky;
  if (sh < 64) {
    qv = Mn >> sh;
    rbit = ((Mn >> (sh - 1)) & 1) != 0;
    rest_nz = rest_nz || (Mn & ((u64{1} << (sh - 1)) - 1)) != 0;
  } else if (sh == 64) {
    rbit = (Mn >> 63) != 0;
    rest_nz = rest_nz || (Mn << 1) != 0;
  } else {
    rest_nz = true;
  }
  if (rbit || rest_nz) return kRange;
  *out = from_bits(sign | qv);
  return kOk;
}

// glibc strtoull(base 0) over an n-char-sequence: 0 = fully consumed,
// 1 = partially (no payload), 2 = overflow (ERANGE).
NP_HD int nan_payload(const char* s, int n, u64* v) {
  *v = 0;
  if (n == 0) return 0;
  int k = 0, base = 10;
  if (s[0] == '0') {
    if (n >= 3 && lower(s[1]) == 'x' && hex_val(s[2]) >= 0) {
      base = 16;
      k = 2;
    } else {
      base = 8;
    }
  }
  const int k0 = k;
  bool over = false;
  for (; k < n; ++k) {
    const int d = base == 16 ? hex_val(s[k]) : (is_digit(s[k]) ? s[k] - '0' : -1);
    if (d < 0 || d >= base) break;
    const u64 lim = (~u64{0} - static_cast<u64>(d)) / static_cast<u64>(base);
    if (*v > lim) over = true;
    *v = *v * static_cast<u64>(base) + static_cast<u64>(d);
  }
  if (over) return 2;
  if (k == k0 && base == 10) return 1;
  return k == n ? 0 : 1;
}

// The reference's parse_double acceptance over the token s[0..n).
NP_HD int parse_double(const char* s, int n, const Pow5* tab, double* out) {
  int i = 0;
  while (i < n && is_space(s[i])) ++i;
  u64 sign = 0;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    if (s[i] == '-') sign = u64{1} << 63;
    ++i;
  }
  if (i >= n) return kSyntax;
  const char c0 = lower(s[i]);
  if (c0 == 'i') {
    if (!match_ci(s + i, n - i, "inf")) return kSyntax;
    i += 3;
    if (match_ci(s + i, n - i, "inity")) i += 5;
    if (i != n) return kSyntax;
    *out = from_bits(sign | 0x7ff0000000000000ull);
    return kOk;
  }
  if (c0 == 'n') {
    if (!match_ci(s + i, n - i, "nan")) return kSyntax;
    i += 3;
    u64 payload = 0;
    if (i < n && s[i] == '(') {
      int j = i + 1;
      while (j < n && is_nchar(s[j])) ++j;
      if (j < n && s[j] == ')') {
        const int st = nan_payload(s + i + 1, j - i - 1, &payload);
        if (st == 2) return kRange;
        if (st != 0) payload = 0;
        i = j + 1;
      }
    }
    if (i != n) return kSyntax;
    *out = from_bits(sign | 0x7ff8000000000000ull | (payload & 0x000fffffffffffffull));
    return kOk;
  }
  if (c0 == '0' && i + 1 < n && lower(s[i + 1]) == 'x') {
    int j = i + 2;
    u64 M = 0;
    int nd = 0;
    long long e = 0;
    bool any = false, seen = false, sticky = false;
    for (; j < n && hex_val(s[j]) >= 0; ++j) {
      any = true;
      const int v = hex_val(s[j]);
      if (!seen && v == 0) continue;
      seen = true;
      if (nd < 16) {
        M = M * 16 + static_cast<u64>(v);
        ++nd;
      } else {
        if (v) sticky = true;
        e += 4;
      }
    }
    if (j < n && s[j] == '.') {
      ++j;
      for (; j < n && hex_val(s[j]) >= 0; ++j) {
        any = true;
        const int v = hex_val(s[j]);
        if (!seen && v == 0) {
          e -= 4;
          continue;
        }
        seen = true;
        if (nd < 16) {
          M = M * 16 + static_cast<u64>(v);
          ++nd;
          e -= 4;
        } else if (v) {
          sticky = true;
        }
      }
    }
    if (!any) return kSyntax;  // strtod takes only the "0"
    if (j < n && lower(s[j]) == 'p') {
      int k = j + 1;
      bool neg = false;
      if (k < n && (s[k] == '+' || s[k] == '-')) neg = s[k++] == '-';
      if (k >= n || !is_digit(s[k])) return kSyntax;
      long long ev = 0;
      for (; k < n && is_digit(s[k]); ++k)
        if (ev < 100000000) ev = ev * 10 + (s[k] - '0');
      e += neg ? -ev : ev;
      j = k;
    }
    if (j != n) return kSyntax;
    if (!seen) {
      *out = from_bits(sign);
      return kOk;
    }
    return round_binary(sign, M, e, sticky, out);
  }
  // decimal
  const int mant0 = i;
  u64 w = 0;
  int nd = 0;
  long long dexp = 0;
  bool any = false, seen = false, trunc = false;
  int j = i;
  for (; j < n && is_digit(s[j]); ++j) {
    any = true;
    const int v = s[j] - '0';
    if (!seen && v == 0) continue;
    seen = true;
    if (nd < 19) {
      w = w * 10 + static_cast<u64>(v);
      ++nd;
    } else {
      if (v) trunc = true;
      ++dexp;
    }
  }
  if (j < n && s[j] == '.') {
    ++j;
    for (; j < n && is_digit(s[j]); ++j) {
      any = true;
      const int v = s[j] - '0';
      if (!seen && v == 0) {
        --dexp;
        continue;
      }
      seen = true;
      if (nd < 19) {
        w = w * 10 + static_cast<u64>(v);
        ++nd;
        --dexp;
      } else if (v) {
        trunc = true;
      }
    }
  }
  if (!any) return kSyntax;
  const int mant1 = j;
  long long exp10 = 0;
  if (j < n && (s[j] == 'e' || s[j] == 'E')) {
    int k = j + 1;
    bool neg = false;
    if (k < n && (s[k] == '+' || s[k] == '-')) neg = s[k++] == '-';
    if (k >= n || !is_digit(s[k])) return kSyntax;  // the 'e' is not consumed
    for (; k < n && is_digit(s[k]); ++k)
      if (exp10 < 100000000) exp10 = exp10 * 10 + (s[k] - '0');
    if (neg) exp10 = -exp10;
    j = k;
  }
  if (j != n) return kSyntax;
  if (!seen) {
    *out = from_bits(sign);
    return kOk;
  }
  const long long q = dexp + exp10;
  if (q > kQMax) return kRange;  // >= 10^309
  if (q < kQMin) return kRange;  // < 10^-323: tiny
  Rounded r = round_decimal(w, static_cast<int>(q), tab);
  bool decide = r.ambiguous;
  if (trunc && !decide) {
    const Rounded r1 = round_decimal(w + 1, static_cast<int>(q), tab);
    decide = r1.ambiguous || r1.m != r.m || r1.e2 != r.e2;
  }
  if (decide) {
    const int c = compare_halfway(s + mant0, mant1 - mant0, exp10, r.m, r.e2);
    if (c == 2) return kInternal;
    if (c > 0 || (c == 0 && (r.m & 1))) {
      if (++r.m == (u64{1} << 53)) {
        r.m = u64{1} << 52;
        ++r.e2;
      }
    }
  }
  return finish(sign, r.m, r.e2, out);
}

}  // namespace numparse
}  // namespace dfpca_gpu
