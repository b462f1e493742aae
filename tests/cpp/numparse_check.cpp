// TEST HARNESS: the long-format number parser (csrc/numparse.cuh, compiled
// here for the host) against glibc strtod under the reference's acceptance
// rule (io.hpp:39-46: whole token consumed, nonempty, errno != ERANGE).
// Prints "<cases> cases, <mismatches> mismatches" and the first mismatches.
#include <cerrno>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

static long g_compare = 0;
#define NP_TRACE_COMPARE() (++g_compare)
#include "numparse.cuh"

using namespace dfpca_gpu::numparse;

static const Pow5 kTab[] = {
#include "pow5_128.inc"
};

static long g_cases = 0, g_bad = 0;

static void check(const std::string& tok) {
  ++g_cases;
  errno = 0;
  char* end = nullptr;
  const double ref = std::strtod(tok.c_str(), &end);
  const bool ref_ok = end != tok.c_str() && *end == '\0' && errno != ERANGE;
  double got = 0.0;
  const int st = parse_double(tok.data(), static_cast<int>(tok.size()), kTab, &got);
  bool same = (st == kOk) == ref_ok;
  if (same && ref_ok) same = std::memcmp(&ref, &got, 8) == 0;
  if (!same) {
    if (++g_bad <= 20) {
      unsigned long long a, b;
      std::memcpy(&a, &ref, 8);
      std::memcpy(&b, &got, 8);
      std::printf("MISMATCH '%s': ref ok=%d %016llx got st=%d %016llx\n", tok.substr(0, 120).c_str(), ref_ok, a,
                  st, b);
    }
  }
}

static std::string fmt(const char* f, double v) {
  char buf[1200];
  std::snprintf(buf, sizeof buf, f, v);
  return buf;
}
static std::string fmtl(const char* f, long double v) {
  char buf[1200];
  std::snprintf(buf, sizeof buf, f, v);
  return buf;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 200000;
  std::mt19937_64 rng(20261018);
  auto rand_double = [&]() {
    for (;;) {
      unsigned long long b = rng();
      double d;
      std::memcpy(&d, &b, 8);
      if (std::isfinite(d)) return d;
    }
  };
  const char* fmts[] = {"%.17g", "%.16g", "%.15g", "%.1g", "%.3g", "%.9g", "%.20g", "%.25g", "%.17e", "%a",
                        "%.40e", "%.13a", "%.2a"};
  for (long i = 0; i < n; ++i) {
    double d = rand_double();
    if (i % 3 == 1) d = std::ldexp(d / std::pow(2.0, std::ilogb(d)), static_cast<int>(rng() % 80) - 40);
    for (const char* f : fmts) check(fmt(f, d));
    // halfway point to the next double, exact in long double (normal range)
    if (std::fabs(d) > 1e-300 && std::fabs(d) < 1e300) {
      const long double mid = (static_cast<long double>(d) + std::nextafter(d, INFINITY)) / 2;
      const std::string ex = fmtl("%.780Le", mid);  // exact expansion
      const auto epos = ex.find('e');
      std::string mant = ex.substr(0, epos), ex10 = ex.substr(epos);
      while (mant.size() > 2 && mant.back() == '0') mant.pop_back();
      check(mant + ex10);                         // exactly halfway: ties to even
      check(mant + "0000000001" + ex10);          // just above
      for (int digits : {17, 18, 19, 20, 21, 25, 30}) {
        const std::string t = fmtl(("%." + std::to_string(digits) + "Le").c_str(), mid);
        check(t);
      }
      // just below: truncate the exact expansion at a random length
      const std::size_t cut = 3 + rng() % (mant.size() > 3 ? mant.size() - 3 : 1);
      check(mant.substr(0, cut) + ex10);
    }
  }
  // boundaries
  const double edges[] = {DBL_MIN, DBL_MAX, DBL_TRUE_MIN, std::nextafter(DBL_MIN, 0.0), 1.0, 0.1, 5e-324, 1e-310,
                          2.2250738585072014e-308, 9007199254740993.0};
  for (double e : edges)
    for (int digits = 1; digits < 30; ++digits) {
      check(fmt(("%." + std::to_string(digits) + "g").c_str(), e));
      check(fmt(("%." + std::to_string(digits) + "g").c_str(), -e));
    }
  const char* fixed[] = {"2.2250738585072013e-308", "2.2250738585072012e-308", "2.2250738585072011e-308",
                         "1.7976931348623158e308", "1.7976931348623159e308", "1e309", "1e-400", "0e-999",
                         "-0", "+0.0", "nan", "-nan", "NaN(123)", "nan(0x8)", "nan(abc)", "nan(-1)", "nan(012)",
                         "nan()", "nan(0x)", "nan(08)", "nan(99999999999999999999)", "nan(1", "inf", "-Infinity",
                         "infin", "INFINITYx", "0x1.8p3", "0X1P-1074", "0x1p-1075", "0x1.fffffffffffff8p1023",
                         "0x1.fffffffffffff7p1023", "0x.8p1", "0x1p+", "0x1p", "0x", "0x.p1", " 1.5", "\t-2",
                         "+2", "1.5 ", ".5", "5.", "e5", "1e", "1e+", "-.e1", "1_0", "", " ", "-", "+.", ".",
                         "4503599627370496.5", "4503599627370497.5", "9007199254740993", "9007199254740995",
                         "0.000000000000000000000000000000000000000000001e300",
                         "100000000000000000000000000000000000000e-20", "1e-99999999999999999999",
                         "1e99999999999999999999", "0e99999999999999999999", "0x1.0000000000000800000001p0",
                         "0x1.00000000000008p0", "0x1.00000000000018p0", "0x0.0000000000001p-1022",
                         "0x1.fffffffffffffp-1023", "0x1p-1022", "0x0.fffffffffffff8p-1022"};
  for (const char* t : fixed) check(t);
  // grammar fuzz
  const char alpha[] = "0123456789.eE+-xXpPabcfinINFtyAN()_ \t";
  for (long i = 0; i < n * 4; ++i) {
    std::string t;
    const int len = 1 + static_cast<int>(rng() % 12);
    for (int k = 0; k < len; ++k) t.push_back(alpha[rng() % (sizeof alpha - 1)]);
    check(t);
  }
  // long digit strings
  for (long i = 0; i < n / 10; ++i) {
    std::string t = (rng() & 1) ? "0." : "";
    const int len = 20 + static_cast<int>(rng() % 300);
    for (int k = 0; k < len; ++k) t.push_back(static_cast<char>('0' + rng() % 10));
    if (rng() & 1) t += "e" + std::to_string(static_cast<int>(rng() % 700) - 350);
    check(t);
  }
  std::printf("%ld cases, %ld mismatches (%ld exact comparisons)\n", g_cases, g_bad, g_compare);
  return g_bad ? 1 : 0;
}
