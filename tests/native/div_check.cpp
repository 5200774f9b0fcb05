// Host check: lc::div1000 (csrc/lc_fastdiv.cuh) equals IEEE x / 1000.0 bit for bit.
// Usage: div_check <n_random> <seed>   -> prints "<n_checked> <n_mismatch>"
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <random>
#include "../../paper_2601_06288_b200/csrc/lc_fastdiv.cuh"

static long long n_checked = 0, n_bad = 0;
static void chk(double x) {
  volatile double ref = x / 1000.0;
  const double got = lc::div1000(x);
  ++n_checked;
  if (std::memcmp((const void*)&ref, &got, 8) && !(std::isnan(got) && std::isnan(ref))) {
    if (n_bad < 10) std::fprintf(stderr, "div1000(%a): ref %a got %a\n", x, (double)ref, got);
    ++n_bad;
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  std::mt19937_64 rng(argc > 2 ? std::atoll(argv[2]) : 1);
  const double specials[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, 1e-320, 0x1p-1000, 0x1p-1000 * 0.999999,
                             0x1p1000, 0x1p1000 * 1.0000001, 1.0, 1000.0, 999.0, 1001.0, 1e300, 1e308};
  for (double x : specials) { chk(x); chk(-x); }
  for (long long i = 1; i <= 2000000; ++i) { chk((double)i); chk((double)i / 64.0); chk((double)i * 1000.0 + 1.0); }
  for (long long i = 0; i < n; ++i) {
    uint64_t b = rng();
    switch (i & 3) {
      case 0: b = (b & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(1003 + rng() % 80) << 52); break;  // latency-like
      case 1: b = (b & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(1 + rng() % 2046) << 52); break;  // every normal exponent
      case 2: { double v = (double)(rng() % 100000000ull) * (double)(rng() % 4096 + 1); std::memcpy(&b, &v, 8); } break;
      default: { double v = std::ldexp((double)(rng() >> 11), -(int)(rng() % 60)); std::memcpy(&b, &v, 8); }
    }
    double x;
    std::memcpy(&x, &b, 8);
    chk(x);
  }
  std::printf("%lld %lld\n", n_checked, n_bad);
  return 0;
}
