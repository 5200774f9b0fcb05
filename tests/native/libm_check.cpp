// Host check: the device restatement of glibc log/exp (csrc/glibc_libm.cuh),
// compiled here for the CPU, must equal this machine's libm bit for bit.
// Usage: libm_check <n_random> <seed>   -> prints "<n_checked> <n_mismatch>"
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <random>
#include "../../paper_2601_06288_b200/csrc/glibc_libm.cuh"

static const double LOG_TAB[256] = GLIBC_LOG_TAB_INIT;
static const uint64_t EXP_TAB[256] = GLIBC_EXP_TAB_INIT;

static long long n_checked = 0, n_bad = 0;
static void chk_log(double x) {
  volatile double ref = std::log(x);
  double got = glibc::log_fma(x, LOG_TAB);
  ++n_checked;
  if (glibc::as_u64(got) != glibc::as_u64(ref)) {
    if (n_bad < 10) std::fprintf(stderr, "log(%a): ref %a got %a\n", x, (double)ref, got);
    ++n_bad;
  }
}
static void chk_exp(double x) {
  volatile double ref = std::exp(x);
  double got = glibc::exp_fma(x, EXP_TAB);
  ++n_checked;
  if (glibc::as_u64(got) != glibc::as_u64(ref) && !(std::isnan(got) && std::isnan(ref))) {
    if (n_bad < 10) std::fprintf(stderr, "exp(%a): ref %a got %a\n", x, (double)ref, got);
    ++n_bad;
  }
}

int main(int argc, char** argv) {
  long long n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  unsigned seed = argc > 2 ? (unsigned)std::atoi(argv[2]) : 1;
  // every integer coordinate in [2, 2^22) plus a strided sweep up to 2^34
  for (long long v = 2; v < (1ll << 22); ++v) chk_log((double)v);
  for (long long v = (1ll << 22); v < (1ll << 34); v += 4099) chk_log((double)v);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-40.0, 60.0), w(-745.0, 709.0), big(1.07, 1e15);
  for (long long i = 0; i < n; ++i) {
    chk_exp(u(rng));
    if ((i & 7) == 0) chk_exp(w(rng));
    if ((i & 3) == 0) chk_log(big(rng));
  }
  const double specials[] = {0.0, -0.0, 1e-300, -1e-300, 709.78, 709.79, -745.2, -708.5, -720.3,
                             710.0, 1000.0, -1000.0, INFINITY, -INFINITY, 5e-17, -5e-17, 512.5, -512.5};
  for (double s : specials) chk_exp(s);
  std::printf("%lld %lld\n", n_checked, n_bad);
  return n_bad ? 1 : 0;
}
