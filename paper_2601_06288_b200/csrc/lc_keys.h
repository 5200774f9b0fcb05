// Integer keys that sort like the reference's config-key strings.
//
// ParallelConfig.key() is "tp{tp}pp{pp}ep{ep}dp{dp}b{batch}" (model.py:205-206),
// and _pool_rank breaks rate ties by that string (search.py:276-277).  Python
// compares strings code point by code point; the literal parts are equal, so two
// keys first differ inside the first numeric field whose decimal strings differ:
// a digit against a digit, or -- one decimal string a prefix of the other -- a
// digit against the following literal letter (which sorts after every digit) or,
// for the batch field, against the end of the string (which sorts first).
//
// Each field is therefore encoded as its decimal digits, left-aligned and padded
// to a fixed width with a filler that sorts after the digits (tp/pp/ep/dp: filler
// 10) or before them (batch: digits + 1, filler 0), as a base-11 number.  The
// combo fields pack into one 56-bit code (values up to 9999), the batch into a
// 35-bit code (values up to 9,999,999,999).  lc_space_upload ranks the combos by
// their code, so a candidate's key is rank << 36 | batch code: one 64-bit
// integer compare instead of formatting two strings.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LC_HD __host__ __device__ __forceinline__
#else
#define LC_HD static inline
#endif

#define LC_KEY_FIELD_MAX 9999ll
#define LC_KEY_BATCH_MAX 9999999999ll

// tp / pp / ep / dp field (a letter follows): 4 base-11 places, filler 10
LC_HD uint64_t lc_field_code(int64_t v) {
  char d[4];
  int n = 0;
  int64_t p = 1;
  while (v / p >= 10) p *= 10;
  for (; p > 0 && n < 4; p /= 10) d[n++] = (char)((v / p) % 10);
  uint64_t code = 0;
  for (int i = 0; i < 4; ++i) code = code * 11u + (uint64_t)(i < n ? d[i] : 10);
  return code;
}

// batch field (the string ends): 10 base-11 places, digit + 1, filler 0
LC_HD uint64_t lc_batch_code(int64_t v) {
  char d[10];
  int n = 0;
  int64_t p = 1;
  while (v / p >= 10) p *= 10;
  for (; p > 0 && n < 10; p /= 10) d[n++] = (char)((v / p) % 10);
  uint64_t code = 0;
  for (int i = 0; i < 10; ++i) code = code * 11u + (uint64_t)(i < n ? d[i] + 1 : 0);
  return code;
}

// (tp, pp, ep, dp) in string order: 4 fields x 4 places = 11^16 < 2^56
LC_HD uint64_t lc_combo_code(int64_t tp, int64_t pp, int64_t ep, int64_t dp) {
  const uint64_t w = 14641u;  // 11^4
  return ((lc_field_code(tp) * w + lc_field_code(pp)) * w + lc_field_code(ep)) * w + lc_field_code(dp);
}
