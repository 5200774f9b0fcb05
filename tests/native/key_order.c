/* Reads "tp pp ep dp batch" lines, prints "combo_code batch_code" per line: the
 * integer keys of csrc/lc_keys.h, checked against Python string order by
 * tests/test_native_abi.py. */
#include <stdio.h>
#include "../../paper_2601_06288_b200/csrc/lc_keys.h"

int main(void) {
  long long tp, pp, ep, dp, b;
  while (scanf("%lld %lld %lld %lld %lld", &tp, &pp, &ep, &dp, &b) == 5)
    printf("%llu %llu\n", (unsigned long long)lc_combo_code(tp, pp, ep, dp), (unsigned long long)lc_batch_code(b));
  return 0;
}
