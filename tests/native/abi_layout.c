/* Prints sizeof / offsetof of the C-ABI structs as JSON, for tests/test_native_abi.py. */
#include <stddef.h>
#include <stdio.h>

#include "../../include/llmconf_b200.h"

#define F(T, f) printf("\"%s.%s\": %zu, ", #T, #f, offsetof(T, f))
#define S(T) printf("\"%s\": %zu, ", #T, sizeof(T))

int main(void) {
  printf("{");
  S(lc_db_desc); S(lc_entry); S(lc_combo); S(lc_slot); S(lc_space_desc); S(lc_search_desc);
  S(lc_search_result); S(lc_batch_totals); S(lc_fetch_req); S(lc_query); S(lc_gen_grid); S(lc_dbgen_desc);
  S(lc_step_req); S(lc_step_out);
  F(lc_search_desc, static_stride); F(lc_step_req, batch); F(lc_step_req, load); F(lc_step_out, c1);
  F(lc_step_out, entry_ms); F(lc_step_out, entry_label);
  F(lc_entry, repeat); F(lc_entry, d); F(lc_combo, weight_bytes); F(lc_slot, step); F(lc_slot, pair);
  F(lc_search_desc, budgets); F(lc_search_desc, ctx_capacity); F(lc_search_desc, load);
  F(lc_search_result, best); F(lc_search_result, n_survivors); F(lc_search_result, n_feasible_plans); F(lc_batch_totals, kernel_ms);
  F(lc_batch_totals, n_cells); F(lc_query, d); F(lc_query, kv_len); F(lc_gen_grid, cell_off);
  F(lc_gen_grid, d); F(lc_gen_grid, offset); F(lc_dbgen_desc, amplitude); F(lc_dbgen_desc, compute);
  F(lc_db_desc, compute); F(lc_db_desc, policy); F(lc_space_desc, gclass_of);
  printf("\"end\": 0}\n");
  return 0;
}
