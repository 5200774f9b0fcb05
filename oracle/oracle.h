/* CPU ORACLE (test infrastructure only) -- plain-C restatement of the reference
 * llmconf configuration-search path, used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs as the CHECKER and the
 * CPU baseline.  The product (paper_2601_06288_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks it against the golden reports that
 * tests/golden/make_golden.py produced from the unmodified reference.
 *
 * Inputs are raw database records (not the product's flattened grids), the
 * model / workload / space / disagg scalars, and the MoE popularity weights
 * drawn by numpy on the host (the RNG draw is the one numpy piece not
 * restated).  Arithmetic uses this machine's libm log/exp exactly as CPython's
 * math module does; the library is compiled with -ffp-contract=off.
 */
#ifndef LLMCONF_ORACLE_H
#define LLMCONF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OK_KIND_GEMM, OK_KIND_ATTN_CTX, OK_KIND_ATTN_GEN, OK_KIND_ALLREDUCE, OK_KIND_ALLGATHER,
       OK_KIND_ALLTOALL, OK_KIND_P2P, OK_KIND_MOE_DISPATCH, OK_KIND_MOE_COMBINE, OK_KIND_MOE_GEMM,
       OK_KIND_EMBEDDING, OK_NKINDS };

typedef struct {
  int32_t n;
  const int32_t* kind;     /* OK_KIND_* */
  const int32_t* quant;    /* 0 fp16, 1 fp8, 2 int8, 3 int4 */
  const int32_t* attn;     /* 0 none, 1 MHA, 2 GQA, 3 MLA */
  const int64_t* dims;     /* [n][5] in the kind's canonical order (see oracle.c kind_dims) */
  const double* latency;   /* us */
  /* hardware */
  const char* hw_name;
  double gpu_memory, mem_bw, intra_bw, inter_bw;
  int32_t gpus_per_node;
  double compute[4];       /* per quant; <= 0 means absent */
  int32_t policy;          /* 0 default, 1 strict, 2 clamp, 3 sol */
  const char* backend;
} or_db;

typedef struct {
  const char* name;
  int64_t num_layers, hidden, heads, kv_heads, head_dim, inter, vocab;
  int32_t attn;            /* 1 MHA 2 GQA 3 MLA */
  int64_t mla_kv_dim;
  int32_t is_moe;
  int64_t n_experts, topk, expert_inter, shared_inter;
  int32_t wq, kq;
  int64_t params;          /* ModelSpec.params() */
  /* moe load (only when is_moe): weights from numpy, already float64 */
  const double* moe_weights;
  int32_t moe_n_weights;
} or_model;

typedef struct {
  int64_t isl, osl, prefix;
  int32_t has_ttft; double ttft_limit;
  int32_t has_floor; double speed_floor;   /* WorkloadSpec.speed_floor() */
  int32_t has_tpot_cap; double tpot_cap;   /* WorkloadSpec.tpot_ceiling() */
  int32_t n_budgets; const int64_t* budgets;
  int32_t mode_static, mode_agg, mode_disagg;
  /* candidate space, already in the reference iteration order */
  int32_t n_tp; const int64_t* tp;
  int32_t n_pp; const int64_t* pp;
  int32_t n_ep; const int64_t* ep;
  int32_t n_dp; const int64_t* dp;
  int32_t n_b; const int64_t* batch;
  int32_t has_ctx_capacity; int64_t ctx_capacity;
  int32_t chunked_prefill;
  double kv_mem_fraction;
  int32_t prefill_pool_cap, decode_pool_cap;
  /* disagg constants */
  double ttft_headroom, prefill_util, decode_util;
  int32_t max_x, max_y;
  int32_t static_stride;   /* estimate_static's decode stride (serving_modes.py:236); <= 0: 32 */
} or_search;

/* one evaluated row (static / aggregated estimate or disaggregated plan) */
typedef struct {
  int32_t mode;            /* 0 static, 1 aggregated, 2 disaggregated */
  int32_t cand;            /* candidate index (static/agg) */
  int32_t p_worker, d_worker, x, y;   /* disagg: worker indices into the worker list */
  int64_t gpus;
  double ttft, tpot, speed, thru, r_sys;
  int32_t feasible, frontier;
} or_row;

typedef struct {
  int32_t mode;            /* 0 static 1 agg 2 disagg/prefill 3 disagg/decode */
  int32_t cand;            /* candidate index (modes 0,1) or worker index (2,3) */
  char reason[512];
} or_skip;

typedef struct {
  int64_t tp, pp, ep, dp, batch;
} or_cfg;

typedef struct {
  int32_t n_cand; or_cfg* cand;          /* caller frees with or_free */
  int32_t n_work; or_cfg* work;
  int32_t n_rows; or_row* rows;
  int32_t n_skip; or_skip* skip;
  int32_t n_front; int32_t* front;       /* row indices, frontier order */
  int32_t best;                          /* row index or -1 */
  int32_t nearest;                       /* row index or -1 (only when best < 0) */
  double nearest_violation;
  int64_t n_queries;                     /* query_latency calls the reference would make */
} or_result;

int or_run_search(const or_db* db, const or_model* m, const or_search* s, or_result* out);

/* estimate_static / estimate_aggregated for one config (serving_modes.py:231-341):
 * mode 0 static, 1 aggregated; returns 0 and fills out[4] = ttft, tpot, speed, thru,
 * or a nonzero status with the reference's "Type: message" in reason. */
int or_estimate(const or_db* db, const or_model* m, const or_search* s, const or_cfg* cfg, int mode, double* out,
                char* reason, int reason_len);
void or_free(or_result* r);

/* query_latency (perfdb.py:539-580) for n queries: dims [n][5] in canonical order,
 * kv_len NULL or [n] (<= 0: seq_len), policy -1 = the database's; status 0 ok,
 * 1 missing key, 2 extrapolation, 3 unsupported; msgs NULL or [n][msg_len]. */
int or_query_batch(const or_db* db, int32_t n, const int32_t* kind, const int32_t* quant, const int32_t* attn,
                   const int64_t* dims, const int64_t* kv_len, int32_t policy, double* out, int32_t* status,
                   char* msgs, int32_t msg_len);

/* pieces exposed for unit KATs */
double or_neumaier_sum(const double* xs, int n);
int64_t or_busiest_shard(const double* weights, int e, int64_t total, int64_t topk, int64_t ep,
                         int64_t* counts_out);

#ifdef __cplusplus
}
#endif
#endif
