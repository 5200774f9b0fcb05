/* llmconf_b200 -- C ABI of the B200 configuration-search engine.
 *
 * Drop-in boundary.  The reference has no plugin registry: its seam is the
 * Python function llmconf.search.run_search(db, model, workload, space, jobs,
 * disagg_constants) (/root/reference/pkg/src/llmconf/search.py:280-358), called
 * by the CLI (cli.py:239, 286) and the HTTP service (service.py:230).  The
 * host shim paper_2601_06288_b200.run_search keeps that signature and crosses
 * into this library through ctypes; the entry points below are what that
 * binding (or any other FFI) calls.  Plain pointers and sizes only.
 *
 *   reference piece                              replaced by
 *   ------------------------------------------   -----------------------------------
 *   PerfDatabase._grids (perfdb.py:283-355)      lc_db_upload   (SoA grids in HBM/smem)
 *   decompose (model.py:271-406) per (tp,pp,ep)  lc_space_upload (host-compiled plan templates)
 *   enumerate_candidates (search.py:82-113)      K0 inside lc_search_batch
 *   busiest_shard_tokens (moe_load.py:141-147)   K3 inside lc_search_batch
 *   get_step_latency / estimate_static /         K2 inside lc_search_batch
 *     estimate_aggregated / *_candidate
 *     (estimator.py:71-156, serving_modes.py:231-381)
 *   _pool_rank top-k, estimate_disaggregated     K5 inside lc_search_batch
 *     (search.py:276-277, 338-341; serving_modes.py:449-494)
 *   meets_sla / pareto_filter / select_best /    K4 inside lc_search_batch
 *     nearest_miss (search.py:129-208)
 *
 * Threading: one lc_ctx per host thread (it owns a CUDA stream and workspace).
 * lc_db / lc_space handles are immutable after upload and may be shared by
 * contexts on the same device.  Every function returns LC_OK (0) or a negative
 * code; lc_last_error() describes the last failure on the calling thread.
 */
#ifndef LLMCONF_B200_H
#define LLMCONF_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LC_ABI_VERSION 3
#define LC_MAX_ENTRIES 16   /* plan entries per (tp, pp, ep) template */
#define LC_MAX_BUDGETS 16
#define LC_MAX_EXPERTS 1024

enum { LC_OK = 0, LC_ERR_ARG = -1, LC_ERR_CUDA = -2, LC_ERR_STATE = -3 };

/* extrapolation policy (perfdb.py:46) */
enum { LC_POLICY_DEFAULT = 0, LC_POLICY_STRICT = 1, LC_POLICY_CLAMP = 2, LC_POLICY_SOL = 3 };

/* operator kinds (perfdb.py:27-39) */
enum {
  LC_KIND_GEMM = 0, LC_KIND_ATTN_CTX, LC_KIND_ATTN_GEN, LC_KIND_ALLREDUCE, LC_KIND_ALLGATHER,
  LC_KIND_ALLTOALL, LC_KIND_P2P, LC_KIND_MOE_DISPATCH, LC_KIND_MOE_COMBINE, LC_KIND_MOE_GEMM,
  LC_KIND_EMBEDDING
};

/* plan entry labels, in decompose order (model.py:313-404) */
enum {
  LC_LBL_EMBEDDING = 0, LC_LBL_QKV, LC_LBL_CTX_ATTN, LC_LBL_GEN_ATTN, LC_LBL_OUT_PROJ, LC_LBL_MLP_UP,
  LC_LBL_MLP_DOWN, LC_LBL_ROUTER, LC_LBL_SHARED_UP, LC_LBL_SHARED_DOWN, LC_LBL_EXPERT_FFN,
  LC_LBL_DISPATCH, LC_LBL_COMBINE, LC_LBL_ATTN_AR, LC_LBL_MLP_AR, LC_LBL_STAGE_BOUNDARY
};

/* how an entry's interpolated coordinates follow from (n_ctx, n_gen, seq) */
enum {
  LC_COORD_TOKENS = 0,  /* d0 = n_ctx + n_gen                              */
  LC_COORD_MSG = 1,     /* d0 = (n_ctx + n_gen) * hidden * 2               */
  LC_COORD_CTX = 2,     /* (d0, d1) = (n_ctx/seq, seq) or (1, n_ctx) mixed */
  LC_COORD_GEN = 3,     /* (d0, d1) = (n_gen, seq)                         */
  LC_COORD_EXPERT = 4   /* d0 = expert tokens (balanced or skewed)         */
};

/* lc_search_desc.modes bits */
enum { LC_MODE_STATIC = 1, LC_MODE_AGGREGATED = 2, LC_MODE_DISAGGREGATED = 4,
       LC_MODE_FORCE = 16 /* skip the memory-fit and budget filters (single-config estimates) */,
       LC_MODE_NO_PLANS = 32 /* disaggregated pools are selected (lc_fetch_pools) but no plans are built:
                                the per-rank pass of a search sharded across GPUs */ };

/* per-row status codes; the failing entry's label sits in bits 8..15 */
enum {
  LC_ST_OK = 0, LC_ST_MISSING_KEY = 1, LC_ST_EXTRAPOLATION = 2, LC_ST_UNSUPPORTED = 3,
  LC_ST_INFEASIBLE_CHUNK_OFF = 4, LC_ST_INFEASIBLE_NO_DECODE_SLOT = 5, LC_ST_NOT_EVALUATED = 255
};

/* ---------------------------------------------------------------- database */
typedef struct {
  int32_t n_grids;
  const int32_t* grid_ndim;      /* [n_grids] 1 or 2 */
  const int32_t* grid_axis_off;  /* [n_grids*2] offset into axis_val/axis_log */
  const int32_t* grid_axis_len;  /* [n_grids*2] */
  const int32_t* grid_cell_off;  /* [n_grids] offset into cell/cell_log, row-major (axis 0 major) */
  int32_t n_axis;
  const int64_t* axis_val;       /* sorted per grid */
  const double* axis_log;        /* math.log(axis_val), computed by the host like the reference */
  int32_t n_cells;
  const double* cell;            /* latency_us */
  const double* cell_log;        /* math.log(cell) */
  double mem_bandwidth, intra_node_bandwidth, inter_node_bandwidth, gpu_memory;
  int32_t gpus_per_node;
  double compute[4];             /* FLOP/s for fp16, fp8, int8, int4; <= 0 = absent */
  int32_t policy;                /* LC_POLICY_* */
} lc_db_desc;

/* ------------------------------------------- model x candidate-space plan */
typedef struct {
  int32_t label, kind, quant, grid;  /* grid < 0: no grid for this key (MissingKeyError) */
  int32_t coord, _pad;
  int64_t repeat;
  int64_t d[5];                      /* canonical dims; fixed ones filled, axes set on device */
} lc_entry;

typedef struct {
  int64_t tp, pp, ep, dp, gpus;
  int32_t tp_i, ep_i;                /* indices into the sorted tp / ep value lists */
  int32_t tmpl;                      /* template index */
  int32_t _pad;
  double weight_bytes;               /* memory_footprint().weight_bytes (model.py:446) */
  double kv_token_bytes;             /* memory_footprint().kv_bytes_per_token (model.py:448-452) */
} lc_combo;

/* a query family priced once per (search, batch): one step kind, one grid, one
 * coordinate recipe (latency is a pure function of grid and coordinates) */
enum { LC_STEP_PREFILL = 0, LC_STEP_GEN = 1, LC_STEP_MIXED = 2 };
typedef struct {
  lc_entry e;                        /* grid, kind, quant, fixed dims, coordinate recipe */
  int32_t step;                      /* LC_STEP_* */
  int32_t pair;                      /* expert recipe: tp_i * n_ep + ep_i, else -1 */
} lc_slot;

typedef struct {
  int64_t hidden, topk, n_experts;
  int32_t is_moe;
  int32_t n_combos;                  /* consistent (tp,pp,ep,dp) in the reference's nested order */
  const lc_combo* combos;
  int32_t n_tmpl;
  const int32_t* tmpl_n_entries;     /* [n_tmpl] */
  const lc_entry* entries;           /* [n_tmpl * LC_MAX_ENTRIES] */
  int32_t n_tp, n_ep;                /* sizes of the tp / ep value lists */
  int32_t n_slots;
  const lc_slot* slots;
  const int32_t* slot_of;            /* [n_tmpl * LC_MAX_ENTRIES * 3]: slot per (template, entry, step), -1 absent */
  int32_t n_gen_classes;             /* distinct generation-attention grids (static decode series) */
  const lc_entry* gen_classes;
  const int32_t* gclass_of;          /* [n_tmpl] */
} lc_space_desc;

/* ------------------------------------------------------------------ search */
typedef struct {
  int64_t isl, osl, prefix;
  int32_t has_ttft, has_floor;
  double ttft_limit, speed_floor, tpot_cap;   /* tpot_cap = 1000/speed_floor (serving_modes.py:109-111) */
  int32_t modes;                     /* bit0 static, bit1 aggregated, bit2 disaggregated, LC_MODE_FORCE */
  int32_t n_budgets;
  int64_t budgets[LC_MAX_BUDGETS];
  int32_t b_off, n_b;                /* sorted batch sizes in the shared batch array */
  int32_t has_ctx_capacity, chunked_prefill;
  int64_t ctx_capacity;
  double kv_mem_fraction;
  int32_t prefill_cap, decode_cap;
  double ttft_headroom, prefill_util, decode_util;
  int32_t max_x, max_y;
  int32_t load;                      /* MoE load vector index (-1 dense) */
  int32_t static_stride;             /* estimate_static's decode stride (serving_modes.py:236); <= 0: 32 */
} lc_search_desc;

typedef struct {
  int32_t n_units;                   /* evaluated units (worker set if disaggregated, else candidates) */
  int32_t unit_off;
  int32_t n_enumerated;              /* counts.enumerated */
  int32_t n_rows, n_feasible, n_skipped;
  int32_t n_front, front_off;
  int32_t n_plans, plan_off;
  int64_t best;                      /* row key (mode << 32 | index) or -1 */
  int64_t nearest;                   /* row key or -1; only when best < 0 */
  double nearest_violation;
  double best_thru, best_speed;
  int64_t queries_1d, queries_2d;    /* reference-equivalent query_latency calls (memoised) */
  int32_t n_survivors;               /* rows left for the exact Pareto scan after bucket pruning */
  int32_t n_feasible_plans;          /* of n_feasible, disaggregated plan rows */
} lc_search_result;

typedef struct {
  int64_t n_units, n_plans, n_front;
  float kernel_ms[6];                /* K0 enumerate, K3 tails, K2 evaluate (tables + cells + expand), K5a pools, K5b disagg, K4 front */
  int64_t n_raw;                     /* raw (tp,pp,ep,dp,batch) tuples examined */
  int64_t n_launches;                /* kernels launched by the device pipeline (K0..K4) */
  int64_t n_table_queries;           /* distinct queries priced: query-table + decode-series entries */
  int64_t n_table_queries_2d;        /* of which 2-D (attention) */
  int64_t n_cells;                   /* (search, template, batch) cells */
} lc_batch_totals;

/* per-unit / per-plan / front arrays to copy back (any pointer may be NULL) */
typedef struct {
  int32_t* unit_search; int32_t* unit_combo; int32_t* unit_batch; uint8_t* unit_in_budget;
  int32_t* st_status; double* st_ttft; double* st_tpot; double* st_speed; double* st_thru;
  int32_t* ag_status; double* ag_ttft; double* ag_tpot; double* ag_speed; double* ag_thru;
  int32_t* pf_status; double* pf_lat; double* pf_rate;
  int32_t* dc_status; double* dc_lat; double* dc_rate;
  int64_t* err_c0; int64_t* err_c1;  /* [n_units*4]: failing coords for st, ag, pf, dc */
  int32_t* plan_p; int32_t* plan_d; int32_t* plan_x; int32_t* plan_y; int64_t* plan_gpus;
  double* plan_r_sys; double* plan_ttft; double* plan_tpot; double* plan_speed; double* plan_thru;
  int64_t* front;                    /* row keys */
} lc_fetch_req;

typedef struct lc_ctx lc_ctx;
typedef struct lc_db lc_db;
typedef struct lc_space lc_space;

int lc_abi_version(void);
const char* lc_last_error(void);

int lc_open(int device, lc_ctx** out);
int lc_close(lc_ctx* ctx);

int lc_db_upload(lc_ctx* ctx, const lc_db_desc* desc, lc_db** out);
int lc_db_free(lc_db* db);

int lc_space_upload(lc_ctx* ctx, const lc_space_desc* desc, lc_space** out);
int lc_space_free(lc_space* sp);

/* Evaluate n_search searches of one (db, model x space) in one pass.
 * batches: shared sorted batch array; loads: n_loads vectors of n_experts
 * {q_i = w_i / sum(w)} (numpy) followed by the by-weight order as doubles.
 * Results stay on the device until lc_fetch / the next batch. */
int lc_search_batch(lc_ctx* ctx, const lc_db* db, const lc_space* sp, int32_t n_search,
                    const lc_search_desc* searches, int32_t n_batches, const int64_t* batches,
                    int32_t n_loads, const double* loads, lc_search_result* results,
                    lc_batch_totals* totals);

int lc_fetch(lc_ctx* ctx, const lc_fetch_req* req);

/* Kernels only (no H2D/D2H): re-run the last batch's device pipeline
 * `iters` times and report the mean per-kernel times; for benchmarks. */
int lc_replay_last(lc_ctx* ctx, int32_t iters, lc_batch_totals* totals);

/* Asynchronous variant: enqueue the last batch's device pipeline (K0..K4) on the
 * context's stream and return immediately (no per-kernel timing). */
int lc_replay_async(lc_ctx* ctx);

/* Restrict the raw (tp,pp,ep,dp,batch) tuples of the following lc_search_batch
 * calls (and replays): tuple r of the batch -- searches concatenated, each
 * n_combos x n_b in enumeration order -- is considered only if lo <= r < hi and
 * (mask == NULL or mask[r - lo] != 0).  Every other tuple is treated as filtered
 * out by enumerate_candidates (search.py:82-113).  hi < 0 clears the filter.
 * A search sharded across GPUs runs each rank on a contiguous block [lo, hi) of
 * its candidates, then one merge pass on the union mask of the
 * ranks' local front / best / nearest-miss / pool top-k candidates. */
int lc_set_raw_filter(lc_ctx* ctx, int64_t lo, int64_t hi, const uint8_t* mask);

/* Disaggregated pool selections of the last batch (search.py:336-339):
 * pool_units[s*128 + k] (k < 64: prefill, 64 + k: decode) are unit indices in
 * pool-rank order, pool_counts[2s], [2s+1] the number of each.  Either pointer
 * may be NULL. */
int lc_fetch_pools(lc_ctx* ctx, int32_t* pool_units, int32_t* pool_counts);

/* raw[i] = raw tuple index (as in lc_set_raw_filter) of unit units[i] of the last
 * batch, -1 if out of range: identifies a candidate across ranks and passes. */
int lc_unit_raw(lc_ctx* ctx, int32_t n, const int32_t* units, int64_t* raw);

/* The context's CUDA stream (cudaStream_t), for callers that order or time work
 * against it (e.g. CUDA events across several contexts). */
int lc_stream(lc_ctx* ctx, void** stream);

/* Scheduling priority of the context's stream (and of the kernels of the batch
 * graphs captured on it from now on): 0 is the default, negative values are
 * higher priority, clamped to the device's range.  Several contexts sharing one
 * GPU can so give the longest pipeline first claim on free SMs. */
int lc_set_priority(lc_ctx* ctx, int priority);

/* ------------------------------------------------ single-operator queries */
/* One query_latency(db, query, policy) call (perfdb.py:539-580).  The host
 * resolves the query's grid key (OperatorQuery.grid_key, perfdb.py:239-244) to a
 * grid id of the uploaded database and writes the shape in canonical order. */
typedef struct {
  int32_t grid;                      /* grid id; < 0: no grid for the key (MissingKeyError) */
  int32_t kind, quant;               /* LC_KIND_*, index into fp16/fp8/int8/int4 */
  int32_t policy;                    /* LC_POLICY_*, or -1: the database's policy */
  int64_t d[5];                      /* required dims in _KIND_DIMS order (perfdb.py:51-69) */
  int64_t kv_len;                    /* attention_generation: shape kv_len, or -1 = seq_len */
} lc_query;                          /* 64 bytes */

/* Price n queries: latency_us[i] in microseconds and status[i] = LC_ST_OK,
 * LC_ST_MISSING_KEY, LC_ST_EXTRAPOLATION or LC_ST_UNSUPPORTED.  Host arrays in
 * and out; returns after the results are copied back.
 * Replaces query_latency (perfdb.py:539-580) and, for in-grid coordinates,
 * _interp_cells (perfdb.py:509-536); sol_estimate (perfdb.py:431-484) above the grid. */
int lc_query_batch(lc_ctx* ctx, const lc_db* db, int32_t n, const lc_query* queries, double* latency_us,
                   int32_t* status);

/* ------------------------------------------------ step latency with breakdown */
typedef struct {
  int32_t tmpl;                      /* (tp, pp, ep) template index of the space plan */
  int32_t phase;                     /* 0 prefill, 1 decode, 2 mixed (model.py PHASES) */
  int64_t n_ctx, n_gen, seq;         /* decompose's token arguments (model.py:271-285) */
  int64_t batch;                     /* cfg.batch: the pipeline bubble's microbatches (estimator.py:83) */
  int32_t load;                      /* MoE load vector index; -1: no skew (dense model) */
  int32_t _pad;
} lc_step_req;                       /* 48 bytes */

typedef struct {
  double total_ms;                   /* sum(breakdown.values()), CPython float sum (estimator.py:95) */
  int32_t status;                    /* code | label << 8 of the first failing entry in plan order; 0 ok */
  int32_t n_entries;                 /* template entries (plan order) */
  int64_t c0, c1;                    /* the failing query's interpolated coordinates */
  double entry_ms[LC_MAX_ENTRIES];   /* 0.0 + ms * bubble per entry (estimator.py:93) */
  int32_t entry_label[LC_MAX_ENTRIES]; /* label id per entry; -1: entry absent from this step */
} lc_step_out;

/* Step latencies with per-label breakdown for n requests: one warp per request
 * computes the expert-tail token count (busiest EP shard, moe_load.py:141-147),
 * every plan entry's coordinates and interpolated latency, and the bubble-scaled
 * sum in plan order.  Host arrays in and out; returns after the copy back.
 * Replaces get_step_latency / _step_latency_cached (estimator.py:71-110) and
 * through them get_mix_latency / get_gen_latency (estimator.py:117-156). */
int lc_step_latency(lc_ctx* ctx, const lc_db* db, const lc_space* sp, int32_t n, const lc_step_req* reqs,
                    int32_t n_loads, const double* loads, lc_step_out* out);

/* ------------------------------------------------ report rows (host) */
/* Column view of a search's report rows (fastreport.Columns). */
typedef struct {
  int64_t n;                         /* rows */
  const int32_t* mode;               /* 0 static, 1 aggregated, 2 disaggregated */
  const int64_t* cfg;                /* [n*5] tp, pp, ep, dp, batch (static / aggregated rows) */
  const int64_t* gpus;
  const double* ttft; const double* tpot; const double* speed; const double* thru;
  const uint8_t* feasible; const uint8_t* frontier;
  const int64_t* pcfg; const int64_t* dcfg;  /* [n*5] prefill / decode worker (disaggregated rows) */
  const int64_t* x; const int64_t* y;        /* replicas */
  const double* r_sys;
  const char* model_json;            /* json.dumps(model name) */
  const char* runtime[6];            /* the runtime object, json.dumps(sort_keys, indent=2), re-indented per depth */
} lc_report_cols;

/* Write the JSON list of rows (rows[0..n_sel) or, when rows is NULL, all rows)
 * as SearchReport.to_json() prints the "rows" / "frontier" lists at list depth
 * `depth` (search.py:224-264): the same bytes as json.dumps(sort_keys=True,
 * indent=2).  Returns the byte count (writes only if it fits in cap), or < 0. */
int64_t lc_report_rows(const lc_report_cols* cols, const int64_t* rows, int64_t n_sel, int32_t depth, int32_t flags,
                       char* out, int64_t cap);

/* ------------------------------------------------ synthetic database generation */
/* One grid of generate_synthetic_db (perfdb.py:641-666): GridAxes (perfdb.py:586-614)
 * with its per-key hash constants already evaluated by the host. */
typedef struct {
  int32_t kind, quant;               /* LC_KIND_*, quant index */
  int32_t n_axes, _pad;              /* 1 or 2 interpolated axes */
  int32_t axis_dim[2];               /* canonical dim index each axis fills */
  int32_t axis_off[2], axis_len[2];  /* into axis_val / axis_term */
  int64_t cell_off;                  /* first cell; grids are contiguous and in order */
  int64_t d[5];                      /* fixed dims in canonical order (axis slots ignored) */
  double offset;                     /* (_hash_unit(seed, key, "offset") - 0.5) * 0.3 */
} lc_gen_grid;                       /* 96 bytes */

typedef struct {
  int32_t n_grids;
  const lc_gen_grid* grids;
  int32_t n_axis;
  const int64_t* axis_val;           /* axis values */
  const double* axis_term;           /* math.sin(omega * math.log2(value) + phase) per value (perfdb.py:637) */
  int64_t n_cells;
  double amplitude;                  /* efficiency_amplitude */
  double mem_bandwidth, intra_node_bandwidth, inter_node_bandwidth;
  int32_t gpus_per_node;
  double compute[4];                 /* FLOP/s for fp16, fp8, int8, int4; <= 0 = absent */
} lc_dbgen_desc;

/* Fill latency_us[n_cells] (roofline x efficiency, row-major per grid, axis 0
 * major) and latency_log[n_cells] (natural log; NaN where glibc's near-1 path
 * applies, for the host to recompute).  status[n_grids] = LC_ST_UNSUPPORTED for
 * a grid whose quant has no compute rate (UnsupportedOperatorError). */
int lc_dbgen(lc_ctx* ctx, const lc_dbgen_desc* desc, double* latency_us, double* latency_log, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif
