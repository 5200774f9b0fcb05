// llmconf_b200: B200 kernels for the llmconf configuration-search hot path and
// the C ABI declared in include/llmconf_b200.h.
//
// Pipeline for one lc_search_batch (many searches of one model x space):
//   K0  k_enum_flags / k_scan_* / k_scatter : enumerate_candidates (search.py:82-113)
//   K3  k_tails                            : MoE busiest-shard tokens (moe_load.py:67-147)
//   K2  k_eval                             : static / aggregated / pool steps per unit
//   K5a k_pools                            : pool top-k by (-rate/gpus, key) (search.py:338-339)
//   K5b k_disagg                           : x*y replica sweep per pairing + plan sort (serving_modes.py:449-494)
//   K4  k_front                            : SLA, Pareto front, best, nearest miss (search.py:129-208)
// Build with --fmad=false: bit-exact parity with CPython needs unfused arithmetic.
#include <cuda_pipeline.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>
#include <mutex>
#include <array>
#include <chrono>
#include <string>
#include <vector>

#include "../../include/llmconf_b200.h"
#include "glibc_libm.cuh"
#include "lc_eval.cuh"
#include "lc_tails.cuh"
#include "lc_keys.h"
#include "lc_report.h"

using namespace lc;

// ============================================================================ host-side state
namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(LC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// largest database image staged into shared memory; larger ones are read from global memory
constexpr size_t kDbStageMax = 200 * 1024;

// While a pipeline is being captured into a CUDA graph no allocation may happen:
// a buffer that would have to grow marks the capture as unusable instead, and the
// caller runs the pipeline directly (which allocates) -- see launch_pipeline.
static thread_local bool tl_capturing = false, tl_capture_grow = false;

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool view = false;  // p points into another buffer (not owned)
  template <class T>
  T* get(size_t n, cudaError_t* err) {
    size_t bytes = n * sizeof(T);
    if (bytes == 0) bytes = 16;
    if (bytes > cap && tl_capturing) {
      tl_capture_grow = true;
      return (T*)p;
    }
    if (bytes > cap) {
      if (p && !view) cudaFree(p);
      p = nullptr;
      cap = 0;
      view = false;
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) { *err = e; return nullptr; }
      cap = bytes;
    }
    return (T*)p;
  }
  void release() {
    if (p && !view) cudaFree(p);
    p = nullptr;
    cap = 0;
    view = false;
  }
  void set_view(void* q, size_t bytes) {
    if (p && !view) cudaFree(p);
    p = q;
    cap = bytes;
    view = true;
  }
};

const double LOG_TAB_H[256] = GLIBC_LOG_TAB_INIT;
const uint64_t EXP_TAB_H[256] = GLIBC_EXP_TAB_INIT;
}  // namespace

struct lc_db {
  int device;
  int32_t n_grids, n_axis, n_cells;
  DevGrid* grids;
  int64_t* axv;
  double* axl;
  double* cell;
  double* clog;
  double* logtab;
  uint64_t* exptab;
  double mem_bw, intra_bw, inter_bw, gpu_memory, compute[4];
  int32_t gpn, policy;
  size_t smem_bytes;  // staged size
  int32_t staged;     // 1: fits the shared-memory staging budget; 0: kernels read it from global memory
};

struct lc_space {
  int device;
  int64_t hidden, topk, n_experts;
  int32_t is_moe, n_combos, n_tmpl, n_tp, n_ep;
  lc_combo* combos;
  int32_t* tmpl_n;
  lc_entry* entries;
  int64_t* tp_vals;  // [n_tp] from combos
  int64_t* ep_vals;  // [n_ep]
  int64_t max_ep_h;  // host copy: largest ep value
  uint8_t* pair_used;  // [n_tp*n_ep]
  int32_t* pair_canon; // [n_tp*n_ep] first pair with the same (max(1, ep/tp), ep): identical tails
  struct TmplInfo* tmpl_info;  // [n_tmpl]
  int32_t n_slots, n_gclass;
  lc_slot* slots;
  int32_t* slot_of;    // [n_tmpl][16][3]: class << 16 | index within class
  int32_t* class_slots;  // global slot id per (class, index), class c at class_off[c]
  int32_t class_n[4], class_off[4], class_n2d[4];
  lc_entry* gclasses;
  int32_t* gclass_of;  // [n_tmpl]
  int32_t* tmpl_cidx_off;  // [n_tmpl + 1] into tmpl_cidx
  int32_t* tmpl_cidx;      // combo indices of each template
  uint64_t* combo_rank;    // [n_combos] rank of (tp, pp, ep, dp) in config-key string order << 36 (lc_keys.h)
};

// Query-table sharing.  A slot's inputs are (grid, coordinates); which search
// inputs the coordinates depend on splits slots into four classes:
//   0 prefill steps:            (context length, batch list, MoE load)
//   1 decode, non-attention:    (batch list, MoE load)
//   2 decode, attention:        (KV midpoint isl + osl/2, batch list)
//   3 mixed steps:              the whole search
// Searches that agree on a class's inputs share one table for that class.
struct QtGroup {
  int64_t off;
  int32_t cls, search, n_slots, _pad;
};

// a decode-series table shared by the searches with the same (isl, batch list)
struct DsGroup {
  int64_t off, isl;
  int32_t b_off, n_b, n_steps, stride;  // stride: estimate_static's decode stride (32 by default)
};

// estimate_static's decode stride (serving_modes.py:236, STATIC_DECODE_STRIDE = 32)
__host__ __device__ __forceinline__ int64_t static_stride(const lc_search_desc& S) {
  return S.static_stride > 0 ? (int64_t)S.static_stride : 32;
}

// Static decode loops shared across output lengths.  The KV samples isl + 32k + 1
// and the decode step terms depend on (isl, batch list, MoE load), not on osl, and
// the loop accumulates t_gen in sample order, so a search with a shorter osl sees a
// prefix of a longer one's partial sums: one thread per (group, template, batch)
// walks the samples once and hands every member its own total.
struct SeriesGroup {
  int64_t off;                    // first thread index
  int32_t rep;                    // representative search (query / decode-series table offsets)
  int32_t m_off, n_m;             // members, sorted by n_steps
  int32_t _pad;
};
struct SeriesMember {
  int32_t search, n_steps;
};
struct SdOut {
  double t_gen;                   // sum of step * run over the member's samples
  int32_t status;                 // code | label << 8
  int32_t qsd;                    // reference-equivalent query counts (q1 | q2 << 16)
  int64_t c0, c1;                 // failing query coordinates
};

// Prefill steps shared by the searches of one prefill query-table group: the
// step's inputs (context, batch list, MoE load -> tails, query table) are the
// group key, so its total is the same for every member (estimator.py:71-110).
struct PGroup {
  int64_t off;   // first entry: [template][b_i]
  int32_t rep;   // representative search
  int32_t n_b;
};
struct PStep {
  double total;
  int32_t status;  // code | label << 8
  int32_t q;       // query counts q1 | q2 << 16
  int64_t c0, c1;  // failing query coordinates
};

// one priced query (decode-series tables)
struct QVal {
  double lat;
  int32_t status;
  int32_t _pad;
};

// One priced query of the shared query tables in 8 bytes: the latency, or for a
// failed query a signalling-NaN pattern carrying its status (exponent all ones,
// quiet bit clear, tag bits 0x7FF4 in the top 16).  Device arithmetic only ever
// yields the canonical quiet NaN and lc_db_upload quiets any NaN database cell,
// so no latency can carry the tag.  Half the bytes of a QVal: the K2 cell kernel
// stages a whole step's values in shared memory per thread.
constexpr unsigned long long kBoxTag = 0x7FF4000000000000ull;
__host__ __device__ __forceinline__ bool is_boxed(unsigned long long bits) { return (bits >> 48) == (kBoxTag >> 48); }
__device__ __forceinline__ double box_status(int st) {
  return __longlong_as_double((long long)(kBoxTag | (unsigned long long)(unsigned)st));
}
__device__ __forceinline__ QVal unbox(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return is_boxed(b) ? QVal{0.0, (int32_t)(b & 0xffffu), 0} : QVal{v, 0, 0};
}

// One MoE tail table: [tp_i * n_ep + ep_i][b_i].  Prefill-type tables depend on
// (batch list, load, context length), decode-type on (batch list, load) only,
// mixed-type on the whole search -- so sweeps share most of them.
struct TailTable {
  int64_t off;
  int32_t type;    // 0 prefill (b * chunk), 1 decode (b), 2 mixed (chunk + n_mix_gen)
  int32_t search;  // representative search (workload for the mixed schedule)
  int32_t b_off, n_b, load, _pad;
  int64_t chunk;
};

struct TmplInfo {
  int64_t tp, pp, ep;
  int32_t tp_i, ep_i;
};

// per-search bookkeeping computed on the host / device
struct SearchMeta {
  int64_t raw_off, n_raw;
  int64_t cell_off;
  int64_t tail_off[3];  // per tail type
  int64_t qt_off[4];    // query tables per slot class [slot-in-class][b_i] (classes in QtGroup)
  int64_t ds_off;       // decode-series table [gclass][b_i][step], shared by searches with equal (isl, batches)
  int32_t n_steps;      // static decode samples (ceil((osl-1)/stride), 0 without static mode)
  int32_t ds_stride;    // steps stored per (gclass, batch) in the shared table (max over its searches)
  int64_t mark_off;     // offset of this search's batches in the mixed-token marking pass
  int32_t _pad2;
  int32_t unit_off, n_units;
  int32_t plan_off, plan_cap;
  int32_t pool_off;  // into pool selection arrays (64 slots per role)
  int32_t n_pre, n_dec;
  int64_t pstep_off;  // this search's prefill-group table of step totals (PStep), -1 none
};

// Per-search row accounting, accumulated by k_expand (static / aggregated rows)
// and k_disagg (plan rows) for K4: counts (search.py:343-358 report counts),
// query totals and the range of feasible speeds (IEEE bit patterns; the
// minimum is kept complemented so that a zeroed record is the empty state).
struct SearchAcc {
  unsigned long long q1, q2, smin_c, smax;
  int32_t feas, rows, enums, skips, fplans, _pad;
};

// fixed-size keys of the host-side table grouping (lc_search_batch)
using Key5 = std::array<int64_t, 5>;

struct lc_ctx {
  int device;
  cudaStream_t stream;
  cudaEvent_t ev[8];
  cudaGraphExec_t gexec = nullptr;  // the last K0..K4 pipeline as an instantiated CUDA graph
  bool graph_ok = false;            // gexec holds the pipeline of the current batch
  bool capturing = false;
  DBuf searches, batches, batch_code, loads, meta, results;
  DBuf flags, pos, block_sums;
  DBuf u_search, u_combo, u_batch, u_budget;
  DBuf st_status, st_v, ag_status, ag_v, pf_status, pf_v, dc_status, dc_v, err_c, front_flags, cell_ctr;
  DBuf inputs;  // one block holding the batch's host inputs (searches .. batch codes are views into it)
  DBuf step_in, step_out, step_loads, pool_key, qt_groups, ds_groups, front_compact, pool_part, front_meta, buckets, surv, n_surv, qt, ds, m_used, tail_tables, tails, tail_hash, pool_sel, plans_i, plans_d, front, u_queries, cell_flags, cells, cell_err;
  DBuf q_in, q_lat, q_st;  // lc_query_batch
  DBuf sgroups, smembers, sd;  // shared static decode loops
  DBuf pgroups, psteps;        // shared prefill step totals
  DBuf acc;                    // SearchAcc per search
  DBuf plan_scratch;           // K5b pairing results [search][256]
  DBuf pool_seed;              // K5a seed thresholds [search][2]
  DBuf pool_sample;            // K5a seed sample [search * combo][2]
  std::vector<PGroup> hpg;
  std::vector<uint64_t> hbatch_code;  // config-key batch-field codes of the batches array (lc_keys.h)
  int64_t n_pstep = 0;
  DBuf raw_mask;               // lc_set_raw_filter: optional keep-mask over [filt_lo, filt_hi)
  int64_t filt_lo = 0, filt_hi = -1;  // filt_hi < 0: no raw-tuple filter
  bool filt_mask = false;
  std::vector<SeriesGroup> hsg;
  std::vector<SeriesMember> hsm;
  int64_t n_series = 0;
  // last batch
  const lc_db* db = nullptr;
  const lc_space* sp = nullptr;
  int32_t n_search = 0, n_batches = 0, n_loads = 0;
  int64_t n_raw = 0, n_cap = 0, n_units = 0, n_tails = 0, n_plan_slots = 0, n_front_slots = 0, n_cells = 0;
  int64_t n_qt = 0, n_ds = 0, n_pd_tails = 0, m_tmax = 0, n_marks = 0;
  bool tails_dedup_ok = false;  // K3 keys (load << 48 | pooled tokens) fit: see k_tails_keys
  int64_t launches = 0;  // kernels launched by the last pipeline run
  int64_t n_qt_2d = 0;   // 2-D entries among the query tables
  int64_t n_total_idx = 0;  // index of the unit total inside block_sums
  std::vector<SearchMeta> hmeta;
  std::vector<TailTable> htables;
  std::vector<DsGroup> hds;
  int64_t* pinned_front = nullptr;  // page-locked staging for front D2H
  size_t pinned_front_cap = 0;
  int32_t* pinned_plans_i = nullptr;  // page-locked copies of the plan slots
  double* pinned_plans_d = nullptr;
  size_t pinned_plans_cap = 0;
  bool staged = false;  // fronts + plans of the last batch already copied to the pinned buffers
  bool batches_sorted = false;  // every search's batch list is non-decreasing: K0 in closed form
  bool enum_fit = false;        // the last K0 ran in closed form (block_sums = per-(search, combo) unit offsets)
  std::vector<int32_t> hsearch_nb;
  unsigned char* arena = nullptr;  // page-locked staging for the batch's inputs and summaries
  size_t arena_cap = 0, arena_used = 0;
  DBuf pair_inb, cmax;          // K0 closed form: per (search, combo) budget flag; per (search, template) fit maxima
  std::vector<QtGroup> hqt;
  std::vector<lc_search_result> hres;
};

// ============================================================================ device kernels
// rel / d and rel % d for an offset inside one search / table group: every such
// offset is below 2^31 (lc_search_batch bounds the batch), so 32-bit unsigned
// arithmetic replaces the 64-bit software division.
__device__ __forceinline__ int div32(int64_t rel, int64_t d) { return (int)((uint32_t)rel / (uint32_t)d); }
__device__ __forceinline__ int mod32(int64_t rel, int64_t d) { return (int)((uint32_t)rel % (uint32_t)d); }

namespace {

constexpr int kScanBlock = 1024;

struct EvalParams {
  // db (global copies; staged to smem)
  const DevGrid* grids; const int64_t* axv; const double* axl; const double* cell; const double* clog;
  const double* logtab; const uint64_t* exptab;
  int32_t n_grids, n_axis, n_cells;
  double mem_bw, intra_bw, inter_bw, gpu_memory, compute[4];
  int32_t gpn, policy;
  int32_t db_global;                 // database too large to stage: read it from global memory (L1/L2)
  int32_t surv_cap;                  // K4 survivors kept for the sorted front scan (kSurvivorCap; lower only in tests)
  unsigned long long* cell_ctr;      // k_eval_cells' chunk counter (zeroed before each launch)
  // space
  const lc_combo* combos; const int32_t* tmpl_n; const lc_entry* entries; int32_t sp_n_combos;
  int64_t hidden, topk, n_experts; int32_t is_moe, n_tp, n_ep;
  const int64_t* tp_vals; const int64_t* ep_vals; const uint8_t* pair_used; const int32_t* pair_canon;
  const TailTable* tail_tables; int32_t n_tail_tables;
  int64_t n_pd_tails;                // prefill/decode tables; the dense mixed region follows
  int64_t m_tmax;                    // mixed tokens index range [0, m_tmax]
  uint8_t* m_used;                   // [n_loads][m_tmax + 1] mixed token counts in use
  const lc_slot* slots; int32_t n_slots; const int32_t* slot_of;
  const int32_t* class_slots; int32_t class_off[4];
  const QtGroup* qt_groups; int32_t n_qt_groups;
  const lc_entry* gclasses; int32_t n_gclass; const int32_t* gclass_of;
  double* qt; int64_t n_qt;           // boxed (box_status)
  QVal* ds; int64_t n_ds;
  const DsGroup* ds_groups; int32_t n_ds_groups;
  const SeriesGroup* sgroups; int32_t n_sgroups; const SeriesMember* smembers; SdOut* sd; int64_t n_series;
  const PGroup* pgroups; int32_t n_pgroups; PStep* psteps; int64_t n_pstep;
  // batch
  const lc_search_desc* searches; const SearchMeta* meta; int32_t n_search;
  int64_t raw_lo, raw_hi; const uint8_t* raw_mask;  // raw-tuple filter (sharded searches)
  const int64_t* batches; const double* loads;
  // units
  const int32_t* u_search; const int32_t* u_combo; const int32_t* u_batch; const uint8_t* u_budget;
  int64_t n_cap;                     // unit capacity (= raw tuples); stride of the SoA planes
  const int32_t* d_total;            // unit count, written by K0 on the device
  const int64_t* tails;
  // outputs
  int32_t* st_status; double* st_v;  // v: [4][n_units] ttft,tpot,speed,thru
  int32_t* ag_status; double* ag_v;
  int32_t* pf_status; double* pf_v;  // [2][n_units] lat, rate
  int32_t* dc_status; double* dc_v;
  int64_t* err_c;                    // [8][n_units]: (c0,c1) x (st,ag,pf,dc)
  uint8_t* front_flags;              // [n_units] bit0 / bit1: the static / aggregated row is SLA-feasible
  double* pool_key;                  // [2][n_cap]: (-rate)/gpus per pool role (search.py:276-277), +inf if skipped
  // cells (search x template x batch)
  const struct TmplInfo* tmpl_info;
  uint32_t* cell_flags;              // bit0: some candidate in budget, bit1: pool worker
  struct CellOut* cells;
  int64_t* cell_err;                 // [cell][8]
  int64_t n_cells_total;
  lc_search_result* results;
  SearchAcc* acc;                    // [n_search]
  unsigned long long* fbuckets;      // [n_search][kSpeedBuckets]: K4 speed-bucket maxima of throughput
  const uint64_t* combo_rank;        // [n_combos] config-key string rank << 36 (lc_keys.h)
  const uint64_t* batch_code;        // [n_batches] config-key batch-field code (lc_keys.h)
  // closed-form K0 (fused candidate rows): unit offsets per (search, combo), budget flags, template combos
  const int32_t* pair_off;           // [n_search * n_combos + 1], nullptr otherwise
  const uint8_t* pair_inb;
  double* pool_sample;               // [n_search * n_combos][2]: pool keys of each pair's last unit (K5a seed)
  const int32_t* tmpl_cidx_off; const int32_t* tmpl_cidx;
};

__device__ __forceinline__ int find_search(const SearchMeta* meta, int n, int64_t r) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (meta[mid].raw_off <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---- K0: enumeration flags: bit0 keep (unit), bit1 in budget
__global__ void k_enum_flags(EvalParams P, int64_t n_raw, uint8_t* flags) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_raw; r += (int64_t)gridDim.x * blockDim.x) {
    // lc_set_raw_filter: a rank's block of a sharded search, or the merge pass's union set
    if (r < P.raw_lo || r >= P.raw_hi || (P.raw_mask && !P.raw_mask[r - P.raw_lo])) {
      flags[r] = 0;
      continue;
    }
    const int s = find_search(P.meta, P.n_search, r);
    const lc_search_desc& S = P.searches[s];
    const int64_t rel = r - P.meta[s].raw_off;
    const int ci = div32(rel, S.n_b), bi = mod32(rel, S.n_b);
    const lc_combo c = P.combos[ci];
    const int64_t b = P.batches[S.b_off + bi];
    uint8_t f = 0;
    // LC_MODE_FORCE: evaluate every consistent tuple (single-config estimates,
    // serving_modes.estimate_static / estimate_aggregated apply no memory or budget filter)
    const bool force = (S.modes & LC_MODE_FORCE) != 0;
    if (force || fits_memory(c, S, P.gpu_memory, P.hidden, b)) {
      const bool inb = force || in_budget(S, c.gpus);
      if (inb || (S.modes & 4)) {  // workers skip the budget (search.py:323)
        f = 1 | (inb ? 2 : 0);
        atomicOr(&P.cell_flags[P.meta[s].cell_off + (int64_t)c.tmpl * S.n_b + bi],
                 (inb ? 1u : 0u) | ((S.modes & 4) ? 2u : 0u));
      }
    }
    flags[r] = f;
  }
}

__global__ void k_scan_blocks(const uint8_t* flags, int64_t n, int32_t* block_sums) {
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  int v = (i < n) ? (flags[i] & 1) : 0;
  v = __syncthreads_count(v);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
}

__global__ void k_scan_top(int32_t* block_sums, int n) {
  // single block exclusive scan, in place; block_sums[n] = total.  Tiles of 8
  // consecutive elements per thread (two coalesced 16-byte loads), a serial scan
  // in registers, then one block scan of the per-thread totals per tile.
  __shared__ int32_t warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = (int)(blockDim.x >> 5);
  const bool vec = ((uintptr_t)block_sums & 15) == 0;
  int carry = 0;
  for (int base = 0; base < n; base += (int)blockDim.x * 8) {
    const int i0 = base + tid * 8;
    int v[8];
    if (vec && i0 + 8 <= n) {
      const int4 a = *(const int4*)(block_sums + i0), b = *(const int4*)(block_sums + i0 + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = i0 + k < n ? block_sums[i0 + k] : 0;
    }
    int sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { const int t = v[k]; v[k] = sum; sum += t; }
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const int excl = x - sum + (w ? warp_tot[w - 1] : 0) + carry;
    if (vec && i0 + 8 <= n) {
      *(int4*)(block_sums + i0) = make_int4(v[0] + excl, v[1] + excl, v[2] + excl, v[3] + excl);
      *(int4*)(block_sums + i0 + 4) = make_int4(v[4] + excl, v[5] + excl, v[6] + excl, v[7] + excl);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k < n) block_sums[i0 + k] = v[k] + excl;
    }
    carry += warp_tot[nw - 1];
    __syncthreads();
  }
  if (tid == 0) block_sums[n] = carry;
}

__global__ void k_scatter(EvalParams P, const uint8_t* flags, int64_t n, const int32_t* block_sums, int32_t* pos,
                          int32_t* u_search, int32_t* u_combo, int32_t* u_batch, uint8_t* u_budget) {
  __shared__ int32_t warp_tot[32];
  const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const uint8_t f = i < n ? flags[i] : 0;
  const int v = f & 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  const int p = block_sums[blockIdx.x] + x - v + (w ? warp_tot[w - 1] : 0);
  if (i < n) {
    pos[i] = p;
    if (v) {
      const int s = find_search(P.meta, P.n_search, i);
      const lc_search_desc& S = P.searches[s];
      const int64_t rel = i - P.meta[s].raw_off;
      u_search[p] = s;
      u_combo[p] = div32(rel, S.n_b);
      u_batch[p] = mod32(rel, S.n_b);
      u_budget[p] = (f >> 1) & 1;
    }
  }
}

__global__ void k_unit_offsets(SearchMeta* meta, int n_search, const int32_t* pos, int64_t n_raw,
                               const int32_t* d_total) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_search) return;
  const int32_t total = *d_total;
  const int64_t r0 = meta[s].raw_off, r1 = r0 + meta[s].n_raw;
  const int32_t a = r0 < n_raw ? pos[r0] : total;
  const int32_t b = r1 < n_raw ? pos[r1] : total;
  meta[s].unit_off = a;
  meta[s].n_units = b - a;
}

#ifndef LC_TAIL_MIN_BLOCKS
#define LC_TAIL_MIN_BLOCKS 3  // 80 registers: no spills of the per-lane expert counts and keys (measured best)
#endif
#ifndef LC_TAIL8_MIN_BLOCKS
#define LC_TAIL8_MIN_BLOCKS 3  // k_tails<8> and up (8 experts per lane)
#endif
// ---- K0 in closed form.  fits_memory (model.py:440-479) is monotone in the
// batch size: the activation term grows with it, so the static footprint grows
// and the KV budget shrinks, while the KV need grows -- and each step is a
// monotone IEEE operation.  Over a search's sorted batch list the fitting
// batches of a (tp,pp,ep,dp) combo are therefore a prefix, found by binary
// search; the budget filter does not depend on the batch.  Units (the kept
// candidates in the reference's order) are then a concatenation of prefixes.
__global__ void k_enum_fit(EvalParams P, int64_t n_pairs, int32_t* counts, uint8_t* pair_inb, int32_t* cmax,
                           int32_t n_tmpl) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_pairs; p += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(p / P.sp_n_combos);
    const int ci = (int)(p % P.sp_n_combos);
    const lc_search_desc& S = P.searches[s];
    const lc_combo c = P.combos[ci];
    const bool force = (S.modes & LC_MODE_FORCE) != 0;
    int nfit = S.n_b;
    if (!force) {
      int lo = 0, hi = S.n_b;  // first batch index that does not fit
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fits_memory(c, S, P.gpu_memory, P.hidden, P.batches[S.b_off + mid])) lo = mid + 1;
        else hi = mid;
      }
      nfit = lo;
    }
    const bool inb = force || in_budget(S, c.gpus);
    const bool kept = inb || (S.modes & 4);  // workers skip the budget (search.py:323)
    counts[p] = kept ? nfit : 0;
    pair_inb[p] = inb ? 1 : 0;
    if (kept && nfit > 0) {
      int32_t* m = cmax + ((int64_t)s * n_tmpl + c.tmpl) * 2;
      if (inb) atomicMax(&m[0], nfit);
      if (S.modes & 4) atomicMax(&m[1], nfit);
    }
  }
}

// cell flags from the per-(search, template) prefix maxima: bit0 some in-budget
// candidate, bit1 some pool worker (as k_enum_flags sets them tuple by tuple)
__global__ void k_cell_flags_fit(EvalParams P, const int32_t* cmax, int32_t n_tmpl, uint32_t* cell_flags) {
  const int s = blockIdx.y;
  const lc_search_desc& S = P.searches[s];
  const int64_t n = (int64_t)n_tmpl * S.n_b;
  const int64_t off = P.meta[s].cell_off;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = div32(x, S.n_b), bi = mod32(x, S.n_b);  // x < n_tmpl * n_b < 2^31
    const int32_t* m = cmax + ((int64_t)s * n_tmpl + t) * 2;
    cell_flags[off + x] = (bi < m[0] ? 1u : 0u) | (bi < m[1] ? 2u : 0u);
  }
}

// one block per (search, combo): its kept prefix of batch indices, in order
__global__ void k_scatter_fit(EvalParams P, int64_t n_pairs, const int32_t* offs, const uint8_t* pair_inb,
                              int32_t* u_search, int32_t* u_combo, int32_t* u_batch, uint8_t* u_budget) {
  for (int64_t p = blockIdx.x; p < n_pairs; p += gridDim.x) {
    const int32_t o = offs[p], n = offs[p + 1] - o;
    if (n <= 0) continue;
    const int s = (int)(p / P.sp_n_combos);
    const int ci = (int)(p % P.sp_n_combos);
    const uint8_t inb = pair_inb[p];
    for (int bi = threadIdx.x; bi < n; bi += blockDim.x) {
      u_search[o + bi] = s;
      u_combo[o + bi] = ci;
      u_batch[o + bi] = bi;
      u_budget[o + bi] = inb;
    }
  }
}

__global__ void k_unit_offsets_fit(SearchMeta* meta, int n_search, int32_t n_combos, const int32_t* offs) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_search) return;
  const int32_t a = offs[(int64_t)s * n_combos], b = offs[(int64_t)(s + 1) * n_combos];
  meta[s].unit_off = a;
  meta[s].n_units = b - a;
}

// ---- K3: MoE tails table [type P/D/M][tp_i][ep_i][b_i] per search
// entry t of the tails table: whether some candidate reads it, and its
// (pooled tokens, ep index, load model)
__device__ __forceinline__ bool tail_entry(const EvalParams& P, int64_t t, int64_t& pooled, int& ep_i, int& load) {
  const int npair = P.n_tp * P.n_ep;
  bool need = false;
  pooled = 0;
  ep_i = 0;
  load = 0;
  if (t >= P.n_pd_tails) {
    // dense mixed region: (load, pair, tokens)
    int64_t r = t - P.n_pd_tails;
    const int64_t tok = r % (P.m_tmax + 1);
    r /= (P.m_tmax + 1);
    const int pair = (int)(r % npair);
    load = (int)(r / npair);
    const int64_t tp = P.tp_vals[pair / P.n_ep];
    ep_i = pair % P.n_ep;
    const int64_t ep = P.ep_vals[ep_i];
    need = ep > 1 && P.pair_used[pair] && P.pair_canon[pair] == pair &&
           P.m_used[(int64_t)load * (P.m_tmax + 1) + tok];
    const int f = (int)ep / (int)tp;  // tp, ep: small positive parallel degrees
    pooled = tok * (f > 1 ? f : 1);
  } else {
    int lo = 0, hi = P.n_tail_tables - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.tail_tables[mid].off <= t) lo = mid;
      else hi = mid - 1;
    }
    const TailTable T = P.tail_tables[lo];
    const int64_t rel = t - T.off;
    const int bi = mod32(rel, T.n_b);
    const int pair = div32(rel, T.n_b);
    if (pair < npair) {
      const int64_t tp = P.tp_vals[pair / P.n_ep];
      ep_i = pair % P.n_ep;
      const int64_t ep = P.ep_vals[ep_i];
      need = ep > 1 && P.pair_used[pair] && P.pair_canon[pair] == pair && T.load >= 0;
      const int64_t b = P.batches[T.b_off + bi];
      const int64_t tokens = T.type == 0 ? b * T.chunk : b;
      const int f = (int)ep / (int)tp;
      pooled = tokens * (f > 1 ? f : 1);
      load = T.load;
    }
  }
  return need;
}

// General path (any number of ep values): each warp takes 32 consecutive table
// entries, the lanes decide in parallel which are needed, then the warp
// computes the needed ones one after another.
template <int PER>
__global__ void __launch_bounds__(256, PER <= 4 ? LC_TAIL_MIN_BLOCKS : LC_TAIL8_MIN_BLOCKS)
    k_tails(EvalParams P, int64_t n_tails, int64_t* tails) {
  __shared__ int hist_all[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* hist = hist_all[warp];
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int E = (int)P.n_experts;
  for (int64_t chunk = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; chunk * 32 < n_tails; chunk += nw) {
    const int64_t t = chunk * 32 + lane;
    int64_t pooled = 0;
    int ep_i = 0, load = 0;
    const bool need = t < n_tails && tail_entry(P, t, pooled, ep_i, load);
    unsigned mask = __ballot_sync(0xffffffffu, need);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int64_t pl = __shfl_sync(0xffffffffu, pooled, src);
      const int64_t e = P.ep_vals[__shfl_sync(0xffffffffu, ep_i, src)];
      const int ld = __shfl_sync(0xffffffffu, load, src);
      const double* q = P.loads + (int64_t)ld * 2 * E;
      const int64_t result = warp_busiest_shard<PER>(q, q + E, E, pl, P.topk, e, hist);
      if (lane == src) tails[t] = result;
    }
  }
}

// Deduplicated path (n_ep <= 64).  The expert counts depend on (load, pooled
// tokens) only, and many entries share them: (tp, ep) pairs with the same
// max(1, ep/tp), and batch b at ratio 2f pools what batch 2b pools at f.
// K3a inserts every needed entry's (load, pooled) key into an open-addressing
// table (one job per distinct key, with the mask of ep values wanted), K3b
// computes each job's counts once and the busiest block for each wanted ep,
// K3c copies the job results into the tails table.
struct TailHash {
  unsigned long long* keys;      // [cap], ~0 empty; key = load << 48 | pooled
  unsigned long long* epmask;    // [cap] ep indices wanted
  int32_t* job_of_slot;          // [cap] written by the inserting entry
  int32_t* jobs;                 // [1 + cap]: count, then slot per job
  int32_t* slot_of;              // [n_tails] slot << 6 | ep index of each entry, -1 not needed
  int64_t* res;                  // [cap_jobs * n_ep] busiest-block tokens per (job, ep index)
  int64_t cap;                   // power of two
};

__device__ __forceinline__ uint64_t tail_hash(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  return k;
}

__global__ void k_tails_keys(EvalParams P, int64_t n_tails, TailHash H) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tails; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t pooled;
    int ep_i, load;
    int32_t slot = -1;
    if (tail_entry(P, t, pooled, ep_i, load)) {
      const unsigned long long key = ((unsigned long long)load << 48) | (unsigned long long)pooled;
      int64_t h = (int64_t)(tail_hash(key) & (uint64_t)(H.cap - 1));
      for (;;) {
        const unsigned long long prev = atomicCAS(&H.keys[h], ~0ull, key);
        if (prev == ~0ull) {  // first entry with this key: a new job
          const int j = atomicAdd(&H.jobs[0], 1);
          H.jobs[1 + j] = (int32_t)h;
          H.job_of_slot[h] = j;
          break;
        }
        if (prev == key) break;
        h = (h + 1) & (H.cap - 1);
      }
      atomicOr(&H.epmask[h], 1ull << ep_i);
      slot = (int32_t)((h << 6) | ep_i);  // cap <= 2^25 (host check)
    }
    H.slot_of[t] = slot;
  }
}

template <int PER>
__global__ void __launch_bounds__(256, PER <= 4 ? LC_TAIL_MIN_BLOCKS : LC_TAIL8_MIN_BLOCKS)
    k_tails_jobs(EvalParams P, TailHash H) {
  __shared__ int hist_all[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* hist = hist_all[warp];
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int E = (int)P.n_experts;
  const int n = H.jobs[0];
  for (int j = blockIdx.x * (blockDim.x >> 5) + warp; j < n; j += nw) {
    const int32_t h = H.jobs[1 + j];
    const unsigned long long key = H.keys[h];
    const int load = (int)(key >> 48);
    const int64_t pooled = (int64_t)(key & ((1ull << 48) - 1));
    const double* q = P.loads + (int64_t)load * 2 * E;
    int64_t cnt[PER];
    warp_expert_counts<PER>(q, q + E, E, pooled, P.topk, hist, cnt);
    unsigned long long m = H.epmask[h];
    while (m) {
      const int ei = __ffsll((long long)m) - 1;
      m &= m - 1;
      const int64_t r = warp_block_max<PER>(cnt, E, P.ep_vals[ei]);
      if (lane == 0) H.res[(int64_t)j * P.n_ep + ei] = r;
    }
  }
}

__global__ void k_tails_put(EvalParams P, int64_t n_tails, TailHash H, int64_t* tails) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tails; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = H.slot_of[t];
    if (v < 0) continue;
    tails[t] = H.res[(int64_t)H.job_of_slot[v >> 6] * P.n_ep + (v & 63)];
  }
}

// K3 prologue: mark the mixed-step token counts some (search, batch) will look up
__global__ void k_mark_mixed(EvalParams P, int64_t n_items) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_items; x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = P.n_search - 1;  // items are (search, batch index), searches contiguous by b_off order
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.meta[mid].mark_off <= x) lo = mid;
      else hi = mid - 1;
    }
    const lc_search_desc& S = P.searches[lo];
    if (S.load < 0 || !(S.modes & 2)) continue;
    const int bi = (int)(x - P.meta[lo].mark_off);
    const AggSched a = agg_schedule(S, P.batches[S.b_off + bi]);
    if (a.st) continue;
    const int64_t tok = a.chunk_tokens + a.n_mix_gen;
    if (tok <= P.m_tmax) P.m_used[(int64_t)S.load * (P.m_tmax + 1) + tok] = 1;
  }
}

// lc_unit_raw: unit index -> raw tuple index of the batch (inverse of K0's compaction)
__global__ void k_unit_raw(const SearchMeta* meta, const lc_search_desc* searches, const int32_t* u_search,
                           const int32_t* u_combo, const int32_t* u_batch, int32_t n_units, int32_t n,
                           const int32_t* units, int64_t* raw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t u = units[i];
  if (u < 0 || u >= n_units) { raw[i] = -1; return; }
  const int s = u_search[u];
  raw[i] = meta[s].raw_off + (int64_t)u_combo[u] * searches[s].n_b + u_batch[u];
}

// ---- single-operator queries (lc_query_batch): query_latency (perfdb.py:539-580)
// for arbitrary shapes, one thread per query.  The database is read from global
// memory (a few tens of KB, L1/L2 resident after the first touch).
__global__ void k_query(DbView D, int32_t n, const lc_query* __restrict__ qs, double* __restrict__ out,
                        int32_t* __restrict__ status) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const lc_query q = qs[i];
    const int policy = q.policy >= 0 ? q.policy : D.policy;
    int st = LC_ST_OK, n_logs = 0;
    double r = 0.0;
    if (q.grid < 0) {
      st = LC_ST_MISSING_KEY;
    } else {
      const DevGrid G = D.grids[q.grid];
      bool any_oob = false, any_above = false;
      int64_t cl[2] = {q.d[0], q.d[1]};
      for (int a = 0; a < G.ndim; ++a) {  // _axis_position out-of-bounds flags (perfdb.py:490-506)
        const int64_t* v = D.axv + G.ax_off[a];
        const int64_t lo = v[0], hi = v[G.ax_len[a] - 1];
        if (q.d[a] < lo) { any_oob = true; cl[a] = lo; }
        if (q.d[a] > hi) { any_oob = any_above = true; cl[a] = hi; }
      }
      if (!any_oob) {
        r = interp_cells(D, G, q.d[0], q.d[1], &n_logs);
      } else if (policy == LC_POLICY_STRICT) {
        st = LC_ST_EXTRAPOLATION;
      } else {
        const bool use_sol = policy == LC_POLICY_SOL || (policy == LC_POLICY_DEFAULT && any_above);
        const double edge = interp_cells(D, G, cl[0], cl[1], &n_logs);
        if (policy == LC_POLICY_CLAMP || !use_sol) {
          r = edge;
        } else {
          // edge query = query.with_coords(clamped); generation attention streams
          // kv_len (default seq_len) keys, which with_coords leaves as given
          int64_t de[5], dq[5];
          for (int k = 0; k < 5; ++k) de[k] = dq[k] = q.d[k];
          for (int a = 0; a < G.ndim; ++a) de[a] = cl[a];
          if (q.kind == LC_KIND_ATTN_GEN && q.kv_len > 0) de[1] = dq[1] = q.kv_len;
          const double sol_edge = sol_us(D, q.kind, q.quant, de, &st);
          if (!st) {
            const double eff = edge / sol_edge;
            const double sol_q = sol_us(D, q.kind, q.quant, dq, &st);
            if (!st) r = sol_q * eff;
          }
        }
      }
    }
    out[i] = st ? 0.0 : r;
    status[i] = st;
  }
}

// ---- synthetic database generation (lc_dbgen): generate_synthetic_db
// (perfdb.py:641-666).  One thread per grid cell: roofline latency of the cell's
// query (sol_estimate, perfdb.py:431-484) times the smooth efficiency factor
// (perfdb.py:625-638), whose per-axis sine terms the host evaluates once per
// axis value with CPython's math (they depend on one coordinate each).  The
// cell's natural log is taken here too (glibc __log_fma restated); the few
// latencies on glibc's near-1 path come back NaN and the host recomputes them.
__global__ void k_dbgen(DbView D, const lc_gen_grid* __restrict__ grids, int32_t n_grids,
                        const int64_t* __restrict__ axv, const double* __restrict__ term, int64_t n_cells,
                        double amplitude, double* __restrict__ lat, double* __restrict__ lat_log,
                        int32_t* __restrict__ status) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_cells; x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_grids - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (grids[mid].cell_off <= x) lo = mid;
      else hi = mid - 1;
    }
    const lc_gen_grid& G = grids[lo];
    const int64_t rel = x - G.cell_off;
    int idx[2] = {0, 0};
    if (G.n_axes == 2) { idx[0] = (int)(rel / G.axis_len[1]); idx[1] = (int)(rel % G.axis_len[1]); }
    else idx[0] = (int)rel;
    int64_t d[5] = {G.d[0], G.d[1], G.d[2], G.d[3], G.d[4]};
    double total = 0.0;
    for (int a = 0; a < G.n_axes; ++a) {
      d[G.axis_dim[a]] = axv[G.axis_off[a] + idx[a]];
      total += term[G.axis_off[a] + idx[a]];
    }
    int st = 0;
    const double base = sol_us(D, G.kind, G.quant, d, &st);
    double eff = 2.0;
    if (amplitude != 0.0) eff = 2.0 + G.offset + amplitude * total / (double)G.n_axes;
    const double v = base * eff;
    lat[x] = v;
    lat_log[x] = st ? 0.0 : glibc::log_fma(v, D.logtab);
    if (st) status[lo] = st;  // benign race: every failing cell of a grid writes the same code
  }
}

// ---- K2: evaluate every unit
// GLOBAL: the database is too large to stage and is read through L1/L2.  The
// staged instantiation derives every view pointer from the shared array alone
// (no branch to a global pointer), so the inlined query path compiles to LDS.
template <bool GLOBAL>
__device__ __forceinline__ void stage_db(const EvalParams& P, unsigned char* smem, DbView* V) {
  V->mem_bw = P.mem_bw; V->intra_bw = P.intra_bw; V->inter_bw = P.inter_bw; V->gpu_memory = P.gpu_memory;
  for (int i = 0; i < 4; ++i) V->compute[i] = P.compute[i];
  V->gpn = P.gpn; V->policy = P.policy;
  if (GLOBAL) {
    V->grids = P.grids; V->axv = P.axv; V->axl = P.axl; V->cell = P.cell; V->clog = P.clog;
    V->logtab = P.logtab; V->exptab = P.exptab;
    return;
  }
  unsigned char* p = smem;
  uint64_t* exptab = (uint64_t*)p; p += 256 * 8;
  double* logtab = (double*)p; p += 256 * 8;
  int64_t* axv = (int64_t*)p; p += (size_t)P.n_axis * 8;
  double* axl = (double*)p; p += (size_t)P.n_axis * 8;
  double* cell = (double*)p; p += (size_t)P.n_cells * 8;
  double* clog = (double*)p; p += (size_t)P.n_cells * 8;
  DevGrid* grids = (DevGrid*)p;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { exptab[i] = P.exptab[i]; logtab[i] = P.logtab[i]; }
  for (int i = threadIdx.x; i < P.n_axis; i += blockDim.x) { axv[i] = P.axv[i]; axl[i] = P.axl[i]; }
  for (int i = threadIdx.x; i < P.n_cells; i += blockDim.x) { cell[i] = P.cell[i]; clog[i] = P.clog[i]; }
  for (int i = threadIdx.x; i < P.n_grids; i += blockDim.x) grids[i] = P.grids[i];
  __syncthreads();
  V->grids = grids; V->axv = axv; V->axl = axl; V->cell = cell; V->clog = clog;
  V->logtab = logtab; V->exptab = exptab;
}

// tail lookup: prefill/decode tables by batch index, the mixed region by token count
__device__ __forceinline__ int64_t tail_at(const EvalParams& P, const SearchMeta& M, const lc_search_desc& S, int type,
                                           int pair, int bi, int64_t tokens) {
  const int cp = P.pair_canon[pair];
  if (type < 2) return P.tails[M.tail_off[type] + (int64_t)cp * S.n_b + bi];
  return P.tails[P.n_pd_tails + ((int64_t)S.load * P.n_tp * P.n_ep + cp) * (P.m_tmax + 1) + tokens];
}

__device__ __forceinline__ int64_t expert_tokens(const EvalParams& P, const lc_combo& c, const SearchMeta& M,
                                                 const lc_search_desc& S, int type, int bi, int64_t tokens) {
  if (!P.is_moe) return 0;
  const int64_t f = c.ep / c.tp > 1 ? c.ep / c.tp : 1;
  const int64_t pooled = tokens * f;
  const int64_t balanced = ceil_div_f(pooled * P.topk, c.ep);
  if (c.ep == 1 || S.load < 0) return balanced;
  const int64_t tail = tail_at(P, M, S, type, c.tp_i * P.n_ep + c.ep_i, bi, tokens);
  return balanced > tail ? balanced : tail;
}


// Per-cell results.  A cell is (search, (tp,pp,ep) template, batch): every
// latency of the reference model depends on the parallel config only through
// tp, pp, ep and the batch (decompose, model.py:271-406; pipeline bubble,
// estimator.py:45-48), never through dp, so the dp variants of a candidate
// share one evaluation.  K2b expands cells back to candidates.
struct CellOut {
  int32_t st_status, ag_status, pf_status, dc_status;
  double st_ttft, st_tpot, ag_ttft, ag_tpot, pf_lat, dc_lat;
  int32_t qP, qSD, qM, qG;  // reference-equivalent query counts per step kind (q1 | q2 << 16)
  int32_t st_steps, flags;  // flags bit0: aggregated used the generation step
};

__device__ __forceinline__ void put_cell_err(const EvalParams& P, int kind, int64_t c, const ErrRec& e) {
  P.cell_err[c * 8 + 2 * kind] = e.c0;
  P.cell_err[c * 8 + 2 * kind + 1] = e.c1;
}

__device__ __forceinline__ int find_cell_search(const SearchMeta* meta, int n, int64_t c) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (meta[mid].cell_off <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}


__device__ __forceinline__ int64_t tail_tokens(const EvalParams& P, const SearchMeta& M, const lc_search_desc& S,
                                               int type, int pair, int bi, int64_t tokens) {
  // expert_tokens() for a (tp_i, ep_i) pair index (estimator.py:58-68, model.py:372-373)
  const int64_t tp = P.tp_vals[pair / P.n_ep], ep = P.ep_vals[pair % P.n_ep];
  const int64_t f = ep / tp > 1 ? ep / tp : 1;
  const int64_t pooled = tokens * f;
  const int64_t balanced = ceil_div_f(pooled * P.topk, ep);
  if (ep == 1 || S.load < 0) return balanced;
  const int64_t tail = tail_at(P, M, S, type, pair, bi, tokens);
  return balanced > tail ? balanced : tail;
}

// Table kernels stage the database in shared memory once per block (~38 KB for
// DeepSeek-V3), so blocks are wide: 512 threads, 2 blocks (32 warps) per SM.
#ifndef LC_TABLE_THREADS
#define LC_TABLE_THREADS 512
#endif
#ifndef LC_TABLE_MIN_BLOCKS
#define LC_TABLE_MIN_BLOCKS 2
#endif
// K2a: query tables.  One thread per (search, slot, batch): the latency every
// template entry of that slot sees in that step (query_latency, perfdb.py:539-580).
template <bool GLOBAL>
__global__ void __launch_bounds__(LC_TABLE_THREADS, LC_TABLE_MIN_BLOCKS) k_qtables(EvalParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  DbView V;
  stage_db<GLOBAL>(P, smem, &V);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < P.n_qt; x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = P.n_qt_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.qt_groups[mid].off <= x) lo = mid;
      else hi = mid - 1;
    }
    const QtGroup Gq = P.qt_groups[lo];
    const int s = Gq.search;  // representative: every member agrees on this class's inputs
    const lc_search_desc& S = P.searches[s];
    const SearchMeta& M = P.meta[s];
    const int64_t rel = x - Gq.off;
    const int j = div32(rel, S.n_b), bi = mod32(rel, S.n_b);
    const lc_slot SL = P.slots[P.class_slots[P.class_off[Gq.cls] + j]];
    double out = box_status(LC_ST_NOT_EVALUATED);
    const int64_t b = P.batches[S.b_off + bi];
    const int64_t chunk = S.isl - S.prefix;
    const int64_t kv_mid = S.isl + S.osl / 2;
    bool need = true;
    StepArgs a{PH_DECODE, 0, b, kv_mid, 0};
    int type = 1;
    if (SL.step == LC_STEP_PREFILL) {
      a = StepArgs{PH_PREFILL, b * chunk, 0, chunk, 0};
      type = 0;
    } else if (SL.step == LC_STEP_MIXED) {
      const AggSched sc = agg_schedule(S, b);
      need = !sc.st;
      a = StepArgs{PH_MIXED, sc.chunk_tokens, sc.n_mix_gen, kv_mid, 0};
      type = 2;
    }
    if (need && SL.e.coord == LC_COORD_EXPERT)
      a.expert_tokens = tail_tokens(P, M, S, type, SL.pair, bi, a.n_ctx + a.n_gen);
    int64_t d[5];
    if (need && entry_coords(SL.e, a, P.hidden, d)) {
      int st = 0, nlog = 0;
      const double lat = LC_TABLE_QUERY(V, SL.e.grid, SL.e.kind, SL.e.quant, d[0], d[1], d[2], d[3], d[4], &st, &nlog);
      out = st ? box_status(st) : lat;
    }
    P.qt[x] = out;
  }
}

// K2a': generation-attention latency at every sampled KV length of the static
// decode loop (serving_modes.py:258-265): one thread per (search, grid, batch, sample).
template <bool GLOBAL>
__global__ void __launch_bounds__(LC_TABLE_THREADS, LC_TABLE_MIN_BLOCKS) k_dstables(EvalParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  DbView V;
  stage_db<GLOBAL>(P, smem, &V);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < P.n_ds; x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = P.n_ds_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.ds_groups[mid].off <= x) lo = mid;
      else hi = mid - 1;
    }
    const DsGroup G = P.ds_groups[lo];
    // layout [gclass][sample][batch]: the batch index is fastest, so the threads
    // of a warp in k_dseries (consecutive batches) read consecutive entries
    int64_t rel = x - G.off;
    const int bi = mod32(rel, G.n_b);
    rel = div32(rel, G.n_b);
    const int k = mod32(rel, G.n_steps);
    const int g = div32(rel, G.n_steps);
    const lc_entry e = P.gclasses[g];
    int st = 0, nlog = 0;
    QVal out;
    out.lat = LC_TABLE_QUERY(V, e.grid, e.kind, e.quant, P.batches[G.b_off + bi], G.isl + (int64_t)G.stride * k + 1, e.d[2], e.d[3],
                             e.d[4], &st, &nlog);
    out.status = st;
    out._pad = 0;
    P.ds[x] = out;
  }
}

// One step's total from the query table: sum in plan order of
// ((lat * repeat) / 1000) * bubble, CPython sum() semantics (estimator.py:83-95);
// the first failing entry in plan order decides the error.
__device__ __forceinline__ const double* qt_ptr(const EvalParams& P, const SearchMeta& M, int32_t so, int n_b, int bi) {
  return P.qt + M.qt_off[so >> 16] + (int64_t)(so & 0xffff) * n_b + bi;
}
__device__ __forceinline__ QVal qt_at(const EvalParams& P, const SearchMeta& M, int32_t so, int n_b, int bi) {
  return unbox(*qt_ptr(P, M, so, n_b, bi));
}

__device__ __forceinline__ int table_step(const EvalParams& P, const SearchMeta& M, const lc_entry* E, int ne,
                                          const int32_t* slot_row, int n_b, int bi, const StepArgs& a, double bubble,
                                          double* out, ErrRec* err, int* q1, int* q2) {
  NeumaierSum sum;
  int c1 = 0, c2 = 0;
  for (int i = 0; i < ne; ++i) {
    const lc_entry& e = E[i];
    if (e.coord == LC_COORD_CTX && !a.n_ctx) continue;
    if (e.coord == LC_COORD_GEN && !a.n_gen) continue;
    const QVal q = qt_at(P, M, slot_row[i * 3], n_b, bi);
    if (e.coord == LC_COORD_CTX || e.coord == LC_COORD_GEN) ++c2; else ++c1;
    if (q.status) {
      int64_t d[5];
      entry_coords(e, a, P.hidden, d);
      err->code = q.status; err->label = e.label; err->c0 = d[0]; err->c1 = d[1];
      return q.status;
    }
    const double ms = div1000(q.lat * (double)e.repeat);
    sum.add(0.0 + ms * bubble);
  }
  *out = sum.result();
  *q1 = c1;
  *q2 = c2;
  return 0;
}

// K2 cells stage a step's query values in shared memory before the plan-order
// sum: every entry's 8-byte table value is requested at once (cp.async, one
// column per thread: [entry][thread]), so the ~16 L2 gathers of a step overlap
// instead of forming a chain of dependent round trips.  The sum itself is
// unchanged (table_step's order, skips and first-failure rule).
#ifndef LC_CELL_MIN_BLOCKS
#define LC_CELL_MIN_BLOCKS 5  // 96 registers (measured 5 ~ 6 > 7 > 8 > 4 blocks/SM since the warp step loops: K2 1.88 -> 1.71 ms)
#endif
#ifndef LC_CELL_BUFS
#define LC_CELL_BUFS 0  // staged steps per thread; 0: unstaged (1 measured neutral, 2 slower: K2 1.93 -> 2.08 / 2.43 ms)
#endif
#ifndef LC_FUSED_STEPS
#define LC_FUSED_STEPS 1  // mixed + generation steps in one warp pass (warp_table_step2)
#endif
#ifndef LC_CELL_PREFETCH
#define LC_CELL_PREFETCH 1
#endif
#ifndef LC_CELL_DYNAMIC
#define LC_CELL_DYNAMIC 1
#endif
constexpr int kCellChunk = 512;  // cells per dynamically scheduled chunk of k_eval_cells
#ifndef LC_WARP_STEPS
#define LC_WARP_STEPS 1  // warp-cooperative mixed / generation steps in k_eval_cells (warp_table_step)
#endif
constexpr int kCellThreads = 128;
constexpr int kCellBufs = LC_CELL_BUFS;
__device__ __forceinline__ void stage_step(const EvalParams& P, const SearchMeta& M, int ne, const int32_t* slot_row,
                                           int n_b, int bi, double* col) {
  if (kCellBufs == 0) return;  // unstaged: the sum reads the table directly
#pragma unroll 4
  for (int i = 0; i < ne; ++i) {
    const int32_t so = slot_row[i * 3];
    if (so >= 0) __pipeline_memcpy_async(col + i * kCellThreads, qt_ptr(P, M, so, n_b, bi), sizeof(double));
  }
  __pipeline_commit();
}

// table_step over a staged column (stage_step, completed)
// `xt` yields the step's expert-token count, needed only for a failing expert
// entry's coordinates (the tail lookup stays off the common path)
template <class XT>
__device__ __forceinline__ int table_step_staged(const EvalParams& P, const SearchMeta& M, const lc_entry* E, int ne,
                                                 const int32_t* slot_row, int n_b, int bi, const double* col,
                                                 StepArgs a, XT xt, double bubble, double* out, ErrRec* err, int* q1,
                                                 int* q2) {
  NeumaierSum sum;
  int c1 = 0, c2 = 0;
  for (int i = 0; i < ne; ++i) {
    const lc_entry& e = E[i];
    if (e.coord == LC_COORD_CTX && !a.n_ctx) continue;
    if (e.coord == LC_COORD_GEN && !a.n_gen) continue;
    const QVal q = unbox(kCellBufs ? col[i * kCellThreads] : *qt_ptr(P, M, slot_row[i * 3], n_b, bi));
    if (e.coord == LC_COORD_CTX || e.coord == LC_COORD_GEN) ++c2; else ++c1;
    if (q.status) {
      int64_t d[5];
      a.expert_tokens = xt();
      entry_coords(e, a, P.hidden, d);
      err->code = q.status; err->label = e.label; err->c0 = d[0]; err->c1 = d[1];
      return q.status;
    }
    const double ms = div1000(q.lat * (double)e.repeat);
    sum.add(0.0 + ms * bubble);
  }
  *out = sum.result();
  *q1 = c1;
  *q2 = c2;
  return 0;
}
// table_step_staged for a whole warp of cells.  Lanes are grouped by (search,
// template) -- one group in the common case, batch lists being long -- and per
// group lane j loads entry j's plan metadata once (coordinate recipe, label,
// repeat and the query-table row of its slot); the plan-order loop broadcasts
// it with shuffles.  Each entry then costs one dependent load (the lane's own
// table value, prefetched two entries ahead) instead of the chain slot ->
// class offset -> value.  Lanes with `active` false only take part in the
// shuffles.  Sum order, skips and the first-failure rule are table_step's.
template <class XT>
__device__ __forceinline__ void warp_table_step(const EvalParams& P, int s, int tmpl, int step, int bi, bool active,
                                                StepArgs a, XT xt, double bubble, double* out, ErrRec* err, int* q1,
                                                int* q2) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  unsigned pending = __ballot_sync(full, active);
  NeumaierSum sum;
  int c1 = 0, c2 = 0;
  bool live = active;
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const int sg = __shfl_sync(full, s, leader), tg = __shfl_sync(full, tmpl, leader);
    const bool act = live && s == sg && tmpl == tg;
    pending &= ~__ballot_sync(full, s == sg && tmpl == tg);
    const int n_b = P.searches[sg].n_b;
    const lc_entry* E = P.entries + (int64_t)tg * LC_MAX_ENTRIES;
    const int ne = P.tmpl_n[tg];
    // lane j: entry j packed in two words -- coordinate recipe (bits 0-3), a flag
    // for a repeat count above 2^24 - 1 (bit 4; read from the entry then) and the
    // repeat (bits 8-31); the query-table index of its slot (int32: n_qt is bounded
    // at batch set-up) -- so an entry costs three shuffles
    int my_pk = 0, my_base = -1;
    if (lane < ne) {
      const lc_entry& e = E[lane];
      const bool big = e.repeat < 0 || e.repeat >= (1ll << 24);
      my_pk = e.coord | (big ? 16 : 0) | (big ? 0 : (int)((uint32_t)e.repeat << 8));
      const int32_t so = P.slot_of[((int64_t)tg * LC_MAX_ENTRIES + lane) * 3 + step];
      if (so >= 0) my_base = (int)(P.meta[sg].qt_off[so >> 16] + (int64_t)(so & 0xffff) * n_b);
    }
    auto fetch = [&](int i, bool& pres) -> double {  // entry i's table value for this lane
      const int pk = __shfl_sync(full, my_pk, i & 31);
      const int base = __shfl_sync(full, my_base, i & 31);
      const int coord = pk & 15;
      const bool skip = (coord == LC_COORD_CTX && !a.n_ctx) || (coord == LC_COORD_GEN && !a.n_gen);
      pres = act && i < ne && !skip && base >= 0;
      return pres ? __ldg(P.qt + base + bi) : 0.0;
    };
    bool run = act, p0, p1;
    double v0 = fetch(0, p0), v1 = fetch(1, p1);
    for (int i = 0; i < ne; ++i) {
      const int pk = __shfl_sync(full, my_pk, i);
      const double v = v0;
      const bool pres = p0;
      v0 = v1;
      p0 = p1;
      v1 = fetch(i + 2, p1);
      if (!run || !pres) continue;
      const int coord = pk & 15;
      const QVal q = unbox(v);
      if (coord == LC_COORD_CTX || coord == LC_COORD_GEN) ++c2; else ++c1;
      if (q.status) {
        int64_t d[5];
        a.expert_tokens = xt();
        entry_coords(E[i], a, P.hidden, d);
        err->code = q.status; err->label = E[i].label; err->c0 = d[0]; err->c1 = d[1];
        run = false;
        live = false;
        continue;
      }
      const double rep = (pk & 16) ? (double)E[i].repeat : (double)((uint32_t)pk >> 8);
      const double ms = div1000(q.lat * rep);
      sum.add(0.0 + ms * bubble);
    }
  }
  if (live) {
    *out = sum.result();
    *q1 = c1;
    *q2 = c2;
  }
}

// The mixed and generation steps of a warp of cells in one pass over the plan
// entries (warp_table_step for two steps): the two plan-order sums are
// independent dependency chains, so interleaving them hides each other's FP64
// latency, and the entry metadata is broadcast once for both.  A lane's
// generation step may be computed when its result is not used (its mixed step
// failed): the step is a pure function of the tables, so nothing changes.
struct StepRes {
  double total;
  ErrRec err;
  int q1, q2;
};
template <class XM, class XG>
__device__ __forceinline__ void warp_table_step2(const EvalParams& P, int s, int tmpl, int bi, bool act_m,
                                                 StepArgs am, XM xtm, bool act_g, StepArgs ag, XG xtg,
                                                 double bubble, StepRes& rm, StepRes& rg) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  unsigned pending = __ballot_sync(full, act_m || act_g);
  NeumaierSum sm, sg;
  int m1 = 0, m2 = 0, g1 = 0, g2 = 0;
  bool live_m = act_m, live_g = act_g;
  auto present = [](int coord, const StepArgs& a) {
    return !((coord == LC_COORD_CTX && !a.n_ctx) || (coord == LC_COORD_GEN && !a.n_gen));
  };
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const int sgi = __shfl_sync(full, s, leader), tg = __shfl_sync(full, tmpl, leader);
    const bool in = s == sgi && tmpl == tg;
    pending &= ~__ballot_sync(full, in);
    const int n_b = P.searches[sgi].n_b;
    const lc_entry* E = P.entries + (int64_t)tg * LC_MAX_ENTRIES;
    const int ne = P.tmpl_n[tg];
    const SearchMeta& M = P.meta[sgi];
    // lane j: entry j as in warp_table_step, with the query-table index of its
    // slot in each of the two steps
    int my_pk = 0, my_bm = -1, my_bg = -1;
    if (lane < ne) {
      const lc_entry& e = E[lane];
      const bool big = e.repeat < 0 || e.repeat >= (1ll << 24);
      my_pk = e.coord | (big ? 16 : 0) | (big ? 0 : (int)((uint32_t)e.repeat << 8));
      const int32_t* so = P.slot_of + ((int64_t)tg * LC_MAX_ENTRIES + lane) * 3;
      const int32_t sm_ = so[LC_STEP_MIXED], sg_ = so[LC_STEP_GEN];
      if (sm_ >= 0) my_bm = (int)(M.qt_off[sm_ >> 16] + (int64_t)(sm_ & 0xffff) * n_b);
      if (sg_ >= 0) my_bg = (int)(M.qt_off[sg_ >> 16] + (int64_t)(sg_ & 0xffff) * n_b);
    }
    bool run_m = live_m && in, run_g = live_g && in;
    const bool go_m = run_m, go_g = run_g;
    // entry i's two table values, one entry ahead
    auto fetch = [&](int i, bool& pm, bool& pg, double& vm, double& vg) {
      const int pk = __shfl_sync(full, my_pk, i & 31);
      const int bm = __shfl_sync(full, my_bm, i & 31), bg = __shfl_sync(full, my_bg, i & 31);
      const int coord = pk & 15;
      pm = go_m && i < ne && present(coord, am) && bm >= 0;
      pg = go_g && i < ne && present(coord, ag) && bg >= 0;
      vm = pm ? __ldg(P.qt + bm + bi) : 0.0;
      vg = pg ? __ldg(P.qt + bg + bi) : 0.0;
    };
    bool pm0, pg0;
    double vm0, vg0;
    fetch(0, pm0, pg0, vm0, vg0);
    for (int i = 0; i < ne; ++i) {
      const int pk = __shfl_sync(full, my_pk, i);
      const double vm = vm0, vg = vg0;
      const bool pm = pm0, pg = pg0;
      fetch(i + 1, pm0, pg0, vm0, vg0);
      const int coord = pk & 15;
      const bool c2d = coord == LC_COORD_CTX || coord == LC_COORD_GEN;
      const double rep = (pk & 16) ? (double)E[i].repeat : (double)((uint32_t)pk >> 8);
      if (run_m && pm) {
        const QVal q = unbox(vm);
        if (c2d) ++m2; else ++m1;
        if (q.status) {
          int64_t d[5];
          am.expert_tokens = xtm();
          entry_coords(E[i], am, P.hidden, d);
          rm.err.code = q.status; rm.err.label = E[i].label; rm.err.c0 = d[0]; rm.err.c1 = d[1];
          run_m = live_m = false;
        } else {
          sm.add(0.0 + div1000(q.lat * rep) * bubble);
        }
      }
      if (run_g && pg) {
        const QVal q = unbox(vg);
        if (c2d) ++g2; else ++g1;
        if (q.status) {
          int64_t d[5];
          ag.expert_tokens = xtg();
          entry_coords(E[i], ag, P.hidden, d);
          rg.err.code = q.status; rg.err.label = E[i].label; rg.err.c0 = d[0]; rg.err.c1 = d[1];
          run_g = live_g = false;
        } else {
          sg.add(0.0 + div1000(q.lat * rep) * bubble);
        }
      }
    }
  }
  if (live_m) { rm.total = sm.result(); rm.q1 = m1; rm.q2 = m2; }
  if (live_g) { rg.total = sg.result(); rg.q1 = g1; rg.q2 = g2; }
}

// K2b: static decode loops (serving_modes.py:256-266), one thread per
// (series group, template, batch) shared by the group's output lengths (SeriesGroup).
// Non-attention terms come from the decode-step query slots (same tokens at every
// sample), attention from the decode-series table.  For each member the result is
// its partial sum after n_steps - 1 samples plus the last sample times its run.
#ifndef LC_DSERIES_MIN_BLOCKS
#define LC_DSERIES_MIN_BLOCKS 6  // 80 registers (measured slightly better than 64 / 8 blocks)
#endif
#ifndef LC_DS_RING
#define LC_DS_RING 8
#endif
#ifndef LC_DECODE_CHAINS
#define LC_DECODE_CHAINS 2  // interleaved Neumaier chains (decode samples) per thread
#endif
constexpr int kChains = LC_DECODE_CHAINS;
constexpr int kDsRing = LC_DS_RING;  // decode-series samples in flight per thread
__global__ void __launch_bounds__(128, LC_DSERIES_MIN_BLOCKS) k_dseries(EvalParams P) {
  __shared__ QVal ds_ring[kDsRing * 128];  // [slot][thread], 16 KB
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < P.n_series;
       x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = P.n_sgroups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.sgroups[mid].off <= x) lo = mid;
      else hi = mid - 1;
    }
    const SeriesGroup G = P.sgroups[lo];
    const lc_search_desc& S = P.searches[G.rep];
    const SearchMeta& M = P.meta[G.rep];
    const int64_t rel = x - G.off;
    const int tmpl = div32(rel, S.n_b), bi = mod32(rel, S.n_b);
    const SeriesMember* mem = P.smembers + G.m_off;
    // samples needed: the longest member whose cell is evaluated
    int K = 0;
    for (int j = 0; j < G.n_m; ++j) {
      const int64_t ci = P.meta[mem[j].search].cell_off + (int64_t)tmpl * S.n_b + bi;
      if ((P.cell_flags[ci] & 1) && mem[j].n_steps > K) K = mem[j].n_steps;
    }
    if (!K) continue;
    const TmplInfo ti = P.tmpl_info[tmpl];
    lc_combo c;
    c.tp = ti.tp; c.pp = ti.pp; c.ep = ti.ep; c.tp_i = ti.tp_i; c.ep_i = ti.ep_i;
    const lc_entry* E = P.entries + (int64_t)tmpl * LC_MAX_ENTRIES;
    const int ne = P.tmpl_n[tmpl];
    const int32_t* so = P.slot_of + (int64_t)tmpl * LC_MAX_ENTRIES * 3;
    const int64_t b = P.batches[S.b_off + bi];
    const int64_t mb = b > 1 ? b : 1;
    const double bubble = (double)(mb + ti.pp - 1) / (double)mb;
    const int64_t xt_dec = expert_tokens(P, c, M, S, 1, bi, b);
    const QVal* ds = P.ds + M.ds_off + (int64_t)P.gclass_of[tmpl] * M.ds_stride * S.n_b + bi;  // sample k at ds[k * n_b]
    const int64_t stride = static_stride(S);  // every member of the group shares it (SeriesGroup key)
    const StepArgs a0{PH_DECODE, 0, b, S.isl + 1, xt_dec};
    double term[LC_MAX_ENTRIES];
    int m = 0, gi = -1;
    const lc_entry* ge = nullptr;
    ErrRec e{0, 0, 0, 0};
    for (int i = 0; i < ne && !e.code; ++i) {
      const lc_entry& en = E[i];
      if (en.coord == LC_COORD_CTX) continue;
      QVal q;
      if (en.coord == LC_COORD_GEN) { q = ds[0]; gi = m; ge = &en; }
      else q = qt_at(P, M, so[i * 3 + LC_STEP_GEN], S.n_b, bi);
      if (q.status) {
        int64_t d[5];
        entry_coords(en, a0, P.hidden, d);
        e.code = q.status; e.label = en.label; e.c0 = d[0]; e.c1 = d[1];
        break;
      }
      const double ms = div1000(q.lat * (double)en.repeat);
      term[m++] = 0.0 + ms * bubble;
    }
    int mi = 0;  // next member to receive its total (members ascend in n_steps)
    int trig = G.n_m > 0 ? mem[0].n_steps - 1 : -1;  // ... at this sample
    auto put = [&](int j, double t_gen, int32_t status, int steps, int64_t c0, int64_t c1) {
      const int64_t ci = P.meta[mem[j].search].cell_off + (int64_t)tmpl * S.n_b + bi;
      SdOut o;
      o.t_gen = t_gen;
      o.status = status;
      o.qsd = ((m - 1) * steps & 0xffff) | (steps << 16);
      o.c0 = c0; o.c1 = c1;
      P.sd[ci] = o;
    };
    if (!e.code) {
      NeumaierSum pre;
      for (int i = 0; i < gi; ++i) pre.add(term[i]);
      const double g_rep = ge ? (double)ge->repeat : 0.0;  // loop-invariant (ge points into global memory)
      // the terms after the attention entry, in registers for the sample loop
      constexpr int kPostRegs = 10;
      const int npost = m - gi - 1;
      double post[kPostRegs];
#pragma unroll
      for (int i = 0; i < kPostRegs; ++i) post[i] = i < npost ? term[gi + 1 + i] : 0.0;
      double t_gen = 0.0;
      // The attention latencies of samples 1..K-1 stream from the decode-series
      // table through a per-thread ring in shared memory, kDsRing samples ahead
      // (cp.async: LDGSTS), so the L2 latency of sample sj + kDsRing overlaps the
      // Neumaier chains of sample sj instead of stalling each iteration.
      QVal* ring = ds_ring + threadIdx.x;  // slot k at ring[k * 128]
      auto issue = [&](int k) {
        if (k > 0 && k < K) __pipeline_memcpy_async(ring + (k % kDsRing) * 128, ds + (int64_t)k * S.n_b, sizeof(QVal));
        __pipeline_commit();
      };
#pragma unroll
      for (int k = 0; k < kDsRing; ++k) issue(k);
      for (int step = 0; step < K && !e.code; step += kChains) {
        // groups of samples < step + kChains are complete once at most kDsRing - kChains are pending
        __pipeline_wait_prior(kDsRing - kChains);
        double g[kChains];
        int bad = -1;
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
          const int sj = step + j;
          g[j] = 0.0;
          if (sj >= K || bad >= 0) continue;
          if (sj == 0) { g[j] = term[gi]; continue; }
          const QVal q = ring[(sj % kDsRing) * 128];
          if (q.status) { bad = j; e.code = q.status; e.label = ge->label; e.c0 = b; e.c1 = S.isl + stride * sj + 1; continue; }
          g[j] = 0.0 + div1000(q.lat * g_rep) * bubble;
        }
#pragma unroll
        for (int j = 0; j < kChains; ++j) issue(step + kDsRing + j);
        NeumaierSum sc[kChains];
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
          sc[j] = pre;
          sc[j].add(g[j]);
        }
        if (npost <= kPostRegs) {
#pragma unroll
          for (int i = 0; i < kPostRegs; ++i) {
            if (i >= npost) break;
#pragma unroll
            for (int j = 0; j < kChains; ++j) sc[j].add_next(post[i]);  // the attention term came first
          }
        } else {
          for (int i = gi + 1; i < m; ++i) {
            const double xv = term[i];
#pragma unroll
            for (int j = 0; j < kChains; ++j) sc[j].add_next(xv);
          }
        }
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
          const int sj = step + j;
          if (sj >= K || (bad >= 0 && j >= bad)) continue;
          const double st = sc[j].result();
          // members whose last sample is sj: t_gen + st * run, run = osl - 1 - stride sj
          while (sj == trig) {  // the next member's last sample (members ascend in n_steps)
            const int64_t run = P.searches[mem[mi].search].osl - 1 - stride * sj;
            put(mi, t_gen + st * (double)run, 0, mem[mi].n_steps, 0, 0);
            ++mi;
            trig = mi < G.n_m ? mem[mi].n_steps - 1 : -1;
          }
          t_gen += st * (double)stride;
        }
      }
      __pipeline_wait_prior(0);  // the ring is reused by this thread's next series
    }
    // members not reached: the first failing query decides
    for (; mi < G.n_m; ++mi) put(mi, 0.0, e.code | (e.label << 8), 0, e.c0, e.c1);
  }
}

// K2a'': prefill step totals, one thread per (prefill group, template, batch);
// k_eval_cells reads them instead of re-summing the step for every member.
__global__ void __launch_bounds__(128) k_ptables(EvalParams P) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < P.n_pstep;
       x += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = P.n_pgroups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.pgroups[mid].off <= x) lo = mid;
      else hi = mid - 1;
    }
    const PGroup G = P.pgroups[lo];
    const lc_search_desc& S = P.searches[G.rep];
    const SearchMeta& M = P.meta[G.rep];
    const int64_t rel = x - G.off;
    const int tmpl = div32(rel, G.n_b), bi = mod32(rel, G.n_b);
    const TmplInfo ti = P.tmpl_info[tmpl];
    lc_combo c;
    c.tp = ti.tp; c.pp = ti.pp; c.ep = ti.ep; c.tp_i = ti.tp_i; c.ep_i = ti.ep_i;
    const lc_entry* E = P.entries + (int64_t)tmpl * LC_MAX_ENTRIES;
    const int ne = P.tmpl_n[tmpl];
    const int32_t* so = P.slot_of + (int64_t)tmpl * LC_MAX_ENTRIES * 3;
    const int64_t b = P.batches[S.b_off + bi];
    const int64_t mb = b > 1 ? b : 1;
    const double bubble = (double)(mb + ti.pp - 1) / (double)mb;
    const int64_t chunk = S.isl - S.prefix;
    const StepArgs a{PH_PREFILL, b * chunk, 0, chunk, expert_tokens(P, c, M, S, 0, bi, b * chunk)};
    double total = 0.0;
    ErrRec err{0, 0, 0, 0};
    int q1 = 0, q2 = 0;
    table_step(P, M, E, ne, so + LC_STEP_PREFILL, S.n_b, bi, a, bubble, &total, &err, &q1, &q2);
    PStep o;
    o.total = total;
    o.status = err.code | (err.label << 8);
    o.q = err.code ? 0 : ((q1 & 0xffff) | (q2 << 16));
    o.c0 = err.c0;
    o.c1 = err.c1;
    P.psteps[x] = o;
  }
}

// K4 speed buckets (k_front_*): order-preserving buckets of the IEEE bit pattern
// of a feasible row's speed, holding the best throughput seen in each.  With a
// speed floor every feasible speed is >= the floor, so the buckets can be fixed
// before any row exists -- 256 per binade from the floor's binade up, 16 binades,
// faster rows sharing the top bucket -- and the maxima are accumulated while the
// rows are written (k_eval_cells / k_expand / k_disagg), saving K4 a pass over
// every row.  Without a floor the range pass (k_front_mid / k_front_pass2) runs.
#ifndef LC_BUCKET_PRECHECK
#define LC_BUCKET_PRECHECK 0  // 1: a plain read before the atomic -- measured no gain
#endif
constexpr int kSpeedBuckets = 4096;
constexpr int kFixedShift = 44;
__device__ __forceinline__ bool fixed_buckets(const lc_search_desc& S) {
  return S.has_floor && S.speed_floor > 0.0 && S.speed_floor < INFINITY;
}
__device__ __forceinline__ int fixed_bucket(const lc_search_desc& S, double speed) {
  const unsigned long long base = ((unsigned long long)__double_as_longlong(S.speed_floor)) >> kFixedShift;
  const unsigned long long d = (((unsigned long long)__double_as_longlong(speed)) >> kFixedShift) - base;
  return d < (unsigned long long)kSpeedBuckets ? (int)d : kSpeedBuckets - 1;  // speed >= floor: no wrap
}
__device__ __forceinline__ void bucket_max(unsigned long long* bk, const lc_search_desc& S, double speed, double thru) {
  // most rows do not raise their bucket's maximum once it has settled: a plain
  // read first keeps them off the (same-address, serialising) L2 atomics
  unsigned long long* at = &bk[fixed_bucket(S, speed)];
  const unsigned long long v = (unsigned long long)__double_as_longlong(thru);
  if (LC_BUCKET_PRECHECK && *(volatile unsigned long long*)at >= v) return;
  atomicMax(at, v);
}

// K2: one thread per cell assembles every step from the tables.
// Warp-aggregated per-search accounting: one set of atomics per warp when all
// its units belong to one search (the common case), per lane otherwise.
struct RowAcc {
  unsigned q1, q2;
  int feas, rows, enums, skips;
  unsigned long long smin_c, smax;
  __device__ __forceinline__ void feasible_speed(double speed) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(speed);
    smax = b > smax ? b : smax;
    smin_c = ~b > smin_c ? ~b : smin_c;
  }
};

__device__ __forceinline__ void acc_flush(SearchAcc* A, const RowAcc& r) {
  if (r.q1) atomicAdd(&A->q1, (unsigned long long)r.q1);
  if (r.q2) atomicAdd(&A->q2, (unsigned long long)r.q2);
  if (r.feas) atomicAdd(&A->feas, r.feas);
  if (r.rows) atomicAdd(&A->rows, r.rows);
  if (r.enums) atomicAdd(&A->enums, r.enums);
  if (r.skips) atomicAdd(&A->skips, r.skips);
  if (r.smax) atomicMax(&A->smax, r.smax);
  if (r.smin_c) atomicMax(&A->smin_c, r.smin_c);
}

// What a cell's dp variants share: derive_metrics (serving_modes.py:161-172)
// up to the final division by the gpu count -- speed, and throughput as
// ((1000 / req) * batch) * osl, the reference's left-to-right order -- the pool
// rates (serving_modes.py:366, 380) before their division by gpus, and the
// feasibility tests (speed and TTFT do not depend on gpus).
struct CellRows {
  double st_speed, st_tp, ag_speed, ag_tp, pf_rate, dc_rate;
  bool st_feas, ag_feas, dup;
};
__device__ __forceinline__ CellRows cell_rows(const lc_search_desc& S, const CellOut& o, int64_t b) {
  CellRows R;
  R.st_speed = R.st_tp = R.ag_speed = R.ag_tp = R.pf_rate = R.dc_rate = 0.0;
  R.st_feas = R.ag_feas = false;
  if (o.st_status == 0) {
    R.st_speed = o.st_tpot == 0.0 ? INFINITY : 1000.0 / o.st_tpot;
    const double req = o.st_ttft + (double)(S.osl - 1) * o.st_tpot;
    R.st_tp = 1000.0 / req * (double)b * (double)S.osl;
    R.st_feas = (!S.has_ttft || o.st_ttft <= S.ttft_limit) && (!S.has_floor || R.st_speed >= S.speed_floor);
  }
  if (o.ag_status == 0) {
    R.ag_speed = o.ag_tpot == 0.0 ? INFINITY : 1000.0 / o.ag_tpot;
    const double req = o.ag_ttft + (double)(S.osl - 1) * o.ag_tpot;
    R.ag_tp = 1000.0 / req * (double)b * (double)S.osl;
    R.ag_feas = (!S.has_ttft || o.ag_ttft <= S.ttft_limit) && (!S.has_floor || R.ag_speed >= S.speed_floor);
  }
  if (o.pf_status == 0) R.pf_rate = (double)b * 1000.0 / o.pf_lat;
  if (o.dc_status == 0) R.dc_rate = S.osl == 1 ? INFINITY : (double)b * 1000.0 / ((double)(S.osl - 1) * o.dc_lat);
  // the generation step is a memo hit when a static decode step used the same KV length
  const int64_t k = (S.isl + S.osl / 2) - S.isl - 1;
  const int64_t sstr = static_stride(S);
  R.dup = o.st_status == 0 && S.osl > 1 && k >= 0 && (k % sstr) == 0 && (k / sstr) < o.st_steps;
  return R;
}

// x / g for a gpu count g: when g is a power of two, x * 2^-k is the same single
// correctly rounded operation on the same exact value as x / 2^k (subnormal
// results included), without the division sequence.
struct GpuDiv {
  double g, inv;
  bool p2;
  __device__ __forceinline__ explicit GpuDiv(int64_t gpus) {
    g = (double)gpus;
    p2 = gpus > 0 && (gpus & (gpus - 1)) == 0 && gpus < (1ll << 52);
    inv = p2 ? __longlong_as_double((long long)(1023 - (__ffsll(gpus) - 1)) << 52) : 0.0;
  }
  __device__ __forceinline__ double operator()(double x) const { return p2 ? x * inv : x / g; }
};

// One candidate's rows from its cell's shared values (CellRows) and its gpu
// count, plus its contribution to the per-search accounting.
__device__ __forceinline__ void expand_unit(const EvalParams& P, const lc_search_desc& S, const CellOut& o,
                                            const CellRows& R, int64_t ci, int64_t u, int64_t gpus, bool inb,
                                            RowAcc& ra, unsigned long long* bk, double* seed_at = nullptr) {
  const int64_t n = P.n_cap;
  const bool do_st = (S.modes & 1) && inb, do_ag = (S.modes & 2) && inb, do_dg = (S.modes & 4) != 0;
  const GpuDiv div_g(gpus);
  int fflags = 0;  // K4 reads these instead of the rows' status / ttft / speed
  int32_t q = 0;
  auto add_q = [&](int32_t x) { q += x; };  // packed halves never overflow 16 bits
  if (do_st) {
    P.st_status[u] = o.st_status;
    if (o.st_status) {
      P.err_c[u] = P.cell_err[ci * 8 + 0]; P.err_c[n + u] = P.cell_err[ci * 8 + 1];
    } else {
      const double thru = div_g(R.st_tp);
      P.st_v[u] = o.st_ttft; P.st_v[n + u] = o.st_tpot; P.st_v[2 * n + u] = R.st_speed; P.st_v[3 * n + u] = thru;
      ++ra.rows;
      if (R.st_feas) {
        fflags |= 1;
        ++ra.feas;
        ra.feasible_speed(R.st_speed);
        if (bk) bucket_max(bk, S, R.st_speed, thru);
      }
      add_q(o.qSD);
    }
  }
  if (do_ag) {
    P.ag_status[u] = o.ag_status;
    if (o.ag_status) {
      P.err_c[2 * n + u] = P.cell_err[ci * 8 + 2]; P.err_c[3 * n + u] = P.cell_err[ci * 8 + 3];
    } else {
      const double thru = div_g(R.ag_tp);
      P.ag_v[u] = o.ag_ttft; P.ag_v[n + u] = o.ag_tpot; P.ag_v[2 * n + u] = R.ag_speed; P.ag_v[3 * n + u] = thru;
      ++ra.rows;
      if (R.ag_feas) {
        fflags |= 2;
        ++ra.feas;
        ra.feasible_speed(R.ag_speed);
        if (bk) bucket_max(bk, S, R.ag_speed, thru);
      }
    }
    add_q(o.qM);
  }
  if (do_st || do_dg) add_q(o.qP);
  if (do_dg) {
    P.pf_status[u] = o.pf_status;
    if (o.pf_status) {
      P.err_c[4 * n + u] = P.cell_err[ci * 8 + 4]; P.err_c[5 * n + u] = P.cell_err[ci * 8 + 5];
      P.pool_key[u] = INFINITY;
      if (seed_at) seed_at[0] = INFINITY;
    } else {
      P.pf_v[u] = o.pf_lat; P.pf_v[n + u] = R.pf_rate;
      const double r = div_g(-R.pf_rate);
      P.pool_key[u] = r;
      if (seed_at) seed_at[0] = r;
    }
    P.dc_status[u] = o.dc_status;
    if (o.dc_status) {
      P.err_c[6 * n + u] = P.cell_err[ci * 8 + 6]; P.err_c[7 * n + u] = P.cell_err[ci * 8 + 7];
      P.pool_key[n + u] = INFINITY;
      if (seed_at) seed_at[1] = INFINITY;
    } else {
      P.dc_v[u] = o.dc_lat;
      P.dc_v[n + u] = R.dc_rate;
      const double r = div_g(-R.dc_rate);
      P.pool_key[n + u] = r;
      if (seed_at) seed_at[1] = r;
    }
  }
  if (((do_ag && (o.flags & 1)) || do_dg) && !(do_st && R.dup)) add_q(o.qG);
  P.front_flags[u] = (uint8_t)fflags;
  ra.q1 += (unsigned)(q & 0xffff);
  ra.q2 += (unsigned)(q >> 16);
  if (inb) {
    ++ra.enums;
    if ((S.modes & 1) && o.st_status) ++ra.skips;
    if ((S.modes & 2) && o.ag_status) ++ra.skips;
  }
  if (do_dg) ra.skips += (o.pf_status != 0) + (o.dc_status != 0);
}

// One cell: every step from the tables (K2).  With the closed-form K0
// (P.pair_off) the cell also writes the rows of its dp-variant candidates
// (expand_unit) -- the cell stays in registers instead of a k_expand re-read.
// WARP: called by all 32 lanes of a warp whose cells share (search, template)
// (cells with cf == 0 included: they take part in the shuffles, write nothing).
template <bool WARP>
__device__ __forceinline__ void eval_cell(const EvalParams& P, int64_t ci, int s, uint32_t cf, RowAcc& ra,
                                          int& s_out, double* stage) {
  const lc_search_desc& S = P.searches[s];
  const SearchMeta& M = P.meta[s];
  const int64_t rel = ci - M.cell_off;
  const int tmpl = div32(rel, S.n_b), bi = mod32(rel, S.n_b);
  const TmplInfo ti = P.tmpl_info[tmpl];
  lc_combo c;  // the fields expert_tokens() reads
  c.tp = ti.tp; c.pp = ti.pp; c.ep = ti.ep; c.tp_i = ti.tp_i; c.ep_i = ti.ep_i;
  const lc_entry* E = P.entries + (int64_t)tmpl * LC_MAX_ENTRIES;
  const int ne = P.tmpl_n[tmpl];
  const int32_t* so = P.slot_of + (int64_t)tmpl * LC_MAX_ENTRIES * 3;
  const int64_t b = P.batches[S.b_off + bi];
  const bool do_st = (cf & 1) && (S.modes & 1), do_ag = (cf & 1) && (S.modes & 2), do_dg = (cf & 2) != 0;
  const int64_t mb = b > 1 ? b : 1;
  const double bubble = (double)(mb + ti.pp - 1) / (double)mb;
  const int64_t chunk = S.isl - S.prefix;
  const int64_t kv_mid = S.isl + S.osl / 2;
  CellOut o;
  o.st_status = o.ag_status = o.pf_status = o.dc_status = LC_ST_NOT_EVALUATED;
  o.st_ttft = o.st_tpot = o.ag_ttft = o.ag_tpot = o.pf_lat = o.dc_lat = 0.0;
  o.qP = o.qSD = o.qM = o.qG = 0;
  o.st_steps = 0;
  o.flags = 0;
  int q1 = 0, q2 = 0;
  // the mixed and generation steps' table values, requested before anything else
  double* colM = stage;
  double* colG = stage + (kCellBufs > 1 ? LC_MAX_ENTRIES * kCellThreads : 0);
  __pipeline_wait_prior(0);  // the previous cell's copies into these columns have landed
  if (do_ag) stage_step(P, M, ne, so + LC_STEP_MIXED, S.n_b, bi, colM);
  bool g_staged = false;
  if (kCellBufs > 1 && (do_ag || do_dg)) {
    stage_step(P, M, ne, so + LC_STEP_GEN, S.n_b, bi, colG);
    g_staged = true;
  }

  // prefill step: static TTFT and the prefill pool
  double p_total = 0.0;
  ErrRec p_err{0, 0, 0, 0};
  if (do_st || do_dg) {
    if (M.pstep_off >= 0) {  // shared with the other searches of the prefill group (k_ptables)
      const PStep ps = P.psteps[M.pstep_off + rel];
      p_total = ps.total;
      p_err.code = ps.status & 0xff; p_err.label = ps.status >> 8; p_err.c0 = ps.c0; p_err.c1 = ps.c1;
      o.qP = ps.q;
    } else {
      const StepArgs a{PH_PREFILL, b * chunk, 0, chunk, expert_tokens(P, c, M, S, 0, bi, b * chunk)};
      table_step(P, M, E, ne, so + LC_STEP_PREFILL, S.n_b, bi, a, bubble, &p_total, &p_err, &q1, &q2);
      if (!p_err.code) o.qP = (q1 & 0xffff) | (q2 << 16);
    }
    o.pf_status = p_err.code | (p_err.label << 8);
    o.pf_lat = p_total;
    if (p_err.code) put_cell_err(P, 2, ci, p_err);
  }
  bool g_done = false;
  double g_total = 0.0;
  ErrRec g_err{0, 0, 0, 0};
  const StepArgs ga{PH_DECODE, 0, b, kv_mid, 0};
  auto xt_dec = [&]() { return expert_tokens(P, c, M, S, 1, bi, b); };
  auto gen_step = [&]() {
    if (!g_staged) {
      stage_step(P, M, ne, so + LC_STEP_GEN, S.n_b, bi, colG);
      g_staged = true;
    }
    __pipeline_wait_prior(0);
    table_step_staged(P, M, E, ne, so + LC_STEP_GEN, S.n_b, bi, colG, ga, xt_dec, bubble, &g_total, &g_err, &q1, &q2);
  };
  if (do_st) {
    double tpot = 0.0;
    ErrRec e = p_err;
    if (!e.code && S.osl > 1) {
      const SdOut sd = P.sd[ci];  // k_dseries
      if (sd.status) {
        e.code = sd.status & 0xff; e.label = sd.status >> 8; e.c0 = sd.c0; e.c1 = sd.c1;
      } else {
        tpot = sd.t_gen / (double)(S.osl - 1);
        o.qSD = sd.qsd;
        o.st_steps = M.n_steps;
      }
    }
    o.st_status = e.code | (e.label << 8);
    o.st_ttft = p_total;
    o.st_tpot = tpot;
    if (e.code) put_cell_err(P, 0, ci, e);
  }
  if constexpr (WARP) {
    // the mixed step, then the generation step at the KV midpoint for every lane
    // that needs it (aggregated l_gen, the decode pool), each one warp loop
    const AggSched sc = agg_schedule(S, b);
    const bool need_mix = do_ag && !sc.st;
    const StepArgs am{PH_MIXED, sc.chunk_tokens, sc.n_mix_gen, kv_mid, 0};
    auto xt_mix = [&]() { return expert_tokens(P, c, M, S, 2, bi, sc.chunk_tokens + sc.n_mix_gen); };
    double l_mix = 0.0;
    ErrRec em{0, 0, 0, 0};
    int m1 = 0, m2 = 0;
#if LC_FUSED_STEPS
    // both steps in one pass; the generation step for every lane that may use it
    StepRes rm{0.0, {0, 0, 0, 0}, 0, 0}, rg{0.0, {0, 0, 0, 0}, 0, 0};
    warp_table_step2(P, s, tmpl, bi, need_mix, am, xt_mix, (need_mix && (sc.t_gen || b == 1)) || do_dg, ga, xt_dec,
                     bubble, rm, rg);
    l_mix = rm.total; em = rm.err; m1 = rm.q1; m2 = rm.q2;
    g_total = rg.total; g_err = rg.err; q1 = rg.q1; q2 = rg.q2;
    const bool gen_for_ag = need_mix && !em.code && (sc.t_gen || b == 1);
#else
    warp_table_step(P, s, tmpl, LC_STEP_MIXED, bi, need_mix, am, xt_mix, bubble, &l_mix, &em, &m1, &m2);
    const bool gen_for_ag = need_mix && !em.code && (sc.t_gen || b == 1);
    warp_table_step(P, s, tmpl, LC_STEP_GEN, bi, gen_for_ag || do_dg, ga, xt_dec, bubble, &g_total, &g_err, &q1, &q2);
#endif
    const int32_t qg = (q1 & 0xffff) | (q2 << 16);
    if (do_ag) {
      ErrRec e{sc.st, 0, 0, 0};
      double ttft = 0.0, tpot = 0.0;
      if (!sc.st) {
        e = em;
        if (!em.code) o.qM = (m1 & 0xffff) | (m2 << 16);
        double l_gen = 0.0;
        if (gen_for_ag) {
          if (!g_err.code) o.qG = qg;
          o.flags |= 1;
          e = g_err;
          l_gen = g_total;
        }
        if (!e.code) {
          const double raw = 2.0 + (double)(sc.T - 3) * (1.0 / 20.0);
          double F = raw > 2.0 ? raw : 2.0;
          F = F < 4.0 ? F : 4.0;
          ttft = l_mix * (double)sc.cpr * F;
          if (b == 1) tpot = S.osl > 1 ? l_gen : 0.0;
          else if (S.osl == 1) tpot = 0.0;
          else if (sc.t_gen == 0) tpot = l_mix;
          else {
            const int64_t ms = sc.t_mix - 3 > 1 ? sc.t_mix - 3 : 1;
            tpot = (l_mix * (double)ms + l_gen * (double)sc.t_gen) / (double)(ms + sc.t_gen);
          }
        }
      }
      o.ag_status = e.code | (e.label << 8);
      o.ag_ttft = ttft;
      o.ag_tpot = tpot;
      if (e.code) put_cell_err(P, 1, ci, e);
    }
    if (do_dg) {
      if (!g_err.code) o.qG = qg;
      o.dc_status = g_err.code | (g_err.label << 8);
      o.dc_lat = g_total;
      if (g_err.code) put_cell_err(P, 3, ci, g_err);
    }
    if (!cf) return;
  } else {
  // generation step at the KV midpoint: aggregated l_gen and the decode pool
  if (do_ag) {
    const AggSched sc = agg_schedule(S, b);
    ErrRec e{sc.st, 0, 0, 0};
    double ttft = 0.0, tpot = 0.0;
    if (!sc.st) {
      double l_mix = 0.0, l_gen = 0.0;
      const StepArgs a{PH_MIXED, sc.chunk_tokens, sc.n_mix_gen, kv_mid, 0};
      auto xt_mix = [&]() { return expert_tokens(P, c, M, S, 2, bi, sc.chunk_tokens + sc.n_mix_gen); };
      __pipeline_wait_prior(kCellBufs > 1 ? 1 : 0);  // the mixed column (the generation one may still fly)
      table_step_staged(P, M, E, ne, so + LC_STEP_MIXED, S.n_b, bi, colM, a, xt_mix, bubble, &l_mix, &e, &q1, &q2);
      if (!e.code) o.qM = (q1 & 0xffff) | (q2 << 16);
      if (!e.code && (sc.t_gen || b == 1)) {
        gen_step();
        g_done = true;
        if (!g_err.code) o.qG = (q1 & 0xffff) | (q2 << 16);
        o.flags |= 1;
        e = g_err;
        l_gen = g_total;
      }
      if (!e.code) {
        const double raw = 2.0 + (double)(sc.T - 3) * (1.0 / 20.0);
        double F = raw > 2.0 ? raw : 2.0;
        F = F < 4.0 ? F : 4.0;
        ttft = l_mix * (double)sc.cpr * F;
        if (b == 1) tpot = S.osl > 1 ? l_gen : 0.0;
        else if (S.osl == 1) tpot = 0.0;
        else if (sc.t_gen == 0) tpot = l_mix;
        else {
          const int64_t ms = sc.t_mix - 3 > 1 ? sc.t_mix - 3 : 1;
          tpot = (l_mix * (double)ms + l_gen * (double)sc.t_gen) / (double)(ms + sc.t_gen);
        }
      }
    }
    o.ag_status = e.code | (e.label << 8);
    o.ag_ttft = ttft;
    o.ag_tpot = tpot;
    if (e.code) put_cell_err(P, 1, ci, e);
  }
  if (do_dg) {
    if (!g_done) {
      gen_step();
      if (!g_err.code) o.qG = (q1 & 0xffff) | (q2 << 16);
    }
    o.dc_status = g_err.code | (g_err.label << 8);
    o.dc_lat = g_total;
    if (g_err.code) put_cell_err(P, 3, ci, g_err);
  }
  }  // !WARP
  if (P.pair_off) {
    s_out = s;
    unsigned long long* bk = fixed_buckets(S) ? P.fbuckets + (int64_t)s * kSpeedBuckets : nullptr;
    const int64_t pbase = (int64_t)s * P.sp_n_combos;
    const int j1 = P.tmpl_cidx_off[tmpl + 1];
    const CellRows R = cell_rows(S, o, b);
    for (int j = P.tmpl_cidx_off[tmpl]; j < j1; ++j) {
      const int cj = P.tmpl_cidx[j];
      const int64_t pr = pbase + cj;
      const int32_t off = P.pair_off[pr], cnt = P.pair_off[pr + 1] - off;
      if (bi >= cnt) continue;  // this dp variant is not a candidate at this batch
      // the pair's last unit (largest batch) also goes to the K5a seed sample
      double* seed_at = P.pool_sample && bi == cnt - 1 ? P.pool_sample + 2 * pr : nullptr;
      expand_unit(P, S, o, R, ci, (int64_t)off + bi, P.combos[cj].gpus, P.pair_inb[pr] != 0, ra, bk, seed_at);
    }
  } else {
    P.cells[ci] = o;
  }
}

__global__ void __launch_bounds__(kCellThreads, LC_CELL_MIN_BLOCKS) k_eval_cells(EvalParams P) {
  __shared__ double stage[kCellBufs ? kCellBufs * LC_MAX_ENTRIES * kCellThreads : 1];  // [buffer][entry][thread]
  const int64_t ncell = P.n_cells_total;
  const int lane = threadIdx.x & 31;
  // a thread's search index only moves forward (one compare per cell instead of
  // a binary search over the searches)
  int hint = -1;
  auto run_range = [&](int64_t beg, int64_t end) {
  for (int64_t base = beg + threadIdx.x - lane; base < end; base += blockDim.x) {
    const int64_t ci = base + lane;
    RowAcc ra{0, 0, 0, 0, 0, 0, 0ull, 0ull};
    int s = -1;
    const uint32_t cf = ci < end ? P.cell_flags[ci] : 0u;
#if LC_CELL_PREFETCH
    // the next iteration's per-cell inputs start moving now (L1 prefetch): the
    // chain flags -> search -> step totals otherwise starts cold every iteration
    if (ci + (int64_t)blockDim.x < end) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P.cell_flags + ci + blockDim.x));
      if (P.sd) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.sd + ci + blockDim.x));
    }
#endif
    if (LC_WARP_STEPS) {
      // every lane of a warp with work takes part (warp_table_step); lanes past
      // the range stand in as lane 0's cell with nothing to evaluate
      if (!__any_sync(0xffffffffu, cf != 0u)) continue;
      const int64_t cv = ci < end ? ci : base;
      if (hint < 0) hint = find_cell_search(P.meta, P.n_search, cv);
      while (hint + 1 < P.n_search && P.meta[hint + 1].cell_off <= cv) ++hint;
      eval_cell<true>(P, cv, hint, cf, ra, s, stage + threadIdx.x);
    } else if (cf) {
      if (hint < 0) hint = find_cell_search(P.meta, P.n_search, ci);
      while (hint + 1 < P.n_search && P.meta[hint + 1].cell_off <= ci) ++hint;
      eval_cell<false>(P, ci, hint, cf, ra, s, stage + threadIdx.x);
    }
    if (!P.pair_off) continue;  // uniform: k_expand does the accounting
    // warp-aggregated accounting (cells are ordered by search)
    int s0 = -1;
    const unsigned act = __ballot_sync(0xffffffffu, s >= 0);
    if (!act) continue;
    s0 = __shfl_sync(0xffffffffu, s, __ffs(act) - 1);
    if (__all_sync(0xffffffffu, s < 0 || s == s0)) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) {
        ra.q1 += __shfl_xor_sync(0xffffffffu, ra.q1, o2);
        ra.q2 += __shfl_xor_sync(0xffffffffu, ra.q2, o2);
        ra.feas += __shfl_xor_sync(0xffffffffu, ra.feas, o2);
        ra.rows += __shfl_xor_sync(0xffffffffu, ra.rows, o2);
        ra.enums += __shfl_xor_sync(0xffffffffu, ra.enums, o2);
        ra.skips += __shfl_xor_sync(0xffffffffu, ra.skips, o2);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, ra.smax, o2);
        const unsigned long long m = __shfl_xor_sync(0xffffffffu, ra.smin_c, o2);
        ra.smax = a > ra.smax ? a : ra.smax;
        ra.smin_c = m > ra.smin_c ? m : ra.smin_c;
      }
      if (lane == 0) acc_flush(P.acc + s0, ra);
    } else if (s >= 0) {
      acc_flush(P.acc + s, ra);
    }
  }
  };
#if LC_CELL_DYNAMIC
  // chunks of kCellChunk cells handed out in order by a counter (the per-cell
  // cost varies with the cell flags, so static ranges leave a tail); a block's
  // chunks ascend, so its search index still only moves forward
  __shared__ long long next;
  for (;;) {
    if (threadIdx.x == 0) next = (long long)atomicAdd(P.cell_ctr, 1ull);
    __syncthreads();
    const int64_t beg = (int64_t)next * kCellChunk;
    __syncthreads();
    if (beg >= ncell) break;
    run_range(beg, beg + kCellChunk < ncell ? beg + kCellChunk : ncell);
  }
#else
  // each block walks one contiguous range of cells
  const int64_t per = ((ncell + gridDim.x - 1) / gridDim.x + 127) / 128 * 128;
  const int64_t beg = (int64_t)blockIdx.x * per;
  run_range(beg, beg + per < ncell ? beg + per : ncell);
#endif
}

// K2b: candidates from their cells -- derive_metrics with the candidate's gpu
// count (serving_modes.py:161-172) and the pool rates (serving_modes.py:366, 380).
#ifndef LC_EXPAND_MIN_BLOCKS
#define LC_EXPAND_MIN_BLOCKS 4  // 64 registers (measured: 4.11 -> 4.00 ms per step)
#endif
__global__ void __launch_bounds__(256, LC_EXPAND_MIN_BLOCKS) k_expand(EvalParams P) {
  const int64_t total = *P.d_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  __shared__ RowAcc wacc[8];
  for (int64_t bbase = blockIdx.x * (int64_t)blockDim.x; bbase < total; bbase += stride) {
    const int64_t u = bbase + threadIdx.x;
    // units are ordered by search: one set of atomics per block when it lies in one search
    const int64_t last = (bbase + blockDim.x < total ? bbase + blockDim.x : total) - 1;
    const bool block_uniform = P.u_search[bbase] == P.u_search[last];
    RowAcc ra{0, 0, 0, 0, 0, 0, 0ull, 0ull};
    int s = -1;
    if (u < total) {
    s = P.u_search[u];
    const lc_search_desc& S = P.searches[s];
    const int bi = P.u_batch[u];
    const lc_combo c = P.combos[P.u_combo[u]];
    const int64_t ci = P.meta[s].cell_off + (int64_t)c.tmpl * S.n_b + bi;
    const CellOut o = P.cells[ci];
    const int64_t b = P.batches[S.b_off + bi];
    const bool inb = P.u_budget[u] != 0;
    expand_unit(P, S, o, cell_rows(S, o, b), ci, u, c.gpus, inb, ra,
                fixed_buckets(S) ? P.fbuckets + (int64_t)s * kSpeedBuckets : nullptr);
    }
    // per-search accounting for K4 (search.py:343-358 counts, speed range)
    int s0 = __shfl_sync(0xffffffffu, s, 0);
    if (s0 < 0) s0 = P.u_search[bbase];  // a warp entirely past the end of the units
    if (__all_sync(0xffffffffu, s < 0 || s == s0)) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) {
        ra.q1 += __shfl_xor_sync(0xffffffffu, ra.q1, o2);
        ra.q2 += __shfl_xor_sync(0xffffffffu, ra.q2, o2);
        ra.feas += __shfl_xor_sync(0xffffffffu, ra.feas, o2);
        ra.rows += __shfl_xor_sync(0xffffffffu, ra.rows, o2);
        ra.enums += __shfl_xor_sync(0xffffffffu, ra.enums, o2);
        ra.skips += __shfl_xor_sync(0xffffffffu, ra.skips, o2);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, ra.smax, o2);
        const unsigned long long m = __shfl_xor_sync(0xffffffffu, ra.smin_c, o2);
        ra.smax = a > ra.smax ? a : ra.smax;
        ra.smin_c = m > ra.smin_c ? m : ra.smin_c;
      }
      if (block_uniform) {
        if (lane == 0) wacc[warp] = ra;
      } else if (lane == 0) {
        acc_flush(P.acc + s0, ra);
      }
    } else if (s >= 0) {
      acc_flush(P.acc + s, ra);
    }
    if (block_uniform) {
      __syncthreads();
      if (threadIdx.x == 0) {
        RowAcc t = wacc[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
          const RowAcc& o2 = wacc[w];
          t.q1 += o2.q1; t.q2 += o2.q2; t.feas += o2.feas; t.rows += o2.rows; t.enums += o2.enums;
          t.skips += o2.skips;
          t.smax = o2.smax > t.smax ? o2.smax : t.smax;
          t.smin_c = o2.smin_c > t.smin_c ? o2.smin_c : t.smin_c;
        }
        acc_flush(P.acc + P.u_search[bbase], t);
      }
      __syncthreads();
    }
  }
}

// ---- comparison helpers for top-k / best / nearest
struct PoolKey {
  double r;     // -rate / gpus
  uint64_t sk;  // config-key string order (lc_keys.h): combo rank << 36 | batch code
  int32_t unit; // global unit index, -1 = none
};

__device__ __forceinline__ PoolKey pool_key_of(const EvalParams& P, const lc_search_desc& S, double r, int32_t u) {
  return PoolKey{r, P.combo_rank[P.u_combo[u]] | P.batch_code[S.b_off + P.u_batch[u]], u};
}

// ---- K5a: top-k prefill / decode pool members per search
// sorted(pool, key=_pool_rank)[:cap] (search.py:276-277, 338-339): the order is
// (-rate/gpus, config-key string), and the stable sort keeps unit order for
// identical keys (duplicate batch values), so the total order is (r, key, unit).
constexpr int kPoolLocal = 32;  // caps up to 32 take the fast path (one list element per lane)
#ifndef LC_POOL_THREADS
#define LC_POOL_THREADS 256
#endif
constexpr int kPoolThreads = LC_POOL_THREADS;

__device__ __forceinline__ bool pool_before(const EvalParams& P, const PoolKey& a, const PoolKey& b) {
  if (a.unit < 0) return false;
  if (b.unit < 0) return true;
  if (a.r != b.r) return a.r < b.r;
  if (a.sk != b.sk) return a.sk < b.sk;
  return a.unit < b.unit;
}

// A sorted top-`cap` list held across a warp's registers: lane j holds element j
// (absent elements are {0, -1}, which sort last).  A chunk of up to 32 new keys
// is merged in one step -- a warp bitonic sort of the chunk, then the bitonic
// merge of the two sorted lists keeping the 32 smallest -- so a long run of
// improving keys (the pool rate per GPU grows along a combo's batch list) costs
// one merge per chunk, not one serial insertion per key.  No local memory.
__device__ __forceinline__ PoolKey shfl_key(const PoolKey& v, int src) {
  return PoolKey{__shfl_sync(0xffffffffu, v.r, src), (uint64_t)__shfl_sync(0xffffffffu, (unsigned long long)v.sk, src),
                 __shfl_sync(0xffffffffu, v.unit, src)};
}
__device__ __forceinline__ PoolKey shfl_xor_key(const PoolKey& v, int m) {
  return PoolKey{__shfl_xor_sync(0xffffffffu, v.r, m),
                 (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)v.sk, m),
                 __shfl_xor_sync(0xffffffffu, v.unit, m)};
}
// compare-exchange with the partner lane (lane ^ j): the lower lane keeps the
// earlier key when `ascending`, the later one otherwise
__device__ __forceinline__ void warp_cx(const EvalParams& P, PoolKey& v, int j, bool ascending) {
  const int lane = threadIdx.x & 31;
  const PoolKey o = shfl_xor_key(v, j);
  const bool lower = (lane & j) == 0;
  if (lower == ascending ? pool_before(P, o, v) : pool_before(P, v, o)) v = o;
}
__device__ __forceinline__ void warp_sort32(const EvalParams& P, PoolKey& v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) warp_cx(P, v, j, (lane & k) == 0);
}
// v: ascending list; w: ascending list; returns the 32 earliest of both, ascending
__device__ __forceinline__ PoolKey warp_merge32(const EvalParams& P, const PoolKey& v, const PoolKey& w) {
  const int lane = threadIdx.x & 31;
  const PoolKey wr = shfl_key(w, 31 - lane);
  PoolKey m = pool_before(P, wr, v) ? wr : v;  // bitonic: the 32 earliest of v ++ reverse(w)
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) warp_cx(P, m, j, true);
  return m;
}

struct WarpTopK {
  PoolKey mine;
  int n;
  __device__ __forceinline__ void init() { mine = PoolKey{0.0, 0, -1}; n = 0; }
  // key of the cap-th element once the list is full (INFINITY before): a new key
  // with a larger r cannot enter
  __device__ __forceinline__ double thr_r(int cap) const {
    return n < cap ? INFINITY : __shfl_sync(0xffffffffu, mine.r, cap - 1);
  }
  // merge one key per lane (unit < 0: none); warp-uniform call
  __device__ __forceinline__ void merge_chunk(const EvalParams& P, PoolKey x, int cap) {
    const int lane = threadIdx.x & 31;
    const int got = __popc(__ballot_sync(0xffffffffu, x.unit >= 0));
    if (!got) return;
    warp_sort32(P, x);
    mine = warp_merge32(P, mine, x);
    n = n + got < cap ? n + got : cap;
    if (lane >= cap) mine = PoolKey{0.0, 0, -1};
  }
  // merge another warp's sorted list (element j in lane j, `m` elements)
  __device__ __forceinline__ void merge_sorted(const EvalParams& P, const PoolKey& x, int m, int cap) {
    const int lane = threadIdx.x & 31;
    if (!m) return;
    mine = warp_merge32(P, mine, x);
    n = n + m < cap ? n + m : cap;
    if (lane >= cap) mine = PoolKey{0.0, 0, -1};
  }
};

// ---- K5b: replica sweep per pairing and plan sort (block per search)
struct PlanRec {
  int32_t p, d, x, y;  // p/d: global unit index
  int64_t gpus;
  double r_sys, ttft, tpot, speed, thru;
};

// K5b: replica sweep (serving_modes.py:468-488), a warp per pairing; the
// pairings of a search are spread over kDisSplit blocks
constexpr int kDisSplit = 16;
__device__ __forceinline__ void disagg_pools(const EvalParams& P, const lc_search_desc& S, const SearchMeta& M,
                                             const int32_t* pool_sel, int s, int32_t* pre, int32_t* dec, int* npre,
                                             int* ndec) {
  // top-k pools first, then the latency filters (search.py:338-339; serving_modes.py:458-466).
  // Called by the whole block: warp 0 filters the prefill pool, warp 1 the decode
  // pool, 32 candidates at a time, compacted in pool order with a ballot.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const int n = warp == 0 ? M.n_pre : M.n_dec;
    int32_t* out = warp == 0 ? pre : dec;
    int cnt = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      bool keep = false;
      int32_t u = -1;
      if (k < n) {
        u = pool_sel[(int64_t)s * 128 + warp * 64 + k];
        keep = warp == 0 ? (!S.has_ttft || P.pf_v[u] * S.ttft_headroom <= S.ttft_limit)
                         : (!S.has_floor || P.dc_v[u] <= S.tpot_cap);
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) out[cnt + __popc(m & ((1u << lane) - 1u))] = u;
      cnt += __popc(m);
    }
    if (lane == 0) *(warp == 0 ? npre : ndec) = cnt;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_disagg_pairs(EvalParams P, const SearchMeta* meta, const int32_t* pool_sel,
                                                      PlanRec* scratch) {
  const int s = blockIdx.x;
  const lc_search_desc& S = P.searches[s];
  if (!(S.modes & 4) || (S.modes & LC_MODE_NO_PLANS)) return;
  __shared__ int32_t pre[64], dec[64];
  __shared__ int npre, ndec;
  disagg_pools(P, S, meta[s], pool_sel, s, pre, dec, &npre, &ndec);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.y * (blockDim.x >> 5) + warp, nwarp = gridDim.y * (blockDim.x >> 5);
  const int npair = npre * ndec;
  PlanRec* plans = scratch + (int64_t)s * 256;
  for (int pi = gw; pi < npair && pi < 256; pi += nwarp) {
    const int32_t up = pre[pi / ndec], ud = dec[pi % ndec];
    const double rp = P.pf_v[P.n_cap + up], rd = P.dc_v[P.n_cap + ud];
    const int64_t gp = P.combos[P.u_combo[up]].gpus, gd = P.combos[P.u_combo[ud]].gpus;
    bool have = false;
    double bk = 0.0;
    int64_t bg = 0;
    int bx = 0, by = 0;
    for (int x = 1; x <= S.max_x; ++x) {
      const double r_pre = rp * (double)x * S.prefill_util;
      const int64_t g_pre = (int64_t)x * gp;
      for (int y = 1 + lane; y <= S.max_y; y += 32) {
        const int64_t gpus = g_pre + (int64_t)y * gd;
        if (!in_budget(S, gpus)) continue;
        const double r_dec = rd * (double)y * S.decode_util;
        const double r_sys = r_dec < r_pre ? r_dec : r_pre;
        const double k0 = -r_sys * (double)S.osl / (double)gpus;
        const bool better = !have || k0 < bk ||
                            (k0 == bk && (gpus < bg || (gpus == bg && (x < bx || (x == bx && y < by)))));
        if (better) { have = true; bk = k0; bg = gpus; bx = x; by = y; }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int oh = __shfl_xor_sync(0xffffffffu, (int)have, o);
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int64_t og = __shfl_xor_sync(0xffffffffu, bg, o);
      const int ox = __shfl_xor_sync(0xffffffffu, bx, o);
      const int oy = __shfl_xor_sync(0xffffffffu, by, o);
      const bool better = oh && (!have || ok < bk ||
                                 (ok == bk && (og < bg || (og == bg && (ox < bx || (ox == bx && oy < by))))));
      if (better) { have = true; bk = ok; bg = og; bx = ox; by = oy; }
    }
    if (lane == 0 && have) {
      PlanRec r;
      r.p = up; r.d = ud; r.x = bx; r.y = by;
      r.gpus = (int64_t)bx * gp + (int64_t)by * gd;
      const double r_pre = rp * (double)bx * S.prefill_util;
      const double r_dec = rd * (double)by * S.decode_util;
      r.r_sys = r_dec < r_pre ? r_dec : r_pre;
      r.ttft = P.pf_v[up] * S.ttft_headroom;
      r.tpot = P.dc_v[ud];
      r.speed = r.tpot == 0.0 ? INFINITY : 1000.0 / r.tpot;
      r.thru = r.r_sys * (double)S.osl / (double)r.gpus;
      // keep pairing order for the stable sort: slot = pairing index
      plans[pi] = r;
    }
    if (lane == 0 && !have) plans[pi].p = -1;
  }
}

// K5b': compact the pairings' plans in pairing order and rank them stably by
// (-thru, gpus, ttft, x, y) (serving_modes.py:424-427, 493); block per search
__global__ void __launch_bounds__(256) k_disagg(EvalParams P, SearchMeta* meta, const int32_t* pool_sel,
                                                const PlanRec* scratch, int32_t* plan_i, double* plan_d,
                                                lc_search_result* results) {
  const int s = blockIdx.x;
  const lc_search_desc& S = P.searches[s];
  __shared__ int32_t pre[64], dec[64];
  __shared__ int npre, ndec;
  __shared__ int nplan;
  if (!(S.modes & 4) || (S.modes & LC_MODE_NO_PLANS)) {
    if (threadIdx.x == 0) { meta[s].plan_cap = 0; results[s].n_plans = 0; }
    return;
  }
  disagg_pools(P, S, meta[s], pool_sel, s, pre, dec, &npre, &ndec);
  const int npair = npre * ndec;
  __shared__ PlanRec plans[256];
  for (int i = threadIdx.x; i < npair && i < 256; i += blockDim.x) plans[i] = scratch[(int64_t)s * 256 + i];
  __syncthreads();
  // compact in pairing order, then stable rank by (-thru, gpus, ttft, x, y)
  __shared__ int32_t order[256];
  {
    // ordered compaction: warp w owns pairings [32w, 32w + 32)
    __shared__ int wcnt[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = threadIdx.x;
    const bool keep = i < npair && i < 256 && plans[i].p >= 0;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wcnt[warp] = __popc(m);
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += wcnt[w];
    if (keep) order[base + __popc(m & ((1u << lane) - 1u))] = i;
    if (threadIdx.x == 255) nplan = base + __popc(m);
  }
  __syncthreads();
  const int32_t off = meta[s].plan_off;
  for (int i = threadIdx.x; i < nplan; i += blockDim.x) {
    const PlanRec& a = plans[order[i]];
    int rank = 0;
    for (int j = 0; j < nplan; ++j) {
      if (j == i) continue;
      const PlanRec& b = plans[order[j]];
      bool less;
      if (-b.thru != -a.thru) less = -b.thru < -a.thru;
      else if (b.gpus != a.gpus) less = b.gpus < a.gpus;
      else if (b.ttft != a.ttft) less = b.ttft < a.ttft;
      else if (b.x != a.x) less = b.x < a.x;
      else if (b.y != a.y) less = b.y < a.y;
      else less = j < i;
      rank += less;
    }
    const int64_t slot = off + rank;
    plan_i[slot * 4 + 0] = a.p; plan_i[slot * 4 + 1] = a.d; plan_i[slot * 4 + 2] = a.x; plan_i[slot * 4 + 3] = a.y;
    plan_d[slot * 6 + 0] = (double)a.gpus; plan_d[slot * 6 + 1] = a.r_sys; plan_d[slot * 6 + 2] = a.ttft;
    plan_d[slot * 6 + 3] = a.tpot; plan_d[slot * 6 + 4] = a.speed; plan_d[slot * 6 + 5] = a.thru;
    // plan rows in the per-search accounting (k_expand covers the other rows)
    if ((!S.has_ttft || a.ttft <= S.ttft_limit) && (!S.has_floor || a.speed >= S.speed_floor)) {
      SearchAcc* A = P.acc + s;
      atomicAdd(&A->feas, 1);
      atomicAdd(&A->fplans, 1);
      const unsigned long long bits = (unsigned long long)__double_as_longlong(a.speed);
      atomicMax(&A->smax, bits);
      atomicMax(&A->smin_c, ~bits);
      if (fixed_buckets(S)) bucket_max(P.fbuckets + (int64_t)s * kSpeedBuckets, S, a.speed, a.thru);
    }
  }
  if (threadIdx.x == 0) {
    results[s].n_plans = nplan;
    if (nplan) atomicAdd(&P.acc[s].rows, nplan);
  }
}

// ---- K4: feasibility, Pareto front, best, nearest miss (block per search)
struct RowView {
  bool valid;
  int mode;  // 0 static 1 aggregated 2 disaggregated
  double ttft, speed, thru;
  int64_t gpus;
  int64_t key;  // mode << 32 | index
};

__device__ __forceinline__ RowView get_row(const EvalParams& P, const SearchMeta& M, const int32_t* plan_i,
                                           const double* plan_d, int64_t nplan, int64_t r) {
  RowView v;
  v.valid = false;
  const int64_t nu = M.n_units;
  if (r < 2 * nu) {
    const int mode = r < nu ? 0 : 1;
    const int64_t i = mode ? r - nu : r;
    const int64_t u = M.unit_off + i;
    if (!P.u_budget[u]) return v;
    const int32_t* st = mode ? P.ag_status : P.st_status;
    const double* vv = mode ? P.ag_v : P.st_v;
    if (st[u] != 0) return v;
    v.valid = true;
    v.mode = mode;
    v.ttft = vv[u];
    v.speed = vv[2 * P.n_cap + u];
    v.thru = vv[3 * P.n_cap + u];
    v.gpus = -1;  // loaded on demand (row_gpus)
    v.key = ((int64_t)mode << 32) | i;
  } else {
    const int64_t i = r - 2 * nu;
    const int64_t slot = M.plan_off + i;
    v.valid = true;
    v.mode = 2;
    v.gpus = (int64_t)plan_d[slot * 6 + 0];
    v.ttft = plan_d[slot * 6 + 2];
    v.speed = plan_d[slot * 6 + 4];
    v.thru = plan_d[slot * 6 + 5];
    v.key = ((int64_t)2 << 32) | i;
  }
  return v;
}

__device__ __forceinline__ bool feasible(const lc_search_desc& S, const RowView& v) {
  if (S.has_ttft && v.ttft > S.ttft_limit) return false;
  return !S.has_floor || v.speed >= S.speed_floor;
}

__device__ int row_label(const EvalParams& P, const SearchMeta& M, const int32_t* plan_i, int64_t key, char* out) {
  const int mode = (int)(key >> 32);
  const int64_t i = key & 0xffffffffll;
  if (mode < 2) {
    const int64_t u = M.unit_off + i;
    const lc_search_desc& S = P.searches[P.u_search[u]];
    return fmt_cfg_key(out, P.combos[P.u_combo[u]], P.batches[S.b_off + P.u_batch[u]]);
  }
  const int64_t slot = M.plan_off + i;
  const int32_t up = plan_i[slot * 4 + 0], ud = plan_i[slot * 4 + 1];
  const lc_search_desc& S = P.searches[P.u_search[up]];
  int n = 0;
  n += put_str(out + n, "P:"); n += put_int(out + n, plan_i[slot * 4 + 2]); n += put_str(out + n, "x");
  n += fmt_cfg_key(out + n, P.combos[P.u_combo[up]], P.batches[S.b_off + P.u_batch[up]]);
  n += put_str(out + n, "|D:"); n += put_int(out + n, plan_i[slot * 4 + 3]); n += put_str(out + n, "x");
  n += fmt_cfg_key(out + n, P.combos[P.u_combo[ud]], P.batches[S.b_off + P.u_batch[ud]]);
  return n;
}

struct BestKey {
  double nthru, nspeed;
  int64_t gpus;
  int mode_rank;  // "aggregated" < "disaggregated" < "static"
  int64_t key;    // -1 none
};

__device__ __forceinline__ int mode_rank(int mode) { return mode == 1 ? 0 : (mode == 2 ? 1 : 2); }

__device__ bool best_less(const EvalParams& P, const SearchMeta& M, const int32_t* plan_i, const BestKey& a,
                          const BestKey& b) {
  if (a.key < 0) return false;
  if (b.key < 0) return true;
  if (a.nthru != b.nthru) return a.nthru < b.nthru;
  if (a.nspeed != b.nspeed) return a.nspeed < b.nspeed;
  // static / aggregated rows carry gpus = -1 until a tie needs it (plans always carry it)
  const int64_t ga = a.gpus >= 0 ? a.gpus : P.combos[P.u_combo[M.unit_off + (a.key & 0xffffffffll)]].gpus;
  const int64_t gb = b.gpus >= 0 ? b.gpus : P.combos[P.u_combo[M.unit_off + (b.key & 0xffffffffll)]].gpus;
  if (ga != gb) return ga < gb;
  if (a.mode_rank != b.mode_rank) return a.mode_rank < b.mode_rank;
  char la[200], lb[200];
  row_label(P, M, plan_i, a.key, la);
  row_label(P, M, plan_i, b.key, lb);
  const int c = str_cmp(la, lb);
  if (c) return c < 0;
  return a.key < b.key;
}

struct MissKey {
  double viol;
  int64_t key;
};

__device__ bool miss_less(const EvalParams& P, const SearchMeta& M, const int32_t* plan_i, const MissKey& a,
                          const MissKey& b) {
  if (a.key < 0) return false;
  if (b.key < 0) return true;
  if (a.viol != b.viol) return a.viol < b.viol;
  char la[200], lb[200];
  row_label(P, M, plan_i, a.key, la);
  row_label(P, M, plan_i, b.key, lb);
  const int c = str_cmp(la, lb);
  if (c) return c < 0;
  return a.key < b.key;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

struct FrontCand {
  double speed, thru;
  int64_t key;
};

constexpr int kSurvivorCap = 2048;  // front candidates kept in shared memory
#ifndef LC_FRONT_THREADS
#define LC_FRONT_THREADS 256
#endif
constexpr int kFrontThreads = LC_FRONT_THREADS;
#define FRONT_ROW_FILTER(v)                                                          \
  if (!v.valid) continue;                                                            \
  if ((v.mode == 0 && !(S.modes & 1)) || (v.mode == 1 && !(S.modes & 2))) continue;

// ---------------------------------------------------------------------------
// K5a and K4.  Each search's rows are spread over kSplit blocks (grid =
// kSplit x n_search) and small per-search kernels merge the partials.
// K4: (1) counts, select_best (search.py:179-187) and the range of feasible
// speeds; (2) per speed-bucket maximum throughput (buckets = top bits of the
// IEEE pattern, so bucket order is speed order); (3) a row can only be on the
// front if it beats the best throughput of every strictly faster bucket --
// those maxima are real rows that would dominate it -- so only such
// survivors go through the exact reference scan (search.py:156-176).
#ifndef LC_FRONT_SPLIT
#define LC_FRONT_SPLIT 64
#endif
#ifndef LC_POOL_SPLIT
#define LC_POOL_SPLIT 16
#endif
constexpr int kSplit = LC_FRONT_SPLIT;     // blocks per search for the Pareto passes
constexpr int kPoolSplit = LC_POOL_SPLIT;  // blocks per search for the pool top-k
constexpr int kCompactFront = 2048;  // fixed-stride copy of each front for one-shot D2H (= survivor cap)

struct PoolPartial {
  PoolKey k[2][kPoolLocal];
  int32_t n[2];
};

__device__ __forceinline__ void slice_of(int64_t n, int parts, int part, int64_t* lo, int64_t* hi) {
  *lo = n * part / parts;
  *hi = n * (part + 1) / parts;
}

// Seed thresholds for K5a: per (search, role), the cap-th smallest key r among
// the last unit of every (search, combo) pair -- written by k_eval_cells into
// pool_sample (closed-form K0 only).  The pool rate per GPU grows along a combo's
// batch list, so these are nearly the search's best keys.  Any cap units with
// r <= T leave no room in the top-k for a unit with r > T, so the cap-th smallest
// sampled r bounds the search's cap-th from above (ties are kept: r <= T passes).
// One warp per (search, role): a sorted 32-list of doubles, bitonic merges.
__device__ __forceinline__ double warp_sort32_d(double v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v, j);
      const bool lower = (lane & j) == 0, asc = (lane & k) == 0;
      v = (lower == asc) ? fmin(v, o) : fmax(v, o);
    }
  return v;
}
// 32 smallest of two ascending warp lists (bitonic merge of a with reversed b)
__device__ __forceinline__ double warp_merge32_d(double a, double b) {
  const int lane = threadIdx.x & 31;
  double m = fmin(a, __shfl_sync(0xffffffffu, b, 31 - lane));
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, m, j);
    m = (lane & j) == 0 ? fmin(m, o) : fmax(m, o);
  }
  return m;
}
// block per (search, role): 8 warps take every 8th chunk of 32 combos, then the
// warps' ascending 32-lists are merged as a tree in shared memory
constexpr int kSeedThreads = 256;
// doubles as order-preserving unsigned keys (k_pools_seed / k_pools_partial share
// each search's pool threshold through atomicMin on these)
__device__ __forceinline__ unsigned long long ord_key(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}
__global__ void __launch_bounds__(kSeedThreads) k_pools_seed(EvalParams P, unsigned long long* seed) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kSeedThreads / 32;
  const int s = blockIdx.x >> 1, role = blockIdx.x & 1;
  __shared__ double lists[kSeedThreads / 32][32];
  const lc_search_desc& S = P.searches[s];
  const int cap = role == 0 ? S.prefill_cap : S.decode_cap;
  const bool on = (S.modes & 4) && cap > 0 && cap <= kPoolLocal;  // block-uniform
  double best = INFINITY;  // lane j: the j-th smallest so far (ascending)
  if (on) {
    const int32_t* po = P.pair_off + (int64_t)s * P.sp_n_combos;
    const double* smp = P.pool_sample + (int64_t)s * P.sp_n_combos * 2 + role;
    for (int c0 = warp * 32; c0 < P.sp_n_combos; c0 += nw * 32) {
      const int c = c0 + lane;
      double r = INFINITY;
      if (c < P.sp_n_combos && po[c + 1] > po[c]) {
        r = smp[2 * c];
        if (!(r <= INFINITY)) r = INFINITY;  // NaN keys never enter a pool (k_pools_partial)
      }
      if (!__any_sync(0xffffffffu, r != INFINITY)) continue;
      best = warp_merge32_d(best, warp_sort32_d(r));
    }
  }
  lists[warp][lane] = best;
  __syncthreads();
  for (int width = nw / 2; width >= 1; width >>= 1) {
    if (warp < width) best = warp_merge32_d(best, lists[warp + width][lane]);
    __syncthreads();
    if (warp < width) lists[warp][lane] = best;
    __syncthreads();
  }
  if (threadIdx.x == 0) seed[2 * s + role] = ord_key(on ? lists[0][cap - 1] : INFINITY);
}

__global__ void __launch_bounds__(kPoolThreads) k_pools_partial(EvalParams P, const SearchMeta* meta,
                                                                 PoolPartial* part, unsigned long long* seed) {
  const int s = blockIdx.y, bx = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const lc_search_desc& S = P.searches[s];
  if (!(S.modes & 4)) return;
  constexpr int kWarps = kPoolThreads / 32;
  __shared__ PoolKey wout[kWarps][kPoolLocal];
  __shared__ int wn[kWarps];
  int64_t lo, hi;
  slice_of(meta[s].n_units, kPoolSplit, bx, &lo, &hi);
  const int64_t u0 = meta[s].unit_off;
  PoolPartial* dst = part + (int64_t)s * kPoolSplit + bx;
  for (int role = 0; role < 2; ++role) {
    const int cap = role == 0 ? S.prefill_cap : S.decode_cap;
    if (cap > kPoolLocal || cap <= 0) { if (tid == 0) dst->n[role] = 0; continue; }
    const double* keys = P.pool_key + (int64_t)role * P.n_cap;
    WarpTopK tk;
    tk.init();
    // warp-strided chunks of 32 consecutive units (coalesced); a key can enter only if
    // not after the current cap-th element (r <= thr; exact order in the merge).  The
    // threshold starts at the search's seed (k_pools_seed): with it most chunks hold
    // no candidate and cost one coalesced load.
    // Any block's cap-th smallest key bounds the search's cap-th from above (cap
    // units are at or before it), so the blocks of a search share their
    // thresholds: atomicMin after each merge, re-read every few chunks.
    unsigned long long* shared_thr = seed ? seed + 2 * s + role : nullptr;
    double thr = shared_thr ? ord_val(*shared_thr) : INFINITY;
    int since = 0;
    // the next chunk's keys are loaded before this chunk is tested (one merge site:
    // unrolled copies of the merge code measured slower)
    const int64_t step = kPoolThreads;
    int64_t base = lo + (int64_t)warp * 32;
    double r_next = base + lane < hi ? keys[u0 + base + lane] : INFINITY;
    for (; base < hi; base += step) {
      const double r = r_next;  // INFINITY: pool candidate skipped
      const int64_t nb = base + step + lane;
      r_next = nb < hi ? keys[u0 + nb] : INFINITY;
#ifdef LC_COUNT_MERGES
      if ((threadIdx.x & 31) == 0) atomicAdd(P.cell_ctr, 1ull);
#endif
      if (shared_thr && ++since == 8) {
        since = 0;
        thr = fmin(thr, ord_val(*(volatile unsigned long long*)shared_thr));
      }
      const bool cand = r != INFINITY && r <= thr;
      if (!__any_sync(0xffffffffu, cand)) continue;
      const int64_t i = base + lane;
#ifdef LC_COUNT_MERGES  // diagnostics build: merges and chunks scanned
      if ((threadIdx.x & 31) == 0) atomicAdd(P.cell_ctr, 1ull << 32);
#endif
      tk.merge_chunk(P, cand ? pool_key_of(P, S, r, (int32_t)(u0 + i)) : PoolKey{0.0, 0, -1}, cap);
      const double mine = tk.thr_r(cap);
      if (mine < thr) {
        thr = mine;
        if (shared_thr && lane == 0) atomicMin(shared_thr, ord_key(mine));
      }
    }
    wout[warp][lane] = tk.mine;
    if (lane == 0) wn[warp] = tk.n;
    __syncthreads();
    // the warps' lists merged as a tree
    for (int width = kWarps / 2; width >= 1; width >>= 1) {
      if (warp < width) tk.merge_sorted(P, wout[warp + width][lane], wn[warp + width], cap);
      __syncthreads();
      if (warp < width) {
        wout[warp][lane] = tk.mine;
        if (lane == 0) wn[warp] = tk.n;
      }
      __syncthreads();
    }
    if (warp == 0) {
      if (lane < tk.n) dst->k[role][lane] = tk.mine;
      if (lane == 0) dst->n[role] = tk.n;
    }
    __syncthreads();
  }
}

// Per search: the kPoolSplit partial top-k lists of each role merged as a tree
// (8 warps per role: 2 partials each, then 4 -> 2 -> 1), 5 dependent merges
// instead of 16 per role; the top-k under the strict total order does not
// depend on the merge order.
constexpr int kPoolFinalThreads = 512;
static_assert(kPoolSplit == 16, "k_pools_final's merge tree assumes 16 partials per search");
__global__ void __launch_bounds__(kPoolFinalThreads) k_pools_final(EvalParams P, SearchMeta* meta,
                                                                   const PoolPartial* part, int32_t* pool_sel) {
  const int s = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef LC_COUNT_MERGES
  if (s == 0 && tid == 0)
    printf("k_pools_partial: %llu chunk merges of %llu chunks scanned\n", *P.cell_ctr >> 32,
           *P.cell_ctr & 0xffffffffull);
#endif
  const lc_search_desc& S = P.searches[s];
  if (!(S.modes & 4)) return;
  __shared__ PoolKey red[kPoolFinalThreads];
  __shared__ PoolKey lists[2][8][32];
  __shared__ int ln[2][8];
  {
    const int role = warp >> 3, w = warp & 7;
    const int cap = role == 0 ? S.prefill_cap : S.decode_cap;
    const bool small = cap <= kPoolLocal;  // uniform per role
    WarpTopK t;
    t.init();
    if (small) {
      for (int b = 2 * w; b < 2 * w + 2; ++b) {
        const PoolPartial& pp = part[(int64_t)s * kPoolSplit + b];
        const int m = pp.n[role];
        t.merge_sorted(P, lane < m ? pp.k[role][lane] : PoolKey{0.0, 0, -1}, m, cap);
      }
      lists[role][w][lane] = t.mine;
      if (lane == 0) ln[role][w] = t.n;
    }
    __syncthreads();
    for (int width = 4; width >= 1; width >>= 1) {
      if (small && w < width) t.merge_sorted(P, lists[role][w + width][lane], ln[role][w + width], cap);
      __syncthreads();
      if (small && w < width) {
        lists[role][w][lane] = t.mine;
        if (lane == 0) ln[role][w] = t.n;
      }
      __syncthreads();
    }
    if (small && w == 0) {
      if (lane < t.n) pool_sel[(int64_t)s * 128 + role * 64 + lane] = t.mine.unit;
      if (lane == 0) {
        if (role == 0) meta[s].n_pre = t.n;
        else meta[s].n_dec = t.n;
      }
    }
  }
  for (int role = 0; role < 2; ++role) {
    const int cap = role == 0 ? S.prefill_cap : S.decode_cap;
    if (cap <= kPoolLocal) continue;
    int got = 0;
    // large caps (33..64): rounds over all units (rare)
    const int32_t u0 = meta[s].unit_off, nu = meta[s].n_units;
    const double* keys = P.pool_key + (int64_t)role * P.n_cap;
    PoolKey prev{0.0, 0, -1};
    for (int k = 0; k < cap && k < 64; ++k) {
      PoolKey best{0.0, 0, -1};
      for (int i = tid; i < nu; i += blockDim.x) {
        const int32_t u = u0 + i;
        const double r = keys[u];
        if (r == INFINITY) continue;
        const PoolKey key = pool_key_of(P, S, r, u);
        if (prev.unit >= 0 && !pool_before(P, prev, key)) continue;
        if (pool_before(P, key, best)) best = key;
      }
      red[tid] = best;
      __syncthreads();
      for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (tid < w && pool_before(P, red[tid + w], red[tid])) red[tid] = red[tid + w];
        __syncthreads();
      }
      const PoolKey sel = red[0];
      __syncthreads();
      if (sel.unit < 0) break;
      if (tid == 0) pool_sel[(int64_t)s * 128 + role * 64 + k] = sel.unit;
      prev = sel;
      ++got;
    }
    if (tid == 0) {
      if (role == 0) meta[s].n_pre = got;
      else meta[s].n_dec = got;
    }
    __syncthreads();
  }
}


struct FrontMeta {
  int32_t shift, any;
  unsigned long long base;
  int32_t fixed, _pad;  // fixed: buckets from the speed floor, filled while the rows were written
};

__global__ void __launch_bounds__(kFrontThreads) k_front_mid(EvalParams P, const SearchMeta* meta,
                                                             const int32_t* plan_i, const double* plan_d,
                                                             lc_search_result* results,
                                                             FrontMeta* fmeta, unsigned long long* buckets,
                                                             int32_t* n_surv) {
  const int s = blockIdx.x, tid = threadIdx.x;
  const lc_search_desc& S = P.searches[s];
  const SearchMeta& M = meta[s];
  __shared__ MissKey mred[kFrontThreads];
  (void)buckets;  // zeroed at the start of the pipeline; fixed-geometry searches are filled by now
  if (tid == 0) {
    const SearchAcc A = P.acc[s];  // k_expand + k_disagg
    const unsigned long long lo = ~A.smin_c, hi = A.smax, q1 = A.q1, q2 = A.q2;
    const int feas = A.feas, rows = A.rows, enums = A.enums, skips = A.skips, fplans = A.fplans;
    const BestKey best{0, 0, 0, 0, -1};  // select_best: from the front, in k_front_final
    lc_search_result& R = results[s];
    R.n_enumerated = enums; R.n_rows = rows; R.n_feasible = feas; R.n_skipped = skips;
    R.n_feasible_plans = fplans;
    R.queries_1d = (int64_t)q1; R.queries_2d = (int64_t)q2;
    R.best = best.key;
    R.best_thru = best.key >= 0 ? -best.nthru : 0.0;
    R.best_speed = best.key >= 0 ? -best.nspeed : 0.0;
    R.nearest = -1;
    R.nearest_violation = 0.0;
    R.front_off = (int32_t)((int64_t)M.unit_off * 2 + M.plan_off);
    R.n_front = 0;
    const bool fixed = fixed_buckets(S);
    int shift = 0;
    if (fixed) shift = kFixedShift;
    else if (feas) while (shift < 63 && ((hi >> shift) - (lo >> shift)) >= (unsigned long long)kSpeedBuckets) ++shift;
    fmeta[s].shift = shift;
    fmeta[s].any = feas > 0;
    fmeta[s].fixed = fixed;
    fmeta[s].base = fixed ? ((unsigned long long)__double_as_longlong(S.speed_floor)) >> kFixedShift
                          : (feas ? (lo >> shift) : 0ull);
    n_surv[s] = 0;
  }
  __syncthreads();
  if (fmeta[s].any) return;
  // nearest miss (search.py:190-208) when nothing is feasible: rare, one block
  const int64_t nplan = results[s].n_plans;
  const int64_t nrows_all = 2 * (int64_t)M.n_units + nplan;
  MissKey miss{0, -1};
  for (int64_t r = tid; r < nrows_all; r += blockDim.x) {
    const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
    FRONT_ROW_FILTER(v)
    double worst = 1.0;
    if (S.has_ttft && v.ttft > S.ttft_limit) { const double x = v.ttft / S.ttft_limit; if (x > worst) worst = x; }
    if (S.has_floor && v.speed < S.speed_floor) {
      const double x = v.speed == 0.0 ? INFINITY : S.speed_floor / v.speed;
      if (x > worst) worst = x;
    }
    if (miss.key < 0 || worst <= miss.viol) {
      MissKey mk{worst, v.key};
      if (miss_less(P, M, plan_i, mk, miss)) miss = mk;
    }
  }
  mred[tid] = miss;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (tid < w && miss_less(P, M, plan_i, mred[tid + w], mred[tid])) mred[tid] = mred[tid + w];
    __syncthreads();
  }
  if (tid == 0) { results[s].nearest = mred[0].key; results[s].nearest_violation = mred[0].viol; }
}

__global__ void __launch_bounds__(kFrontThreads) k_front_pass2(EvalParams P, const SearchMeta* meta,
                                                               const int32_t* plan_i, const double* plan_d,
                                                               const lc_search_result* results, const FrontMeta* fmeta,
                                                               unsigned long long* buckets) {
  const int s = blockIdx.y, bx = blockIdx.x, tid = threadIdx.x;
  const FrontMeta fm = fmeta[s];
  if (!fm.any || fm.fixed) return;  // fixed geometry: filled while the rows were written
  const lc_search_desc& S = P.searches[s];
  const SearchMeta& M = meta[s];
  const int64_t nplan = results[s].n_plans;
  const int64_t nrows_all = 2 * (int64_t)M.n_units + nplan;
  unsigned long long* bk = buckets + (int64_t)s * kSpeedBuckets;
  int64_t lo, hi;
  slice_of(nrows_all, kSplit, bx, &lo, &hi);
  for (int64_t r = lo + tid; r < hi; r += blockDim.x) {
    const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
    FRONT_ROW_FILTER(v)
    if (!feasible(S, v)) continue;
    const int b = (int)((((unsigned long long)__double_as_longlong(v.speed)) >> fm.shift) - fm.base);
    atomicMax(&bk[b], (unsigned long long)__double_as_longlong(v.thru));
  }
}

__global__ void __launch_bounds__(kFrontThreads) k_front_suffix(const FrontMeta* fmeta, unsigned long long* buckets) {
  const int s = blockIdx.x, tid = threadIdx.x;
  if (!fmeta[s].any) return;
  unsigned long long* bk = buckets + (int64_t)s * kSpeedBuckets;
  // exclusive suffix maximum: per-thread runs of `per` buckets, then a warp
  // shuffle scan and a scan over the warps' maxima for the part above
  __shared__ unsigned long long wmax[kFrontThreads / 32];
  constexpr int per = kSpeedBuckets / kFrontThreads;
  const int lane = tid & 31, w = tid >> 5;
  unsigned long long loc[per];
  unsigned long long run = 0;
#pragma unroll
  for (int j = per - 1; j >= 0; --j) { loc[j] = run; const unsigned long long x = bk[tid * per + j]; run = x > run ? x : run; }
  unsigned long long inc = run;  // inclusive suffix max over lanes >= lane
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_down_sync(0xffffffffu, inc, o);
    if (lane + o < 32) inc = y > inc ? y : inc;
  }
  if (lane == 0) wmax[w] = inc;
  unsigned long long above = __shfl_down_sync(0xffffffffu, inc, 1);
  if (lane == 31) above = 0;
  __syncthreads();
  for (int v = w + 1; v < kFrontThreads / 32; ++v) above = wmax[v] > above ? wmax[v] : above;
#pragma unroll
  for (int j = 0; j < per; ++j) bk[tid * per + j] = loc[j] > above ? loc[j] : above;
}

__global__ void __launch_bounds__(kFrontThreads) k_front_pass3(EvalParams P, const SearchMeta* meta,
                                                               const int32_t* plan_i, const double* plan_d,
                                                               const lc_search_result* results, const FrontMeta* fmeta,
                                                               const unsigned long long* buckets, FrontCand* surv,
                                                               int32_t* n_surv) {
  const int s = blockIdx.y, bx = blockIdx.x, tid = threadIdx.x;
  const FrontMeta fm = fmeta[s];
  if (!fm.any) return;
  const lc_search_desc& S = P.searches[s];
  const SearchMeta& M = meta[s];
  const int64_t nplan = results[s].n_plans;
  const unsigned long long* bk = buckets + (int64_t)s * kSpeedBuckets;
  auto test = [&](double speed, double thru, int64_t key) {
    const int b = fm.fixed ? fixed_bucket(S, speed)
                           : (int)((((unsigned long long)__double_as_longlong(speed)) >> fm.shift) - fm.base);
    if (bk[b] != 0ull && thru <= __longlong_as_double((long long)bk[b])) return;
    const int k = atomicAdd(&n_surv[s], 1);
    if (k < P.surv_cap) surv[(int64_t)s * kSurvivorCap + k] = FrontCand{speed, thru, key};
  };
  // unit rows: the feasibility byte written with the rows (expand_unit) -- only the
  // feasible rows' speed and throughput are read
  int64_t lo, hi;
  slice_of(M.n_units, kSplit, bx, &lo, &hi);
  int f_next = lo + tid < hi ? P.front_flags[M.unit_off + lo + tid] : 0;
  for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
    const int64_t u = M.unit_off + i;
    const int f = f_next;  // loaded one iteration ahead
    f_next = i + blockDim.x < hi ? P.front_flags[u + blockDim.x] : 0;
    if (!f) continue;
    if (f & 1) test(P.st_v[2 * P.n_cap + u], P.st_v[3 * P.n_cap + u], i);
    if (f & 2) test(P.ag_v[2 * P.n_cap + u], P.ag_v[3 * P.n_cap + u], ((int64_t)1 << 32) | i);
  }
  // plan rows
  slice_of(nplan, kSplit, bx, &lo, &hi);
  for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
    const RowView v = get_row(P, M, plan_i, plan_d, nplan, 2 * (int64_t)M.n_units + i);
    if (!feasible(S, v)) continue;
    test(v.speed, v.thru, v.key);
  }
}

#ifndef LC_FINAL_THREADS
#define LC_FINAL_THREADS 512
#endif
constexpr int kFinalThreads = LC_FINAL_THREADS;
__global__ void __launch_bounds__(kFinalThreads) k_front_final(EvalParams P, const SearchMeta* meta,
                                                               const int32_t* plan_i, const double* plan_d,
                                                               lc_search_result* results, const FrontMeta* fmeta,
                                                               const FrontCand* surv, const int32_t* n_surv,
                                                               int64_t* front, int64_t* compact) {
  const int s = blockIdx.x, tid = threadIdx.x;
  if (!fmeta[s].any) return;
  extern __shared__ __align__(16) unsigned char fsm2[];
  FrontCand* sorted = (FrontCand*)fsm2;                     // kSurvivorCap
  FrontCand* staged = sorted + kSurvivorCap;                // kSurvivorCap
  int64_t* keys_out = (int64_t*)(staged + kSurvivorCap);    // kSurvivorCap
  __shared__ double dred[32];
  __shared__ int nfront, nlvl;
  const lc_search_desc& S = P.searches[s];
  const SearchMeta& M = meta[s];
  const int64_t nplan = results[s].n_plans;
  const int64_t nrows_all = 2 * (int64_t)M.n_units + nplan;
  const int64_t foff = (int64_t)M.unit_off * 2 + M.plan_off;
  const int nsv = n_surv[s];
  if (tid == 0) results[s].n_survivors = nsv;
  if (nsv <= P.surv_cap) {
    // bitonic sort of the survivors by (speed desc, row key asc), padded to a power of two
    const FrontCand* svg = surv + (int64_t)s * kSurvivorCap;
    int np2 = 1;
    while (np2 < nsv) np2 <<= 1;
    for (int i = tid; i < np2; i += blockDim.x)
      sorted[i] = i < nsv ? svg[i] : FrontCand{-INFINITY, 0.0, INT64_MAX};
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < np2; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const FrontCand a = sorted[i], b = sorted[l];
            const bool a_first = (a.speed > b.speed) || (a.speed == b.speed && a.key < b.key);
            const bool up = (i & k) == 0;
            if (up != a_first) { sorted[i] = b; sorted[l] = a; }
          }
        }
        // a distance below 32 pairs elements of one warp (i = tid + r * blockDim):
        // a warp barrier suffices unless this or the next substep crosses warps
        const int jn = j > 1 ? j >> 1 : k;  // the next substep's distance
        if (j >= 32 || jn >= 32) __syncthreads();
        else __syncwarp();
      }
    }
    __syncthreads();
    // group maxima and the running maximum of all faster rows, in parallel
    // inclusive prefix max of thru over sorted order: runs of consecutive elements
    // per thread, a warp shuffle scan and a scan over the warps' maxima
    double* pm = (double*)staged;
    {
      __shared__ double wmx[kFinalThreads / 32];
      const int lane = tid & 31, wid = tid >> 5;
      const int per = (nsv + (int)blockDim.x - 1) / (int)blockDim.x;
      const int a0 = tid * per, a1 = a0 + per < nsv ? a0 + per : nsv;
      double run = -INFINITY;
      for (int i = a0; i < a1; ++i) run = fmax(run, sorted[i].thru);
      double inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = fmax(inc, y);
      }
      if (lane == 31) wmx[wid] = inc;
      double ex = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) ex = -INFINITY;
      __syncthreads();
      for (int w = 0; w < wid; ++w) ex = fmax(ex, wmx[w]);
      for (int i = a0; i < a1; ++i) {
        ex = fmax(ex, sorted[i].thru);
        pm[i] = ex;
      }
      __syncthreads();
    }
    int* flag = (int*)keys_out;  // front membership, then output positions
    for (int i = tid; i < nsv; i += blockDim.x) {
      int g0 = i;
      while (g0 > 0 && sorted[g0 - 1].speed == sorted[i].speed) --g0;
      int g1 = i;
      while (g1 + 1 < nsv && sorted[g1 + 1].speed == sorted[i].speed) ++g1;
      double top = -INFINITY;
      for (int j = g0; j <= g1; ++j) top = fmax(top, sorted[j].thru);
      const double faster = g0 > 0 ? pm[g0 - 1] : -INFINITY;
      flag[i] = (sorted[i].thru == top && top > faster) ? 1 : 0;
    }
    __syncthreads();
    // select_best (search.py:179-187) on the front, where the best row always is:
    // highest throughput, then highest speed (block maxima), then the full key
    double tmax = -INFINITY;
    for (int i = tid; i < nsv; i += blockDim.x)
      if (flag[i]) tmax = fmax(tmax, sorted[i].thru);
    tmax = block_max(tmax, dred);
    double smax = -INFINITY;
    for (int i = tid; i < nsv; i += blockDim.x)
      if (flag[i] && sorted[i].thru == tmax) smax = fmax(smax, sorted[i].speed);
    smax = block_max(smax, dred);
    // ordered compaction of the front rows: contiguous runs per thread + block scan
    const int per = (nsv + (int)blockDim.x - 1) / (int)blockDim.x;
    const int i0 = tid * per, i1 = i0 + per < nsv ? i0 + per : nsv;
    int cnt = 0;
    for (int i = i0; i < i1; ++i) cnt += flag[i];
    __shared__ int wsum[kFinalThreads / 32];
    const int lane = tid & 31, wid = tid >> 5;
    const int wex = warp_excl_scan(cnt, lane);
    if (lane == 31) wsum[wid] = wex + cnt;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wid; ++w) base += wsum[w];
    int pos = base + wex;
    BestKey best{0, 0, 0, 0, -1};
    for (int i = i0; i < i1; ++i) {
      if (!flag[i]) continue;
      const int64_t key = sorted[i].key;
      front[foff + pos] = key;
      compact[(int64_t)s * kCompactFront + pos] = key;
      ++pos;
      if (sorted[i].thru != tmax || sorted[i].speed != smax) continue;
      const int mode = (int)(key >> 32);
      const BestKey k{-sorted[i].thru, -sorted[i].speed,
                      mode == 2 ? (int64_t)plan_d[(M.plan_off + (key & 0xffffffffll)) * 6 + 0] : -1,
                      mode_rank(mode), key};
      if (best_less(P, M, plan_i, k, best)) best = k;
    }
    // tied candidates are rare: warp leaders collect, thread 0 picks by the full key
    __shared__ BestKey wbest[kFinalThreads];
    wbest[tid] = best;
    __syncthreads();
    if (tid < 32) {
      // warp 0 finds the threads holding a candidate by ballots; lane 0 compares them
      for (int base = 0; base < (int)blockDim.x; base += 32) {
        unsigned m = __ballot_sync(0xffffffffu, wbest[base + tid].key >= 0);
        if (tid == 0) {
          while (m) {
            const int t = base + __ffs(m) - 1;
            m &= m - 1;
            if (best_less(P, M, plan_i, wbest[t], best)) best = wbest[t];
          }
        }
      }
    }
    if (tid == 0) {
      int m = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m += wsum[w];
      results[s].n_front = m;
      results[s].best = best.key;
      results[s].best_thru = best.key >= 0 ? -best.nthru : 0.0;
      results[s].best_speed = best.key >= 0 ? -best.nspeed : 0.0;
    }
    return;
  }
  // survivor overflow: iterative staircase over all rows (one block)
  BestKey obest{0, 0, 0, 0, -1};
  if (tid == 0) nfront = 0;
  __syncthreads();
  double best_thru = -INFINITY;
  while (true) {
    double sm = -INFINITY;
    bool any = false;
    for (int64_t r = tid; r < nrows_all; r += blockDim.x) {
      const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
      FRONT_ROW_FILTER(v)
      if (!feasible(S, v)) continue;
      if (v.thru > best_thru) { any = true; sm = fmax(sm, v.speed); }
    }
    if (!__syncthreads_or(any)) break;
    const double sp = block_max(any ? sm : -INFINITY, dred);
    double tmax = -INFINITY;
    for (int64_t r = tid; r < nrows_all; r += blockDim.x) {
      const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
      FRONT_ROW_FILTER(v)
      if (!feasible(S, v)) continue;
      if (v.speed == sp) tmax = fmax(tmax, v.thru);
    }
    const double top = block_max(tmax, dred);
    // this level's rows (speed sp, throughput top), collected in parallel and
    // emitted in row order (row order is key order); a level with more ties
    // than the buffer holds is emitted by one thread scanning the rows
    int64_t* lvl = (int64_t*)fsm2;  // the fast path's sort buffers are free here
    constexpr int kLevelCap = 8192;  // a power of two (the sort pads to one) within the 112 KB buffer
    static_assert(kLevelCap * sizeof(int64_t) <= (2 * sizeof(FrontCand) + 8) * kSurvivorCap, "level buffer");
    if (tid == 0) nlvl = 0;
    __syncthreads();
    for (int64_t r = tid; r < nrows_all; r += blockDim.x) {
      const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
      FRONT_ROW_FILTER(v)
      if (!feasible(S, v)) continue;
      if (v.speed == sp && v.thru == top) {
        const int k = atomicAdd(&nlvl, 1);
        if (k < kLevelCap) lvl[k] = v.key;
      }
    }
    __syncthreads();
    const int nl = nlvl;
    if (nl <= kLevelCap) {
      int np2 = 1;
      while (np2 < nl) np2 <<= 1;
      for (int i = nl + tid; i < np2; i += blockDim.x) lvl[i] = INT64_MAX;
      __syncthreads();
      for (int k = 2; k <= np2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < np2; i += blockDim.x) {
            const int l = i ^ j;
            if (l > i) {
              const int64_t a = lvl[i], b = lvl[l];
              if (((i & k) == 0) == (a > b)) { lvl[i] = b; lvl[l] = a; }
            }
          }
          __syncthreads();
        }
      if (tid == 0) {
        for (int i = 0; i < nl; ++i) {
          const int64_t key = lvl[i];
          const int mode = (int)(key >> 32);
          if (nfront < kCompactFront) compact[(int64_t)s * kCompactFront + nfront] = key;
          front[foff + nfront++] = key;
          const int64_t g = mode == 2 ? (int64_t)plan_d[(M.plan_off + (key & 0xffffffffll)) * 6 + 0] : -1;
          const BestKey k{-top, -sp, g, mode_rank(mode), key};
          if (best_less(P, M, plan_i, k, obest)) obest = k;
        }
      }
    } else if (tid == 0) {
      for (int64_t r = 0; r < nrows_all; ++r) {
        const RowView v = get_row(P, M, plan_i, plan_d, nplan, r);
        FRONT_ROW_FILTER(v)
        if (!feasible(S, v)) continue;
        if (v.speed == sp && v.thru == top) {
          if (nfront < kCompactFront) compact[(int64_t)s * kCompactFront + nfront] = v.key;
          front[foff + nfront++] = v.key;
          const BestKey k{-v.thru, -v.speed, v.gpus, mode_rank(v.mode), v.key};
          if (best_less(P, M, plan_i, k, obest)) obest = k;
        }
      }
    }
    __syncthreads();
    best_thru = top;
  }
  if (tid == 0) {
    results[s].n_front = nfront;
    results[s].best = obest.key;
    results[s].best_thru = obest.key >= 0 ? -obest.nthru : 0.0;
    results[s].best_speed = obest.key >= 0 ? -obest.nspeed : 0.0;
  }
}

}  // namespace

template <class T>
static int upload(T** dst, const T* src, size_t n, cudaStream_t st) {
  size_t bytes = n * sizeof(T);
  CK(cudaMalloc((void**)dst, bytes ? bytes : 16));
  if (bytes) CK(cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st));
  return LC_OK;
}

struct StepView {  // what k_step reads of a space plan
  const lc_entry* entries;
  const int32_t* tmpl_n;
  const TmplInfo* tmpl_info;
  int64_t hidden, topk, n_experts;
  int32_t is_moe, n_tmpl;
};

// get_step_latency (estimator.py:71-110), one warp per request: the expert-tail
// token count (busiest EP shard, a warp apportionment), then the plan entries
// across the lanes -- coordinates (decompose, model.py:302-404), latency
// (query_latency), 0.0 + ms * bubble -- and lane 0 sums them in plan order with
// CPython's float sum; the first failing entry in plan order decides the error.
template <int PER>
__global__ void __launch_bounds__(128) k_step(DbView V, StepView T, int32_t n, const lc_step_req* __restrict__ reqs,
                                              const double* __restrict__ loads, lc_step_out* __restrict__ out) {
  __shared__ int hist_all[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; r < n; r += nw) {
    const lc_step_req R = reqs[r];
    const TmplInfo ti = T.tmpl_info[R.tmpl];
    const int64_t tokens = R.n_ctx + R.n_gen;
    int64_t xt = 0;
    if (T.is_moe) {  // _skewed_expert_tokens (estimator.py:58-68)
      const int64_t f = ti.ep / ti.tp > 1 ? ti.ep / ti.tp : 1;
      const int64_t pooled = tokens * f;
      xt = ceil_div_f(pooled * T.topk, ti.ep);
      if (ti.ep > 1 && R.load >= 0) {
        const int E = (int)T.n_experts;
        const double* q = loads + (int64_t)R.load * 2 * E;
        const int64_t tail = warp_busiest_shard<PER>(q, q + E, E, pooled, T.topk, ti.ep, hist_all[warp]);
        xt = tail > xt ? tail : xt;
      }
    }
    const StepArgs a{R.phase, R.n_ctx, R.n_gen, R.seq, xt};
    const int ne = T.tmpl_n[R.tmpl];
    const int64_t mb = R.batch > 1 ? R.batch : 1;
    const double bubble = (double)(mb + ti.pp - 1) / (double)mb;  // pipeline_bubble (estimator.py:45-48)
    double val = 0.0;
    int st = 0, label = -1;
    int64_t d[5] = {0, 0, 0, 0, 0};
    if (lane < ne) {
      const lc_entry e = T.entries[(int64_t)R.tmpl * LC_MAX_ENTRIES + lane];
      if (entry_coords(e, a, T.hidden, d)) {
        label = e.label;
        int nlog = 0;
        const double lat = query_body<true>(V, e.grid, e.kind, e.quant, d[0], d[1], d[2], d[3], d[4], &st, &nlog);
        val = 0.0 + div1000(lat * (double)e.repeat) * bubble;
      }
    }
    lc_step_out* o = out + r;
    if (lane < LC_MAX_ENTRIES) {
      o->entry_ms[lane] = st ? 0.0 : val;
      o->entry_label[lane] = lane < ne ? label : -1;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, label >= 0 && st != 0);
    if (bad) {  // the first failing entry in plan order raises (query_latency)
      const int src = __ffs(bad) - 1;
      const int bst = __shfl_sync(0xffffffffu, st, src);
      const int blb = __shfl_sync(0xffffffffu, label, src);
      const int64_t c0 = __shfl_sync(0xffffffffu, d[0], src), c1 = __shfl_sync(0xffffffffu, d[1], src);
      if (lane == 0) { o->status = bst | (blb << 8); o->c0 = c0; o->c1 = c1; o->total_ms = 0.0; o->n_entries = ne; }
      continue;
    }
    NeumaierSum sum;
    for (int i = 0; i < ne; ++i) {
      const double v = __shfl_sync(0xffffffffu, val, i);
      const int lb = __shfl_sync(0xffffffffu, label, i);
      if (lb >= 0) sum.add(v);
    }
    if (lane == 0) { o->status = 0; o->c0 = o->c1 = 0; o->total_ms = sum.result(); o->n_entries = ne; }
  }
}

// ============================================================================ C ABI
extern "C" {

int lc_abi_version(void) { return LC_ABI_VERSION; }
const char* lc_last_error(void) { return g_err.c_str(); }

int lc_open(int device, lc_ctx** out) {
  if (!out) return fail(LC_ERR_ARG, "lc_open: out is NULL");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(LC_ERR_ARG, "lc_open: bad device index");
  CK(cudaSetDevice(device));
  // kernel attributes are per process and device: set them once, to the largest
  // shared-memory staging any database may need, so concurrent contexts never race
  {
    static std::mutex mu;
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lock(mu);
    if (device < 64 && !done[device]) {
      const int big = (int)kDbStageMax;
      CK(cudaFuncSetAttribute(k_qtables<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
      CK(cudaFuncSetAttribute(k_dstables<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
      CK(cudaFuncSetAttribute(k_front_final, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)((2 * sizeof(FrontCand) + 8) * kSurvivorCap)));
      done[device] = true;
    }
  }
  lc_ctx* c = new lc_ctx();
  c->device = device;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  for (auto& e : c->ev) CK(cudaEventCreate(&e));
  *out = c;
  return LC_OK;
}

int lc_close(lc_ctx* c) {
  if (!c) return LC_OK;
  cudaSetDevice(c->device);
  DBuf* bufs[] = {&c->searches, &c->batches, &c->batch_code, &c->loads, &c->meta, &c->results, &c->flags, &c->pos,
                  &c->block_sums, &c->u_search, &c->u_combo, &c->u_batch, &c->u_budget, &c->st_status,
                  &c->st_v, &c->ag_status, &c->ag_v, &c->pf_status, &c->pf_v, &c->dc_status, &c->dc_v,
                  &c->err_c, &c->u_queries, &c->cell_flags, &c->cells, &c->cell_err, &c->step_in, &c->step_out, &c->step_loads, &c->pool_key, &c->qt_groups, &c->ds_groups, &c->front_compact, &c->pool_part, &c->front_meta, &c->buckets, &c->surv, &c->n_surv, &c->qt, &c->ds, &c->m_used, &c->tail_tables, &c->tails, &c->tail_hash, &c->pool_sel, &c->plans_i, &c->plans_d, &c->front, &c->q_in, &c->q_lat, &c->q_st, &c->sgroups, &c->smembers, &c->sd, &c->raw_mask, &c->pair_inb, &c->cmax, &c->pgroups, &c->psteps, &c->acc, &c->plan_scratch, &c->pool_seed, &c->pool_sample, &c->front_flags, &c->cell_ctr, &c->inputs};
  for (DBuf* b : bufs) b->release();
  for (auto& e : c->ev) cudaEventDestroy(e);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->pinned_front) cudaFreeHost(c->pinned_front);
  if (c->pinned_plans_i) cudaFreeHost(c->pinned_plans_i);
  if (c->pinned_plans_d) cudaFreeHost(c->pinned_plans_d);
  if (c->arena) cudaFreeHost(c->arena);
  cudaStreamDestroy(c->stream);
  delete c;
  return LC_OK;
}

int lc_db_upload(lc_ctx* c, const lc_db_desc* d, lc_db** out) {
  if (!c || !d || !out) return fail(LC_ERR_ARG, "lc_db_upload: NULL argument");
  CK(cudaSetDevice(c->device));
  lc_db* db = new lc_db();
  db->device = c->device;
  db->n_grids = d->n_grids; db->n_axis = d->n_axis; db->n_cells = d->n_cells;
  std::vector<DevGrid> g(d->n_grids);
  for (int i = 0; i < d->n_grids; ++i) {
    g[i].ndim = d->grid_ndim[i];
    if (g[i].ndim != 1 && g[i].ndim != 2) { delete db; return fail(LC_ERR_ARG, "grid ndim must be 1 or 2"); }
    for (int a = 0; a < 2; ++a) { g[i].ax_off[a] = d->grid_axis_off[2 * i + a]; g[i].ax_len[a] = d->grid_axis_len[2 * i + a]; }
    g[i].cell_off = d->grid_cell_off[i];
  }
  int rc;
  if ((rc = upload(&db->grids, g.data(), g.size(), c->stream))) return rc;
  if ((rc = upload(&db->axv, d->axis_val, d->n_axis, c->stream))) return rc;
  if ((rc = upload(&db->axl, d->axis_log, d->n_axis, c->stream))) return rc;
  // NaN cells are quieted (repr / JSON print every NaN alike): the query tables'
  // status boxes are signalling-NaN patterns no latency may carry (box_status)
  std::vector<double> cells(d->cell, d->cell + d->n_cells);
  for (double& x : cells) {
    uint64_t b;
    memcpy(&b, &x, 8);
    if (std::isnan(x) && is_boxed(b)) { b |= 0x0008000000000000ull; memcpy(&x, &b, 8); }
  }
  if ((rc = upload(&db->cell, cells.data(), d->n_cells, c->stream))) return rc;
  if ((rc = upload(&db->clog, d->cell_log, d->n_cells, c->stream))) return rc;
  if ((rc = upload(&db->logtab, LOG_TAB_H, 256, c->stream))) return rc;
  if ((rc = upload(&db->exptab, EXP_TAB_H, 256, c->stream))) return rc;
  db->mem_bw = d->mem_bandwidth; db->intra_bw = d->intra_node_bandwidth; db->inter_bw = d->inter_node_bandwidth;
  db->gpu_memory = d->gpu_memory;
  for (int i = 0; i < 4; ++i) db->compute[i] = d->compute[i];
  db->gpn = d->gpus_per_node; db->policy = d->policy;
  db->smem_bytes = 256 * 16 + (size_t)d->n_axis * 16 + (size_t)d->n_cells * 16 + (size_t)d->n_grids * sizeof(DevGrid);
  db->staged = db->smem_bytes <= (size_t)kDbStageMax && !getenv("LC_DB_GLOBAL");
  CK(cudaStreamSynchronize(c->stream));
  *out = db;
  return LC_OK;
}

int lc_db_free(lc_db* db) {
  if (!db) return LC_OK;
  cudaSetDevice(db->device);
  cudaFree(db->grids); cudaFree(db->axv); cudaFree(db->axl); cudaFree(db->cell); cudaFree(db->clog);
  cudaFree(db->logtab); cudaFree(db->exptab);
  delete db;
  return LC_OK;
}

int lc_space_upload(lc_ctx* c, const lc_space_desc* d, lc_space** out) {
  if (!c || !d || !out) return fail(LC_ERR_ARG, "lc_space_upload: NULL argument");
  if (d->n_experts > LC_MAX_EXPERTS) return fail(LC_ERR_ARG, "too many experts");
  CK(cudaSetDevice(c->device));
  lc_space* sp = new lc_space();
  sp->device = c->device;
  sp->hidden = d->hidden; sp->topk = d->topk; sp->n_experts = d->n_experts; sp->is_moe = d->is_moe;
  sp->n_combos = d->n_combos; sp->n_tmpl = d->n_tmpl; sp->n_tp = d->n_tp; sp->n_ep = d->n_ep;
  std::vector<int64_t> tpv(d->n_tp > 0 ? d->n_tp : 1, 1), epv(d->n_ep > 0 ? d->n_ep : 1, 1);
  std::vector<uint8_t> used((size_t)(d->n_tp > 0 ? d->n_tp : 1) * (d->n_ep > 0 ? d->n_ep : 1), 0);
  std::vector<TmplInfo> tinfo(d->n_tmpl > 0 ? d->n_tmpl : 1, TmplInfo{1, 1, 1, 0, 0});
  for (int i = 0; i < d->n_combos; ++i) {
    const lc_combo& k = d->combos[i];
    if (k.tp_i < 0 || k.tp_i >= d->n_tp || k.ep_i < 0 || k.ep_i >= d->n_ep || k.tmpl < 0 || k.tmpl >= d->n_tmpl)
      return fail(LC_ERR_ARG, "lc_space_upload: combo index out of range");
    tpv[k.tp_i] = k.tp; epv[k.ep_i] = k.ep;
    used[(size_t)k.tp_i * d->n_ep + k.ep_i] = 1;
    tinfo[k.tmpl] = TmplInfo{k.tp, k.pp, k.ep, k.tp_i, k.ep_i};
  }
  for (int t = 0; t < d->n_tmpl; ++t)
    if (d->tmpl_n_entries[t] > LC_MAX_ENTRIES) return fail(LC_ERR_ARG, "template has too many entries");
  int rc;
  if ((rc = upload(&sp->combos, d->combos, d->n_combos, c->stream))) return rc;
  if ((rc = upload(&sp->tmpl_n, d->tmpl_n_entries, d->n_tmpl, c->stream))) return rc;
  if ((rc = upload(&sp->entries, d->entries, (size_t)d->n_tmpl * LC_MAX_ENTRIES, c->stream))) return rc;
  if ((rc = upload(&sp->tp_vals, tpv.data(), tpv.size(), c->stream))) return rc;
  if ((rc = upload(&sp->ep_vals, epv.data(), epv.size(), c->stream))) return rc;
  sp->max_ep_h = 1;
  for (int64_t v : epv) sp->max_ep_h = v > sp->max_ep_h ? v : sp->max_ep_h;
  if ((rc = upload(&sp->pair_used, used.data(), used.size(), c->stream))) return rc;
  if ((rc = upload(&sp->tmpl_info, tinfo.data(), tinfo.size(), c->stream))) return rc;
  std::vector<int32_t> canon(used.size(), 0);
  for (int a = 0; a < (d->n_tp > 0 ? d->n_tp : 1); ++a)
    for (int e = 0; e < (d->n_ep > 0 ? d->n_ep : 1); ++e) {
      const int idx = a * d->n_ep + e;
      canon[idx] = idx;
      const int64_t f = epv[e] / tpv[a] > 1 ? epv[e] / tpv[a] : 1;
      for (int a2 = 0; a2 < a; ++a2) {
        const int64_t f2 = epv[e] / tpv[a2] > 1 ? epv[e] / tpv[a2] : 1;
        if (f2 == f && used[a2 * d->n_ep + e]) { canon[idx] = a2 * d->n_ep + e; break; }
      }
    }
  if ((rc = upload(&sp->pair_canon, canon.data(), canon.size(), c->stream))) return rc;
  sp->n_slots = d->n_slots;
  sp->n_gclass = d->n_gen_classes;
  if ((rc = upload(&sp->slots, d->slots, d->n_slots > 0 ? d->n_slots : 0, c->stream))) return rc;
  {
    std::vector<int32_t> cls(d->n_slots > 0 ? d->n_slots : 1, 0), idx(d->n_slots > 0 ? d->n_slots : 1, 0);
    std::vector<int32_t> lists[4];
    int32_t n2d[4] = {0, 0, 0, 0};
    for (int k = 0; k < d->n_slots; ++k) {
      const lc_slot& sl = d->slots[k];
      const int c0 = sl.step == LC_STEP_PREFILL ? 0 : sl.step == LC_STEP_MIXED ? 3 : (sl.e.coord == LC_COORD_GEN ? 2 : 1);
      cls[k] = c0;
      idx[k] = (int32_t)lists[c0].size();
      if (sl.e.coord == LC_COORD_CTX || sl.e.coord == LC_COORD_GEN) ++n2d[c0];
      lists[c0].push_back(k);
    }
    std::vector<int32_t> all;
    for (int c0 = 0; c0 < 4; ++c0) {
      sp->class_off[c0] = (int32_t)all.size();
      sp->class_n[c0] = (int32_t)lists[c0].size();
      sp->class_n2d[c0] = n2d[c0];
      all.insert(all.end(), lists[c0].begin(), lists[c0].end());
    }
    const size_t n_so = (size_t)(d->n_tmpl > 0 ? d->n_tmpl : 1) * LC_MAX_ENTRIES * 3;
    std::vector<int32_t> so(n_so, -1);
    for (size_t i = 0; i < n_so && d->n_tmpl > 0; ++i) {
      const int32_t g = d->slot_of[i];
      so[i] = g < 0 ? -1 : ((cls[g] << 16) | idx[g]);
    }
    if ((rc = upload(&sp->slot_of, so.data(), so.size(), c->stream))) return rc;
    if ((rc = upload(&sp->class_slots, all.data(), all.size(), c->stream))) return rc;
  }
  if ((rc = upload(&sp->gclasses, d->gen_classes, d->n_gen_classes > 0 ? d->n_gen_classes : 0, c->stream))) return rc;
  if ((rc = upload(&sp->gclass_of, d->gclass_of, d->n_tmpl > 0 ? d->n_tmpl : 1, c->stream))) return rc;
  {
    std::vector<int32_t> off((size_t)(d->n_tmpl > 0 ? d->n_tmpl : 0) + 1, 0), idx;
    for (int t = 0; t < d->n_tmpl; ++t) {
      off[t] = (int32_t)idx.size();
      for (int i = 0; i < d->n_combos; ++i)
        if (d->combos[i].tmpl == t) idx.push_back(i);
    }
    off[d->n_tmpl > 0 ? d->n_tmpl : 0] = (int32_t)idx.size();
    if (idx.empty()) idx.push_back(0);
    if ((rc = upload(&sp->tmpl_cidx_off, off.data(), off.size(), c->stream))) return rc;
    if ((rc = upload(&sp->tmpl_cidx, idx.data(), idx.size(), c->stream))) return rc;
  }
  {
    // string-order rank of each combo's (tp, pp, ep, dp) (lc_keys.h): the pool-rank tie break
    std::vector<uint64_t> code(d->n_combos > 0 ? d->n_combos : 1, 0), rank(code.size(), 0);
    for (int i = 0; i < d->n_combos; ++i) {
      const lc_combo& k = d->combos[i];
      if (k.tp > LC_KEY_FIELD_MAX || k.pp > LC_KEY_FIELD_MAX || k.ep > LC_KEY_FIELD_MAX || k.dp > LC_KEY_FIELD_MAX)
        return fail(LC_ERR_ARG, "lc_space_upload: tp/pp/ep/dp values above 9999 are not supported");
      code[i] = lc_combo_code(k.tp, k.pp, k.ep, k.dp);
    }
    std::vector<uint64_t> sorted(code.begin(), code.begin() + (d->n_combos > 0 ? d->n_combos : 0));
    std::sort(sorted.begin(), sorted.end());
    sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
    for (int i = 0; i < d->n_combos; ++i)
      rank[i] = (uint64_t)(std::lower_bound(sorted.begin(), sorted.end(), code[i]) - sorted.begin()) << 36;
    if ((rc = upload(&sp->combo_rank, rank.data(), rank.size(), c->stream))) return rc;
  }
  CK(cudaStreamSynchronize(c->stream));
  *out = sp;
  return LC_OK;
}

int lc_space_free(lc_space* sp) {
  if (!sp) return LC_OK;
  cudaSetDevice(sp->device);
  cudaFree(sp->combos); cudaFree(sp->tmpl_n); cudaFree(sp->entries); cudaFree(sp->tp_vals); cudaFree(sp->ep_vals);
  cudaFree(sp->pair_used);
  cudaFree(sp->tmpl_info);
  cudaFree(sp->pair_canon);
  cudaFree(sp->slots); cudaFree(sp->slot_of); cudaFree(sp->class_slots); cudaFree(sp->gclasses); cudaFree(sp->gclass_of);
  cudaFree(sp->tmpl_cidx_off); cudaFree(sp->tmpl_cidx); cudaFree(sp->combo_rank);
  delete sp;
  return LC_OK;
}

static EvalParams make_params(lc_ctx* c) {
  EvalParams P;
  memset(&P, 0, sizeof(P));
  const lc_db* db = c->db;
  const lc_space* sp = c->sp;
  P.grids = db->grids; P.axv = db->axv; P.axl = db->axl; P.cell = db->cell; P.clog = db->clog;
  P.logtab = db->logtab; P.exptab = db->exptab;
  P.n_grids = db->n_grids; P.n_axis = db->n_axis; P.n_cells = db->n_cells;
  P.mem_bw = db->mem_bw; P.intra_bw = db->intra_bw; P.inter_bw = db->inter_bw; P.gpu_memory = db->gpu_memory;
  for (int i = 0; i < 4; ++i) P.compute[i] = db->compute[i];
  P.gpn = db->gpn; P.policy = db->policy;
  P.db_global = db->staged ? 0 : 1;
  {
    // LC_SURVIVOR_CAP (tests only) lowers the cap so small searches take K4's overflow path
    static const int cap_env = getenv("LC_SURVIVOR_CAP") ? atoi(getenv("LC_SURVIVOR_CAP")) : 0;
    P.surv_cap = cap_env > 0 && cap_env < kSurvivorCap ? cap_env : kSurvivorCap;
  }
  P.combos = sp->combos; P.tmpl_n = sp->tmpl_n; P.entries = sp->entries; P.sp_n_combos = sp->n_combos;
  P.hidden = sp->hidden; P.topk = sp->topk; P.n_experts = sp->n_experts; P.is_moe = sp->is_moe;
  P.n_tp = sp->n_tp; P.n_ep = sp->n_ep; P.tp_vals = sp->tp_vals; P.ep_vals = sp->ep_vals; P.pair_used = sp->pair_used;
  P.pair_canon = sp->pair_canon;
  P.tail_tables = (const TailTable*)c->tail_tables.p;
  P.n_tail_tables = (int32_t)c->htables.size();
  P.n_pd_tails = c->n_pd_tails;
  P.m_tmax = c->m_tmax;
  P.m_used = (uint8_t*)c->m_used.p;
  P.slots = sp->slots; P.n_slots = sp->n_slots; P.slot_of = sp->slot_of;
  P.class_slots = sp->class_slots;
  for (int k = 0; k < 4; ++k) P.class_off[k] = sp->class_off[k];
  P.qt_groups = (const QtGroup*)c->qt_groups.p; P.n_qt_groups = (int32_t)c->hqt.size();
  P.gclasses = sp->gclasses; P.n_gclass = sp->n_gclass; P.gclass_of = sp->gclass_of;
  P.qt = (double*)c->qt.p; P.n_qt = c->n_qt;
  P.ds = (QVal*)c->ds.p; P.n_ds = c->n_ds;
  P.ds_groups = (const DsGroup*)c->ds_groups.p; P.n_ds_groups = (int32_t)c->hds.size();
  P.sgroups = (const SeriesGroup*)c->sgroups.p; P.n_sgroups = (int32_t)c->hsg.size();
  P.smembers = (const SeriesMember*)c->smembers.p; P.sd = (SdOut*)c->sd.p; P.n_series = c->n_series;
  P.pgroups = (const PGroup*)c->pgroups.p; P.n_pgroups = (int32_t)c->hpg.size();
  P.psteps = (PStep*)c->psteps.p; P.n_pstep = c->n_pstep;
  P.searches = (const lc_search_desc*)c->searches.p;
  P.meta = (const SearchMeta*)c->meta.p;
  P.n_search = c->n_search;
  if (c->filt_hi >= 0) {
    P.raw_lo = c->filt_lo;
    P.raw_hi = c->filt_hi;
    P.raw_mask = c->filt_mask ? (const uint8_t*)c->raw_mask.p : nullptr;
  } else {
    P.raw_lo = 0;
    P.raw_hi = INT64_MAX;
    P.raw_mask = nullptr;
  }
  P.batches = (const int64_t*)c->batches.p;
  P.loads = (const double*)c->loads.p;
  P.u_search = (const int32_t*)c->u_search.p; P.u_combo = (const int32_t*)c->u_combo.p;
  P.u_batch = (const int32_t*)c->u_batch.p; P.u_budget = (const uint8_t*)c->u_budget.p;
  P.n_cap = c->n_cap;
  P.d_total = (const int32_t*)c->block_sums.p + c->n_total_idx;
  P.tails = (const int64_t*)c->tails.p;
  P.st_status = (int32_t*)c->st_status.p; P.st_v = (double*)c->st_v.p;
  P.ag_status = (int32_t*)c->ag_status.p; P.ag_v = (double*)c->ag_v.p;
  P.pf_status = (int32_t*)c->pf_status.p; P.pf_v = (double*)c->pf_v.p;
  P.dc_status = (int32_t*)c->dc_status.p; P.dc_v = (double*)c->dc_v.p;
  P.err_c = (int64_t*)c->err_c.p;
  P.front_flags = (uint8_t*)c->front_flags.p;
  P.cell_ctr = (unsigned long long*)c->cell_ctr.p;
  P.pool_key = (double*)c->pool_key.p;
  P.tmpl_info = sp->tmpl_info;
  P.cell_flags = (uint32_t*)c->cell_flags.p;
  P.cells = (CellOut*)c->cells.p;
  P.cell_err = (int64_t*)c->cell_err.p;
  P.n_cells_total = c->n_cells;
  P.results = (lc_search_result*)c->results.p;
  P.acc = (SearchAcc*)c->acc.p;
  P.fbuckets = (unsigned long long*)c->buckets.p;
  P.combo_rank = c->sp ? c->sp->combo_rank : nullptr;
  P.batch_code = (const uint64_t*)c->batch_code.p;
#ifndef LC_NO_FUSE_EXPAND
  P.pair_off = c->enum_fit ? (const int32_t*)c->block_sums.p : nullptr;
#else
  P.pair_off = nullptr;
#endif
  P.pair_inb = (const uint8_t*)c->pair_inb.p;
#ifndef LC_NO_POOL_SEED
  P.pool_sample = P.pair_off ? (double*)c->pool_sample.p : nullptr;
#else
  P.pool_sample = nullptr;
#endif
  P.tmpl_cidx_off = sp->tmpl_cidx_off; P.tmpl_cidx = sp->tmpl_cidx;
  return P;
}

static int sm_count(int dev) {
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

// stage boundary events: inside a graph capture they become event-record nodes
static cudaError_t record_ev(lc_ctx* c, int k) {
  return cudaEventRecordWithFlags(c->ev[k], c->stream, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

// Everything after the unit list is known: K3, K2, K5a, K5b, K4.
static int run_eval_pipeline(lc_ctx* c, lc_batch_totals* totals) {
  cudaError_t err = cudaSuccess;
  const int64_t n = c->n_cap;
  c->st_status.get<int32_t>(n, &err); c->st_v.get<double>(4 * n, &err);
  c->ag_status.get<int32_t>(n, &err); c->ag_v.get<double>(4 * n, &err);
  c->pf_status.get<int32_t>(n, &err); c->pf_v.get<double>(2 * n, &err);
  c->dc_status.get<int32_t>(n, &err); c->dc_v.get<double>(2 * n, &err);
  c->err_c.get<int64_t>(8 * n, &err);
  c->front_flags.get<uint8_t>(n, &err);
  c->cell_ctr.get<unsigned long long>(1, &err);
  c->pool_key.get<double>(2 * n, &err);
  c->cells.get<CellOut>(c->n_cells, &err);
  c->qt.get<double>(c->n_qt, &err);
  c->ds.get<QVal>(c->n_ds, &err);
  c->cell_err.get<int64_t>(8 * c->n_cells, &err);
  c->pool_sel.get<int32_t>((size_t)c->n_search * 128, &err);
  c->plans_i.get<int32_t>((size_t)c->n_plan_slots * 4, &err);
  c->plans_d.get<double>((size_t)c->n_plan_slots * 6, &err);
  c->front.get<int64_t>((size_t)c->n_front_slots, &err);
  c->tails.get<int64_t>((size_t)(c->n_tails > 0 ? c->n_tails : 1), &err);
  const int64_t n_mark_bytes = (int64_t)(c->n_loads > 0 ? c->n_loads : 1) * (c->m_tmax + 1);
  c->m_used.get<uint8_t>(n_mark_bytes, &err);
  if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(err));
  // per-search result accumulators (queries are summed by K4)
  CK(cudaMemsetAsync(c->results.p, 0, sizeof(lc_search_result) * c->n_search, c->stream));
  {
    SearchAcc* acc = c->acc.get<SearchAcc>(c->n_search > 0 ? c->n_search : 1, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "accumulator allocation");
    CK(cudaMemsetAsync(acc, 0, sizeof(SearchAcc) * (c->n_search > 0 ? c->n_search : 1), c->stream));
  }
  {
    // K4 speed buckets: zeroed here, filled by K2 / K5b for fixed-geometry searches
    c->buckets.get<unsigned long long>((size_t)c->n_search * kSpeedBuckets, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "bucket allocation");
    CK(cudaMemsetAsync(c->buckets.p, 0, sizeof(unsigned long long) * kSpeedBuckets * c->n_search, c->stream));
  }
  EvalParams P = make_params(c);
  const int sms = sm_count(c->device);
  CK(record_ev(c, 1));
  if (c->n_tails > c->n_pd_tails) {
    P.m_used = (uint8_t*)c->m_used.p;
    CK(cudaMemsetAsync(c->m_used.p, 0, n_mark_bytes, c->stream));
    int blocks = (int)((c->n_marks + 255) / 256);
    if (blocks < 1) blocks = 1;
    ++c->launches;
    k_mark_mixed<<<blocks, 256, 0, c->stream>>>(P, c->n_marks);
    CK(cudaGetLastError());
  }
  if (c->n_tails > 0) {
#ifndef LC_TAILS_NODEDUP
    const bool dedup = c->tails_dedup_ok;
#else
    const bool dedup = false;
#endif
    const int res_blocks = sms * (c->sp->n_experts <= 128 ? LC_TAIL_MIN_BLOCKS : LC_TAIL8_MIN_BLOCKS);
    if (dedup) {
      TailHash H;
      H.cap = 1;
      while (H.cap < 2 * c->n_tails) H.cap <<= 1;
      const size_t n_jobs_cap = (size_t)c->n_tails;
      const size_t b_keys = 8 * H.cap, b_mask = 8 * H.cap, b_jos = 4 * H.cap, b_jobs = 4 * (1 + n_jobs_cap),
                   b_slot = 4 * (size_t)c->n_tails, b_res = 8 * n_jobs_cap * c->sp->n_ep;
      auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
      cudaError_t err2 = cudaSuccess;
      unsigned char* base = c->tail_hash.get<unsigned char>(al(b_keys) + al(b_mask) + al(b_jos) + al(b_jobs) +
                                                                 al(b_slot) + al(b_res), &err2);
      if (err2 != cudaSuccess) return fail(LC_ERR_CUDA, "tail hash allocation");
      size_t o = 0;
      H.keys = (unsigned long long*)(base + o); o += al(b_keys);
      H.epmask = (unsigned long long*)(base + o); o += al(b_mask);
      H.job_of_slot = (int32_t*)(base + o); o += al(b_jos);
      H.jobs = (int32_t*)(base + o); o += al(b_jobs);
      H.slot_of = (int32_t*)(base + o); o += al(b_slot);
      H.res = (int64_t*)(base + o);
      CK(cudaMemsetAsync(H.keys, 0xff, b_keys, c->stream));
      CK(cudaMemsetAsync(H.epmask, 0, b_mask, c->stream));
      CK(cudaMemsetAsync(H.jobs, 0, sizeof(int32_t), c->stream));
      int eblocks = (int)((c->n_tails + 255) / 256);
      if (eblocks > sms * 8) eblocks = sms * 8;
      ++c->launches;
      k_tails_keys<<<eblocks, 256, 0, c->stream>>>(P, c->n_tails, H);
      CK(cudaGetLastError());
      ++c->launches;
      // persistent: the resident warps take the jobs in turn (their count is on the device)
      if (c->sp->n_experts <= 128) k_tails_jobs<4><<<res_blocks, 256, 0, c->stream>>>(P, H);
      else if (c->sp->n_experts <= 256) k_tails_jobs<8><<<res_blocks, 256, 0, c->stream>>>(P, H);
      else k_tails_jobs<32><<<res_blocks, 256, 0, c->stream>>>(P, H);
      CK(cudaGetLastError());
      ++c->launches;
      k_tails_put<<<eblocks, 256, 0, c->stream>>>(P, c->n_tails, H, (int64_t*)c->tails.p);
    } else {
      const int64_t warps = (c->n_tails + 31) / 32;  // a warp per 32 consecutive entries
      int blocks = (int)((warps + 7) / 8);
      if (blocks > sms * 16) blocks = sms * 16;
      ++c->launches;
      // experts per lane: 8 covers E <= 256 (DeepSeek-V3, GPT-OSS) at a quarter of the registers
      if (c->sp->n_experts <= 128) k_tails<4><<<blocks, 256, 0, c->stream>>>(P, c->n_tails, (int64_t*)c->tails.p);
      else if (c->sp->n_experts <= 256) k_tails<8><<<blocks, 256, 0, c->stream>>>(P, c->n_tails, (int64_t*)c->tails.p);
      else k_tails<32><<<blocks, 256, 0, c->stream>>>(P, c->n_tails, (int64_t*)c->tails.p);
    }
    CK(cudaGetLastError());
  }
  CK(record_ev(c, 2));
  {
    EvalParams P2 = make_params(c);  // table pointers are valid only after the allocations above
    P = P2;
  }
  const size_t smem = c->db->staged ? c->db->smem_bytes : 0;
  auto launch_tables = [&](auto kern, int64_t n_items) -> int {
    if (n_items <= 0) return LC_OK;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LC_TABLE_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (n_items + LC_TABLE_THREADS - 1) / LC_TABLE_THREADS;
    const int64_t cap = (int64_t)sms * per_sm;
    if (blocks > cap) blocks = cap;
    ++c->launches;
    kern<<<(int)blocks, LC_TABLE_THREADS, smem, c->stream>>>(P);
    CK(cudaGetLastError());
    return LC_OK;
  };
  const bool staged = c->db->staged;
  int rc2 = launch_tables(staged ? k_qtables<false> : k_qtables<true>, c->n_qt);
  if (rc2) return rc2;
  rc2 = launch_tables(staged ? k_dstables<false> : k_dstables<true>, c->n_ds);
  if (rc2) return rc2;
  if (c->n_series > 0) {
    int64_t blocks = (c->n_series + 127) / 128;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    ++c->launches;
    k_dseries<<<(int)blocks, 128, 0, c->stream>>>(P);
    CK(cudaGetLastError());
  }
  if (c->n_pstep > 0) {
    int64_t blocks = (c->n_pstep + 127) / 128;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    ++c->launches;
    k_ptables<<<(int)blocks, 128, 0, c->stream>>>(P);
    CK(cudaGetLastError());
  }
  if (c->n_cells > 0) {
    int64_t blocks = (c->n_cells + 127) / 128;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    ++c->launches;
    CK(cudaMemsetAsync(c->cell_ctr.p, 0, sizeof(unsigned long long), c->stream));
    k_eval_cells<<<(int)blocks, 128, 0, c->stream>>>(P);
    CK(cudaGetLastError());
  }
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    if (!P.pair_off) {  // otherwise k_eval_cells wrote the candidate rows
      ++c->launches;
      k_expand<<<(int)blocks, 256, 0, c->stream>>>(P);  // also the per-search accounting (SearchAcc)
    }
    CK(cudaGetLastError());
  }
  CK(record_ev(c, 3));
  {
    PoolPartial* pp = c->pool_part.get<PoolPartial>((size_t)c->n_search * kPoolSplit, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "pool partial allocation");
    ++c->launches;
    unsigned long long* seed = nullptr;
#ifndef LC_NO_POOL_SEED
    if (P.pool_sample) {
      unsigned long long* sd = c->pool_seed.get<unsigned long long>((size_t)c->n_search * 2, &err);
      if (err != cudaSuccess) return fail(LC_ERR_CUDA, "pool seed allocation");
      ++c->launches;
      k_pools_seed<<<2 * c->n_search, kSeedThreads, 0, c->stream>>>(P, sd);
      seed = sd;
    }
#endif
    k_pools_partial<<<dim3(kPoolSplit, c->n_search), kPoolThreads, 0, c->stream>>>(P, (const SearchMeta*)c->meta.p, pp,
                                                                                    seed);
    ++c->launches;
    k_pools_final<<<c->n_search, kPoolFinalThreads, 0, c->stream>>>(P, (SearchMeta*)c->meta.p, pp,
                                                                   (int32_t*)c->pool_sel.p);
    CK(cudaGetLastError());
  }
  CK(record_ev(c, 4));
  ++c->launches;
  {
    PlanRec* scr = c->plan_scratch.get<PlanRec>((size_t)c->n_search * 256, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "plan scratch allocation");
    k_disagg_pairs<<<dim3(c->n_search, kDisSplit), 256, 0, c->stream>>>(P, (const SearchMeta*)c->meta.p,
                                                                       (const int32_t*)c->pool_sel.p, scr);
    ++c->launches;
    k_disagg<<<c->n_search, 256, 0, c->stream>>>(P, (SearchMeta*)c->meta.p, (const int32_t*)c->pool_sel.p, scr,
                                                 (int32_t*)c->plans_i.p, (double*)c->plans_d.p,
                                                 (lc_search_result*)c->results.p);
  }
  CK(cudaGetLastError());
  CK(record_ev(c, 5));
  {
    FrontMeta* fm = c->front_meta.get<FrontMeta>(c->n_search, &err);
    unsigned long long* bk = c->buckets.get<unsigned long long>((size_t)c->n_search * kSpeedBuckets, &err);
    FrontCand* sv = c->surv.get<FrontCand>((size_t)c->n_search * kSurvivorCap, &err);
    int32_t* ns = c->n_surv.get<int32_t>(c->n_search, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "front workspace allocation");
    const SearchMeta* meta = (const SearchMeta*)c->meta.p;
    const int32_t* pi = (const int32_t*)c->plans_i.p;
    const double* pd = (const double*)c->plans_d.p;
    lc_search_result* res = (lc_search_result*)c->results.p;
    const dim3 g(kSplit, c->n_search);
    ++c->launches;
    k_front_mid<<<c->n_search, kFrontThreads, 0, c->stream>>>(P, meta, pi, pd, res, fm, bk, ns);
    ++c->launches;
    k_front_pass2<<<g, kFrontThreads, 0, c->stream>>>(P, meta, pi, pd, res, fm, bk);
    ++c->launches;
    k_front_suffix<<<c->n_search, kFrontThreads, 0, c->stream>>>(fm, bk);
    ++c->launches;
    k_front_pass3<<<g, kFrontThreads, 0, c->stream>>>(P, meta, pi, pd, res, fm, bk, sv, ns);
    const size_t fsmem = (2 * sizeof(FrontCand) + 8) * kSurvivorCap;
    ++c->launches;
    int64_t* fc = c->front_compact.get<int64_t>((size_t)c->n_search * kCompactFront, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, "front workspace allocation");
    k_front_final<<<c->n_search, kFinalThreads, fsmem, c->stream>>>(P, meta, pi, pd, res, fm, sv, ns,
                                                                      (int64_t*)c->front.p, fc);
    CK(cudaGetLastError());
  }
  CK(record_ev(c, 6));
  (void)totals;
  return LC_OK;
}

static int run_enum_fit(lc_ctx* c) {
  cudaError_t err = cudaSuccess;
  const int64_t n_raw = c->n_raw;
  const int32_t nc = c->sp->n_combos, nt = c->sp->n_tmpl;
  const int64_t n_pairs = (int64_t)c->n_search * nc;
  int32_t* bs = c->block_sums.get<int32_t>(n_pairs + 1, &err);
  uint8_t* inb = c->pair_inb.get<uint8_t>(n_pairs > 0 ? n_pairs : 1, &err);
  c->pool_sample.get<double>((size_t)(n_pairs > 0 ? n_pairs : 1) * 2, &err);  // K5a seed sample (k_eval_cells)
  int32_t* cmax = c->cmax.get<int32_t>((size_t)c->n_search * (nt > 0 ? nt : 1) * 2 + 1, &err);
  uint32_t* cflags = c->cell_flags.get<uint32_t>(c->n_cells, &err);
  c->n_cap = n_raw;
  int32_t* us = c->u_search.get<int32_t>(n_raw, &err);
  int32_t* uc = c->u_combo.get<int32_t>(n_raw, &err);
  int32_t* ub = c->u_batch.get<int32_t>(n_raw, &err);
  uint8_t* ubud = c->u_budget.get<uint8_t>(n_raw, &err);
  if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(err));
  EvalParams P = make_params(c);
  const int sms = sm_count(c->device);
  c->n_total_idx = n_pairs;
  if (n_pairs == 0) {
    CK(cudaMemsetAsync(bs, 0, sizeof(int32_t), c->stream));
  } else {
    CK(cudaMemsetAsync(cmax, 0, sizeof(int32_t) * (size_t)c->n_search * (nt > 0 ? nt : 1) * 2, c->stream));
    int blocks = (int)((n_pairs + 127) / 128);
    if (blocks > sms * 8) blocks = sms * 8;
    ++c->launches;
    k_enum_fit<<<blocks, 128, 0, c->stream>>>(P, n_pairs, bs, inb, cmax, nt);
    if (c->n_cells) {
      int32_t nbmax = 1;
      for (int s = 0; s < c->n_search; ++s) nbmax = c->hsearch_nb[s] > nbmax ? c->hsearch_nb[s] : nbmax;
      const int64_t per = (int64_t)nt * nbmax;
      int bx = (int)((per + 255) / 256);
      if (bx > 64) bx = 64;
      ++c->launches;
      k_cell_flags_fit<<<dim3(bx, c->n_search), 256, 0, c->stream>>>(P, cmax, nt, cflags);
    }
    ++c->launches;
    k_scan_top<<<1, 1024, 0, c->stream>>>(bs, (int)n_pairs);
    ++c->launches;
    int sb = (int)(n_pairs < (int64_t)sms * 32 ? n_pairs : (int64_t)sms * 32);
    k_scatter_fit<<<sb, 128, 0, c->stream>>>(P, n_pairs, bs, inb, us, uc, ub, ubud);
    CK(cudaGetLastError());
  }
  ++c->launches;
  k_unit_offsets_fit<<<(c->n_search + 127) / 128, 128, 0, c->stream>>>((SearchMeta*)c->meta.p, c->n_search, nc, bs);
  CK(cudaGetLastError());
  return LC_OK;
}

static int run_enum(lc_ctx* c) {
  c->enum_fit = c->batches_sorted && c->filt_hi < 0 && !getenv("LC_ENUM_FLAGS");
  if (c->enum_fit) return run_enum_fit(c);
  cudaError_t err = cudaSuccess;
  const int64_t n_raw = c->n_raw;
  const int64_t nblk = (n_raw + kScanBlock - 1) / kScanBlock;
  uint8_t* flags = c->flags.get<uint8_t>(n_raw, &err);
  int32_t* pos = c->pos.get<int32_t>(n_raw, &err);
  int32_t* bs = c->block_sums.get<int32_t>(nblk + 1, &err);
  uint32_t* cflags = c->cell_flags.get<uint32_t>(c->n_cells, &err);
  if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(err));
  if (c->n_cells) CK(cudaMemsetAsync(cflags, 0, sizeof(uint32_t) * c->n_cells, c->stream));
  EvalParams P = make_params(c);
  const int sms = sm_count(c->device);
  if (n_raw > 0) {
    int blocks = (int)((n_raw + 255) / 256);
    if (blocks > sms * 32) blocks = sms * 32;
    ++c->launches;
    k_enum_flags<<<blocks, 256, 0, c->stream>>>(P, n_raw, flags);
    ++c->launches;
    k_scan_blocks<<<(int)nblk, kScanBlock, 0, c->stream>>>(flags, n_raw, bs);
    ++c->launches;
    k_scan_top<<<1, 1024, 0, c->stream>>>(bs, (int)nblk);
    CK(cudaGetLastError());
  } else {
    CK(cudaMemsetAsync(bs, 0, sizeof(int32_t), c->stream));
  }
  c->n_total_idx = nblk;
  c->n_cap = n_raw;
  int32_t* us = c->u_search.get<int32_t>(n_raw, &err);
  int32_t* uc = c->u_combo.get<int32_t>(n_raw, &err);
  int32_t* ub = c->u_batch.get<int32_t>(n_raw, &err);
  uint8_t* ubud = c->u_budget.get<uint8_t>(n_raw, &err);
  if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(err));
  if (n_raw > 0) {
    ++c->launches;
    k_scatter<<<(int)nblk, kScanBlock, 0, c->stream>>>(P, flags, n_raw, bs, pos, us, uc, ub, ubud);
    CK(cudaGetLastError());
  }
  ++c->launches;
  k_unit_offsets<<<(c->n_search + 127) / 128, 128, 0, c->stream>>>((SearchMeta*)c->meta.p, c->n_search, pos, n_raw,
                                                                   bs + nblk);
  CK(cudaGetLastError());
  return LC_OK;
}

// K0 .. K4 of the current batch.  The launch sequence (~25 kernels and memsets)
// is captured into a CUDA graph and launched as one unit: the GPU then runs the
// dependent kernels back to back without per-launch gaps.  A previous graph is
// updated in place (cudaGraphExecUpdate) when only parameters changed.  A
// capture that would have to grow a workspace buffer is discarded and the
// pipeline runs directly once (allocating); LC_NO_GRAPH=1 always runs directly.
static int run_direct(lc_ctx* c, lc_batch_totals* totals) {
  CK(cudaEventRecord(c->ev[0], c->stream));
  c->launches = 0;
  int rc = run_enum(c);
  if (rc) return rc;
  c->n_front_slots = 2 * c->n_cap + c->n_plan_slots;
  return run_eval_pipeline(c, totals);
}

static int launch_pipeline(lc_ctx* c, lc_batch_totals* totals) {
  static const bool no_graph = getenv("LC_NO_GRAPH") != nullptr;
  c->graph_ok = false;
  if (no_graph) return run_direct(c, totals);
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  tl_capturing = true;
  tl_capture_grow = false;
  c->capturing = true;
  c->launches = 0;
  int rc = (int)record_ev(c, 0) == (int)cudaSuccess ? LC_OK : LC_ERR_CUDA;
  if (!rc) rc = run_enum(c);
  if (!rc) {
    c->n_front_slots = 2 * c->n_cap + c->n_plan_slots;
    rc = run_eval_pipeline(c, totals);
  }
  tl_capturing = false;
  c->capturing = false;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  if (rc || e != cudaSuccess || tl_capture_grow || !g) {
    if (g) cudaGraphDestroy(g);
    (void)cudaGetLastError();
    if (rc && !tl_capture_grow) return rc;
    return run_direct(c, totals);  // allocates the workspace; the next batch of this shape is captured
  }
  if (c->gexec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(c->gexec, g, &info) != cudaSuccess) {
      (void)cudaGetLastError();
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
  }
  if (!c->gexec) {
    const cudaError_t ie = cudaGraphInstantiate(&c->gexec, g, 0);
    if (ie != cudaSuccess) {
      cudaGraphDestroy(g);
      c->gexec = nullptr;
      return fail(LC_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
    }
  }
  cudaGraphDestroy(g);
  CK(cudaGraphLaunch(c->gexec, c->stream));
  c->graph_ok = true;
  return LC_OK;
}

int lc_search_batch(lc_ctx* c, const lc_db* db, const lc_space* sp, int32_t n_search,
                    const lc_search_desc* searches, int32_t n_batches, const int64_t* batches, int32_t n_loads,
                    const double* loads, lc_search_result* results, lc_batch_totals* totals) {
  if (!c || !db || !sp || (n_search > 0 && !searches) || n_search < 0)
    return fail(LC_ERR_ARG, "lc_search_batch: bad arguments");
  // LC_HOST_TIMING=1: host-side phases of the call on stderr (plan / launch / wait)
  static const bool host_timing = getenv("LC_HOST_TIMING") != nullptr;
  const auto t_in = std::chrono::steady_clock::now();
  auto ms_since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  CK(cudaSetDevice(c->device));
  c->staged = false;
  c->db = db;
  c->sp = sp;
  c->n_search = n_search;
  if (n_search == 0) {  // nothing to evaluate: empty results, no launches
    c->n_batches = n_batches;
    c->n_loads = n_loads;
    c->n_raw = c->n_cap = c->n_units = c->n_cells = c->n_plan_slots = c->n_front_slots = 0;
    c->n_qt = c->n_ds = c->n_tails = c->n_series = c->n_pstep = 0;
    c->launches = 0;
    c->hres.clear();
    c->hmeta.clear();
    if (totals) memset(totals, 0, sizeof(*totals));
    return LC_OK;
  }
  c->n_batches = n_batches;
  c->n_loads = n_loads;
  // host bookkeeping: raw tuple, tail and plan offsets
  c->hmeta.assign(n_search, SearchMeta{});
  c->batches_sorted = true;
  c->hsearch_nb.assign(n_search, 0);
  for (int s = 0; s < n_search; ++s) {
    const lc_search_desc& S = searches[s];
    c->hsearch_nb[s] = S.n_b;
    if (S.b_off < 0 || S.n_b < 0 || S.b_off + S.n_b > n_batches) continue;  // rejected below
    if (s > 0 && S.b_off == searches[s - 1].b_off && S.n_b == searches[s - 1].n_b) continue;  // same list as the last
    for (int j = 1; j < S.n_b; ++j)
      if (batches[S.b_off + j] < batches[S.b_off + j - 1]) c->batches_sorted = false;
  }
  int64_t raw = 0, tails = 0, plans = 0, cells = 0, qts = 0, dss = 0;
  for (int s = 0; s < n_search; ++s) {
    const lc_search_desc& S = searches[s];
    if (S.n_b < 0 || S.b_off < 0 || S.b_off + S.n_b > n_batches) return fail(LC_ERR_ARG, "batch range out of bounds");
    if (S.n_budgets < 0 || S.n_budgets > LC_MAX_BUDGETS) return fail(LC_ERR_ARG, "too many gpu budgets");
    if (S.load >= n_loads) return fail(LC_ERR_ARG, "load index out of range");
    if (S.prefill_cap > 64 || S.decode_cap > 64) return fail(LC_ERR_ARG, "pool caps above 64 are not supported");
    SearchMeta& M = c->hmeta[s];
    M.raw_off = raw;
    M.n_raw = (int64_t)sp->n_combos * S.n_b;
    raw += M.n_raw;
    M.cell_off = cells;
    cells += (int64_t)sp->n_tmpl * S.n_b;
    M.qt_off[0] = M.qt_off[1] = M.qt_off[2] = M.qt_off[3] = 0;
    M.n_steps = ((S.modes & 1) && S.osl > 1) ? (int32_t)((S.osl - 1 + static_stride(S) - 1) / static_stride(S)) : 0;
    M.tail_off[0] = M.tail_off[1] = M.tail_off[2] = 0;
    M.plan_off = (int32_t)plans;
    const int pc = ((S.modes & 4) && !(S.modes & LC_MODE_NO_PLANS)) ? S.prefill_cap * S.decode_cap : 0;
    if (pc > 256) return fail(LC_ERR_ARG, "prefill_cap * decode_cap above 256 is not supported");
    M.plan_cap = pc;
    plans += pc;
  }
  // unit / cell / plan positions are int32 on the device (K0 scan, unit_off, n_units)
  if (raw > INT32_MAX || cells > INT32_MAX || plans > INT32_MAX)
    return fail(LC_ERR_ARG, "batch too large: more than 2^31-1 raw candidate tuples (or cells, plan slots) in one "
                            "lc_search_batch call; split the workloads over several calls");
  // MoE tail tables, shared between searches with the same inputs
  c->htables.clear();
  if (sp->is_moe) {
    // batch lists are identified by (b_off, n_b): callers that pass one copy per
    // distinct list (the Python engine does) get full sharing
    std::map<Key5, int32_t> tindex;  // (type, b_off, n_b, load, chunk) -> table
    const int64_t per_b = (int64_t)sp->n_tp * sp->n_ep;
    for (int s = 0; s < n_search; ++s) {
      const lc_search_desc& S = searches[s];
      const int32_t cb = S.b_off;
      for (int type = 0; type < 2; ++type) {
        const Key5 key = {type, cb, S.n_b, S.load, type == 0 ? S.isl - S.prefix : 0};
        auto jt = tindex.find(key);
        int32_t ti;
        if (jt == tindex.end()) {
          ti = (int32_t)c->htables.size();
          tindex[key] = ti;
          TailTable T;
          T.off = tails; T.type = type; T.search = s; T.b_off = cb; T.n_b = S.n_b; T.load = S.load; T._pad = 0;
          T.chunk = S.isl - S.prefix;
          c->htables.push_back(T);
          tails += per_b * S.n_b;
        } else {
          ti = jt->second;
        }
        c->hmeta[s].tail_off[type] = c->htables[ti].off;
      }
    }
  }
  // query-table groups per slot class (see QtGroup)
  c->hqt.clear();
  c->n_qt_2d = 0;
  {
    std::map<Key5, int32_t> gidx;
    for (int s = 0; s < n_search; ++s) {
      const lc_search_desc& S = searches[s];
      const int64_t cb = S.b_off;
      const bool need[4] = {(S.modes & 5) != 0, (S.modes & 7) != 0, (S.modes & 6) != 0, (S.modes & 2) != 0};
      for (int cl = 0; cl < 4; ++cl) {
        if (!need[cl] || !sp->class_n[cl]) continue;
        Key5 key;
        if (cl == 0) key = {0, S.isl - S.prefix, cb, S.n_b, S.load};
        else if (cl == 1) key = {1, cb, S.n_b, S.load, 0};
        else if (cl == 2) key = {2, S.isl + S.osl / 2, cb, S.n_b, 0};
        else key = {3, s, 0, 0, 0};
        auto jt = gidx.find(key);
        if (jt == gidx.end()) {
          gidx[key] = (int32_t)c->hqt.size();
          c->hqt.push_back(QtGroup{qts, cl, s, sp->class_n[cl], 0});
          c->n_qt_2d += (int64_t)sp->class_n2d[cl] * S.n_b;
          c->hmeta[s].qt_off[cl] = qts;
          qts += (int64_t)sp->class_n[cl] * S.n_b;
        } else {
          c->hmeta[s].qt_off[cl] = c->hqt[jt->second].off;
        }
      }
    }
  }
  // prefill step tables: one per class-0 query-table group
  c->hpg.clear();
  c->n_pstep = 0;
  for (int s = 0; s < n_search; ++s) c->hmeta[s].pstep_off = -1;
  {
    std::map<int64_t, int64_t> by_table;  // qt offset of the group's table -> pstep offset
    for (int s = 0; s < n_search; ++s) {
      const lc_search_desc& S = searches[s];
      if (!(S.modes & 5) || !sp->class_n[0]) continue;
      const int64_t key = c->hmeta[s].qt_off[0];
      auto it = by_table.find(key);
      if (it == by_table.end()) {
        by_table[key] = c->n_pstep;
        c->hpg.push_back(PGroup{c->n_pstep, s, S.n_b});
        c->hmeta[s].pstep_off = c->n_pstep;
        c->n_pstep += (int64_t)sp->n_tmpl * S.n_b;
      } else {
        c->hmeta[s].pstep_off = it->second;
      }
    }
  }
  // decode-series groups: the KV samples isl + 32k + 1 do not depend on osl
  c->hds.clear();
  {
    std::map<Key5, int32_t> gidx;
    for (int s = 0; s < n_search; ++s) {
      const lc_search_desc& S = searches[s];
      SearchMeta& M = c->hmeta[s];
      M.ds_off = 0;
      M.ds_stride = 0;
      if (!M.n_steps || !sp->n_gclass) continue;
      const int32_t cb = S.b_off;
      const Key5 key = {S.isl, cb, S.n_b, static_stride(S), 0};
      auto jt = gidx.find(key);
      int32_t gi;
      if (jt == gidx.end()) {
        gi = gidx[key] = (int32_t)c->hds.size();
        c->hds.push_back(DsGroup{0, S.isl, cb, S.n_b, 0, (int32_t)static_stride(S)});
      } else {
        gi = jt->second;
      }
      if (M.n_steps > c->hds[gi].n_steps) c->hds[gi].n_steps = M.n_steps;
      M._pad2 = gi;  // group index until offsets are known
    }
    // The attention latency depends on (batch, kv) only, so input lengths whose
    // KV samples continue one another (same batch list and stride, isl equal
    // modulo the stride, next first sample at most one stride past the last)
    // share one merged table: a search starts k0 samples into it.
    const size_t n_g = c->hds.size();
    std::vector<int32_t> ord(n_g), to(n_g);
    std::vector<int64_t> k0(n_g, 0);
    for (size_t i = 0; i < n_g; ++i) ord[i] = (int32_t)i;
    auto gkey = [&](const DsGroup& g) {
      return std::make_tuple(g.b_off, g.n_b, g.stride, g.isl % g.stride, g.isl);
    };
    std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return gkey(c->hds[a]) < gkey(c->hds[b]); });
    std::vector<DsGroup> merged;
    for (int32_t i : ord) {
      const DsGroup& g = c->hds[i];
#ifndef LC_DS_NOMERGE
      if (!merged.empty()) {
#else
      if (false) {
#endif
        DsGroup& m = merged.back();
        if (m.b_off == g.b_off && m.n_b == g.n_b && m.stride == g.stride && m.isl % m.stride == g.isl % g.stride &&
            g.isl <= m.isl + (int64_t)m.stride * m.n_steps) {
          const int64_t k = (g.isl - m.isl) / m.stride;
          if (k + g.n_steps > m.n_steps) m.n_steps = (int32_t)(k + g.n_steps);
          to[i] = (int32_t)merged.size() - 1;
          k0[i] = k;
          continue;
        }
      }
      to[i] = (int32_t)merged.size();
      merged.push_back(g);
    }
    c->hds.swap(merged);
    for (auto& g : c->hds) {
      g.off = dss;
      dss += (int64_t)sp->n_gclass * g.n_b * g.n_steps;
    }
    for (int s = 0; s < n_search; ++s) {
      SearchMeta& M = c->hmeta[s];
      if (!M.n_steps || !sp->n_gclass) continue;
      const DsGroup& G = c->hds[to[M._pad2]];
      M.ds_off = G.off + k0[M._pad2] * G.n_b;
      M.ds_stride = G.n_steps;
    }
  }
  // static decode series: searches that differ only in osl share one loop (SeriesGroup)
  c->hsg.clear();
  c->hsm.clear();
  c->n_series = 0;
  if (sp->n_gclass) {
    std::map<Key5, std::vector<int32_t>> members;
    std::vector<Key5> order;
    for (int s = 0; s < n_search; ++s) {
      const lc_search_desc& S = searches[s];
      if (!c->hmeta[s].n_steps) continue;
      const Key5 key = {S.isl, S.b_off, S.n_b, S.load, static_stride(S)};
      auto it = members.find(key);
      if (it == members.end()) { order.push_back(key); members[key] = {s}; }
      else it->second.push_back(s);
    }
    for (const auto& key : order) {
      std::vector<int32_t>& ms = members[key];
      std::stable_sort(ms.begin(), ms.end(), [&](int32_t a, int32_t b) { return c->hmeta[a].n_steps < c->hmeta[b].n_steps; });
      SeriesGroup g;
      g.off = c->n_series;
      g.rep = ms[0];
      g.m_off = (int32_t)c->hsm.size();
      g.n_m = (int32_t)ms.size();
      g._pad = 0;
      for (int32_t s : ms) c->hsm.push_back(SeriesMember{s, c->hmeta[s].n_steps});
      c->hsg.push_back(g);
      c->n_series += (int64_t)sp->n_tmpl * searches[ms[0]].n_b;
    }
  }
  // dense mixed-step region: tokens = chunk_tokens + n_mix_gen <= context + batch
  c->n_pd_tails = tails;
  c->m_tmax = 0;
  int64_t marks = 0;
  int32_t last_boff = -1, last_nb = -1;
  int64_t last_bmax = 0;
  for (int s = 0; s < n_search; ++s) {
    const lc_search_desc& S = searches[s];
    c->hmeta[s].mark_off = marks;
    marks += S.n_b;
    if (!sp->is_moe || !(S.modes & 2) || S.n_b == 0) continue;
    if (S.b_off != last_boff || S.n_b != last_nb) {  // searches sharing a batch list share its maximum
      last_bmax = 0;
      for (int j = 0; j < S.n_b; ++j) last_bmax = batches[S.b_off + j] > last_bmax ? batches[S.b_off + j] : last_bmax;
      last_boff = S.b_off;
      last_nb = S.n_b;
    }
    const int64_t bmax = last_bmax;
    const int64_t t = (S.isl - S.prefix) + bmax;
    c->m_tmax = t > c->m_tmax ? t : c->m_tmax;
  }
  c->n_marks = marks;
  if (sp->is_moe && n_loads > 0 && c->m_tmax > 0) tails += (int64_t)n_loads * sp->n_tp * sp->n_ep * (c->m_tmax + 1);
  c->n_raw = raw;
  c->n_cells = cells;
  if (qts > INT32_MAX || dss > INT32_MAX)
    return fail(LC_ERR_ARG, "batch too large: more than 2^31-1 query-table entries in one lc_search_batch call; "
                            "split the workloads over several calls");
  c->n_qt = qts;
  c->n_ds = dss;
  c->n_tails = tails;
  {
    // the deduplicated K3 packs (load, pooled tokens) into 64 bits: loads < 2^16,
    // pooled = tokens * max(1, ep / tp) < 2^48 (bounded in doubles: no overflow)
    double max_b = 1.0, max_chunk = 1.0;
    const double max_ep = (double)sp->max_ep_h;
    for (int32_t i = 0; i < n_batches; ++i) max_b = std::max(max_b, (double)batches[i]);
    for (int s = 0; s < n_search; ++s) max_chunk = std::max(max_chunk, (double)(searches[s].isl - searches[s].prefix));
    const double max_tok = std::max(max_b * max_chunk, (double)c->m_tmax);
    static const bool general = getenv("LC_TAILS_GENERAL") != nullptr;  // tests: force the general K3
    c->tails_dedup_ok = !general && n_loads < 65536 && max_tok * max_ep < 1e14 && sp->n_ep <= 64 &&
                        tails <= (1 << 24);
  }
  c->n_plan_slots = plans;
  cudaError_t err = cudaSuccess;
  c->hbatch_code.resize(n_batches > 0 ? n_batches : 1);
  for (int32_t i = 0; i < n_batches; ++i) {
    if (batches[i] > LC_KEY_BATCH_MAX) return fail(LC_ERR_ARG, "batch sizes above 9999999999 are not supported");
    c->hbatch_code[i] = lc_batch_code(batches[i] > 0 ? batches[i] : 1);
  }
  c->psteps.get<PStep>((size_t)c->n_pstep, &err);
  c->sd.get<SdOut>(c->n_series ? (size_t)cells : 0, &err);
  c->results.get<lc_search_result>(n_search, &err);
  if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(err));
  // inputs go through one page-locked arena so every H2D copy is asynchronous
  {
    const size_t sizes[11] = {sizeof(lc_search_desc) * n_search, sizeof(int64_t) * n_batches,
                             (n_loads && sp->n_experts) ? sizeof(double) * n_loads * 2 * sp->n_experts : 0,
                             sizeof(SearchMeta) * n_search, sizeof(TailTable) * c->htables.size(),
                             sizeof(DsGroup) * c->hds.size(), sizeof(QtGroup) * c->hqt.size(),
                             sizeof(SeriesGroup) * c->hsg.size(), sizeof(SeriesMember) * c->hsm.size(),
                             sizeof(PGroup) * c->hpg.size(), sizeof(uint64_t) * n_batches};
    const void* srcs[11] = {searches, batches, loads, c->hmeta.data(), c->htables.data(), c->hds.data(),
                            c->hqt.data(), c->hsg.data(), c->hsm.data(), c->hpg.data(), c->hbatch_code.data()};
    // one device block holds all eleven inputs at the arena's offsets, so a single
    // H2D copy moves them (the buffers are views into it)
    DBuf* bufs[11] = {&c->searches, &c->batches, &c->loads, &c->meta, &c->tail_tables, &c->ds_groups,
                      &c->qt_groups, &c->sgroups, &c->smembers, &c->pgroups, &c->batch_code};
    size_t offs[11], tot = 0;
    for (int k = 0; k < 11; ++k) {
      offs[k] = tot;
      const size_t a = (sizes[k] + 255) & ~(size_t)255;
      tot += a ? a : 256;  // an empty input still gets a valid (unused) address
    }
    unsigned char* base = c->inputs.get<unsigned char>(tot, &err);
    if (err != cudaSuccess) return fail(LC_ERR_CUDA, std::string("input allocation: ") + cudaGetErrorString(err));
    for (int k = 0; k < 11; ++k) bufs[k]->set_view(base + offs[k], (sizes[k] + 255) & ~(size_t)255);
    size_t need = tot;
    need += (sizeof(lc_search_result) + sizeof(SearchMeta)) * (size_t)n_search + 1024;  // summaries coming back
    if (c->arena_cap < need) {
      if (c->arena) cudaFreeHost(c->arena);
      c->arena = nullptr;
      c->arena_cap = 0;
      CK(cudaHostAlloc((void**)&c->arena, need, cudaHostAllocDefault));
      c->arena_cap = need;
    }
    for (int k = 0; k < 11; ++k)
      if (sizes[k]) memcpy(c->arena + offs[k], srcs[k], sizes[k]);
    CK(cudaMemcpyAsync(base, c->arena, tot, cudaMemcpyHostToDevice, c->stream));
    c->arena_used = tot;
  }
  const double t_plan = host_timing ? ms_since(t_in) : 0.0;
  int rc = launch_pipeline(c, totals);
  if (rc) return rc;
  const double t_launch = host_timing ? ms_since(t_in) : 0.0;
  // compact fronts and plan slots ride the same synchronisation as the summaries
  // (page-locked staging; lc_fetch then serves them from host memory)
  c->staged = false;
  if (n_search) {
    const size_t need_f = (size_t)n_search * kCompactFront;
    if (c->pinned_front_cap < need_f) {
      if (c->pinned_front) cudaFreeHost(c->pinned_front);
      c->pinned_front = nullptr;
      c->pinned_front_cap = 0;
      CK(cudaHostAlloc((void**)&c->pinned_front, need_f * 8, cudaHostAllocDefault));
      c->pinned_front_cap = need_f;
    }
    const size_t need_p = (size_t)(c->n_plan_slots > 0 ? c->n_plan_slots : 1);
    if (c->pinned_plans_cap < need_p) {
      if (c->pinned_plans_i) cudaFreeHost(c->pinned_plans_i);
      if (c->pinned_plans_d) cudaFreeHost(c->pinned_plans_d);
      c->pinned_plans_i = nullptr;
      c->pinned_plans_d = nullptr;
      c->pinned_plans_cap = 0;
      CK(cudaHostAlloc((void**)&c->pinned_plans_i, need_p * 4 * sizeof(int32_t), cudaHostAllocDefault));
      CK(cudaHostAlloc((void**)&c->pinned_plans_d, need_p * 6 * sizeof(double), cudaHostAllocDefault));
      c->pinned_plans_cap = need_p;
    }
    CK(cudaMemcpyAsync(c->pinned_front, c->front_compact.p, need_f * 8, cudaMemcpyDeviceToHost, c->stream));
    if (c->n_plan_slots) {
      CK(cudaMemcpyAsync(c->pinned_plans_i, c->plans_i.p, (size_t)c->n_plan_slots * 4 * sizeof(int32_t),
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(c->pinned_plans_d, c->plans_d.p, (size_t)c->n_plan_slots * 6 * sizeof(double),
                         cudaMemcpyDeviceToHost, c->stream));
    }
    c->staged = true;
  }
  c->hres.resize(n_search);
  unsigned char* back = c->arena + c->arena_used;  // page-locked landing zone for the summaries
  lc_search_result* pres = (lc_search_result*)back;
  SearchMeta* pmeta = (SearchMeta*)(back + ((sizeof(lc_search_result) * (size_t)n_search + 255) & ~(size_t)255));
  int32_t* ptotal = (int32_t*)((unsigned char*)pmeta + ((sizeof(SearchMeta) * (size_t)n_search + 255) & ~(size_t)255));
  if (n_search) {
    CK(cudaMemcpyAsync(pres, c->results.p, sizeof(lc_search_result) * n_search, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(pmeta, c->meta.p, sizeof(SearchMeta) * n_search, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaMemcpyAsync(ptotal, (const int32_t*)c->block_sums.p + c->n_total_idx, sizeof(int32_t),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (host_timing)
    fprintf(stderr, "lc_search_batch: %d searches, planned %.3f ms, launched %.3f ms, synchronised %.3f ms\n",
            n_search, t_plan, t_launch, ms_since(t_in));
  if (n_search) {
    memcpy(c->hres.data(), pres, sizeof(lc_search_result) * n_search);
    memcpy(c->hmeta.data(), pmeta, sizeof(SearchMeta) * n_search);
  }
  const int32_t total_units = *ptotal;
  c->n_units = total_units;
  int64_t nfront = 0, nplan = 0;
  for (int s = 0; s < n_search; ++s) {
    lc_search_result& R = c->hres[s];
    R.unit_off = c->hmeta[s].unit_off;
    R.n_units = c->hmeta[s].n_units;
    R.plan_off = c->hmeta[s].plan_off;
    nfront += R.n_front;
    nplan += R.n_plans;
  }
  if (results && n_search) memcpy(results, c->hres.data(), sizeof(lc_search_result) * n_search);
  if (totals) {
    memset(totals, 0, sizeof(*totals));
    totals->n_units = c->n_units;
    totals->n_plans = nplan;
    totals->n_front = nfront;
    totals->n_raw = c->n_raw;
    totals->n_launches = c->launches;
    totals->n_table_queries = c->n_qt + c->n_ds;
    totals->n_table_queries_2d = c->n_qt_2d + c->n_ds;
    totals->n_cells = c->n_cells;
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]); totals->kernel_ms[0] = ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]); totals->kernel_ms[1] = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]); totals->kernel_ms[2] = ms;
    cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]); totals->kernel_ms[3] = ms;
    cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]); totals->kernel_ms[4] = ms;
    cudaEventElapsedTime(&ms, c->ev[5], c->ev[6]); totals->kernel_ms[5] = ms;
  }
  return LC_OK;
}

int lc_replay_last(lc_ctx* c, int32_t iters, lc_batch_totals* totals) {
  if (!c || !c->db || iters < 1) return fail(LC_ERR_STATE, "lc_replay_last: no previous batch");
  CK(cudaSetDevice(c->device));
  if (c->n_search == 0) {
    if (totals) memset(totals, 0, sizeof(*totals));
    return LC_OK;
  }
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    // inputs (descriptors, batches, loads, DB, plan) are resident: K0 .. K4 only
    CK(cudaEventRecord(c->ev[0], c->stream));
    c->launches = 0;
    int rc = run_enum(c);
    if (rc) return rc;
    rc = run_eval_pipeline(c, totals);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 6; ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, c->ev[k], c->ev[k + 1]);
      acc[k] += ms;
    }
  }
  if (totals) {
    for (int k = 0; k < 6; ++k) totals->kernel_ms[k] = (float)(acc[k] / iters);
    totals->n_units = c->n_units;
    totals->n_raw = c->n_raw;
    totals->n_launches = c->launches;
    totals->n_table_queries = c->n_qt + c->n_ds;
    totals->n_table_queries_2d = c->n_qt_2d + c->n_ds;
    totals->n_cells = c->n_cells;
  }
  return LC_OK;
}

int lc_replay_async(lc_ctx* c) {
  if (!c || !c->db) return fail(LC_ERR_STATE, "lc_replay_async: no previous batch");
  CK(cudaSetDevice(c->device));
  if (c->n_search == 0) return LC_OK;
  if (c->graph_ok) {  // inputs and workspace are unchanged: relaunch the batch's graph
    CK(cudaGraphLaunch(c->gexec, c->stream));
    return LC_OK;
  }
  return launch_pipeline(c, nullptr);
}

static DbView db_view(const lc_db* db) {
  DbView V;
  V.grids = db->grids; V.axv = db->axv; V.axl = db->axl; V.cell = db->cell; V.clog = db->clog;
  V.logtab = db->logtab; V.exptab = db->exptab;
  V.mem_bw = db->mem_bw; V.intra_bw = db->intra_bw; V.inter_bw = db->inter_bw; V.gpu_memory = db->gpu_memory;
  for (int i = 0; i < 4; ++i) V.compute[i] = db->compute[i];
  V.gpn = db->gpn; V.policy = db->policy;
  return V;
}

int lc_query_batch(lc_ctx* c, const lc_db* db, int32_t n, const lc_query* queries, double* latency_us,
                   int32_t* status) {
  if (!c || !db || n < 0 || (n > 0 && (!queries || !latency_us || !status)))
    return fail(LC_ERR_ARG, "lc_query_batch: bad argument");
  if (n == 0) return LC_OK;
  CK(cudaSetDevice(c->device));
  for (int32_t i = 0; i < n; ++i) {
    const lc_query& q = queries[i];
    if (q.grid >= db->n_grids || q.kind < 0 || q.kind > LC_KIND_EMBEDDING || q.quant < 0 || q.quant > 3 ||
        q.policy < -1 || q.policy > LC_POLICY_SOL)
      return fail(LC_ERR_ARG, "lc_query_batch: query " + std::to_string(i) + " out of range");
  }
  cudaError_t e = cudaSuccess;
  lc_query* dq = c->q_in.get<lc_query>(n, &e);
  double* dlat = c->q_lat.get<double>(n, &e);
  int32_t* dst = c->q_st.get<int32_t>(n, &e);
  if (e != cudaSuccess) return fail(LC_ERR_CUDA, std::string("lc_query_batch: ") + cudaGetErrorString(e));
  CK(cudaMemcpyAsync(dq, queries, sizeof(lc_query) * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  const DbView V = db_view(db);
  const int threads = 128;
  const int blocks = (int)std::min<int64_t>(((int64_t)n + threads - 1) / threads, 148 * 16);
  k_query<<<blocks, threads, 0, c->stream>>>(V, n, dq, dlat, dst);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(latency_us, dlat, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(status, dst, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LC_OK;
}

int lc_step_latency(lc_ctx* c, const lc_db* db, const lc_space* sp, int32_t n, const lc_step_req* reqs,
                    int32_t n_loads, const double* loads, lc_step_out* out) {
  if (!c || !db || !sp || n < 0 || (n > 0 && (!reqs || !out)) || n_loads < 0 || (n_loads > 0 && !loads))
    return fail(LC_ERR_ARG, "lc_step_latency: bad argument");
  if (n == 0) return LC_OK;
  for (int32_t i = 0; i < n; ++i) {
    const lc_step_req& r = reqs[i];
    if (r.tmpl < 0 || r.tmpl >= sp->n_tmpl || r.phase < 0 || r.phase > 2 || r.n_ctx < 0 || r.n_gen < 0 ||
        r.seq < 1 || r.load >= n_loads || (r.phase == PH_PREFILL && r.n_ctx % r.seq))
      return fail(LC_ERR_ARG, "lc_step_latency: request " + std::to_string(i) + " out of range");
  }
  CK(cudaSetDevice(c->device));
  cudaError_t e = cudaSuccess;
  lc_step_req* dreq = c->step_in.get<lc_step_req>(n, &e);
  lc_step_out* dout = c->step_out.get<lc_step_out>(n, &e);
  double* dload = c->step_loads.get<double>(n_loads > 0 ? (size_t)n_loads * 2 * sp->n_experts : 1, &e);
  if (e != cudaSuccess) return fail(LC_ERR_CUDA, std::string("lc_step_latency: ") + cudaGetErrorString(e));
  CK(cudaMemcpyAsync(dreq, reqs, sizeof(lc_step_req) * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  if (n_loads > 0)
    CK(cudaMemcpyAsync(dload, loads, sizeof(double) * (size_t)n_loads * 2 * sp->n_experts, cudaMemcpyHostToDevice,
                       c->stream));
  StepView T;
  T.entries = sp->entries; T.tmpl_n = sp->tmpl_n; T.tmpl_info = sp->tmpl_info;
  T.hidden = sp->hidden; T.topk = sp->topk; T.n_experts = sp->n_experts; T.is_moe = sp->is_moe;
  T.n_tmpl = sp->n_tmpl;
  const DbView V = db_view(db);
  const int blocks = (int)std::min<int64_t>(((int64_t)n + 3) / 4, 148 * 8);
  if (sp->n_experts <= 128) k_step<4><<<blocks, 128, 0, c->stream>>>(V, T, n, dreq, dload, dout);
  else if (sp->n_experts <= 256) k_step<8><<<blocks, 128, 0, c->stream>>>(V, T, n, dreq, dload, dout);
  else k_step<32><<<blocks, 128, 0, c->stream>>>(V, T, n, dreq, dload, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, dout, sizeof(lc_step_out) * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LC_OK;
}

int lc_dbgen(lc_ctx* c, const lc_dbgen_desc* g, double* latency_us, double* latency_log, int32_t* status) {
  if (!c || !g || !latency_us || !latency_log || !status || g->n_grids < 0 || g->n_cells < 0)
    return fail(LC_ERR_ARG, "lc_dbgen: bad argument");
  for (int32_t i = 0; i < g->n_grids; ++i) status[i] = 0;
  if (g->n_cells == 0 || g->n_grids == 0) return LC_OK;
  int64_t expect = 0;
  for (int32_t i = 0; i < g->n_grids; ++i) {
    const lc_gen_grid& G = g->grids[i];
    if (G.n_axes < 1 || G.n_axes > 2 || G.kind < 0 || G.kind > LC_KIND_EMBEDDING || G.quant < 0 || G.quant > 3 ||
        G.cell_off != expect)
      return fail(LC_ERR_ARG, "lc_dbgen: grid " + std::to_string(i) + " malformed");
    int64_t cells = 1;
    for (int a = 0; a < G.n_axes; ++a) {
      if (G.axis_len[a] < 1 || G.axis_off[a] < 0 || G.axis_off[a] + G.axis_len[a] > g->n_axis ||
          G.axis_dim[a] < 0 || G.axis_dim[a] > 4)
        return fail(LC_ERR_ARG, "lc_dbgen: grid " + std::to_string(i) + " axis out of range");
      cells *= G.axis_len[a];
    }
    expect += cells;
  }
  if (expect != g->n_cells) return fail(LC_ERR_ARG, "lc_dbgen: n_cells does not match the grids");
  CK(cudaSetDevice(c->device));
  lc_gen_grid* dg = nullptr; int64_t* dax = nullptr; double* dterm = nullptr; double* dlogtab = nullptr;
  double* dlat = nullptr; double* dlog = nullptr; int32_t* dst = nullptr;
  int rc = 0;
  if ((rc = upload(&dg, g->grids, (size_t)g->n_grids, c->stream)) || (rc = upload(&dax, g->axis_val, (size_t)g->n_axis, c->stream)) ||
      (rc = upload(&dterm, g->axis_term, (size_t)g->n_axis, c->stream)) ||
      (rc = upload(&dlogtab, LOG_TAB_H, 256, c->stream))) {
    cudaFree(dg); cudaFree(dax); cudaFree(dterm); cudaFree(dlogtab);
    return rc;
  }
  cudaError_t e = cudaMalloc(&dlat, sizeof(double) * (size_t)g->n_cells);
  if (e == cudaSuccess) e = cudaMalloc(&dlog, sizeof(double) * (size_t)g->n_cells);
  if (e == cudaSuccess) e = cudaMalloc(&dst, sizeof(int32_t) * (size_t)g->n_grids);
  if (e == cudaSuccess) e = cudaMemsetAsync(dst, 0, sizeof(int32_t) * (size_t)g->n_grids, c->stream);
  if (e == cudaSuccess) {
    DbView V;
    memset(&V, 0, sizeof(V));
    V.logtab = dlogtab;
    V.mem_bw = g->mem_bandwidth; V.intra_bw = g->intra_node_bandwidth; V.inter_bw = g->inter_node_bandwidth;
    for (int i = 0; i < 4; ++i) V.compute[i] = g->compute[i];
    V.gpn = g->gpus_per_node;
    const int64_t blocks = std::min<int64_t>((g->n_cells + 255) / 256, 148 * 16);
    k_dbgen<<<(int)blocks, 256, 0, c->stream>>>(V, dg, g->n_grids, dax, dterm, g->n_cells, g->amplitude, dlat, dlog, dst);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(latency_us, dlat, sizeof(double) * (size_t)g->n_cells, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(latency_log, dlog, sizeof(double) * (size_t)g->n_cells, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(status, dst, sizeof(int32_t) * (size_t)g->n_grids, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dg); cudaFree(dax); cudaFree(dterm); cudaFree(dlogtab); cudaFree(dlat); cudaFree(dlog); cudaFree(dst);
  if (e != cudaSuccess) return fail(LC_ERR_CUDA, std::string("lc_dbgen: ") + cudaGetErrorString(e));
  return LC_OK;
}

int lc_set_raw_filter(lc_ctx* c, int64_t lo, int64_t hi, const uint8_t* mask) {
  if (!c) return fail(LC_ERR_ARG, "lc_set_raw_filter: NULL context");
  c->graph_ok = false;  // the next pipeline run enumerates under the new filter
  if (hi < 0) {
    c->filt_lo = 0; c->filt_hi = -1; c->filt_mask = false;
    return LC_OK;
  }
  if (lo < 0 || hi < lo) return fail(LC_ERR_ARG, "lc_set_raw_filter: need 0 <= lo <= hi");
  CK(cudaSetDevice(c->device));
  c->filt_lo = lo; c->filt_hi = hi; c->filt_mask = mask != nullptr;
  if (mask && hi > lo) {
    cudaError_t e = cudaSuccess;
    uint8_t* d = c->raw_mask.get<uint8_t>((size_t)(hi - lo), &e);
    if (e != cudaSuccess) return fail(LC_ERR_CUDA, std::string("lc_set_raw_filter: ") + cudaGetErrorString(e));
    CK(cudaMemcpyAsync(d, mask, (size_t)(hi - lo), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return LC_OK;
}

int lc_fetch_pools(lc_ctx* c, int32_t* pool_units, int32_t* pool_counts) {
  if (!c || !c->db) return fail(LC_ERR_STATE, "lc_fetch_pools: no previous batch");
  CK(cudaSetDevice(c->device));
  if (pool_units && c->n_search)
    CK(cudaMemcpyAsync(pool_units, c->pool_sel.p, sizeof(int32_t) * 128 * (size_t)c->n_search,
                       cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (pool_counts)
    for (int s = 0; s < c->n_search; ++s) {
      pool_counts[2 * s] = c->hmeta[s].n_pre;
      pool_counts[2 * s + 1] = c->hmeta[s].n_dec;
    }
  return LC_OK;
}

int lc_unit_raw(lc_ctx* c, int32_t n, const int32_t* units, int64_t* raw) {
  if (!c || !c->db) return fail(LC_ERR_STATE, "lc_unit_raw: no previous batch");
  if (n < 0 || (n > 0 && (!units || !raw))) return fail(LC_ERR_ARG, "lc_unit_raw: bad argument");
  if (n == 0) return LC_OK;
  CK(cudaSetDevice(c->device));
  cudaError_t e = cudaSuccess;
  int32_t* du = c->q_st.get<int32_t>(n, &e);
  int64_t* dr = (int64_t*)c->q_lat.get<double>(n, &e);
  if (e != cudaSuccess) return fail(LC_ERR_CUDA, std::string("lc_unit_raw: ") + cudaGetErrorString(e));
  CK(cudaMemcpyAsync(du, units, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  k_unit_raw<<<(n + 127) / 128, 128, 0, c->stream>>>((const SearchMeta*)c->meta.p, (const lc_search_desc*)c->searches.p,
                                                     (const int32_t*)c->u_search.p, (const int32_t*)c->u_combo.p,
                                                     (const int32_t*)c->u_batch.p, (int32_t)c->n_units, n, du, dr);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(raw, dr, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LC_OK;
}

// ---- report rows (host): the "rows" / "frontier" lists of SearchReport.to_json()
static bool put_row(lcr::Out& o, const lc_report_cols* c, int64_t i, int depth, bool flags) {
  using lcr::Out;
  char f[4][40];
  const double vals[4] = {c->thru[i], c->tpot[i], c->ttft[i], c->mode[i] == 2 ? c->r_sys[i] : 0.0};
  for (int k = 0; k < 4; ++k) {
    if (!std::isfinite(vals[k])) return false;
    lcr::py_repr(vals[k], f[k]);
  }
  char sp[40];
  if (std::isfinite(c->speed[i])) lcr::py_repr(c->speed[i], sp);
  else strcpy(sp, "null");
  auto key = [&](const int64_t* g) {
    o.put("tp"); o.i64(g[0]); o.put("pp"); o.i64(g[1]); o.put("ep"); o.i64(g[2]); o.put("dp"); o.i64(g[3]);
    o.put("b"); o.i64(g[4]);
  };
  auto parallel = [&](const int64_t* g, int d) {  // opening brace at depth d
    o.put("{\n"); o.pad(d + 1); o.put("\"dp\": "); o.i64(g[3]); o.put(",\n");
    o.pad(d + 1); o.put("\"ep\": "); o.i64(g[2]); o.put(",\n");
    o.pad(d + 1); o.put("\"pp\": "); o.i64(g[1]); o.put(",\n");
    o.pad(d + 1); o.put("\"tp\": "); o.i64(g[0]); o.put("\n"); o.pad(d); o.put("}");
  };
  auto flag_lines = [&]() {
    if (!flags) return;
    o.pad(depth + 1); o.put(c->feasible[i] ? "\"feasible\": true,\n" : "\"feasible\": false,\n");
    o.pad(depth + 1); o.put(c->frontier[i] ? "\"frontier\": true,\n" : "\"frontier\": false,\n");
  };
  auto tail = [&]() {
    o.pad(depth + 1); o.put("\"speed\": "); o.puts(sp); o.put(",\n");
    o.pad(depth + 1); o.put("\"throughput_per_gpu\": "); o.puts(f[0]); o.put(",\n");
    o.pad(depth + 1); o.put("\"tpot_ms\": "); o.puts(f[1]); o.put(",\n");
    o.pad(depth + 1); o.put("\"ttft_ms\": "); o.puts(f[2]); o.put("\n");
    o.pad(depth); o.put("}");
  };
  o.put("{\n");
  if (c->mode[i] < 2) {
    const int64_t* g = c->cfg + 5 * i;
    static const char* modes[2] = {"static", "aggregated"};
    o.pad(depth + 1); o.put("\"batch\": "); o.i64(g[4]); o.put(",\n");
    o.pad(depth + 1); o.put("\"config\": \""); key(g); o.put("\",\n");
    flag_lines();
    o.pad(depth + 1); o.put("\"gpus\": "); o.i64(c->gpus[i]); o.put(",\n");
    o.pad(depth + 1); o.put("\"mode\": \""); o.puts(modes[c->mode[i]]); o.put("\",\n");
    o.pad(depth + 1); o.put("\"model\": "); o.puts(c->model_json); o.put(",\n");
    o.pad(depth + 1); o.put("\"parallel\": "); parallel(g, depth + 1); o.put(",\n");
    o.pad(depth + 1); o.put("\"runtime\": "); o.puts(c->runtime[depth + 1]); o.put(",\n");
    tail();
    return true;
  }
  const int64_t* pg = c->pcfg + 5 * i;
  const int64_t* dg = c->dcfg + 5 * i;
  auto side = [&](const int64_t* g, int64_t reps) {  // opening brace at depth + 1
    const int d = depth + 1;
    o.put("{\n");
    o.pad(d + 1); o.put("\"batch\": "); o.i64(g[4]); o.put(",\n");
    o.pad(d + 1); o.put("\"parallel\": "); parallel(g, d + 1); o.put(",\n");
    o.pad(d + 1); o.put("\"replicas\": "); o.i64(reps); o.put(",\n");
    o.pad(d + 1); o.put("\"runtime\": "); o.puts(c->runtime[d + 1]); o.put("\n");
    o.pad(d); o.put("}");
  };
  o.pad(depth + 1); o.put("\"config\": \"P:"); o.i64(c->x[i]); o.put("x"); key(pg); o.put("|D:"); o.i64(c->y[i]);
  o.put("x"); key(dg); o.put("\",\n");
  o.pad(depth + 1); o.put("\"decode\": "); side(dg, c->y[i]); o.put(",\n");
  flag_lines();
  o.pad(depth + 1); o.put("\"gpus\": "); o.i64(c->gpus[i]); o.put(",\n");
  o.pad(depth + 1); o.put("\"mode\": \"disaggregated\",\n");
  o.pad(depth + 1); o.put("\"prefill\": "); side(pg, c->x[i]); o.put(",\n");
  o.pad(depth + 1); o.put("\"r_sys\": "); o.puts(f[3]); o.put(",\n");
  tail();
  return true;
}

int64_t lc_report_rows(const lc_report_cols* c, const int64_t* rows, int64_t n_sel, int32_t depth, int32_t flags,
                       char* out, int64_t cap) {
  if (!c || depth < 0 || depth > 3 || n_sel < 0) {
    fail(LC_ERR_ARG, "lc_report_rows: bad argument");
    return -1;
  }
  lcr::Out o{out, 0, out ? cap : 0};
  const int64_t n = rows ? n_sel : c->n;
  if (n == 0) {
    o.put("[]");
    return o.n;
  }
  o.put("[\n");
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = rows ? rows[k] : k;
    if (i < 0 || i >= c->n) {
      fail(LC_ERR_ARG, "lc_report_rows: row index out of range");
      return -1;
    }
    o.pad(depth + 1);
    if (!put_row(o, c, i, depth + 1, flags != 0)) {
      fail(LC_ERR_ARG, "Out of range float values are not JSON compliant");
      return -2;
    }
    o.put(k + 1 < n ? ",\n" : "\n");
  }
  o.pad(depth);
  o.put("]");
  return o.n;
}

int lc_stream(lc_ctx* c, void** stream) {
  if (!c || !stream) return fail(LC_ERR_ARG, "lc_stream: NULL argument");
  *stream = (void*)c->stream;
  return LC_OK;
}

int lc_set_priority(lc_ctx* c, int priority) {
  if (!c) return fail(LC_ERR_ARG, "lc_set_priority: NULL context");
  CK(cudaSetDevice(c->device));
  int least = 0, greatest = 0;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  const int p = priority < greatest ? greatest : (priority > least ? least : priority);
  CK(cudaStreamSynchronize(c->stream));
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, p));
  CK(cudaStreamDestroy(c->stream));
  c->stream = s;
  // kernel nodes take their priority from the capturing stream: recapture
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
  c->graph_ok = false;
  return LC_OK;
}

int lc_fetch(lc_ctx* c, const lc_fetch_req* r) {
  if (!c || !r) return fail(LC_ERR_ARG, "lc_fetch: NULL argument");
  CK(cudaSetDevice(c->device));
  const int64_t n = c->n_units;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst || !bytes) return LC_OK;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return LC_OK;
  };
  int rc = 0;
  rc |= cp(r->unit_search, c->u_search.p, n * 4);
  rc |= cp(r->unit_combo, c->u_combo.p, n * 4);
  rc |= cp(r->unit_batch, c->u_batch.p, n * 4);
  rc |= cp(r->unit_in_budget, c->u_budget.p, n);
  rc |= cp(r->st_status, c->st_status.p, n * 4);
  rc |= cp(r->ag_status, c->ag_status.p, n * 4);
  rc |= cp(r->pf_status, c->pf_status.p, n * 4);
  rc |= cp(r->dc_status, c->dc_status.p, n * 4);
  const double* stv = (const double*)c->st_v.p;
  const double* agv = (const double*)c->ag_v.p;
  const double* pfv = (const double*)c->pf_v.p;
  const double* dcv = (const double*)c->dc_v.p;
  const int64_t m = c->n_cap;
  rc |= cp(r->st_ttft, stv, n * 8); rc |= cp(r->st_tpot, stv + m, n * 8);
  rc |= cp(r->st_speed, stv + 2 * m, n * 8); rc |= cp(r->st_thru, stv + 3 * m, n * 8);
  rc |= cp(r->ag_ttft, agv, n * 8); rc |= cp(r->ag_tpot, agv + m, n * 8);
  rc |= cp(r->ag_speed, agv + 2 * m, n * 8); rc |= cp(r->ag_thru, agv + 3 * m, n * 8);
  rc |= cp(r->pf_lat, pfv, n * 8); rc |= cp(r->pf_rate, pfv + m, n * 8);
  rc |= cp(r->dc_lat, dcv, n * 8); rc |= cp(r->dc_rate, dcv + m, n * 8);
  if (r->err_c0 || r->err_c1) {
    std::vector<int64_t> e(8 * m);
    if (m) CK(cudaMemcpyAsync(e.data(), c->err_c.p, 8 * m * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 4; ++k)
      for (int64_t u = 0; u < n; ++u) {
        if (r->err_c0) r->err_c0[4 * u + k] = e[(2 * k) * m + u];
        if (r->err_c1) r->err_c1[4 * u + k] = e[(2 * k + 1) * m + u];
      }
  }
  // plans and fronts are copied compactly per search
  std::vector<int32_t> pi_v;
  std::vector<double> pd_v;
  if (c->n_plan_slots && (r->plan_p || r->plan_d || r->plan_x || r->plan_y || r->plan_gpus || r->plan_r_sys ||
                          r->plan_ttft || r->plan_tpot || r->plan_speed || r->plan_thru)) {
    // staged: read the page-locked copies in place (only the used slots are touched)
    const int32_t* pi = c->pinned_plans_i;
    const double* pd = c->pinned_plans_d;
    if (!c->staged) {
      pi_v.resize(c->n_plan_slots * 4);
      pd_v.resize(c->n_plan_slots * 6);
      CK(cudaMemcpyAsync(pi_v.data(), c->plans_i.p, pi_v.size() * 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(pd_v.data(), c->plans_d.p, pd_v.size() * 8, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      pi = pi_v.data();
      pd = pd_v.data();
    }
    int64_t k = 0;
    for (int s = 0; s < c->n_search; ++s) {
      const lc_search_result& R = c->hres[s];
      for (int j = 0; j < R.n_plans; ++j, ++k) {
        const int64_t slot = R.plan_off + j;
        if (r->plan_p) r->plan_p[k] = pi[slot * 4 + 0];
        if (r->plan_d) r->plan_d[k] = pi[slot * 4 + 1];
        if (r->plan_x) r->plan_x[k] = pi[slot * 4 + 2];
        if (r->plan_y) r->plan_y[k] = pi[slot * 4 + 3];
        if (r->plan_gpus) r->plan_gpus[k] = (int64_t)pd[slot * 6 + 0];
        if (r->plan_r_sys) r->plan_r_sys[k] = pd[slot * 6 + 1];
        if (r->plan_ttft) r->plan_ttft[k] = pd[slot * 6 + 2];
        if (r->plan_tpot) r->plan_tpot[k] = pd[slot * 6 + 3];
        if (r->plan_speed) r->plan_speed[k] = pd[slot * 6 + 4];
        if (r->plan_thru) r->plan_thru[k] = pd[slot * 6 + 5];
      }
    }
  }
  if (r->front) {
    bool fits = true;
    for (int s = 0; s < c->n_search; ++s) fits &= c->hres[s].n_front <= kCompactFront;
    if (fits && c->n_search) {
      // copy only up to the longest front of each search row: rows are kCompactFront apart
      int32_t maxf = 0;
      for (int s = 0; s < c->n_search; ++s) maxf = c->hres[s].n_front > maxf ? c->hres[s].n_front : maxf;
      const size_t need = (size_t)c->n_search * kCompactFront;
      if (c->pinned_front_cap < need) {
        if (c->pinned_front) cudaFreeHost(c->pinned_front);
        CK(cudaHostAlloc((void**)&c->pinned_front, need * 8, cudaHostAllocDefault));
        c->pinned_front_cap = need;
      }
      if (maxf > 0 && !c->staged) {
        CK(cudaMemcpy2DAsync(c->pinned_front, kCompactFront * 8, c->front_compact.p, kCompactFront * 8,
                             (size_t)maxf * 8, c->n_search, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
      }
      int64_t k = 0;
      for (int s = 0; s < c->n_search; ++s) {
        memcpy(r->front + k, c->pinned_front + (size_t)s * kCompactFront, 8 * (size_t)c->hres[s].n_front);
        k += c->hres[s].n_front;
      }
    } else {
      int64_t k = 0;
      for (int s = 0; s < c->n_search; ++s) {
        const lc_search_result& R = c->hres[s];
        if (R.n_front)
          CK(cudaMemcpyAsync(r->front + k, (const int64_t*)c->front.p + R.front_off, R.n_front * 8,
                             cudaMemcpyDeviceToHost, c->stream));
        k += R.n_front;
      }
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  return rc ? LC_ERR_CUDA : LC_OK;
}

}  // extern "C"
