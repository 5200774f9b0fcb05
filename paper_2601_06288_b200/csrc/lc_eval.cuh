// Device-side restatement of the reference's per-operator latency model:
// grid lookup / log-log interpolation / extrapolation (perfdb.py:431-580),
// the per-step sum (estimator.py:71-95) and the serving-mode arithmetic
// (serving_modes.py:161-381).  Everything here is bit-exact with CPython on
// x86-64: operations are written in Python's left-to-right order and the
// translation unit is compiled with --fmad=false, so no product is fused
// unless an explicit fma() says so (only inside glibc_libm.cuh).
#pragma once
#include <stdint.h>
#include <math.h>
#include "../../include/llmconf_b200.h"
#include "glibc_libm.cuh"
#include "lc_fastdiv.cuh"

namespace lc {

__device__ __forceinline__ double quant_bytes(int q) {  // perfdb.py:25
  return q == 0 ? 2.0 : (q == 3 ? 0.5 : 1.0);
}

struct DevGrid {
  int32_t ndim;
  int32_t ax_off[2];
  int32_t ax_len[2];
  int32_t cell_off;
};

// Read-only view of the flattened database; every array lives in shared
// memory inside the evaluation kernels (≈35 KB for DeepSeek-V3).
struct DbView {
  const DevGrid* grids;
  const int64_t* axv;
  const double* axl;
  const double* cell;
  const double* clog;
  const double* logtab;
  const uint64_t* exptab;
  double mem_bw, intra_bw, inter_bw, gpu_memory;
  double compute[4];
  int32_t gpn, policy;
};

struct ErrRec {
  int32_t code;   // LC_ST_*
  int32_t label;  // failing entry's label
  int64_t c0, c1; // its interpolated coordinates
};

// CPython 3.12 builtin sum() over a float sequence with int start 0
// (bltinmodule.c: Neumaier compensation, compensation added if finite & nonzero).
struct NeumaierSum {
  double f, c;
  int n;
  __device__ __forceinline__ NeumaierSum() : f(0.0), c(0.0), n(0) {}
  __device__ __forceinline__ void add(double x) {
    if (n++ == 0) { f = 0.0 + x; return; }
    add_next(x);
  }
  // add() once a term has been added: the larger-magnitude operand is selected
  // before the compensation ((a - t) + b), so the branch costs selects instead
  // of both arms' subtractions on the FP64 pipe -- the same operations as
  // CPython's `if fabs(f) >= fabs(x)` arms.
  __device__ __forceinline__ void add_next(double x) {
    const double t = f + x;
    const bool fx = fabs(f) >= fabs(x);
    const double a = fx ? f : x, b = fx ? x : f;
    c += (a - t) + b;
    f = t;
  }
  __device__ __forceinline__ double result() const {
    return (c != 0.0 && isfinite(c)) ? f + c : f;
  }
};

__device__ __forceinline__ int lower_bound_i64(const int64_t* v, int n, int64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// _interp_cells (perfdb.py:509-536) for coordinates inside the box.  At most
// two axes, so the corners are spelled out (no dynamically indexed arrays):
// corner order is axis-major, lo before hi; a corner whose weight factor is
// exactly zero is skipped (t < 1.0 / t > 0.0); weights are the products of the
// per-axis factors (x * 1.0 == x, so exact axes need no special case).
__device__ __forceinline__ void axis_pos(const DbView& D, const DevGrid& G, int a, int64_t x, int* lo, int* hi,
                                         double* t, bool* exact, int* n_log_calls) {
  const int64_t* v = D.axv + G.ax_off[a];
  const double* lv = D.axl + G.ax_off[a];
  const int i = lower_bound_i64(v, G.ax_len[a], x);
  if (v[i] == x) {
    *lo = *hi = i;
    *t = 0.0;
    *exact = true;
  } else {
    *lo = i - 1;
    *hi = i;
    *exact = false;
    const double lx = glibc::log_fma((double)x, D.logtab);
    ++*n_log_calls;
    *t = (lx - lv[i - 1]) / (lv[i] - lv[i - 1]);
  }
}

__device__ __forceinline__ double interp_body(const DbView& D, const DevGrid G, int64_t c0, int64_t c1,
                                              int* n_log_calls) {
  int lo0, hi0, lo1 = 0, hi1 = 0;
  double t0, t1 = 0.0;
  bool ex0, ex1 = true;
  axis_pos(D, G, 0, c0, &lo0, &hi0, &t0, &ex0, n_log_calls);
  if (G.ndim == 2) axis_pos(D, G, 1, c1, &lo1, &hi1, &t1, &ex1, n_log_calls);
  const int n1 = G.ndim == 2 ? G.ax_len[1] : 1;
  const double* cells = D.cell + G.cell_off;
  const double* clogs = D.clog + G.cell_off;
  if (ex0 && ex1) return cells[lo0 * n1 + lo1];
  // corners present per axis: the lo side unless its factor (1 - t) is zero, the hi side if t > 0
  const bool a_lo = ex0 || t0 < 1.0, a_hi = !ex0 && t0 > 0.0;
  const bool b_lo = ex1 || t1 < 1.0, b_hi = !ex1 && t1 > 0.0;
  const double fa_lo = ex0 ? 1.0 : 1.0 - t0, fa_hi = t0;
  const double fb_lo = ex1 ? 1.0 : 1.0 - t1, fb_hi = t1;
  const bool p00 = a_lo && b_lo, p01 = a_lo && b_hi, p10 = a_hi && b_lo, p11 = a_hi && b_hi;
  const int i00 = lo0 * n1 + lo1, i01 = lo0 * n1 + hi1, i10 = hi0 * n1 + lo1, i11 = hi0 * n1 + hi1;
  const int first = p00 ? i00 : (p01 ? i01 : (p10 ? i10 : i11));
  const double v0 = cells[first];
  const int nc = (int)p00 + (int)p01 + (int)p10 + (int)p11;
  if (nc == 1) return v0;
  bool same = true;
  if (p00) same &= cells[i00] == v0;
  if (p01) same &= cells[i01] == v0;
  if (p10) same &= cells[i10] == v0;
  if (p11) same &= cells[i11] == v0;
  if (same) return v0;  // constant cells stay bit-exact
  NeumaierSum s;
  if (p00) s.add((fa_lo * fb_lo) * clogs[i00]);
  if (p01) s.add((fa_lo * fb_hi) * clogs[i01]);
  if (p10) s.add((fa_hi * fb_lo) * clogs[i10]);
  if (p11) s.add((fa_hi * fb_hi) * clogs[i11]);
  return glibc::exp_fma(s.result(), D.exptab);
}

__device__ __noinline__ double interp_cells(const DbView& D, const DevGrid G, int64_t c0, int64_t c1,
                                            int* n_log_calls) {
  return interp_body(D, G, c0, c1, n_log_calls);
}

// sol_estimate (perfdb.py:431-484); d is the canonical dim vector.
__device__ __noinline__ double sol_us(const DbView& D, int kind, int quant, const int64_t* d, int* st) {
  const double b = quant_bytes(quant);
  if (kind >= LC_KIND_ALLREDUCE && kind <= LC_KIND_P2P) {
    const int64_t n = d[1];
    const double link = n <= D.gpn ? D.intra_bw : D.inter_bw;
    double factor;
    if (kind == LC_KIND_ALLREDUCE) factor = 2.0 * (double)(n - 1) / (double)n;
    else if (kind == LC_KIND_P2P) factor = 1.0;
    else factor = (double)(n - 1) / (double)n;
    const double seconds = (double)d[0] * factor / link;
    return seconds * 1e6;
  }
  const double compute = D.compute[quant];
  if (!(compute > 0.0)) { *st = LC_ST_UNSUPPORTED; return 0.0; }
  double flops, bytes_moved;
  if (kind == LC_KIND_GEMM) {
    const int64_t m = d[0], n = d[1], k = d[2];
    flops = 2.0 * (double)m * (double)n * (double)k;
    bytes_moved = b * (double)(m * k + k * n + m * n);
  } else if (kind == LC_KIND_ATTN_CTX) {
    const int64_t B = d[0], s = d[1], H = d[2], KV = d[3], hd = d[4];
    flops = 2.0 * (double)B * (double)H * (double)s * (double)s * (double)hd;
    bytes_moved = b * (double)B * (double)s * (double)(2 * H + 2 * KV) * (double)hd;
  } else if (kind == LC_KIND_ATTN_GEN) {
    const int64_t B = d[0], kv = d[1], H = d[2], KV = d[3], hd = d[4];
    flops = 4.0 * (double)B * (double)H * (double)kv * (double)hd;
    bytes_moved = b * (double)B * (double)kv * 2.0 * (double)KV * (double)hd;
  } else if (kind == LC_KIND_MOE_GEMM) {
    const int64_t t = d[0], e = d[1], h = d[3], i = d[4];
    flops = 3.0 * 2.0 * (double)t * (double)h * (double)i;
    bytes_moved = b * (3.0 * (double)e * (double)h * (double)i + (double)(t * (h + i)));
  } else if (kind == LC_KIND_MOE_DISPATCH || kind == LC_KIND_MOE_COMBINE) {
    const double seconds = b * (double)d[0] * (double)d[2] * (double)d[3] / D.intra_bw;
    return seconds * 1e6;
  } else {  // embedding
    return b * (double)d[0] * (double)d[1] / D.mem_bw * 1e6;
  }
  const double a = flops / compute, c = bytes_moved / D.mem_bw;
  return (c > a ? c : a) * 1e6;
}

// query_latency (perfdb.py:539-580) for one query: grid id, kind, quant and the
// canonical dims d0..d4 (interpolated axes in d0, d1).  Everything is passed by
// value so callers keep their operands in registers.
template <bool INL>
__device__ __forceinline__ double query_body(const DbView& D, int32_t grid, int32_t kind, int32_t quant, int64_t d0,
                                             int64_t d1, int64_t d2, int64_t d3, int64_t d4, int* st, int* n_logs) {
  if (grid < 0) { *st = LC_ST_MISSING_KEY; return 0.0; }
  const DevGrid G = D.grids[grid];
  bool any_oob = false, any_above = false;
  int64_t cl0 = d0, cl1 = d1;
  {
    const int64_t* v = D.axv + G.ax_off[0];
    const int64_t lo = v[0], hi = v[G.ax_len[0] - 1];
    if (d0 < lo) { any_oob = true; cl0 = lo; }
    if (d0 > hi) { any_oob = any_above = true; cl0 = hi; }
  }
  if (G.ndim == 2) {
    const int64_t* v = D.axv + G.ax_off[1];
    const int64_t lo = v[0], hi = v[G.ax_len[1] - 1];
    if (d1 < lo) { any_oob = true; cl1 = lo; }
    if (d1 > hi) { any_oob = any_above = true; cl1 = hi; }
  }
  if (!any_oob) return INL ? interp_body(D, G, d0, d1, n_logs) : interp_cells(D, G, d0, d1, n_logs);
  if (D.policy == LC_POLICY_STRICT) { *st = LC_ST_EXTRAPOLATION; return 0.0; }
  const bool use_sol = D.policy == LC_POLICY_SOL || (D.policy == LC_POLICY_DEFAULT && any_above);
  if (D.policy == LC_POLICY_CLAMP || !use_sol) return interp_cells(D, G, cl0, cl1, n_logs);
  const double edge = interp_cells(D, G, cl0, cl1, n_logs);
  const int64_t de[5] = {cl0, G.ndim == 2 ? cl1 : d1, d2, d3, d4};
  const double sol_edge = sol_us(D, kind, quant, de, st);
  if (*st) return 0.0;
  const double eff = edge / sol_edge;
  const int64_t dq[5] = {d0, d1, d2, d3, d4};
  const double sol_q = sol_us(D, kind, quant, dq, st);
  if (*st) return 0.0;
  return sol_q * eff;
}

__device__ __noinline__ double query(const DbView& D, int32_t grid, int32_t kind, int32_t quant, int64_t d0,
                                    int64_t d1, int64_t d2, int64_t d3, int64_t d4, int* st, int* n_logs) {
  return query_body<false>(D, grid, kind, quant, d0, d1, d2, d3, d4, st, n_logs);
}

// the table kernels have one query site each: inline the common (inside-the-box) path there
#ifdef LC_NO_INLINE_TABLES
#define LC_TABLE_QUERY query
#else
#define LC_TABLE_QUERY query_body<true>
#endif

enum { PH_PREFILL = 0, PH_DECODE = 1, PH_MIXED = 2 };

struct StepArgs {
  int phase;
  int64_t n_ctx, n_gen, seq;
  int64_t expert_tokens;  // final expert_ffn token count for this step
};

// Fill the interpolated coordinates of entry e for a step; false if the entry
// is absent from this step's plan (context attention needs n_ctx > 0,
// generation attention n_gen > 0: model.py:327-357).
__device__ __forceinline__ bool entry_coords(const lc_entry& e, const StepArgs& a, int64_t hidden, int64_t* d) {
  d[0] = e.d[0]; d[1] = e.d[1]; d[2] = e.d[2]; d[3] = e.d[3]; d[4] = e.d[4];
  const int64_t tokens = a.n_ctx + a.n_gen;
  switch (e.coord) {
    case LC_COORD_TOKENS: d[0] = tokens; return true;
    case LC_COORD_MSG: d[0] = tokens * hidden * 2; return true;
    case LC_COORD_CTX:
      if (!a.n_ctx) return false;
      d[0] = a.phase == PH_MIXED ? 1 : a.n_ctx / a.seq;
      d[1] = a.phase == PH_MIXED ? a.n_ctx : a.seq;
      return true;
    case LC_COORD_GEN:
      if (!a.n_gen) return false;
      d[0] = a.n_gen; d[1] = a.seq;
      return true;
    default: d[0] = a.expert_tokens; return true;
  }
}

// derive_metrics (serving_modes.py:161-172)
__device__ __forceinline__ void derive_metrics(double ttft, double tpot, int64_t batch, int64_t osl, int64_t gpus,
                                               double* speed, double* thru) {
  *speed = tpot == 0.0 ? INFINITY : 1000.0 / tpot;
  const double req = ttft + (double)(osl - 1) * tpot;
  *thru = 1000.0 / req * (double)batch * (double)osl / (double)gpus;
}

// math.ceil(a / b) with float division (the reference's ceil(x / y) on ints);
// a power-of-two b divides by an exact multiply (the same correctly rounded value)
__device__ __forceinline__ int64_t ceil_div_f(int64_t a, int64_t b) {
  if (b > 0 && (b & (b - 1)) == 0 && b < (1ll << 52))
    return (int64_t)ceil((double)a * __longlong_as_double((long long)(1023 - (__ffsll(b) - 1)) << 52));
  return (int64_t)ceil((double)a / (double)b);
}

// Aggregated-mode schedule (serving_modes.py:292-320): returns status and the
// mixed-step shape.
struct AggSched {
  int32_t st;
  int64_t c_ctx, chunk_total, T, cpr, chunk_tokens, t_mix, t_gen, n_mix_gen, prefilling;
};

__device__ __forceinline__ AggSched agg_schedule(const lc_search_desc& S, int64_t b) {
  AggSched r;
  r.st = 0;
  r.chunk_total = S.isl - S.prefix;
  r.c_ctx = S.has_ctx_capacity ? S.ctx_capacity : (r.chunk_total > 2048 ? r.chunk_total : 2048);
  r.T = r.cpr = r.chunk_tokens = r.t_mix = r.t_gen = r.n_mix_gen = r.prefilling = 0;
  if (!S.chunked_prefill && r.chunk_total > r.c_ctx) { r.st = LC_ST_INFEASIBLE_CHUNK_OFF; return r; }
  r.T = ceil_div_f(r.chunk_total * b, r.c_ctx);
  r.cpr = ceil_div_f(r.chunk_total, r.c_ctx);
  r.chunk_tokens = r.c_ctx < r.chunk_total ? r.c_ctx : r.chunk_total;
  if (b == 1) {
    r.t_mix = 1; r.t_gen = S.osl - 1; r.n_mix_gen = 0;
  } else if (r.T >= S.osl) {
    int64_t n = (int64_t)((double)(b * S.osl) / (double)r.T);
    r.n_mix_gen = n > 1 ? n : 1;
    r.t_mix = S.osl; r.t_gen = 0;
  } else {
    r.prefilling = ceil_div_f(r.c_ctx, r.chunk_total);
    r.n_mix_gen = b - r.prefilling;
    if (r.n_mix_gen < 1) { r.st = LC_ST_INFEASIBLE_NO_DECODE_SLOT; return r; }
    r.t_mix = r.T; r.t_gen = S.osl - r.T;
  }
  return r;
}

// memory fit for one (combo, batch) (model.py:440-479)
__device__ __forceinline__ bool fits_memory(const lc_combo& c, const lc_search_desc& S, double gpu_memory,
                                            int64_t hidden, int64_t batch) {
  const int64_t cap = S.has_ctx_capacity ? S.ctx_capacity : 2048;
  const int64_t live = batch > cap ? batch : cap;
  const int64_t act = 4 * live * hidden * 2;
  const double overhead = 0.05 * gpu_memory + (double)act;
  const double stat = c.weight_bytes + overhead;
  if (stat > gpu_memory) return false;
  const double kv_budget = S.kv_mem_fraction * (gpu_memory - stat);
  const double kv_need = c.kv_token_bytes * (double)batch * (double)(S.isl + S.osl);
  return kv_need <= kv_budget;
}

__device__ __forceinline__ bool in_budget(const lc_search_desc& S, int64_t g) {
  if (S.n_budgets == 0) return true;
  for (int i = 0; i < S.n_budgets; ++i)
    if (S.budgets[i] == g) return true;
  return false;
}

// ---- config key strings (ParallelConfig.key, model.py:205-206) for tie-breaks
__device__ __forceinline__ int put_int(char* s, int64_t v) {
  char tmp[24];
  int n = 0;
  if (v == 0) tmp[n++] = '0';
  while (v > 0) { tmp[n++] = (char)('0' + v % 10); v /= 10; }
  for (int i = 0; i < n; ++i) s[i] = tmp[n - 1 - i];
  return n;
}

__device__ __forceinline__ int put_str(char* s, const char* t) {
  int n = 0;
  while (t[n]) { s[n] = t[n]; ++n; }
  return n;
}

__device__ __forceinline__ int fmt_cfg_key(char* s, const lc_combo& c, int64_t batch) {
  int n = 0;
  n += put_str(s + n, "tp"); n += put_int(s + n, c.tp);
  n += put_str(s + n, "pp"); n += put_int(s + n, c.pp);
  n += put_str(s + n, "ep"); n += put_int(s + n, c.ep);
  n += put_str(s + n, "dp"); n += put_int(s + n, c.dp);
  n += put_str(s + n, "b"); n += put_int(s + n, batch);
  s[n] = 0;
  return n;
}

__device__ __forceinline__ int str_cmp(const char* a, const char* b) {
  int i = 0;
  while (a[i] && a[i] == b[i]) ++i;
  return (int)(unsigned char)a[i] - (int)(unsigned char)b[i];
}

}  // namespace lc
