/* CPU ORACLE (test infrastructure only; see oracle.h).
 *
 * Plain-C restatement of the reference configuration search, function by
 * function, with the reference location each part follows.  Arithmetic keeps
 * CPython's left-to-right, unfused order (build with -ffp-contract=off), and
 * uses libm log/exp like CPython's math module.  Python's sum() over floats is
 * Neumaier-compensated in CPython >= 3.12; or_neumaier_sum restates it.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double QUANT_BYTES[4] = {2.0, 1.0, 1.0, 0.5}; /* perfdb.py:25 */
static const char* QUANT_NAME[4] = {"fp16", "fp8", "int8", "int4"};
static const char* KIND_NAME[OK_NKINDS] = {
    "gemm", "attention_context", "attention_generation", "allreduce", "allgather", "alltoall",
    "p2p", "moe_dispatch", "moe_combine", "moe_gemm", "embedding"};
static const char* ATTN_NAME[4] = {"", "MHA", "GQA", "MLA"};

/* canonical dim order per kind and which positions are interpolated axes
 * (perfdb.py:51-69).  Fixed dims are printed in sorted-name order in keys. */
typedef struct {
  int ndims;
  const char* names[5];
  int n_axes;
  int axes[2];
  int n_fixed;
  int fixed[4]; /* positions, sorted by name; attention adds attn_kind first */
} kind_info;

static const kind_info KINFO[OK_NKINDS] = {
    /* gemm m n k */ {3, {"m", "n", "k"}, 1, {0}, 2, {2, 1}},
    /* attn ctx */ {5, {"batch", "seq_len", "num_heads", "kv_heads", "head_dim"}, 2, {0, 1}, 3, {4, 3, 2}},
    /* attn gen */ {5, {"batch", "seq_len", "num_heads", "kv_heads", "head_dim"}, 2, {0, 1}, 3, {4, 3, 2}},
    /* allreduce */ {2, {"message_bytes", "participant_count"}, 1, {0}, 1, {1}},
    /* allgather */ {2, {"message_bytes", "participant_count"}, 1, {0}, 1, {1}},
    /* alltoall */ {2, {"message_bytes", "participant_count"}, 1, {0}, 1, {1}},
    /* p2p */ {2, {"message_bytes", "participant_count"}, 1, {0}, 1, {1}},
    /* dispatch */ {5, {"tokens", "experts", "topk", "hidden", "intermediate"}, 1, {0}, 4, {1, 3, 4, 2}},
    /* combine */ {5, {"tokens", "experts", "topk", "hidden", "intermediate"}, 1, {0}, 4, {1, 3, 4, 2}},
    /* moe_gemm */ {5, {"tokens", "experts", "topk", "hidden", "intermediate"}, 1, {0}, 4, {1, 3, 4, 2}},
    /* embedding */ {3, {"tokens", "hidden", "vocab"}, 1, {0}, 2, {1, 2}},
};

static int is_comm(int kind) { return kind >= OK_KIND_ALLREDUCE && kind <= OK_KIND_P2P; }
static int is_attn(int kind) { return kind == OK_KIND_ATTN_CTX || kind == OK_KIND_ATTN_GEN; }

/* ------------------------------------------------------------------------- */
/* CPython 3.12 builtin sum() over floats, start=0 (bltinmodule.c builtin_sum_impl) */
double or_neumaier_sum(const double* xs, int n) {
  if (n == 0) return 0.0;
  double f = 0.0 + xs[0]; /* int 0 + float */
  double c = 0.0;
  for (int i = 1; i < n; ++i) {
    double x = xs[i];
    double t = f + x;
    if (fabs(f) >= fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* ------------------------------------------------------------------------- */
/* grids (perfdb.py:283-355) */
typedef struct {
  int kind, quant, attn;
  int64_t fixed[4];
  int n_axes;
  int64_t* axis[2];
  int axis_len[2];
  double* cells; /* row-major, axis 0 major */
} grid;

typedef struct {
  const or_db* db;
  grid* grids;
  int n_grids;
  int kinds_present[OK_NKINDS];
} gridset;

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int grid_matches(const grid* g, int kind, int quant, int attn, const int64_t* fixed) {
  if (g->kind != kind || g->quant != quant || g->attn != attn) return 0;
  for (int i = 0; i < KINFO[kind].n_fixed; ++i)
    if (g->fixed[i] != fixed[i]) return 0;
  return 1;
}

static int find_grid(const gridset* gs, int kind, int quant, int attn, const int64_t* fixed) {
  for (int i = 0; i < gs->n_grids; ++i)
    if (grid_matches(&gs->grids[i], kind, quant, attn, fixed)) return i;
  return -1;
}

static int axis_index(const int64_t* vals, int n, int64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (vals[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo; /* bisect_left */
}

static void build_grids(const or_db* db, gridset* gs) {
  memset(gs, 0, sizeof(*gs));
  gs->db = db;
  gs->grids = (grid*)calloc((size_t)db->n + 1, sizeof(grid));
  int* owner = (int*)malloc(sizeof(int) * (size_t)db->n);
  for (int r = 0; r < db->n; ++r) {
    int kind = db->kind[r];
    const kind_info* ki = &KINFO[kind];
    int64_t fixed[4] = {0, 0, 0, 0};
    for (int i = 0; i < ki->n_fixed; ++i) fixed[i] = db->dims[r * 5 + ki->fixed[i]];
    int attn = is_attn(kind) ? db->attn[r] : 0;
    int g = find_grid(gs, kind, db->quant[r], attn, fixed);
    if (g < 0) {
      g = gs->n_grids++;
      grid* G = &gs->grids[g];
      G->kind = kind; G->quant = db->quant[r]; G->attn = attn;
      memcpy(G->fixed, fixed, sizeof(fixed));
      G->n_axes = ki->n_axes;
      gs->kinds_present[kind] = 1;
    }
    owner[r] = g;
  }
  for (int g = 0; g < gs->n_grids; ++g) {
    grid* G = &gs->grids[g];
    int cnt = 0;
    for (int r = 0; r < db->n; ++r) cnt += owner[r] == g;
    for (int a = 0; a < G->n_axes; ++a) {
      int64_t* v = (int64_t*)malloc(sizeof(int64_t) * (size_t)cnt);
      int m = 0;
      for (int r = 0; r < db->n; ++r)
        if (owner[r] == g) v[m++] = db->dims[r * 5 + KINFO[G->kind].axes[a]];
      qsort(v, (size_t)m, sizeof(int64_t), cmp_i64);
      int u = 0;
      for (int i = 0; i < m; ++i)
        if (u == 0 || v[u - 1] != v[i]) v[u++] = v[i];
      G->axis[a] = v;
      G->axis_len[a] = u;
    }
    int n1 = G->n_axes == 2 ? G->axis_len[1] : 1;
    G->cells = (double*)calloc((size_t)G->axis_len[0] * (size_t)n1, sizeof(double));
    for (int r = 0; r < db->n; ++r) {
      if (owner[r] != g) continue;
      int i0 = axis_index(G->axis[0], G->axis_len[0], db->dims[r * 5 + KINFO[G->kind].axes[0]]);
      int i1 = G->n_axes == 2 ? axis_index(G->axis[1], G->axis_len[1], db->dims[r * 5 + KINFO[G->kind].axes[1]]) : 0;
      G->cells[(size_t)i0 * n1 + i1] = db->latency[r];
    }
  }
  free(owner);
}

static void free_grids(gridset* gs) {
  for (int g = 0; g < gs->n_grids; ++g) {
    free(gs->grids[g].axis[0]);
    free(gs->grids[g].axis[1]);
    free(gs->grids[g].cells);
  }
  free(gs->grids);
}

/* ------------------------------------------------------------------------- */
/* queries and errors */
typedef struct {
  int kind, quant, attn;
  int64_t d[5]; /* canonical order */
  int64_t kv_len; /* attention_generation shape kv_len; <= 0: seq_len (OperatorQuery.kv_len, perfdb.py:232-234) */
} query;

enum { ST_OK = 0, ST_MISSING = 1, ST_EXTRAP = 2, ST_UNSUPPORTED = 3 };

typedef struct {
  int st;
  char msg[512];
} err_t;

static int fmt_key(char* out, size_t n, const query* q) {
  const kind_info* ki = &KINFO[q->kind];
  int w = snprintf(out, n, "('%s', '%s', (", KIND_NAME[q->kind], QUANT_NAME[q->quant]);
  int items = 0;
  if (is_attn(q->kind)) {
    w += snprintf(out + w, n - (size_t)w, "('attn_kind', '%s')", ATTN_NAME[q->attn]);
    items++;
  }
  for (int i = 0; i < ki->n_fixed; ++i) {
    w += snprintf(out + w, n - (size_t)w, "%s('%s', %lld)", items ? ", " : "", ki->names[ki->fixed[i]],
                  (long long)q->d[ki->fixed[i]]);
    items++;
  }
  w += snprintf(out + w, n - (size_t)w, "%s))", items == 1 ? "," : "");
  return w;
}

/* roofline, perfdb.py:431-484 */
static int sol_estimate(const or_db* db, const query* q, double* out, err_t* err) {
  double b = QUANT_BYTES[q->quant];
  int kind = q->kind;
  const int64_t* d = q->d;
  if (is_comm(kind)) {
    int64_t n = d[1];
    double link = n <= db->gpus_per_node ? db->intra_bw : db->inter_bw;
    double factor;
    if (kind == OK_KIND_ALLREDUCE) factor = 2.0 * (double)(n - 1) / (double)n;
    else if (kind == OK_KIND_P2P) factor = 1.0;
    else factor = (double)(n - 1) / (double)n;
    double seconds = (double)d[0] * factor / link;
    *out = seconds * 1e6;
    return ST_OK;
  }
  double compute = db->compute[q->quant];
  if (!(compute > 0.0)) {
    err->st = ST_UNSUPPORTED;
    snprintf(err->msg, sizeof(err->msg),
             "UnsupportedOperatorError: hardware '%s' has no compute rate for quant '%s'", db->hw_name,
             QUANT_NAME[q->quant]);
    return ST_UNSUPPORTED;
  }
  double flops, bytes_moved;
  if (kind == OK_KIND_GEMM) {
    int64_t m = d[0], n = d[1], k = d[2];
    flops = 2.0 * (double)m * (double)n * (double)k;
    bytes_moved = b * (double)(m * k + k * n + m * n);
  } else if (kind == OK_KIND_ATTN_CTX) {
    int64_t B = d[0], s = d[1], H = d[2], KV = d[3], hd = d[4];
    flops = 2.0 * (double)B * (double)H * (double)s * (double)s * (double)hd;
    bytes_moved = b * (double)B * (double)s * (double)(2 * H + 2 * KV) * (double)hd;
  } else if (kind == OK_KIND_ATTN_GEN) {
    int64_t B = d[0], kv = q->kv_len > 0 ? q->kv_len : d[1], H = d[2], KV = d[3], hd = d[4];
    flops = 4.0 * (double)B * (double)H * (double)kv * (double)hd;
    bytes_moved = b * (double)B * (double)kv * 2.0 * (double)KV * (double)hd;
  } else if (kind == OK_KIND_MOE_GEMM) {
    int64_t t = d[0], e = d[1], h = d[3], i = d[4];
    flops = 3.0 * 2.0 * (double)t * (double)h * (double)i;
    bytes_moved = b * (3.0 * (double)e * (double)h * (double)i + (double)(t * (h + i)));
  } else if (kind == OK_KIND_MOE_DISPATCH || kind == OK_KIND_MOE_COMBINE) {
    int64_t t = d[0], k_ = d[2], h = d[3];
    double seconds = b * (double)t * (double)k_ * (double)h / db->intra_bw;
    *out = seconds * 1e6;
    return ST_OK;
  } else { /* embedding */
    int64_t t = d[0], h = d[1];
    *out = b * (double)t * (double)h / db->mem_bw * 1e6;
    return ST_OK;
  }
  double a = flops / compute, c = bytes_moved / db->mem_bw;
  double seconds = c > a ? c : a; /* Python max(a, c) */
  *out = seconds * 1e6;
  return ST_OK;
}

/* _axis_position, perfdb.py:490-506 */
typedef struct {
  int lo, hi, oob;
  double t;
} axpos;

static axpos axis_position(const int64_t* v, int n, int64_t x) {
  axpos p = {0, 0, 0, 0.0};
  if (x < v[0]) { p.oob = -1; return p; }
  if (x > v[n - 1]) { p.lo = p.hi = n - 1; p.oob = 1; return p; }
  int i = axis_index(v, n, x);
  if (v[i] == x) { p.lo = p.hi = i; return p; }
  p.lo = i - 1; p.hi = i;
  p.t = (log((double)x) - log((double)v[i - 1])) / (log((double)v[i]) - log((double)v[i - 1]));
  return p;
}

/* _interp_cells, perfdb.py:509-536 */
static double interp_cells(const grid* G, const int64_t* coords) {
  axpos pos[2];
  int exact = 1;
  for (int a = 0; a < G->n_axes; ++a) {
    pos[a] = axis_position(G->axis[a], G->axis_len[a], coords[a]);
    if (!(pos[a].oob == 0 && pos[a].lo == pos[a].hi)) exact = 0;
  }
  int n1 = G->n_axes == 2 ? G->axis_len[1] : 1;
  if (exact) {
    int i1 = G->n_axes == 2 ? pos[1].lo : 0;
    return G->cells[(size_t)pos[0].lo * n1 + i1];
  }
  double w[4];
  int idx0[4], idx1[4];
  int nc = 1;
  w[0] = 1.0; idx0[0] = 0; idx1[0] = 0;
  for (int a = 0; a < G->n_axes; ++a) {
    double nw[4];
    int n0[4], n1i[4];
    int m = 0;
    for (int c = 0; c < nc; ++c) {
      if (pos[a].lo == pos[a].hi) {
        nw[m] = w[c]; n0[m] = a == 0 ? pos[a].lo : idx0[c]; n1i[m] = a == 1 ? pos[a].lo : idx1[c]; m++;
      } else {
        if (pos[a].t < 1.0) {
          nw[m] = w[c] * (1.0 - pos[a].t);
          n0[m] = a == 0 ? pos[a].lo : idx0[c]; n1i[m] = a == 1 ? pos[a].lo : idx1[c]; m++;
        }
        if (pos[a].t > 0.0) {
          nw[m] = w[c] * pos[a].t;
          n0[m] = a == 0 ? pos[a].hi : idx0[c]; n1i[m] = a == 1 ? pos[a].hi : idx1[c]; m++;
        }
      }
    }
    nc = m;
    memcpy(w, nw, sizeof(double) * (size_t)m);
    memcpy(idx0, n0, sizeof(int) * (size_t)m);
    memcpy(idx1, n1i, sizeof(int) * (size_t)m);
  }
  double v[4];
  for (int c = 0; c < nc; ++c) v[c] = G->cells[(size_t)idx0[c] * n1 + idx1[c]];
  if (nc == 1) return v[0];
  int same = 1;
  for (int c = 1; c < nc; ++c) same &= v[c] == v[0];
  if (same) return v[0];
  double terms[4];
  for (int c = 0; c < nc; ++c) terms[c] = w[c] * log(v[c]);
  return exp(or_neumaier_sum(terms, nc));
}

/* query_latency, perfdb.py:539-580 */
static int query_latency_p(const gridset* gs, const query* q, int policy, double* out, err_t* err) {
  const or_db* db = gs->db;
  const kind_info* ki = &KINFO[q->kind];
  int64_t fixed[4] = {0, 0, 0, 0};
  for (int i = 0; i < ki->n_fixed; ++i) fixed[i] = q->d[ki->fixed[i]];
  int g = find_grid(gs, q->kind, q->quant, is_attn(q->kind) ? q->attn : 0, fixed);
  if (g < 0) {
    err->st = ST_MISSING;
    int w = snprintf(err->msg, sizeof(err->msg), "MissingKeyError: no grid for key ");
    w += fmt_key(err->msg + w, sizeof(err->msg) - (size_t)w, q);
    w += snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "; database covers kinds [");
    /* sorted kind names */
    const char* names[OK_NKINDS];
    int nn = 0;
    for (int k = 0; k < OK_NKINDS; ++k)
      if (gs->kinds_present[k]) names[nn++] = KIND_NAME[k];
    for (int i = 1; i < nn; ++i)
      for (int j = i; j > 0 && strcmp(names[j - 1], names[j]) > 0; --j) {
        const char* t = names[j]; names[j] = names[j - 1]; names[j - 1] = t;
      }
    for (int i = 0; i < nn; ++i)
      w += snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "%s'%s'", i ? ", " : "", names[i]);
    snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "]");
    return ST_MISSING;
  }
  const grid* G = &gs->grids[g];
  int64_t coords[2];
  int any_oob = 0, any_above = 0;
  for (int a = 0; a < G->n_axes; ++a) {
    coords[a] = q->d[ki->axes[a]];
    axpos p = axis_position(G->axis[a], G->axis_len[a], coords[a]);
    if (p.oob) any_oob = 1;
    if (p.oob > 0) any_above = 1;
  }
  if (!any_oob) {
    *out = interp_cells(G, coords);
    return ST_OK;
  }
  if (policy == 1) { /* strict */
    err->st = ST_EXTRAP;
    int w = snprintf(err->msg, sizeof(err->msg), "ExtrapolationError: query coords {");
    for (int a = 0; a < G->n_axes; ++a)
      w += snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "%s'%s': %lld", a ? ", " : "",
                    ki->names[ki->axes[a]], (long long)coords[a]);
    w += snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "} outside grid box {");
    for (int a = 0; a < G->n_axes; ++a)
      w += snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "%s'%s': (%lld, %lld)", a ? ", " : "",
                    ki->names[ki->axes[a]], (long long)G->axis[a][0],
                    (long long)G->axis[a][G->axis_len[a] - 1]);
    snprintf(err->msg + w, sizeof(err->msg) - (size_t)w, "}");
    return ST_EXTRAP;
  }
  int64_t clamped[2];
  for (int a = 0; a < G->n_axes; ++a) {
    int64_t c = coords[a], lo = G->axis[a][0], hi = G->axis[a][G->axis_len[a] - 1];
    c = c > lo ? c : lo;
    clamped[a] = c < hi ? c : hi;
  }
  int use_sol = policy == 3 || (policy == 0 && any_above);
  if (policy == 2 || !use_sol) {
    *out = interp_cells(G, clamped);
    return ST_OK;
  }
  double edge = interp_cells(G, clamped);
  query eq = *q;
  for (int a = 0; a < G->n_axes; ++a) eq.d[ki->axes[a]] = clamped[a];
  double sol_edge, sol_q;
  if (sol_estimate(db, &eq, &sol_edge, err)) return err->st;
  double eff = edge / sol_edge;
  if (sol_estimate(db, q, &sol_q, err)) return err->st;
  *out = sol_q * eff;
  return ST_OK;
}

static int query_latency(const gridset* gs, const query* q, double* out, err_t* err) {
  return query_latency_p(gs, q, gs->db->policy, out, err);
}

int or_query_batch(const or_db* db, int32_t n, const int32_t* kind, const int32_t* quant, const int32_t* attn,
                   const int64_t* dims, const int64_t* kv_len, int32_t policy, double* out, int32_t* status,
                   char* msgs, int32_t msg_len) {
  gridset gs;
  build_grids(db, &gs);
  for (int32_t i = 0; i < n; ++i) {
    query q;
    memset(&q, 0, sizeof(q));
    q.kind = kind[i]; q.quant = quant[i]; q.attn = attn[i];
    for (int k = 0; k < 5; ++k) q.d[k] = dims[(size_t)i * 5 + k];
    q.kv_len = kv_len ? kv_len[i] : 0;
    err_t err;
    err.st = 0; err.msg[0] = 0;
    out[i] = 0.0;
    status[i] = query_latency_p(&gs, &q, policy >= 0 ? policy : db->policy, &out[i], &err);
    if (msgs && msg_len > 0) snprintf(msgs + (size_t)i * msg_len, (size_t)msg_len, "%s", status[i] ? err.msg : "");
  }
  free_grids(&gs);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* MoE skew, moe_load.py:67-147 */
typedef struct {
  double key; /* frac or weight */
  int idx;
} kidx;

static int cmp_desc_key_idx(const void* a, const void* b) {
  const kidx* x = (const kidx*)a;
  const kidx* y = (const kidx*)b;
  /* lexsort((arange, -key)): ascending -key, then index */
  double nx = -x->key, ny = -y->key;
  if (nx < ny) return -1;
  if (nx > ny) return 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

int64_t or_busiest_shard(const double* weights, int e, int64_t total, int64_t topk, int64_t ep,
                         int64_t* counts_out) {
  /* numpy: weights.sum() is pairwise; weights / s * target elementwise */
  /* pairwise sum restated: numpy pairwise_sum with blocks of 8, unrolled 128 */
  double s;
  {
    /* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) */
    double* tmp = (double*)malloc(sizeof(double) * (size_t)e);
    memcpy(tmp, weights, sizeof(double) * (size_t)e);
    extern double or_np_pairwise_sum(const double* a, int64_t n);
    s = or_np_pairwise_sum(tmp, e);
    free(tmp);
  }
  int64_t target = total * topk;
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)e);
  kidx* fr = (kidx*)malloc(sizeof(kidx) * (size_t)e);
  int64_t csum = 0;
  for (int i = 0; i < e; ++i) {
    double raw = weights[i] / s * (double)target;
    double f = floor(raw);
    cnt[i] = (int64_t)f;
    fr[i].key = raw - (double)cnt[i];
    fr[i].idx = i;
    csum += cnt[i];
  }
  int64_t shortfall = target - csum;
  qsort(fr, (size_t)e, sizeof(kidx), cmp_desc_key_idx);
  for (int64_t j = 0; j < shortfall && j < e; ++j) cnt[fr[j].idx] += 1;
  int64_t surplus = 0;
  for (int i = 0; i < e; ++i)
    if (cnt[i] - total > 0) surplus += cnt[i] - total;
  if (surplus) {
    for (int i = 0; i < e; ++i)
      if (cnt[i] > total) cnt[i] = total;
    for (int i = 0; i < e; ++i) { fr[i].key = weights[i]; fr[i].idx = i; }
    qsort(fr, (size_t)e, sizeof(kidx), cmp_desc_key_idx);
    for (int j = 0; j < e && surplus; ++j) {
      int i = fr[j].idx;
      int64_t room = total - cnt[i];
      int64_t take = room < surplus ? room : surplus;
      cnt[i] += take;
      surplus -= take;
    }
  }
  int64_t best = 0;
  int64_t per = e / ep;
  for (int64_t r = 0; r < ep; ++r) {
    int64_t acc = 0;
    for (int64_t j = 0; j < per; ++j) acc += cnt[r * per + j];
    if (r == 0 || acc > best) best = acc;
  }
  if (counts_out) memcpy(counts_out, cnt, sizeof(int64_t) * (size_t)e);
  free(cnt);
  free(fr);
  return best;
}

/* numpy's pairwise summation for contiguous float64 (PW_BLOCKSIZE 128, 8 accumulators) */
double or_np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8], res;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return or_np_pairwise_sum(a, n2) + or_np_pairwise_sum(a + n2, n - n2);
  }
}

/* ------------------------------------------------------------------------- */
/* model, decompose (model.py:263-406) */
enum {
  L_EMB, L_QKV, L_CTX, L_GEN, L_OUT, L_UP, L_DOWN, L_ROUTER, L_SUP, L_SDOWN, L_EXPERT, L_DISPATCH,
  L_COMBINE, L_AR1, L_AR2, L_P2P, L_N
};

typedef struct {
  query q;
  int64_t repeat;
  int label;
} entry;

typedef struct {
  int64_t tp, pp, ep, dp, batch;
} cfg_t;

static int64_t ceil_div_f(int64_t a, int64_t b) { return (int64_t)ceil((double)a / (double)b); }

static int decompose(const or_model* m, const cfg_t* c, int phase /*0 prefill 1 decode 2 mixed*/,
                     int64_t n_ctx, int64_t n_gen, int64_t seq, entry* out) {
  int n = 0;
  int64_t tokens = n_ctx + n_gen;
  int64_t h = m->hidden;
  int64_t heads = m->heads / c->tp;
  int64_t kvh = m->attn == 3 ? 1 : (m->kv_heads / c->tp > 1 ? m->kv_heads / c->tp : 1);
  int64_t hd = m->attn == 3 ? m->mla_kv_dim : m->head_dim;
  int64_t layers = ceil_div_f(m->num_layers, c->pp);
#define ADD(K, QN, LBL, REP, D0, D1, D2, D3, D4)                                              \
  do {                                                                                      \
    entry* e_ = &out[n++];                                                                  \
    e_->q.kind = (K); e_->q.quant = (QN); e_->q.attn = m->attn; e_->q.kv_len = 0;          \
    e_->q.d[0] = (D0); e_->q.d[1] = (D1); e_->q.d[2] = (D2); e_->q.d[3] = (D3); e_->q.d[4] = (D4); \
    e_->repeat = (REP); e_->label = (LBL);                                                  \
  } while (0)
  ADD(OK_KIND_EMBEDDING, m->wq, L_EMB, 1, tokens, h, m->vocab, 0, 0);
  int64_t qkv_n = m->attn == 3 ? heads * m->head_dim + m->mla_kv_dim : (heads + 2 * kvh) * m->head_dim;
  ADD(OK_KIND_GEMM, m->wq, L_QKV, layers, tokens, qkv_n, h, 0, 0);
  if (n_ctx) {
    int64_t cb = phase == 2 ? 1 : n_ctx / seq;
    int64_t cs = phase == 2 ? n_ctx : seq;
    ADD(OK_KIND_ATTN_CTX, m->kq, L_CTX, layers, cb, cs, heads, kvh, hd);
  }
  if (n_gen) ADD(OK_KIND_ATTN_GEN, m->kq, L_GEN, layers, n_gen, seq, heads, kvh, hd);
  ADD(OK_KIND_GEMM, m->wq, L_OUT, layers, tokens, h, heads * m->head_dim, 0, 0);
  if (!m->is_moe) {
    int64_t inter = m->inter / c->tp > 1 ? m->inter / c->tp : 1;
    ADD(OK_KIND_GEMM, m->wq, L_UP, layers, tokens, 2 * inter, h, 0, 0);
    ADD(OK_KIND_GEMM, m->wq, L_DOWN, layers, tokens, h, inter, 0, 0);
  } else {
    ADD(OK_KIND_GEMM, m->wq, L_ROUTER, layers, tokens, m->n_experts, h, 0, 0);
    if (m->shared_inter) {
      int64_t sh = m->shared_inter / c->tp > 1 ? m->shared_inter / c->tp : 1;
      ADD(OK_KIND_GEMM, m->wq, L_SUP, layers, tokens, 2 * sh, h, 0, 0);
      ADD(OK_KIND_GEMM, m->wq, L_SDOWN, layers, tokens, h, sh, 0, 0);
    }
    int64_t f = c->ep / c->tp > 1 ? c->ep / c->tp : 1;
    int64_t pooled = tokens * f;
    int64_t et = ceil_div_f(pooled * m->topk, c->ep);
    int64_t g = c->tp / c->ep > 1 ? c->tp / c->ep : 1;
    ADD(OK_KIND_MOE_GEMM, m->wq, L_EXPERT, layers, et, m->n_experts / c->ep, m->topk, h, m->expert_inter / g);
    if (c->ep > 1) {
      ADD(OK_KIND_MOE_DISPATCH, 0, L_DISPATCH, layers, tokens, m->n_experts, m->topk, h, m->expert_inter);
      ADD(OK_KIND_MOE_COMBINE, 0, L_COMBINE, layers, tokens, m->n_experts, m->topk, h, m->expert_inter);
    }
  }
  if (c->tp > 1) {
    ADD(OK_KIND_ALLREDUCE, 0, L_AR1, layers, tokens * h * 2, c->tp, 0, 0, 0);
    ADD(OK_KIND_ALLREDUCE, 0, L_AR2, layers, tokens * h * 2, c->tp, 0, 0, 0);
  }
  if (c->pp > 1) ADD(OK_KIND_P2P, 0, L_P2P, c->pp - 1, tokens * h * 2, 2, 0, 0, 0);
#undef ADD
  return n;
}

typedef struct {
  const gridset* gs;
  const or_model* m;
  const or_search* s;
  int64_t n_queries;
} ctx_t;

/* _step_latency_cached, estimator.py:71-95 */
static int step_latency(ctx_t* X, const cfg_t* c, int phase, int64_t n_ctx, int64_t n_gen, int64_t seq,
                        double* total, err_t* err) {
  entry ent[L_N];
  int n = decompose(X->m, c, phase, n_ctx, n_gen, seq, ent);
  int64_t mb = c->batch > 1 ? c->batch : 1;
  double bubble = (double)(mb + c->pp - 1) / (double)mb;
  int64_t total_tokens = n_ctx + n_gen;
  double terms[L_N];
  for (int i = 0; i < n; ++i) {
    query q = ent[i].q;
    if (ent[i].label == L_EXPERT && X->m->is_moe && c->ep > 1) {
      int64_t f = c->ep / c->tp > 1 ? c->ep / c->tp : 1;
      int64_t pooled = total_tokens * f;
      int64_t balanced = ceil_div_f(pooled * X->m->topk, c->ep);
      int64_t tail = or_busiest_shard(X->m->moe_weights, X->m->moe_n_weights, pooled, X->m->topk, c->ep, NULL);
      q.d[0] = balanced > tail ? balanced : tail;
    }
    double lat = 0.0;
    X->n_queries++;
    if (query_latency(X->gs, &q, &lat, err)) return err->st;
    double ms = lat * (double)ent[i].repeat / 1000.0;
    terms[i] = 0.0 + ms * bubble;
  }
  *total = or_neumaier_sum(terms, n);
  return ST_OK;
}

/* ------------------------------------------------------------------------- */
/* serving modes, serving_modes.py:161-494 */
static void derive_metrics(double ttft, double tpot, int64_t batch, int64_t osl, int64_t gpus, double* speed,
                           double* thru) {
  *speed = tpot == 0.0 ? INFINITY : 1000.0 / tpot;
  double req = ttft + (double)(osl - 1) * tpot;
  *thru = 1000.0 / req * (double)batch * (double)osl / (double)gpus;
}

typedef struct {
  double ttft, tpot, speed, thru;
} est_t;

static int estimate_static(ctx_t* X, const cfg_t* c, est_t* e, err_t* err) {
  const or_search* s = X->s;
  int64_t b = c->batch, isl = s->isl, osl = s->osl, chunk = s->isl - s->prefix;
  double ttft, t_gen = 0.0;
  if (step_latency(X, c, 0, b * chunk, 0, chunk, &ttft, err)) return err->st;
  int64_t k = 0;
  while (k < osl - 1) {
    int64_t kv = isl + k + 1;
    double step;
    if (step_latency(X, c, 1, 0, b, kv, &step, err)) return err->st;
    const int64_t stride = s->static_stride > 0 ? s->static_stride : 32; /* STATIC_DECODE_STRIDE */
    int64_t run = osl - 1 - k < stride ? osl - 1 - k : stride;
    t_gen += step * (double)run;
    k += run;
  }
  double tpot = osl > 1 ? t_gen / (double)(osl - 1) : 0.0;
  e->ttft = ttft; e->tpot = tpot;
  derive_metrics(ttft, tpot, b, osl, c->tp * c->pp * c->dp, &e->speed, &e->thru);
  return ST_OK;
}

enum { ST_INFEASIBLE = 4 };

static int64_t ctx_capacity(const or_search* s) {
  if (s->has_ctx_capacity) return s->ctx_capacity;
  int64_t e = s->isl - s->prefix;
  return e > 2048 ? e : 2048;
}

static int estimate_aggregated(ctx_t* X, const cfg_t* c, est_t* e, err_t* err) {
  const or_search* s = X->s;
  int64_t b = c->batch, isl = s->isl, osl = s->osl;
  int64_t chunk_total = isl - s->prefix;
  int64_t c_ctx = ctx_capacity(s);
  if (!s->chunked_prefill && chunk_total > c_ctx) {
    err->st = ST_INFEASIBLE;
    snprintf(err->msg, sizeof(err->msg),
             "InfeasibleConfigError: context of %lld tokens exceeds capacity %lld and chunking is off",
             (long long)chunk_total, (long long)c_ctx);
    return ST_INFEASIBLE;
  }
  int64_t T = ceil_div_f(chunk_total * b, c_ctx);
  int64_t cpr = ceil_div_f(chunk_total, c_ctx);
  int64_t chunk_tokens = c_ctx < chunk_total ? c_ctx : chunk_total;
  int64_t t_mix, t_gen, n_mix_gen;
  if (b == 1) {
    t_mix = 1; t_gen = osl - 1; n_mix_gen = 0;
  } else if (T >= osl) {
    n_mix_gen = (int64_t)((double)(b * osl) / (double)T);
    if (n_mix_gen < 1) n_mix_gen = 1;
    t_mix = osl; t_gen = 0;
  } else {
    int64_t prefilling = ceil_div_f(c_ctx, chunk_total);
    n_mix_gen = b - prefilling;
    if (n_mix_gen < 1) {
      err->st = ST_INFEASIBLE;
      snprintf(err->msg, sizeof(err->msg),
               "InfeasibleConfigError: batch %lld too small to decode alongside %lld prefilling requests",
               (long long)b, (long long)prefilling);
      return ST_INFEASIBLE;
    }
    t_mix = T; t_gen = osl - T;
  }
  int64_t kv = isl + osl / 2;
  double l_mix, l_gen = 0.0;
  if (step_latency(X, c, 2, chunk_tokens, n_mix_gen, kv, &l_mix, err)) return err->st;
  if (t_gen || b == 1)
    if (step_latency(X, c, 1, 0, b, kv, &l_gen, err)) return err->st;
  double raw = 2.0 + (double)(T - 3) * (1.0 / 20.0);
  double F = raw > 2.0 ? raw : 2.0;
  F = F < 4.0 ? F : 4.0;
  double ttft = l_mix * (double)cpr * F;
  double tpot;
  if (b == 1) tpot = osl > 1 ? l_gen : 0.0;
  else if (osl == 1) tpot = 0.0;
  else if (t_gen == 0) tpot = l_mix;
  else {
    int64_t ms = t_mix - 3 > 1 ? t_mix - 3 : 1;
    tpot = (l_mix * (double)ms + l_gen * (double)t_gen) / (double)(ms + t_gen);
  }
  e->ttft = ttft; e->tpot = tpot;
  derive_metrics(ttft, tpot, b, osl, c->tp * c->pp * c->dp, &e->speed, &e->thru);
  return ST_OK;
}

/* ------------------------------------------------------------------------- */
/* enumeration: search.py:82-113, model.py:209-236, 440-479 */
static int consistent(const or_model* m, const cfg_t* c) {
  if (m->heads % c->tp) return 0;
  if (c->pp > m->num_layers) return 0;
  if (!m->is_moe) {
    if (c->ep != 1) return 0;
    if (c->tp <= m->inter && m->inter % c->tp) return 0;
  } else {
    if (m->n_experts % c->ep) return 0;
    if (c->ep > c->tp * c->dp) return 0;
    int64_t hi = c->ep > c->tp ? c->ep : c->tp, lo = c->ep < c->tp ? c->ep : c->tp;
    if (hi % lo) return 0;
    if (c->tp > c->ep && m->expert_inter % (c->tp / c->ep)) return 0;
    if (m->shared_inter && c->tp <= m->shared_inter && m->shared_inter % c->tp) return 0;
  }
  return 1;
}

static int fits_memory(const or_db* db, const or_model* m, const or_search* s, const cfg_t* c) {
  double bw = QUANT_BYTES[m->wq], bkv = QUANT_BYTES[m->kq];
  int64_t expert = m->is_moe ? m->num_layers * m->n_experts * 3 * m->hidden * m->expert_inter : 0;
  int64_t dense = m->params - expert > 0 ? m->params - expert : 0;
  int64_t mx = c->ep > c->tp ? c->ep : c->tp;
  double weight = bw * ((double)dense / (double)c->tp + (double)expert / (double)mx) / (double)c->pp;
  int64_t layers = ceil_div_f(m->num_layers, c->pp);
  double kv_token;
  if (m->attn == 3) kv_token = (double)(layers * m->mla_kv_dim) * bkv;
  else {
    int64_t kvh = m->kv_heads / c->tp > 1 ? m->kv_heads / c->tp : 1;
    kv_token = (double)(2 * layers * kvh * m->head_dim) * bkv;
  }
  int64_t cap = s->has_ctx_capacity ? s->ctx_capacity : 2048;
  int64_t live = c->batch > cap ? c->batch : cap;
  int64_t act = 4 * live * m->hidden * 2;
  double overhead = 0.05 * db->gpu_memory + (double)act;
  double stat = weight + overhead;
  if (stat > db->gpu_memory) return 0;
  double kv_budget = s->kv_mem_fraction * (db->gpu_memory - stat);
  double kv_need = kv_token * (double)c->batch * (double)(s->isl + s->osl);
  return kv_need <= kv_budget;
}

static int in_budget(const or_search* s, int64_t g) {
  if (s->n_budgets == 0) return 1;
  for (int i = 0; i < s->n_budgets; ++i)
    if (s->budgets[i] == g) return 1;
  return 0;
}

static int enumerate(const or_db* db, const or_model* m, const or_search* s, int enforce_budget, or_cfg** out) {
  int cap = 64, n = 0;
  or_cfg* v = (or_cfg*)malloc(sizeof(or_cfg) * (size_t)cap);
  for (int a = 0; a < s->n_tp; ++a)
    for (int p = 0; p < s->n_pp; ++p)
      for (int e = 0; e < s->n_ep; ++e)
        for (int d = 0; d < s->n_dp; ++d)
          for (int bi = 0; bi < s->n_b; ++bi) {
            cfg_t c = {s->tp[a], s->pp[p], s->ep[e], s->dp[d], s->batch[bi]};
            if (c.tp < 1 || c.pp < 1 || c.ep < 1 || c.dp < 1 || c.batch < 1) continue;
            if (!consistent(m, &c)) continue;
            if (enforce_budget && !in_budget(s, c.tp * c.pp * c.dp)) continue;
            if (!fits_memory(db, m, s, &c)) continue;
            if (n == cap) { cap *= 2; v = (or_cfg*)realloc(v, sizeof(or_cfg) * (size_t)cap); }
            v[n].tp = c.tp; v[n].pp = c.pp; v[n].ep = c.ep; v[n].dp = c.dp; v[n].batch = c.batch;
            n++;
          }
  *out = v;
  return n;
}

static int key_str(char* out, const or_cfg* c) {
  return sprintf(out, "tp%lldpp%lldep%llddp%lldb%lld", (long long)c->tp, (long long)c->pp, (long long)c->ep,
                 (long long)c->dp, (long long)c->batch);
}

/* ------------------------------------------------------------------------- */
/* disaggregated: serving_modes.py:347-494, search.py:276-277, 322-341 */
typedef struct {
  int worker;
  double lat, rate;
  int64_t gpus;
  char key[96];
} pool_t;

static int cmp_pool(const void* a, const void* b) {
  const pool_t* x = (const pool_t*)a;
  const pool_t* y = (const pool_t*)b;
  double kx = -x->rate / (double)x->gpus, ky = -y->rate / (double)y->gpus;
  if (kx < ky) return -1;
  if (kx > ky) return 1;
  return strcmp(x->key, y->key);
}

typedef struct {
  int p, d; /* pool positions */
  int64_t x, y, gpus;
  double r_sys, ttft, tpot, speed, thru;
  int order;
} plan_t;

static int cmp_plan(const void* a, const void* b) {
  const plan_t* x = (const plan_t*)a;
  const plan_t* y = (const plan_t*)b;
  double tx = -x->thru, ty = -y->thru;
  if (tx != ty) return tx < ty ? -1 : 1;
  if (x->gpus != y->gpus) return x->gpus < y->gpus ? -1 : 1;
  if (x->ttft != y->ttft) return x->ttft < y->ttft ? -1 : 1;
  if (x->x != y->x) return x->x < y->x ? -1 : 1;
  if (x->y != y->y) return x->y < y->y ? -1 : 1;
  return (x->order > y->order) - (x->order < y->order); /* stable */
}

/* ------------------------------------------------------------------------- */
static void push_skip(or_result* r, int* cap, int mode, int cand, const char* msg) {
  if (r->n_skip == *cap) {
    *cap = *cap ? *cap * 2 : 64;
    r->skip = (or_skip*)realloc(r->skip, sizeof(or_skip) * (size_t)*cap);
  }
  or_skip* s = &r->skip[r->n_skip++];
  s->mode = mode; s->cand = cand;
  snprintf(s->reason, sizeof(s->reason), "%s", msg);
}

static void push_row(or_result* r, int* cap, const or_row* row) {
  if (r->n_rows == *cap) {
    *cap = *cap ? *cap * 2 : 64;
    r->rows = (or_row*)realloc(r->rows, sizeof(or_row) * (size_t)*cap);
  }
  r->rows[r->n_rows++] = *row;
}

static void row_label(const or_result* r, const or_row* row, char* out) {
  if (row->mode < 2) {
    key_str(out, &r->cand[row->cand]);
  } else {
    char a[96], b[96];
    key_str(a, &r->work[row->p_worker]);
    key_str(b, &r->work[row->d_worker]);
    sprintf(out, "P:%dx%s|D:%dx%s", row->x, a, row->y, b);
  }
}

static int meets_sla(const or_search* s, const or_row* row) {
  if (s->has_ttft && row->ttft > s->ttft_limit) return 0;
  return !s->has_floor || row->speed >= s->speed_floor;
}

static const char* MODE_STR[3] = {"static", "aggregated", "disaggregated"};

int or_run_search(const or_db* db, const or_model* m, const or_search* s, or_result* out) {
  memset(out, 0, sizeof(*out));
  out->best = -1;
  out->nearest = -1;
  gridset gs;
  build_grids(db, &gs);
  ctx_t X = {&gs, m, s, 0};
  int row_cap = 0, skip_cap = 0;

  out->n_cand = enumerate(db, m, s, 1, &out->cand);
  for (int mode = 0; mode < 2; ++mode) {
    if (mode == 0 && !s->mode_static) continue;
    if (mode == 1 && !s->mode_agg) continue;
    for (int i = 0; i < out->n_cand; ++i) {
      cfg_t c = {out->cand[i].tp, out->cand[i].pp, out->cand[i].ep, out->cand[i].dp, out->cand[i].batch};
      est_t e = {0, 0, 0, 0};
      err_t err = {0, {0}};
      int st = mode == 0 ? estimate_static(&X, &c, &e, &err) : estimate_aggregated(&X, &c, &e, &err);
      if (st) { push_skip(out, &skip_cap, mode, i, err.msg); continue; }
      or_row row;
      memset(&row, 0, sizeof(row));
      row.mode = mode; row.cand = i; row.p_worker = row.d_worker = -1;
      row.gpus = c.tp * c.pp * c.dp;
      row.ttft = e.ttft; row.tpot = e.tpot; row.speed = e.speed; row.thru = e.thru;
      push_row(out, &row_cap, &row);
    }
  }

  if (s->mode_disagg) {
    out->n_work = enumerate(db, m, s, 0, &out->work);
    pool_t* pre = (pool_t*)malloc(sizeof(pool_t) * (size_t)(out->n_work + 1));
    pool_t* dec = (pool_t*)malloc(sizeof(pool_t) * (size_t)(out->n_work + 1));
    int npre = 0, ndec = 0;
    int64_t chunk = s->isl - s->prefix;
    for (int i = 0; i < out->n_work; ++i) {
      cfg_t c = {out->work[i].tp, out->work[i].pp, out->work[i].ep, out->work[i].dp, out->work[i].batch};
      int64_t g = c.tp * c.pp * c.dp;
      double lat = 0.0;
      err_t err = {0, {0}};
      if (step_latency(&X, &c, 0, c.batch * chunk, 0, chunk, &lat, &err)) {
        push_skip(out, &skip_cap, 2, i, err.msg);
      } else {
        pool_t* p = &pre[npre++];
        p->worker = i; p->lat = lat; p->rate = (double)c.batch * 1000.0 / lat; p->gpus = g;
        key_str(p->key, &out->work[i]);
      }
      err.st = 0;
      if (step_latency(&X, &c, 1, 0, c.batch, s->isl + s->osl / 2, &lat, &err)) {
        push_skip(out, &skip_cap, 3, i, err.msg);
      } else {
        pool_t* p = &dec[ndec++];
        p->worker = i; p->lat = lat; p->gpus = g;
        p->rate = s->osl == 1 ? INFINITY : (double)c.batch * 1000.0 / ((double)(s->osl - 1) * lat);
        key_str(p->key, &out->work[i]);
      }
    }
    qsort(pre, (size_t)npre, sizeof(pool_t), cmp_pool);
    qsort(dec, (size_t)ndec, sizeof(pool_t), cmp_pool);
    if (npre > s->prefill_pool_cap) npre = s->prefill_pool_cap;
    if (ndec > s->decode_pool_cap) ndec = s->decode_pool_cap;
    plan_t* plans = (plan_t*)malloc(sizeof(plan_t) * (size_t)(npre * ndec + 1));
    int nplan = 0;
    for (int pi = 0; pi < npre; ++pi) {
      const pool_t* p = &pre[pi];
      if (s->has_ttft && !(p->lat * s->ttft_headroom <= s->ttft_limit)) continue;
      for (int di = 0; di < ndec; ++di) {
        const pool_t* d = &dec[di];
        if (s->has_tpot_cap && !(d->lat <= s->tpot_cap)) continue;
        int have = 0;
        double bk0 = 0; int64_t bg = 0, bx = 0, by = 0;
        for (int64_t x = 1; x <= s->max_x; ++x) {
          double r_pre = p->rate * (double)x * s->prefill_util;
          int64_t g_pre = x * p->gpus;
          for (int64_t y = 1; y <= s->max_y; ++y) {
            int64_t gpus = g_pre + y * d->gpus;
            if (!in_budget(s, gpus)) continue;
            double r_dec = d->rate * (double)y * s->decode_util;
            double r_sys = r_dec < r_pre ? r_dec : r_pre;
            double k0 = -r_sys * (double)s->osl / (double)gpus;
            int better = !have || k0 < bk0 || (k0 == bk0 && (gpus < bg || (gpus == bg && (x < bx || (x == bx && y < by)))));
            if (better) { have = 1; bk0 = k0; bg = gpus; bx = x; by = y; }
          }
        }
        if (!have) continue;
        plan_t* P = &plans[nplan];
        P->p = pi; P->d = di; P->x = bx; P->y = by; P->order = nplan;
        P->gpus = bx * p->gpus + by * d->gpus;
        double r_pre = p->rate * (double)bx * s->prefill_util;
        double r_dec = d->rate * (double)by * s->decode_util;
        P->r_sys = r_dec < r_pre ? r_dec : r_pre;
        P->ttft = p->lat * s->ttft_headroom;
        P->tpot = d->lat;
        P->speed = P->tpot == 0.0 ? INFINITY : 1000.0 / P->tpot;
        P->thru = P->r_sys * (double)s->osl / (double)P->gpus;
        nplan++;
      }
    }
    qsort(plans, (size_t)nplan, sizeof(plan_t), cmp_plan);
    for (int i = 0; i < nplan; ++i) {
      or_row row;
      memset(&row, 0, sizeof(row));
      row.mode = 2; row.cand = -1;
      row.p_worker = pre[plans[i].p].worker; row.d_worker = dec[plans[i].d].worker;
      row.x = (int32_t)plans[i].x; row.y = (int32_t)plans[i].y; row.gpus = plans[i].gpus;
      row.ttft = plans[i].ttft; row.tpot = plans[i].tpot; row.speed = plans[i].speed;
      row.thru = plans[i].thru; row.r_sys = plans[i].r_sys;
      push_row(out, &row_cap, &row);
    }
    free(plans); free(pre); free(dec);
  }

  /* feasibility, pareto_filter over feasible rows (search.py:156-176, 343-344) */
  int nr = out->n_rows;
  for (int i = 0; i < nr; ++i) out->rows[i].feasible = meets_sla(s, &out->rows[i]);
  int* order = (int*)malloc(sizeof(int) * (size_t)(nr + 1));
  int nf = 0;
  for (int i = 0; i < nr; ++i)
    if (out->rows[i].feasible) order[nf++] = i;
  /* stable insertion sort by speed descending */
  for (int i = 1; i < nf; ++i) {
    int v = order[i], j = i;
    while (j > 0 && out->rows[order[j - 1]].speed < out->rows[v].speed) { order[j] = order[j - 1]; --j; }
    order[j] = v;
  }
  out->front = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf + 1));
  double best_thru = -INFINITY;
  for (int a = 0; a < nf;) {
    int b = a;
    double sp = out->rows[order[a]].speed, top = -INFINITY;
    while (b < nf && out->rows[order[b]].speed == sp) {
      if (b == a || out->rows[order[b]].thru > top) top = out->rows[order[b]].thru;
      ++b;
    }
    if (top > best_thru) {
      for (int j = a; j < b; ++j)
        if (out->rows[order[j]].thru == top) {
          out->front[out->n_front++] = order[j];
          out->rows[order[j]].frontier = 1;
        }
      best_thru = top;
    }
    a = b;
  }
  free(order);

  /* select_best (search.py:179-187) */
  char la[256], lb[256];
  for (int i = 0; i < nr; ++i) {
    const or_row* r = &out->rows[i];
    if (!r->feasible) continue;
    if (out->best < 0) { out->best = i; continue; }
    const or_row* b = &out->rows[out->best];
    int better = 0;
    if (-r->thru != -b->thru) better = -r->thru < -b->thru;
    else if (-r->speed != -b->speed) better = -r->speed < -b->speed;
    else if (r->gpus != b->gpus) better = r->gpus < b->gpus;
    else {
      int c = strcmp(MODE_STR[r->mode], MODE_STR[b->mode]);
      if (c) better = c < 0;
      else {
        row_label(out, r, la); row_label(out, b, lb);
        better = strcmp(la, lb) < 0;
      }
    }
    if (better) out->best = i;
  }
  /* nearest_miss (search.py:190-208) */
  if (out->best < 0 && nr > 0) {
    double bv = 0;
    for (int i = 0; i < nr; ++i) {
      const or_row* r = &out->rows[i];
      double worst = 1.0;
      if (s->has_ttft && r->ttft > s->ttft_limit) {
        double v = r->ttft / s->ttft_limit;
        if (v > worst) worst = v;
      }
      if (s->has_floor && r->speed < s->speed_floor) {
        double v = r->speed == 0.0 ? INFINITY : s->speed_floor / r->speed;
        if (v > worst) worst = v;
      }
      int better = out->nearest < 0 || worst < bv;
      if (!better && worst == bv) {
        row_label(out, r, la); row_label(out, &out->rows[out->nearest], lb);
        better = strcmp(la, lb) < 0;
      }
      if (better) { out->nearest = i; bv = worst; }
    }
    out->nearest_violation = bv;
  }
  out->n_queries = X.n_queries;
  free_grids(&gs);
  return 0;
}

void or_free(or_result* r) {
  free(r->cand); free(r->work); free(r->rows); free(r->skip); free(r->front);
  memset(r, 0, sizeof(*r));
}

int or_estimate(const or_db* db, const or_model* m, const or_search* s, const or_cfg* cfg, int mode, double* out,
                char* reason, int reason_len) {
  gridset gs;
  build_grids(db, &gs);
  ctx_t X = {&gs, m, s, 0};
  cfg_t c = {cfg->tp, cfg->pp, cfg->ep, cfg->dp, cfg->batch};
  est_t e = {0, 0, 0, 0};
  err_t err = {0, {0}};
  const int st = mode == 0 ? estimate_static(&X, &c, &e, &err) : estimate_aggregated(&X, &c, &e, &err);
  if (st) snprintf(reason, (size_t)reason_len, "%s", err.msg);
  else { out[0] = e.ttft; out[1] = e.tpot; out[2] = e.speed; out[3] = e.thru; }
  free_grids(&gs);
  return st;
}
