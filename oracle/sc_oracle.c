/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Not part of the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load liboracle.so, and only as the checker.
 *
 * A plain-C restatement of the reference hot path (/root/reference/proj/src),
 * written independently, so it can travel to the GPU box (where
 * /root/reference does not exist).  It is pinned against the unmodified
 * reference (oracle/_ref/libslicecraft_ref.so via ref_shim.cpp) by
 * tests/test_oracle_pin.py and against the committed golden vectors in
 * tests/golden/.
 *
 * Every function names the reference lines it restates.  Arithmetic order is
 * part of the contract wherever it is floating point:
 *   - f64 summed-area table:  T = ((v + L) + U) - UL   (cost.cpp:97-115)
 *   - rect sum:               ((d - b) - c) + a        (cost.hpp:75-81)
 *   - layout time:            worst = max(0.0, ...)    (search.cpp:77-83)
 *   - slice SSE:              (double)(i128 num) / (double)count (texture.cpp:83-88)
 *   - layout SSE:             total = 0.0; total += sse in slice order (search.cpp:85-91)
 * Compiled with -ffp-contract=off so no FMA can change a rounding.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_COLS 64
#define ORC_MAX_SLICES 128

enum {
  ORC_OK = 0,
  ORC_ERR_GEOMETRY = 1,
  ORC_ERR_FORMAT = 7,
  ORC_ERR_CONFIG = 8,
  ORC_ERR_NO_CANDIDATE = 10,
  ORC_ERR_SIZE = 11,
};

/* ---- grid (grid.cpp:9-32) ------------------------------------------------ */
static int grid_make(int fw, int fh, int ctu, int* cols, int* rows) {
  if (ctu != 32 && ctu != 64 && ctu != 128) return ORC_ERR_GEOMETRY;
  if (fw < 1 || fh < 1) return ORC_ERR_GEOMETRY;
  *cols = (fw + ctu - 1) / ctu;
  *rows = (fh + ctu - 1) / ctu;
  return ORC_OK;
}
static int cell_w(int fw, int ctu, int x) { int r = fw - x * ctu; return r < ctu ? r : ctu; }
static int cell_h(int fh, int ctu, int y) { int r = fh - y * ctu; return r < ctu ? r : ctu; }

/* rectangle index shared with the product:
 * xw(x0,w) major (x0 outer, w inner), yh(y0,h) minor. */
static long xw_index(int cols, int x0, int w) { return (long)x0 * cols - (long)x0 * (x0 - 1) / 2 + (w - 1); }
static long yh_index(int rows, int y0, int h) { return (long)y0 * rows - (long)y0 * (y0 - 1) / 2 + (h - 1); }

/* ---- texture (texture.cpp:145-169) --------------------------------------- */
/* Per-CTU count/sum/sumsq, exact u64, over the true pixel extent of each CTU.
 * `luma` is bps-byte little-endian samples with a row pitch in bytes. */
int orc_ctu_stats(const void* luma, int bps, int fw, int fh, size_t pitch, int ctu,
                  uint64_t* out) {
  int cols, rows;
  int st = grid_make(fw, fh, ctu, &cols, &rows);
  if (st) return st;
  if (bps != 1 && bps != 2) return ORC_ERR_FORMAT;
  const unsigned char* base = (const unsigned char*)luma;
  for (int cy = 0; cy < rows; ++cy) {
    for (int cx = 0; cx < cols; ++cx) {
      uint64_t cnt = 0, sum = 0, sq = 0;
      int x1 = cx * ctu, y1 = cy * ctu;
      int x2 = x1 + cell_w(fw, ctu, cx), y2 = y1 + cell_h(fh, ctu, cy);
      for (int y = y1; y < y2; ++y) {
        const unsigned char* row = base + (size_t)y * pitch;
        for (int x = x1; x < x2; ++x) {
          uint64_t v = bps == 1 ? row[x] : ((const uint16_t*)row)[x];
          cnt += 1;
          sum += v;
          sq += v * v;
        }
      }
      uint64_t* r = out + 3 * ((size_t)cy * cols + cx);
      r[0] = cnt;
      r[1] = sum;
      r[2] = sq;
    }
  }
  return ORC_OK;
}

/* TextureStats ctor validation (texture.cpp:90-111). */
int orc_texture_validate(int fw, int fh, int ctu, const uint64_t* rec) {
  int cols, rows;
  int st = grid_make(fw, fh, ctu, &cols, &rows);
  if (st) return st;
  for (int y = 0; y < rows; ++y)
    for (int x = 0; x < cols; ++x) {
      const uint64_t* r = rec + 3 * ((size_t)y * cols + x);
      if (r[0] != (uint64_t)cell_w(fw, ctu, x) * (uint64_t)cell_h(fh, ctu, y)) return ORC_ERR_FORMAT;
      __int128 lhs = (__int128)r[0] * r[2];
      __int128 rhs = (__int128)r[1] * r[1];
      if (lhs < rhs) return ORC_ERR_FORMAT;
    }
  return ORC_OK;
}

/* ---- summed-area tables -------------------------------------------------- */
/* f64 SAT, row-major recurrence order of cost.cpp:97-112. */
static void sat_f64(const double* v, int cols, int rows, double* t) {
  size_t stride = (size_t)cols + 1;
  memset(t, 0, sizeof(double) * stride * (rows + 1));
  for (int y = 0; y < rows; ++y)
    for (int x = 0; x < cols; ++x) {
      size_t i = (size_t)(y + 1) * stride + (x + 1);
      t[i] = v[(size_t)y * cols + x] + t[i - 1] + t[i - stride] - t[i - stride - 1];
    }
}
/* cost.hpp:75-81 */
static double rect_sum(const double* t, int cols, int x0, int y0, int w, int h) {
  size_t s = (size_t)cols + 1;
  return t[(size_t)(y0 + h) * s + (x0 + w)] - t[(size_t)y0 * s + (x0 + w)] -
         t[(size_t)(y0 + h) * s + x0] + t[(size_t)y0 * s + x0];
}
/* u64 SATs, texture.cpp:113-129 (modular; order-free). */
static void sat_u64(const uint64_t* rec, int cols, int rows, uint64_t* t /* 3 tables */) {
  size_t stride = (size_t)cols + 1, cells = stride * (rows + 1);
  memset(t, 0, sizeof(uint64_t) * 3 * cells);
  for (int k = 0; k < 3; ++k) {
    uint64_t* p = t + k * cells;
    for (int y = 0; y < rows; ++y)
      for (int x = 0; x < cols; ++x) {
        size_t i = (size_t)(y + 1) * stride + (x + 1);
        p[i] = rec[3 * ((size_t)y * cols + x) + k] + p[i - 1] + p[i - stride] - p[i - stride - 1];
      }
  }
}
/* SliceMoments::sse (texture.cpp:83-88); GCC __int128 -> double is RNE. */
static double moments_sse(uint64_t c, uint64_t s, uint64_t q) {
  if (c == 0) return 0.0;
  __int128 num = (__int128)c * (__int128)q - (__int128)s * (__int128)s;
  return (double)num / (double)c;
}
static double rect_sse(const uint64_t* t, int cols, int rows, int x0, int y0, int w, int h) {
  size_t stride = (size_t)cols + 1, cells = stride * (rows + 1);
  size_t a = (size_t)y0 * stride + x0, b = (size_t)y0 * stride + (x0 + w);
  size_t c = (size_t)(y0 + h) * stride + x0, d = (size_t)(y0 + h) * stride + (x0 + w);
  uint64_t m[3];
  for (int k = 0; k < 3; ++k) {
    const uint64_t* p = t + k * cells;
    m[k] = p[d] - p[b] - p[c] + p[a];
  }
  return moments_sse(m[0], m[1], m[2]);
}

int orc_sat_f64(const double* v, int cols, int rows, double* t) {
  sat_f64(v, cols, rows, t);
  return ORC_OK;
}

/* Every rectangle's time, product order. */
int orc_rect_times(const double* times, int cols, int rows, double* out) {
  double* t = malloc(sizeof(double) * (cols + 1) * (rows + 1));
  sat_f64(times, cols, rows, t);
  for (int x0 = 0; x0 < cols; ++x0)
    for (int w = 1; w <= cols - x0; ++w)
      for (int y0 = 0; y0 < rows; ++y0)
        for (int h = 1; h <= rows - y0; ++h)
          out[xw_index(cols, x0, w) * (long)(rows * (rows + 1) / 2) + yh_index(rows, y0, h)] =
              rect_sum(t, cols, x0, y0, w, h);
  free(t);
  return ORC_OK;
}

/* Every rectangle's SSE, product order (validates like the TextureStats ctor). */
int orc_rect_sse(int fw, int fh, int ctu, const uint64_t* rec, double* out) {
  int cols, rows;
  int st = grid_make(fw, fh, ctu, &cols, &rows);
  if (st) return st;
  st = orc_texture_validate(fw, fh, ctu, rec);
  if (st) return st;
  uint64_t* t = malloc(sizeof(uint64_t) * 3 * (cols + 1) * (rows + 1));
  sat_u64(rec, cols, rows, t);
  for (int x0 = 0; x0 < cols; ++x0)
    for (int w = 1; w <= cols - x0; ++w)
      for (int y0 = 0; y0 < rows; ++y0)
        for (int h = 1; h <= rows - y0; ++h)
          out[xw_index(cols, x0, w) * (long)(rows * (rows + 1) / 2) + yh_index(rows, y0, h)] =
              rect_sse(t, cols, rows, x0, y0, w, h);
  free(t);
  return ORC_OK;
}

/* ---- cost model (cost.cpp:28-38, 66-95) ----------------------------------- */
int orc_temporal_layer(int poc, int gop, int* tl) {
  if (gop < 1 || (gop & (gop - 1)) != 0) return ORC_ERR_CONFIG;
  if (poc < 0) return ORC_ERR_CONFIG;
  unsigned rem = (unsigned)poc % (unsigned)gop;
  if (rem == 0) { *tl = 0; return ORC_OK; }
  *tl = __builtin_ctz((unsigned)gop) - __builtin_ctz(rem);
  return ORC_OK;
}

/* ---- ColumnSplit search (search.cpp:110-405) ------------------------------ */
typedef struct {
  int32_t n_cols;
  int32_t col_widths[ORC_MAX_COLS];
  int32_t runs_per_col[ORC_MAX_COLS];
  int32_t run_heights[ORC_MAX_SLICES];
} orc_layout;

typedef struct {
  double t_min_us;
  uint64_t candidates_step1;
  orc_layout argmin1;
  double t_best_us;
  double sse_best;
  uint64_t candidates_step2;
  orc_layout best;
} orc_result;

typedef struct {
  int cols, rows, n, ncols_max, coverage, step;
  double k, budget;
  const double* sat;       /* f64 SAT */
  const uint64_t* usat;    /* 3 u64 SATs (step 2) */
  /* current layout */
  int c;
  int w[ORC_MAX_COLS], r[ORC_MAX_COLS], h[ORC_MAX_SLICES];
  int nh;
  /* results */
  uint64_t count;
  int found;
  double best_t, best_sse;
  orc_layout best;
} dfs_t;

static double layout_time(const dfs_t* d) {
  double worst = 0.0;
  int x = 0, run = 0;
  for (int col = 0; col < d->c; ++col) {
    int y = 0;
    for (int j = 0; j < d->r[col]; ++j, ++run) {
      double v = rect_sum(d->sat, d->cols, x, y, d->w[col], d->h[run]);
      worst = worst < v ? v : worst; /* std::max(worst, v) */
      y += d->h[run];
    }
    x += d->w[col];
  }
  return worst;
}

static double layout_sse(const dfs_t* d) {
  double total = 0.0;
  int x = 0, run = 0;
  for (int col = 0; col < d->c; ++col) {
    int y = 0;
    for (int j = 0; j < d->r[col]; ++j, ++run) {
      total += rect_sse(d->usat, d->cols, d->rows, x, y, d->w[col], d->h[run]);
      y += d->h[run];
    }
    x += d->w[col];
  }
  return total;
}

static void snapshot(dfs_t* d) {
  memset(&d->best, 0, sizeof(d->best));
  d->best.n_cols = d->c;
  for (int i = 0; i < d->c; ++i) {
    d->best.col_widths[i] = d->w[i];
    d->best.runs_per_col[i] = d->r[i];
  }
  for (int i = 0; i < d->n; ++i) d->best.run_heights[i] = d->h[i];
}

/* sink + reduce of run_step1 (search.cpp:280-289) / step 2 (search.cpp:375-394) */
static void leaf(dfs_t* d) {
  d->count++;
  double t = layout_time(d);
  if (d->step == 1) {
    if (t < d->best_t) { d->best_t = t; d->found = 1; snapshot(d); }
  } else {
    if (t <= d->budget) {
      double sse = layout_sse(d);
      if (sse < d->best_sse || (sse == d->best_sse && t < d->best_t)) {
        d->best_sse = sse; d->best_t = t; d->found = 1; snapshot(d);
      }
    }
  }
}

/* rec_heights (search.cpp:163-190) */
static void rec_heights(dfs_t* d, int col, int run, int rows_left, int64_t amin, int64_t amax) {
  if (col == d->c) { leaf(d); return; }
  int runs = d->r[col];
  if (run == runs) { rec_heights(d, col + 1, 0, d->rows, amin, amax); return; }
  int w = d->w[col];
  int runs_left = runs - run;
  int lo = runs_left == 1 ? rows_left : 1;
  int hi = rows_left - (runs_left - 1);
  for (int h = lo; h <= hi; ++h) {
    int64_t area = (int64_t)w * h;
    int64_t na = amin < area ? amin : area;
    int64_t nx = amax > area ? amax : area;
    if (!(d->k * (double)na > (double)nx)) continue;
    d->h[d->nh++] = h;
    rec_heights(d, col, run + 1, rows_left - h, na, nx);
    d->nh--;
  }
}

/* rec_runs (search.cpp:145-161) */
static void rec_runs(dfs_t* d, int col, int slices_left) {
  if (col == d->c) {
    if (slices_left == 0) { d->nh = 0; rec_heights(d, 0, 0, d->rows, INT64_MAX, 0); }
    return;
  }
  int after = d->c - col - 1;
  int lo = slices_left - after * d->rows; if (lo < 1) lo = 1;
  int hi = slices_left - after; if (hi > d->rows) hi = d->rows;
  for (int r = lo; r <= hi; ++r) { d->r[col] = r; rec_runs(d, col + 1, slices_left - r); }
}

/* rec_widths (search.cpp:133-143): note the reference does NOT require the
 * widths to sum to the grid width (compat); coverage=1 keeps only Σw == cols. */
static void rec_widths(dfs_t* d, int col, int cols_left) {
  if (col == d->c) {
    if (d->coverage && cols_left != 0) return;
    rec_runs(d, 0, d->n);
    return;
  }
  int max_w = cols_left - (d->c - col - 1);
  for (int w = 1; w <= max_w; ++w) { d->w[col] = w; rec_widths(d, col + 1, cols_left - w); }
}

static int check_cfg(int n, double lambda, double k, int max_cols) {
  /* SearchConfig::check (search.cpp:28-36) */
  if (n < 1) return ORC_ERR_CONFIG;
  if (!(k > 1.0)) return ORC_ERR_CONFIG;
  if (!(lambda >= 0.0) || !isfinite(lambda)) return ORC_ERR_CONFIG;
  if (max_cols < 0) return ORC_ERR_CONFIG;
  return ORC_OK;
}

static void run_generator(dfs_t* d) {
  /* ColumnSplitGenerator::run (search.cpp:120-128) */
  int maxc = d->n;
  if (d->ncols_max < maxc) maxc = d->ncols_max;
  if (d->cols < maxc) maxc = d->cols;
  for (int c = 1; c <= maxc; ++c) { d->c = c; rec_widths(d, 0, d->cols); }
}

/* two_step_partition minus the estimate (search.cpp:407-434); the estimate is
 * the caller's est map.  step: 1 = step 1 only; 2 = step 2 only with t_min_in;
 * 3 = both.  coverage: 0 = reference (Σw <= cols), 1 = covering (Σw == cols). */
int orc_search(int fw, int fh, int ctu, const double* est, const uint64_t* rec, int n,
               double lambda, double k, int max_tile_cols, int coverage, int step,
               double t_min_in, orc_result* out) {
  int cols, rows;
  int st = grid_make(fw, fh, ctu, &cols, &rows);
  if (st) return st;
  st = check_cfg(n, lambda, k, max_tile_cols);
  if (st) return st;
  if (n > cols * rows) return ORC_ERR_GEOMETRY;
  if (n > ORC_MAX_SLICES) return ORC_ERR_SIZE;
  memset(out, 0, sizeof(*out));
  double* sat = malloc(sizeof(double) * (cols + 1) * (rows + 1));
  sat_f64(est, cols, rows, sat);
  uint64_t* usat = NULL;
  dfs_t* d = calloc(1, sizeof(dfs_t));
  d->cols = cols; d->rows = rows; d->n = n; d->k = k; d->coverage = coverage;
  d->ncols_max = max_tile_cols > 0 ? max_tile_cols : n;
  d->sat = sat;
  double t_min = t_min_in;
  if (step & 1) {
    d->step = 1; d->count = 0; d->found = 0; d->best_t = INFINITY;
    run_generator(d);
    if (!d->found) { free(sat); free(d); return ORC_ERR_NO_CANDIDATE; }
    out->t_min_us = d->best_t;
    out->candidates_step1 = d->count;
    out->argmin1 = d->best;
    t_min = d->best_t;
  }
  if (step & 2) {
    st = orc_texture_validate(fw, fh, ctu, rec);
    if (st) { free(sat); free(d); return st; }
    usat = malloc(sizeof(uint64_t) * 3 * (cols + 1) * (rows + 1));
    sat_u64(rec, cols, rows, usat);
    d->usat = usat;
    d->step = 2; d->count = 0; d->found = 0;
    d->best_t = INFINITY; d->best_sse = INFINITY;
    d->budget = t_min * (1.0 + lambda); /* search.cpp:344 */
    run_generator(d);
    if (!d->found) { free(sat); free(usat); free(d); return ORC_ERR_NO_CANDIDATE; }
    if (!(step & 1)) out->t_min_us = t_min;
    out->t_best_us = d->best_t;
    out->sse_best = d->best_sse;
    out->candidates_step2 = d->count;
    out->best = d->best;
  }
  free(sat); free(usat); free(d);
  return ORC_OK;
}

/* Count-only walk of the same family (for_each_candidate, search.cpp:302-319). */
static void count_heights(dfs_t* d, int col, int run, int rows_left, int64_t amin, int64_t amax) {
  if (col == d->c) { d->count++; return; }
  int runs = d->r[col];
  if (run == runs) { count_heights(d, col + 1, 0, d->rows, amin, amax); return; }
  int w = d->w[col], runs_left = runs - run;
  int lo = runs_left == 1 ? rows_left : 1, hi = rows_left - (runs_left - 1);
  for (int h = lo; h <= hi; ++h) {
    int64_t area = (int64_t)w * h;
    int64_t na = amin < area ? amin : area, nx = amax > area ? amax : area;
    if (!(d->k * (double)na > (double)nx)) continue;
    count_heights(d, col, run + 1, rows_left - h, na, nx);
  }
}
static void count_runs(dfs_t* d, int col, int slices_left) {
  if (col == d->c) { if (slices_left == 0) count_heights(d, 0, 0, d->rows, INT64_MAX, 0); return; }
  int after = d->c - col - 1;
  int lo = slices_left - after * d->rows; if (lo < 1) lo = 1;
  int hi = slices_left - after; if (hi > d->rows) hi = d->rows;
  for (int r = lo; r <= hi; ++r) { d->r[col] = r; count_runs(d, col + 1, slices_left - r); }
}
static void count_widths(dfs_t* d, int col, int cols_left) {
  if (col == d->c) { if (d->coverage && cols_left != 0) return; count_runs(d, 0, d->n); return; }
  int max_w = cols_left - (d->c - col - 1);
  for (int w = 1; w <= max_w; ++w) { d->w[col] = w; count_widths(d, col + 1, cols_left - w); }
}
int orc_count(int cols, int rows, int n, double k, int max_tile_cols, int coverage, uint64_t* count) {
  dfs_t* d = calloc(1, sizeof(dfs_t));
  d->cols = cols; d->rows = rows; d->n = n; d->k = k; d->coverage = coverage;
  d->ncols_max = max_tile_cols > 0 ? max_tile_cols : n;
  int maxc = n;
  if (d->ncols_max < maxc) maxc = d->ncols_max;
  if (cols < maxc) maxc = cols;
  for (int c = 1; c <= maxc; ++c) { d->c = c; count_widths(d, 0, cols); }
  *count = d->count;
  free(d);
  return ORC_OK;
}

/* ---- exact branch-and-bound restatement (configs 4/5) ---------------------
 * The reference DFS (rec_widths / rec_runs / rec_heights, search.cpp:133-190)
 * in the reference's order, scoring like run_step1 / the step-2 reduction
 * (search.cpp:283-289, 386-394), but skipping a subtree when no candidate in
 * it can win under the reference's strict comparisons:
 *   step 1: a lower bound LB >= best_t (ties later in order never replace),
 *   step 2: LB > budget (infeasible).
 * LB is the running max of the slices already fixed, tightened at the widths
 * and runs levels by colLB(x0, w, r): the minimum over all compositions of the
 * column into r runs of its slowest run (area constraint relaxed), from a DP
 * over rows.  Written independently of the GPU walk; counts are not
 * enumerated (the caller takes them from the exact DP). */
typedef struct {
  dfs_t d;
  double* lb;   /* lb[(xw * (rmax+1) + r)] exact r */
  double* lbm;  /* prefix min over r' <= r */
  int rmax;
} bb_t;

static double rt_clamped(const dfs_t* d, int x0, int y0, int w, int h) {
  double v = rect_sum(d->sat, d->cols, x0, y0, w, h);
  return v > 0.0 ? v : 0.0; /* layout_time's max from 0.0 (search.cpp:78-81) */
}

static void bb_bounds(bb_t* b) {
  dfs_t* d = &b->d;
  int cols = d->cols, rows = d->rows, R = b->rmax;
  int nxw = cols * (cols + 1) / 2;
  b->lb = malloc(sizeof(double) * nxw * (R + 1));
  b->lbm = malloc(sizeof(double) * nxw * (R + 1));
  double* prev = malloc(sizeof(double) * (rows + 1));
  double* cur = malloc(sizeof(double) * (rows + 1));
  for (int x0 = 0; x0 < cols; ++x0)
    for (int w = 1; w <= cols - x0; ++w) {
      long xw = xw_index(cols, x0, w);
      for (int y = 0; y <= rows; ++y) prev[y] = y == 0 ? 0.0 : INFINITY;
      double runmin = INFINITY;
      b->lb[xw * (R + 1)] = INFINITY;
      b->lbm[xw * (R + 1)] = INFINITY;
      for (int r = 1; r <= R; ++r) {
        for (int y = 0; y <= rows; ++y) {
          double best = INFINITY;
          for (int y0 = 0; y0 < y; ++y0) {
            if (prev[y0] == INFINITY) continue;
            double v = rt_clamped(d, x0, y0, w, y - y0);
            double m = prev[y0] > v ? prev[y0] : v;
            if (m < best) best = m;
          }
          cur[y] = best;
        }
        b->lb[xw * (R + 1) + r] = cur[rows];
        if (cur[rows] < runmin) runmin = cur[rows];
        b->lbm[xw * (R + 1) + r] = runmin;
        memcpy(prev, cur, sizeof(double) * (rows + 1));
      }
    }
  free(prev);
  free(cur);
}

static int bb_dead(const bb_t* b, double lbv) {
  const dfs_t* d = &b->d;
  return d->step == 1 ? !(lbv < d->best_t) : (lbv > d->budget);
}

static void bb_heights(bb_t* b, int col, int run, int rows_left, int64_t amin, int64_t amax,
                       int x, double P) {
  dfs_t* d = &b->d;
  if (col == d->c) {
    leaf(d);
    return;
  }
  int runs = d->r[col];
  if (run == runs) {
    bb_heights(b, col + 1, 0, d->rows, amin, amax, x + d->w[col], P);
    return;
  }
  int w = d->w[col], runs_left = runs - run;
  int lo = runs_left == 1 ? rows_left : 1, hi = rows_left - (runs_left - 1);
  int y0 = d->rows - rows_left;
  for (int h = lo; h <= hi; ++h) {
    int64_t area = (int64_t)w * h;
    int64_t na = amin < area ? amin : area, nx = amax > area ? amax : area;
    if (!(d->k * (double)na > (double)nx)) continue;
    double v = rt_clamped(d, x, y0, w, h);
    double Pn = P > v ? P : v;
    if (bb_dead(b, Pn)) continue;
    d->h[d->nh++] = h;
    bb_heights(b, col, run + 1, rows_left - h, na, nx, x, Pn);
    d->nh--;
  }
}

static void bb_runs(bb_t* b, int col, int slices_left, int x, double PR) {
  dfs_t* d = &b->d;
  if (col == d->c) {
    if (slices_left == 0) {
      d->nh = 0;
      bb_heights(b, 0, 0, d->rows, INT64_MAX, 0, 0, 0.0);
    }
    return;
  }
  int after = d->c - col - 1;
  int lo = slices_left - after * d->rows; if (lo < 1) lo = 1;
  int hi = slices_left - after; if (hi > d->rows) hi = d->rows;
  long xw = xw_index(d->cols, x, d->w[col]);
  for (int r = lo; r <= hi; ++r) {
    double v = r <= b->rmax ? b->lb[xw * (b->rmax + 1) + r] : 0.0;
    double P = PR > v ? PR : v;
    if (bb_dead(b, P)) continue;
    d->r[col] = r;
    bb_runs(b, col + 1, slices_left - r, x + d->w[col], P);
  }
}

static void bb_widths(bb_t* b, int col, int cols_left, double PW, int rmax_c) {
  dfs_t* d = &b->d;
  if (col == d->c) {
    if (d->coverage && cols_left != 0) return;
    bb_runs(b, 0, d->n, 0, PW);
    return;
  }
  int max_w = cols_left - (d->c - col - 1);
  int x = d->cols - cols_left;
  for (int w = 1; w <= max_w; ++w) {
    double v = b->lbm[xw_index(d->cols, x, w) * (b->rmax + 1) + rmax_c];
    double P = PW > v ? PW : v;
    if (bb_dead(b, P)) continue;
    d->w[col] = w;
    bb_widths(b, col + 1, cols_left - w, P, rmax_c);
  }
}

static void bb_generator(bb_t* b) {
  dfs_t* d = &b->d;
  int maxc = d->n;
  if (d->ncols_max < maxc) maxc = d->ncols_max;
  if (d->cols < maxc) maxc = d->cols;
  for (int c = 1; c <= maxc; ++c) {
    d->c = c;
    int rmax_c = d->n - c + 1;
    if (rmax_c > d->rows) rmax_c = d->rows;
    if (rmax_c > b->rmax) rmax_c = b->rmax;
    bb_widths(b, 0, d->cols, 0.0, rmax_c);
  }
}

/* Same contract as orc_search (steps, outputs), counts left at 0. */
int orc_search_pruned(int fw, int fh, int ctu, const double* est, const uint64_t* rec, int n,
                      double lambda, double k, int max_tile_cols, int coverage, int step,
                      double t_min_in, orc_result* out) {
  int cols, rows;
  int st = grid_make(fw, fh, ctu, &cols, &rows);
  if (st) return st;
  st = check_cfg(n, lambda, k, max_tile_cols);
  if (st) return st;
  if (n > cols * rows) return ORC_ERR_GEOMETRY;
  if (n > ORC_MAX_SLICES) return ORC_ERR_SIZE;
  memset(out, 0, sizeof(*out));
  bb_t* b = calloc(1, sizeof(bb_t));
  dfs_t* d = &b->d;
  double* sat = malloc(sizeof(double) * (cols + 1) * (rows + 1));
  sat_f64(est, cols, rows, sat);
  uint64_t* usat = NULL;
  d->cols = cols; d->rows = rows; d->n = n; d->k = k; d->coverage = coverage;
  d->ncols_max = max_tile_cols > 0 ? max_tile_cols : n;
  d->sat = sat;
  b->rmax = n < rows ? n : rows;
  bb_bounds(b);
  double t_min = t_min_in;
  if (step & 1) {
    d->step = 1; d->found = 0; d->best_t = INFINITY;
    bb_generator(b);
    if (!d->found) { st = ORC_ERR_NO_CANDIDATE; goto done; }
    out->t_min_us = d->best_t;
    out->argmin1 = d->best;
    t_min = d->best_t;
  }
  if (step & 2) {
    st = orc_texture_validate(fw, fh, ctu, rec);
    if (st) goto done;
    usat = malloc(sizeof(uint64_t) * 3 * (cols + 1) * (rows + 1));
    sat_u64(rec, cols, rows, usat);
    d->usat = usat;
    d->step = 2; d->found = 0;
    d->best_t = INFINITY; d->best_sse = INFINITY;
    d->budget = t_min * (1.0 + lambda);
    bb_generator(b);
    if (!d->found) { st = ORC_ERR_NO_CANDIDATE; goto done; }
    if (!(step & 1)) out->t_min_us = t_min;
    out->t_best_us = d->best_t;
    out->sse_best = d->best_sse;
    out->best = d->best;
  }
done:
  free(sat); free(usat); free(b->lb); free(b->lbm); free(b);
  return st;
}
