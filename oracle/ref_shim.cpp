// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (the `slicecraft`
// sources under /root/reference/proj/src, compiled in place by
// oracle/Makefile into oracle/_ref/libslicecraft_ref.so).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
// load it.  Every function forwards to the reference entry point named in its
// comment; exceptions are mapped to the same status codes the product C-ABI
// uses (include/slicecraft_b200.h, SC_ERR_*), so tests can compare error
// behaviour one-for-one.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "slicecraft/cost.hpp"
#include "slicecraft/errors.hpp"
#include "slicecraft/grid.hpp"
#include "slicecraft/search.hpp"
#include "slicecraft/texture.hpp"

using namespace slicecraft;

namespace {

thread_local std::string g_err;

// Same numbering as sc_status in include/slicecraft_b200.h.
int map_exception() {
  try {
    throw;
  } catch (const GeometryError& e) { g_err = e.what(); return 1; }
  catch (const OverlapError& e) { g_err = e.what(); return 2; }
  catch (const CoverageError& e) { g_err = e.what(); return 3; }
  catch (const StructureError& e) { g_err = e.what(); return 4; }
  catch (const IoError& e) { g_err = e.what(); return 5; }
  catch (const RangeError& e) { g_err = e.what(); return 6; }
  catch (const FormatError& e) { g_err = e.what(); return 7; }
  catch (const ConfigError& e) { g_err = e.what(); return 8; }
  catch (const TraceError& e) { g_err = e.what(); return 9; }
  catch (const NoCandidateError& e) { g_err = e.what(); return 10; }
  catch (const SizeError& e) { g_err = e.what(); return 11; }
  catch (const UsageError& e) { g_err = e.what(); return 12; }
  catch (const std::exception& e) { g_err = e.what(); return 99; }
  catch (...) { g_err = "unknown"; return 99; }
}

// Flat layout record shared with oracle/oracle.py (ctypes mirror).
struct RefLayout {
  int32_t n_cols;
  int32_t n_slices;
  int32_t col_widths[64];
  int32_t row_heights[64];
  int32_t n_tile_rows;
  int32_t slices[128][5];  // x0, y0, w, h, id
};

struct RefOutcome {
  double t_min_us, t_best_us, sse_best;
  uint64_t candidates_evaluated, candidates_step1, candidates_step2;
  double search_time_us, time_min_step_us, clustering_step_us;
  int32_t est_source, est_source_poc;
  RefLayout best;
};

void to_layout(const Partition& p, RefLayout* out) {
  std::memset(out, 0, sizeof(*out));
  out->n_cols = static_cast<int32_t>(p.tiles.col_widths.size());
  out->n_tile_rows = static_cast<int32_t>(p.tiles.row_heights.size());
  out->n_slices = p.slice_count();
  for (size_t i = 0; i < p.tiles.col_widths.size() && i < 64; ++i)
    out->col_widths[i] = p.tiles.col_widths[i];
  for (size_t i = 0; i < p.tiles.row_heights.size() && i < 64; ++i)
    out->row_heights[i] = p.tiles.row_heights[i];
  for (size_t i = 0; i < p.slices.size() && i < 128; ++i) {
    const RectSlice& s = p.slices[i];
    out->slices[i][0] = s.x0;
    out->slices[i][1] = s.y0;
    out->slices[i][2] = s.w;
    out->slices[i][3] = s.h;
    out->slices[i][4] = s.id;
  }
}

SearchConfig make_cfg(int n, double lambda, double k, int family, int max_cols,
                      int workers) {
  SearchConfig c;
  c.n_slices = n;
  c.lambda = lambda;
  c.k_area = k;
  c.family = family == 1 ? CandidateFamily::UniformOnly : CandidateFamily::ColumnSplit;
  c.max_tile_cols = max_cols;
  c.workers = workers;
  return c;
}

CostMap make_map(const CtuGrid& g, const double* times, int poc, int tl) {
  CostMap m;
  m.grid = g;
  m.times_us.assign(times, times + g.cell_count());
  m.poc = poc;
  m.temporal_layer = tl;
  return m;
}

TextureStats make_stats(const CtuGrid& g, const uint64_t* rec, int poc) {
  std::vector<CtuRecord> r(static_cast<size_t>(g.cell_count()));
  for (size_t i = 0; i < r.size(); ++i) {
    r[i].count = rec[3 * i];
    r[i].sum = rec[3 * i + 1];
    r[i].sumsq = rec[3 * i + 2];
  }
  return TextureStats(g, std::move(r), poc);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

size_t ref_layout_size() { return sizeof(RefLayout); }
size_t ref_outcome_size() { return sizeof(RefOutcome); }

// CtuGrid::make (grid.cpp:9-24)
int ref_grid_make(int w, int h, int ctu, int* cols, int* rows) {
  try {
    CtuGrid g = CtuGrid::make(w, h, ctu);
    *cols = g.cols;
    *rows = g.rows;
    return 0;
  } catch (...) { return map_exception(); }
}

// ctu_stats (texture.cpp:145-169) on a uint16 plane; records out as
// {count, sum, sumsq} triplets, row-major over the CTU grid.
int ref_ctu_stats(const uint16_t* samples, int w, int h, int bit_depth, int ctu,
                  int poc, uint64_t* out) {
  try {
    CtuGrid g = CtuGrid::make(w, h, ctu);
    LumaPlane p;
    p.width = w;
    p.height = h;
    p.bit_depth = bit_depth;
    p.samples.assign(samples, samples + static_cast<size_t>(w) * h);
    TextureStats st = ctu_stats(p, g, poc);
    const auto& r = st.records();
    for (size_t i = 0; i < r.size(); ++i) {
      out[3 * i] = r[i].count;
      out[3 * i + 1] = r[i].sum;
      out[3 * i + 2] = r[i].sumsq;
    }
    return 0;
  } catch (...) { return map_exception(); }
}

// TextureStats ctor validation (texture.cpp:90-111) on caller records.
int ref_texture_validate(int w, int h, int ctu, const uint64_t* rec) {
  try {
    CtuGrid g = CtuGrid::make(w, h, ctu);
    make_stats(g, rec, 0);
    return 0;
  } catch (...) { return map_exception(); }
}

// PrefixSumTable::rect_sum (cost.hpp:75-81) for every rectangle, in the
// product's rectangle order: xw(x0,w) major, yh(y0,h) minor, x0/y0 outer.
int ref_rect_times(const double* times, int cols, int rows, double* out) {
  try {
    std::vector<double> v(times, times + static_cast<size_t>(cols) * rows);
    PrefixSumTable t(v, cols, rows);
    size_t i = 0;
    for (int x0 = 0; x0 < cols; ++x0)
      for (int w = 1; w <= cols - x0; ++w)
        for (int y0 = 0; y0 < rows; ++y0)
          for (int h = 1; h <= rows - y0; ++h) out[i++] = t.rect_sum(x0, y0, w, h);
    return 0;
  } catch (...) { return map_exception(); }
}

// TextureStats::rect_moments(...).sse() (texture.cpp:83-88, 132-143), same order.
int ref_rect_sse(int fw, int fh, int ctu, const uint64_t* rec, double* out,
                 uint64_t* moments_out) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    TextureStats st = make_stats(g, rec, 0);
    size_t i = 0;
    for (int x0 = 0; x0 < g.cols; ++x0)
      for (int w = 1; w <= g.cols - x0; ++w)
        for (int y0 = 0; y0 < g.rows; ++y0)
          for (int h = 1; h <= g.rows - y0; ++h) {
            SliceMoments m = st.rect_moments(x0, y0, w, h);
            if (moments_out) {
              moments_out[3 * i] = m.count;
              moments_out[3 * i + 1] = m.sum;
              moments_out[3 * i + 2] = m.sumsq;
            }
            out[i++] = m.sse();
          }
    return 0;
  } catch (...) { return map_exception(); }
}

// for_each_candidate (search.cpp:302-319): count, and optionally the first
// `max_out` layouts.
int ref_enumerate(int fw, int fh, int ctu, int n, double k, int family, int max_cols,
                  uint64_t* count, RefLayout* out, uint64_t max_out) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    SearchConfig c = make_cfg(n, 0.0, k, family, max_cols, 1);
    uint64_t cnt = 0;
    for_each_candidate(g, c, [&](const Partition& p) {
      if (out && cnt < max_out) to_layout(p, &out[cnt]);
      ++cnt;
    });
    *count = cnt;
    return 0;
  } catch (...) { return map_exception(); }
}

// min_time_search (search.cpp:328-332)
int ref_min_time_search(int fw, int fh, int ctu, const double* est, int n,
                        double lambda, double k, int family, int max_cols, int workers,
                        double* t_min, RefLayout* argmin) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    CostMap m = make_map(g, est, 0, 0);
    auto r = min_time_search(m, make_cfg(n, lambda, k, family, max_cols, workers));
    *t_min = r.first;
    to_layout(r.second, argmin);
    return 0;
  } catch (...) { return map_exception(); }
}

// constrained_clustering_search (search.cpp:334-405)
int ref_constrained_clustering(int fw, int fh, int ctu, const double* est,
                               const uint64_t* rec, double t_min, int n, double lambda,
                               double k, int family, int max_cols, int workers,
                               RefOutcome* out) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    CostMap m = make_map(g, est, 0, 0);
    TextureStats st = make_stats(g, rec, 0);
    SearchOutcome o = constrained_clustering_search(
        m, st, t_min, make_cfg(n, lambda, k, family, max_cols, workers));
    std::memset(out, 0, sizeof(*out));
    out->t_min_us = o.t_min_us;
    out->t_best_us = o.t_best_us;
    out->sse_best = o.sse_best;
    out->candidates_evaluated = o.candidates_evaluated;
    out->candidates_step1 = o.candidates_step1;
    out->candidates_step2 = o.candidates_step2;
    to_layout(o.best, &out->best);
    return 0;
  } catch (...) { return map_exception(); }
}

// two_step_partition (search.cpp:407-434) over a history built with
// CostHistory::append (cost.cpp:56-75): `n_maps` maps of cells doubles each,
// with their pocs and temporal layers, in encode order.
int ref_two_step(int fw, int fh, int ctu, int gop, int n_maps, const double* maps,
                 const int* pocs, const int* tls, const uint64_t* rec, int poc, int n,
                 double lambda, double k, int family, int max_cols, int workers,
                 RefOutcome* out) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    CostHistory hist(g, gop);
    for (int i = 0; i < n_maps; ++i)
      hist.append(make_map(g, maps + static_cast<size_t>(i) * g.cell_count(), pocs[i],
                           tls[i]));
    TextureStats st = make_stats(g, rec, poc);
    SearchOutcome o =
        two_step_partition(hist, st, poc, make_cfg(n, lambda, k, family, max_cols, workers));
    std::memset(out, 0, sizeof(*out));
    out->t_min_us = o.t_min_us;
    out->t_best_us = o.t_best_us;
    out->sse_best = o.sse_best;
    out->candidates_evaluated = o.candidates_evaluated;
    out->candidates_step1 = o.candidates_step1;
    out->candidates_step2 = o.candidates_step2;
    out->search_time_us = o.search_time_us;
    out->time_min_step_us = o.time_min_step_us;
    out->clustering_step_us = o.clustering_step_us;
    out->est_source = static_cast<int32_t>(o.est_source);
    out->est_source_poc = o.est_source_poc;
    to_layout(o.best, &out->best);
    return 0;
  } catch (...) { return map_exception(); }
}

// temporal_layer_of_poc (cost.cpp:28-38)
int ref_temporal_layer(int poc, int gop, int* tl) {
  try {
    *tl = temporal_layer_of_poc(poc, gop);
    return 0;
  } catch (...) { return map_exception(); }
}

// estimate_ctu_times (cost.cpp:66-95)
int ref_estimate(int fw, int fh, int ctu, int gop, int n_maps, const double* maps,
                 const int* pocs, const int* tls, int poc, double* est, int* source,
                 int* source_poc) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    CostHistory hist(g, gop);
    for (int i = 0; i < n_maps; ++i)
      hist.append(make_map(g, maps + static_cast<size_t>(i) * g.cell_count(), pocs[i],
                           tls[i]));
    CostMap e = estimate_ctu_times(hist, poc);
    std::memcpy(est, e.times_us.data(), e.times_us.size() * sizeof(double));
    *source = static_cast<int>(e.source);
    *source_poc = e.source_poc;
    return 0;
  } catch (...) { return map_exception(); }
}

// uniform_partition (grid.cpp:186-262)
int ref_uniform_partition(int fw, int fh, int ctu, int n, RefLayout* out) {
  try {
    to_layout(uniform_partition(CtuGrid::make(fw, fh, ctu), n), out);
    return 0;
  } catch (...) { return map_exception(); }
}

// partition_time (cost.cpp:117-145) and partition_sse (texture.cpp:183-189)
// on a partition given as tile widths + slices; optionally validated first
// (validate_partition, grid.cpp:86-184).
int ref_partition_eval(int fw, int fh, int ctu, int n_cols, const int* col_widths,
                       int n_rows, const int* row_heights, int n_slices,
                       const int* slices, const double* times, const uint64_t* rec,
                       int validate, double* max_us, double* total_us, int64_t* argmax,
                       double* sse) {
  try {
    CtuGrid g = CtuGrid::make(fw, fh, ctu);
    TileGrid t;
    t.col_widths.assign(col_widths, col_widths + n_cols);
    t.row_heights.assign(row_heights, row_heights + n_rows);
    std::vector<RectSlice> s(static_cast<size_t>(n_slices));
    for (int i = 0; i < n_slices; ++i)
      s[i] = RectSlice{slices[5 * i], slices[5 * i + 1], slices[5 * i + 2],
                       slices[5 * i + 3], slices[5 * i + 4]};
    Partition p;
    if (validate) {
      p = validate_partition(g, t, s);
    } else {  // compat-mode candidates do not cover the grid (search.cpp:133-143)
      p.grid = g;
      p.tiles = t;
      p.slices = s;
    }
    if (times) {
      SliceTimeTable tt = partition_time(make_map(g, times, 0, 0), p);
      *max_us = tt.max_us;
      *total_us = tt.total_us;
      *argmax = static_cast<int64_t>(tt.argmax);
    }
    if (rec) *sse = partition_sse(make_stats(g, rec, 0), p);
    return 0;
  } catch (...) { return map_exception(); }
}

// yuv_frame_count (texture.cpp:25-40) and load_yuv_frame (texture.cpp:42-81)
int ref_yuv_frame_count(const char* path, int w, int h, int bit_depth, int* out) {
  try {
    *out = yuv_frame_count(path, w, h, bit_depth);
    return 0;
  } catch (...) { return map_exception(); }
}

int ref_load_yuv_frame(const char* path, int w, int h, int poc, int bit_depth, uint16_t* out) {
  try {
    const LumaPlane p = load_yuv_frame(path, w, h, poc, bit_depth);
    std::memcpy(out, p.samples.data(), p.samples.size() * sizeof(uint16_t));
    return 0;
  } catch (...) { return map_exception(); }
}

}  // extern "C"
