// Drop-in binding of the B200 partitioner core for code written against the
// reference `slicecraft` API (proj/include/slicecraft/*.hpp).
//
// Compile it together with the reference headers (the API contract) and link
// libslicecraft_dropin.so (dropin/slicecraft_api.cpp: every out-of-line
// function those headers declare, on the C-ABI) + libslicecraft_b200.so; no
// reference library is needed.  Every function takes and returns the
// reference's own types and throws the reference's own exception classes
// (errors.hpp:10-85); the compute runs in the sm_100a kernels behind
// include/slicecraft_b200.h.  The functions below take an explicit Context
// and search mode; the unqualified slicecraft:: functions use the implicit
// per-thread context.
//
//   slicecraft::ctu_stats(luma, grid, poc)              -> b200::ctu_stats(ctx, ...)
//   slicecraft::min_time_search(est, cfg)               -> b200::min_time_search(ctx, ...)
//   slicecraft::constrained_clustering_search(...)      -> b200::constrained_clustering_search(ctx, ...)
//   slicecraft::two_step_partition(history, stats, ...) -> b200::two_step_partition(ctx, ...)
//   slicecraft::uniform_partition(grid, n)              -> b200::uniform_partition(grid, n)
//   slicecraft::partition_time(costs, p)                -> b200::partition_time(ctx, costs, p)
//   slicecraft::partition_sse(stats, p)                 -> b200::partition_sse(ctx, stats, p)
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "slicecraft/cost.hpp"
#include "slicecraft/errors.hpp"
#include "slicecraft/grid.hpp"
#include "slicecraft/search.hpp"
#include "slicecraft/texture.hpp"
#include "slicecraft_b200.h"

namespace slicecraft {
namespace b200 {

// sc_status -> the reference exception class (errors.hpp:10-85).
[[noreturn]] inline void rethrow(sc_status s) {
  const std::string m = sc_last_error();
  switch (s) {
    case SC_ERR_GEOMETRY: throw GeometryError(m);
    case SC_ERR_OVERLAP: throw OverlapError(m);
    case SC_ERR_COVERAGE: throw CoverageError(m);
    case SC_ERR_STRUCTURE: throw StructureError(m);
    case SC_ERR_IO: throw IoError(m);
    case SC_ERR_RANGE: throw RangeError(m);
    case SC_ERR_FORMAT: throw FormatError(m);
    case SC_ERR_CONFIG: throw ConfigError(m);
    case SC_ERR_TRACE: throw TraceError(m);
    case SC_ERR_NO_CANDIDATE: throw NoCandidateError(m);
    case SC_ERR_SIZE: throw SizeError(m);
    case SC_ERR_USAGE: throw UsageError(m);
    default: throw Error(m);
  }
}
inline void check(sc_status s) {
  if (s != SC_OK) rethrow(s);
}

class Context;
// The implicit context behind the reference-API functions of the link-level
// drop-in (dropin/slicecraft_api.cpp, libslicecraft_dropin.so): one per host
// thread on device SLICECRAFT_B200_DEVICE (default 0), searching in
// SLICECRAFT_B200_MODE (exhaustive, or pruned) unless set here.
void set_default_device(int device);
void set_default_mode(int mode);  // SC_MODE_EXHAUSTIVE / SC_MODE_PRUNED
int default_mode();
Context& default_context();

// One device context (streams, device tables, cached search plans).
class Context {
 public:
  explicit Context(int device = 0) { check(sc_ctx_create(device, &ctx_)); }
  ~Context() { sc_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  sc_ctx* get() const { return ctx_; }

 private:
  sc_ctx* ctx_ = nullptr;
};

inline sc_grid to_c(const CtuGrid& g) {
  return sc_grid{g.frame_width, g.frame_height, g.ctu_size, g.cols, g.rows};
}

// SearchConfig (search.hpp:22-34); the B200 fields default to the reference
// family (widths summing to <= cols) and the exhaustive walk.
inline sc_search_cfg to_c(const SearchConfig& c, int mode = SC_MODE_EXHAUSTIVE) {
  sc_search_cfg r;
  r.n_slices = c.n_slices;
  r.lambda = c.lambda;
  r.k_area = c.k_area;
  r.family = c.family == CandidateFamily::UniformOnly ? SC_FAMILY_UNIFORM_ONLY
                                                      : SC_FAMILY_COLUMN_SPLIT;
  r.max_tile_cols = c.max_tile_cols;
  r.workers = c.workers;
  r.coverage = SC_COVERAGE_REFERENCE;
  r.mode = mode;
  return r;
}

// layout_to_partition (search.cpp:63-75).
inline Partition to_partition(const CtuGrid& g, const sc_layout& L) {
  Partition p;
  p.grid = g;
  p.origin = PartitionOrigin::Proposed;
  p.tiles.col_widths.assign(L.col_widths, L.col_widths + L.n_cols);
  p.tiles.row_heights = {g.rows};
  int x = 0, run = 0, id = 0;
  for (int c = 0; c < L.n_cols; ++c) {
    int y = 0;
    for (int j = 0; j < L.runs_per_col[c]; ++j, ++run) {
      p.slices.push_back(RectSlice{x, y, L.col_widths[c], L.run_heights[run], id++});
      y += L.run_heights[run];
    }
    x += L.col_widths[c];
  }
  return p;
}

// uniform_partition (grid.cpp:186-262) through sc_uniform_partition_n.
inline Partition uniform_partition(const CtuGrid& g, int n_slices) {
  const sc_grid cg = to_c(g);
  const std::size_t n = static_cast<std::size_t>(n_slices > 0 ? n_slices : 1);
  std::vector<int32_t> cw(n), rh(n);
  std::vector<sc_rect> s(n);
  int32_t nc = 0, nr = 0;
  check(sc_uniform_partition_n(&cg, n_slices, cw.data(), &nc, rh.data(), &nr, s.data()));
  Partition p;
  p.grid = g;
  p.origin = PartitionOrigin::Uniform;
  p.tiles.col_widths.assign(cw.begin(), cw.begin() + nc);
  p.tiles.row_heights.assign(rh.begin(), rh.begin() + nr);
  for (int i = 0; i < n_slices; ++i)
    p.slices.push_back(RectSlice{s[i].x0, s[i].y0, s[i].w, s[i].h, s[i].id});
  return p;
}

// A search result's partition: the ColumnSplit layout, or the uniform one.
inline Partition result_partition(const CtuGrid& g, const sc_search_result& r,
                                  const sc_layout& L) {
  if (r.origin == SC_ORIGIN_UNIFORM) return b200::uniform_partition(g, L.n_slices);
  return to_partition(g, L);
}

static_assert(sizeof(CtuRecord) == sizeof(sc_ctu_record), "CtuRecord layout");

inline std::vector<sc_rect> to_rects(const Partition& p) {
  std::vector<sc_rect> r;
  for (const RectSlice& s : p.slices) r.push_back(sc_rect{s.x0, s.y0, s.w, s.h, s.id});
  return r;
}

// partition_time (cost.hpp:102-105) on the device: SliceTimeTable of one
// partition (slice times by id, first-strict-> argmax, total in id order).
inline SliceTimeTable partition_time(Context& ctx, const CostMap& costs, const Partition& p) {
  if (costs.grid != p.grid) throw GeometryError("cost map grid does not match the partition grid");
  const sc_grid g = to_c(p.grid);
  const std::vector<sc_rect> r = to_rects(p);
  sc_partition_stats st;
  SliceTimeTable out;
  out.slice_times_us.resize(r.size());
  check(sc_partition_eval(ctx.get(), &g, r.data(), static_cast<int32_t>(r.size()),
                          costs.times_us.data(), nullptr, 1, &st, out.slice_times_us.data(),
                          nullptr));
  out.max_us = st.max_us;
  out.total_us = st.total_us;
  out.argmax = static_cast<std::size_t>(st.argmax);
  return out;
}

// partition_sse (texture.hpp:92) on the device.
inline double partition_sse(Context& ctx, const TextureStats& stats, const Partition& p) {
  if (stats.grid() != p.grid)
    throw GeometryError("texture stats grid does not match the partition grid");
  const sc_grid g = to_c(p.grid);
  const std::vector<sc_rect> r = to_rects(p);
  sc_partition_stats st;
  check(sc_partition_eval(ctx.get(), &g, r.data(), static_cast<int32_t>(r.size()), nullptr,
                          reinterpret_cast<const sc_ctu_record*>(stats.records().data()), 1, &st,
                          nullptr, nullptr));
  return st.sse;
}

// ctu_stats (texture.hpp:83): K1 on the plane's uint16 samples.
inline TextureStats ctu_stats(Context& ctx, const LumaPlane& luma, const CtuGrid& grid,
                              int poc = 0) {
  if (luma.width != grid.frame_width || luma.height != grid.frame_height)
    throw GeometryError("plane dimensions do not match the grid");
  std::vector<CtuRecord> rec(static_cast<size_t>(grid.cell_count()));
  check(sc_texture_moments(ctx.get(), luma.samples.data(), 2, luma.width, luma.height,
                           static_cast<size_t>(luma.width) * 2,
                           static_cast<size_t>(luma.width) * luma.height * 2, grid.ctu_size, 1,
                           reinterpret_cast<sc_ctu_record*>(rec.data())));
  return TextureStats(grid, std::move(rec), poc);
}

// min_time_search (search.hpp:66-67).
inline std::pair<double, Partition> min_time_search(Context& ctx, const CostMap& est,
                                                    const SearchConfig& cfg,
                                                    int mode = SC_MODE_EXHAUSTIVE) {
  const sc_grid g = to_c(est.grid);
  const sc_search_cfg c = to_c(cfg, mode);
  sc_search_result r;
  check(sc_min_time_search(ctx.get(), &g, &c, est.times_us.data(), 1, &r));
  return {r.t_min_us, result_partition(est.grid, r, r.argmin)};
}

inline SearchOutcome to_outcome(const CtuGrid& g, const sc_search_result& r) {
  SearchOutcome o;
  o.best = result_partition(g, r, r.best);
  o.t_min_us = r.t_min_us;
  o.t_best_us = r.t_best_us;
  o.sse_best = r.sse_best;
  o.candidates_evaluated = r.candidates_evaluated;
  o.candidates_step1 = r.candidates_step1;
  o.candidates_step2 = r.candidates_step2;
  o.search_time_us = r.search_time_us;
  o.time_min_step_us = r.time_min_step_us;
  o.clustering_step_us = r.clustering_step_us;
  return o;
}

// constrained_clustering_search (search.hpp:72-75).
inline SearchOutcome constrained_clustering_search(Context& ctx, const CostMap& est,
                                                   const TextureStats& stats, double t_min_us,
                                                   const SearchConfig& cfg,
                                                   int mode = SC_MODE_EXHAUSTIVE) {
  if (stats.grid() != est.grid)
    throw GeometryError("texture stats grid does not match the cost map grid");
  const sc_grid g = to_c(est.grid);
  const sc_search_cfg c = to_c(cfg, mode);
  sc_search_result r;
  check(sc_constrained_clustering(ctx.get(), &g, &c, est.times_us.data(),
                                  reinterpret_cast<const sc_ctu_record*>(stats.records().data()),
                                  &t_min_us, 1, &r));
  return to_outcome(est.grid, r);
}

// two_step_partition (search.hpp:80-82): host estimate (cost.cpp:66-95), then
// both steps on the device.
inline SearchOutcome two_step_partition(Context& ctx, const CostHistory& history,
                                        const TextureStats& stats, int poc,
                                        const SearchConfig& cfg, int mode = SC_MODE_EXHAUSTIVE) {
  if (stats.grid() != history.grid())
    throw GeometryError("texture stats grid does not match the history grid");
  const CostMap est = estimate_ctu_times(history, poc);
  const sc_grid g = to_c(history.grid());
  const sc_search_cfg c = to_c(cfg, mode);
  sc_search_result r;
  check(sc_two_step(ctx.get(), &g, &c, est.times_us.data(),
                    reinterpret_cast<const sc_ctu_record*>(stats.records().data()), 1, &r));
  SearchOutcome o = to_outcome(history.grid(), r);
  o.candidates_step1 = r.candidates_step1;
  o.est_source = est.source;
  o.est_source_poc = est.source_poc;
  return o;
}

}  // namespace b200
}  // namespace slicecraft
