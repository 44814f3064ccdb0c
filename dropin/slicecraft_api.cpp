// Link-level drop-in for the reference partitioner API (proj/include/slicecraft).
//
// Compiled against the caller's copy of the reference headers -- the API
// contract -- this file defines every out-of-line function and member those
// headers declare, on top of the C-ABI in include/slicecraft_b200.h.  A VTM-side
// caller that was linked against the reference library links
//   libslicecraft_dropin.so + libslicecraft_b200.so
// instead and runs unchanged: the texture map (K1), the time / SSE tables
// (K2/K3), the ColumnSplit search (K4/K5), partition_time / partition_sse and
// validate_partition run on the B200; the O(cells) host model (cost history,
// estimator, summed-area tables) comes from the same library's host code.
// Nothing here links or includes reference sources.
//
// Device and search mode of the implicit per-thread context:
//   SLICECRAFT_B200_DEVICE (default 0), SLICECRAFT_B200_MODE=pruned|exhaustive
// or explicitly through slicecraft::b200::set_default_device / _mode.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "slicecraft_b200.hpp"

namespace slicecraft {
namespace b200 {

namespace {
int g_device = -1;  // -1: from the environment
int g_mode = -1;
thread_local std::unique_ptr<Context> t_ctx;
thread_local int t_ctx_device = -1;

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}
}  // namespace

void set_default_device(int device) { g_device = device; }
void set_default_mode(int mode) { g_mode = mode; }

int default_mode() {
  if (g_mode >= 0) return g_mode;
  const char* v = std::getenv("SLICECRAFT_B200_MODE");
  return v && std::string(v) == "pruned" ? SC_MODE_PRUNED : SC_MODE_EXHAUSTIVE;
}

// The calling thread's context (one per host thread, as the C-ABI asks).
Context& default_context() {
  const int dev = g_device >= 0 ? g_device : env_int("SLICECRAFT_B200_DEVICE", 0);
  if (!t_ctx || t_ctx_device != dev) {
    t_ctx.reset(new Context(dev));
    t_ctx_device = dev;
  }
  return *t_ctx;
}

}  // namespace b200

// ---- grid.hpp ------------------------------------------------------------------
CtuGrid CtuGrid::make(int frame_width, int frame_height, int ctu_size) {
  sc_grid g;
  b200::check(sc_grid_make(frame_width, frame_height, ctu_size, &g));
  CtuGrid r;
  r.frame_width = g.frame_width;
  r.frame_height = g.frame_height;
  r.ctu_size = g.ctu_size;
  r.cols = g.cols;
  r.rows = g.rows;
  return r;
}

int CtuGrid::cell_width(int x) const { return std::min(ctu_size, frame_width - x * ctu_size); }
int CtuGrid::cell_height(int y) const { return std::min(ctu_size, frame_height - y * ctu_size); }

std::string to_string(PartitionOrigin origin) {
  switch (origin) {
    case PartitionOrigin::Uniform: return "Uniform";
    case PartitionOrigin::Proposed: return "Proposed";
    default: return "Custom";
  }
}

PartitionOrigin partition_origin_from_string(const std::string& s) {
  for (PartitionOrigin o : {PartitionOrigin::Uniform, PartitionOrigin::Proposed,
                            PartitionOrigin::Custom})
    if (s == to_string(o)) return o;
  throw FormatError("unknown partition origin: " + s);
}

std::vector<int> split_even(int total, int parts) {
  std::vector<int> out(static_cast<std::size_t>(std::max(parts, 0)));
  b200::check(sc_split_even(total, parts, out.data()));
  return out;
}

// The device post-check (validate.cu): tile / bound / id checks, exact
// disjoint cover and structure, with the reference's classes and messages.
Partition validate_partition(const CtuGrid& grid, TileGrid tiles, std::vector<RectSlice> slices,
                             PartitionOrigin origin) {
  const sc_grid g = b200::to_c(grid);
  std::vector<sc_rect> r;
  r.reserve(slices.size());
  for (const RectSlice& s : slices) r.push_back(sc_rect{s.x0, s.y0, s.w, s.h, s.id});
  b200::check(sc_validate_partition(b200::default_context().get(), &g,
                                    static_cast<int32_t>(tiles.col_widths.size()),
                                    tiles.col_widths.data(),
                                    static_cast<int32_t>(tiles.row_heights.size()),
                                    tiles.row_heights.data(), r.data(),
                                    static_cast<int32_t>(r.size()), nullptr));
  Partition p;
  p.grid = grid;
  p.tiles = std::move(tiles);
  p.slices = std::move(slices);
  p.origin = origin;
  return p;
}

Partition uniform_partition(const CtuGrid& grid, int n_slices) {
  return b200::uniform_partition(grid, n_slices);
}

double area_ratio(const Partition& p) {
  std::int64_t amin = p.slices.front().area(), amax = amin;
  for (const RectSlice& s : p.slices) {
    amin = std::min(amin, s.area());
    amax = std::max(amax, s.area());
  }
  return static_cast<double>(amax) / static_cast<double>(amin);
}

// One character per cell: later slices paint over earlier ones, uncovered
// cells stay '?' (grid.cpp:264-288).
std::string render_ascii(const Partition& p) {
  static const char kSym[] = "0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz";
  const int cols = p.grid.cols, rows = p.grid.rows;
  std::vector<char> cell(static_cast<std::size_t>(cols) * rows, '?');
  for (const RectSlice& s : p.slices) {
    const char c = s.id >= 0 && s.id < 62 ? kSym[s.id] : '#';
    for (int y = std::max(s.y0, 0); y < std::min(s.y0 + s.h, rows); ++y)
      for (int x = std::max(s.x0, 0); x < std::min(s.x0 + s.w, cols); ++x)
        cell[static_cast<std::size_t>(y) * cols + x] = c;
  }
  std::string out;
  out.reserve(static_cast<std::size_t>(cols + 1) * rows);
  for (int y = 0; y < rows; ++y) {
    out.append(cell.begin() + static_cast<std::ptrdiff_t>(y) * cols,
               cell.begin() + static_cast<std::ptrdiff_t>(y + 1) * cols);
    out.push_back('\n');
  }
  return out;
}

// ---- texture.hpp ---------------------------------------------------------------
int yuv_frame_count(const std::filesystem::path& path, int frame_w, int frame_h, int bit_depth) {
  int32_t n = 0;
  b200::check(sc_yuv_frame_count(path.string().c_str(), frame_w, frame_h, bit_depth, &n));
  return n;
}

LumaPlane load_yuv_frame(const std::filesystem::path& path, int frame_w, int frame_h, int poc,
                         int bit_depth) {
  LumaPlane p;
  p.width = frame_w;
  p.height = frame_h;
  p.bit_depth = bit_depth;
  p.samples.resize(static_cast<std::size_t>(std::max(frame_w, 0)) * std::max(frame_h, 0));
  b200::check(sc_yuv_load_luma(path.string().c_str(), frame_w, frame_h, poc, bit_depth,
                               p.samples.data()));
  return p;
}

double SliceMoments::sse() const {
  const sc_ctu_record m{count, sum, sumsq};
  double out = 0.0;
  b200::check(sc_moments_sse(&m, &out));
  return out;
}

TextureStats::TextureStats(CtuGrid grid, std::vector<CtuRecord> records, int poc)
    : grid_(grid), poc_(poc), records_(std::move(records)) {
  const sc_grid g = b200::to_c(grid_);
  const std::size_t n = static_cast<std::size_t>(grid_.cols + 1) * (grid_.rows + 1);
  pre_count_.resize(n);
  pre_sum_.resize(n);
  pre_sumsq_.resize(n);
  b200::check(sc_texture_tables(&g, reinterpret_cast<const sc_ctu_record*>(records_.data()),
                                static_cast<int64_t>(records_.size()), pre_count_.data(),
                                pre_sum_.data(), pre_sumsq_.data()));
}

SliceMoments TextureStats::rect_moments(int x0, int y0, int w, int h) const {
  const std::size_t s = static_cast<std::size_t>(grid_.cols) + 1;
  const std::size_t a = y0 * s + x0, b = y0 * s + x0 + w, c = (y0 + h) * s + x0,
                    d = (y0 + h) * s + x0 + w;
  SliceMoments m;
  m.count = pre_count_[d] - pre_count_[b] - pre_count_[c] + pre_count_[a];
  m.sum = pre_sum_[d] - pre_sum_[b] - pre_sum_[c] + pre_sum_[a];
  m.sumsq = pre_sumsq_[d] - pre_sumsq_[b] - pre_sumsq_[c] + pre_sumsq_[a];
  return m;
}

TextureStats ctu_stats(const LumaPlane& luma, const CtuGrid& grid, int poc) {
  return b200::ctu_stats(b200::default_context(), luma, grid, poc);
}

double partition_sse(const TextureStats& stats, const Partition& p) {
  return b200::partition_sse(b200::default_context(), stats, p);
}

std::vector<SliceMoments> slice_moments(const TextureStats& stats, const Partition& p) {
  if (stats.grid() != p.grid)
    throw GeometryError("texture stats grid does not match the partition grid");
  const sc_grid g = b200::to_c(p.grid);
  const std::vector<sc_rect> r = b200::to_rects(p);
  sc_partition_stats st;
  std::vector<SliceMoments> out(r.size());
  static_assert(sizeof(SliceMoments) == sizeof(sc_ctu_record), "SliceMoments layout");
  b200::check(sc_partition_eval(b200::default_context().get(), &g, r.data(),
                                static_cast<int32_t>(r.size()), nullptr,
                                reinterpret_cast<const sc_ctu_record*>(stats.records().data()), 1,
                                &st, nullptr, reinterpret_cast<sc_ctu_record*>(out.data())));
  return out;
}

// ---- cost.hpp ------------------------------------------------------------------
std::string to_string(CostSource source) {
  switch (source) {
    case CostSource::CoTemporalLayer: return "CoTemporalLayer";
    case CostSource::MostRecentAny: return "MostRecentAny";
    case CostSource::Uniform: return "Uniform";
    default: return "Measured";
  }
}

double CostMap::total_us() const {
  double t = 0.0;
  for (double v : times_us) t += v;
  return t;
}

int temporal_layer_of_poc(int poc, int gop_size) {
  int32_t tl = 0;
  b200::check(sc_temporal_layer(poc, gop_size, &tl));
  return tl;
}

CostHistory::CostHistory(CtuGrid grid, int gop_size) : grid_(grid), gop_(gop_size) {
  temporal_layer_of_poc(0, gop_size);  // the gop is validated eagerly
}

void CostHistory::append(CostMap map) {
  const sc_grid hg = b200::to_c(grid_), mg = b200::to_c(map.grid);
  std::vector<int32_t> pocs;
  pocs.reserve(maps_.size());
  for (const CostMap& m : maps_) pocs.push_back(m.poc);
  b200::check(sc_cost_map_check(&hg, &mg, map.times_us.data(),
                                static_cast<int64_t>(map.times_us.size()), map.poc, pocs.data(),
                                static_cast<int32_t>(pocs.size())));
  maps_.push_back(std::move(map));
}

CostMap estimate_ctu_times(const CostHistory& history, int poc) {
  const auto& maps = history.maps();
  std::vector<const double*> ptrs;
  std::vector<int32_t> pocs, tls;
  for (const CostMap& m : maps) {
    ptrs.push_back(m.times_us.data());
    pocs.push_back(m.poc);
    tls.push_back(m.temporal_layer);
  }
  const sc_grid g = b200::to_c(history.grid());
  CostMap est;
  est.grid = history.grid();
  est.times_us.resize(static_cast<std::size_t>(history.grid().cell_count()));
  int32_t src = 0, src_poc = -1, tl = 0;
  b200::check(sc_estimate_ctu_times(&g, history.gop_size(), static_cast<int32_t>(maps.size()),
                                    ptrs.data(), pocs.data(), tls.data(), poc,
                                    est.times_us.data(), &src, &src_poc, &tl));
  for (const CostMap& m : maps)  // the copied map's remaining fields (cost.cpp:71-84)
    if (src != SC_SOURCE_UNIFORM && m.poc == src_poc) est.qp = m.qp;
  est.poc = poc;
  est.temporal_layer = tl;
  est.source = static_cast<CostSource>(src);
  est.source_poc = src_poc;
  return est;
}

PrefixSumTable::PrefixSumTable(const std::vector<double>& values, int cols, int rows)
    : cols_(cols), rows_(rows) {
  table_.resize(static_cast<std::size_t>(std::max(cols, 0) + 1) * (std::max(rows, 0) + 1));
  b200::check(sc_prefix_sum_table(values.data(), static_cast<int64_t>(values.size()), cols, rows,
                                  table_.data()));
}

PrefixSumTable::PrefixSumTable(const CostMap& costs)
    : PrefixSumTable(costs.times_us, costs.grid.cols, costs.grid.rows) {}

// Against a caller's table: its own rect_sum (cost.hpp:75-81) per slice, the
// first strict maximum and the id-order total (cost.cpp:117-139).
SliceTimeTable partition_time(const PrefixSumTable& table, const Partition& p) {
  if (table.cols() != p.grid.cols || table.rows() != p.grid.rows)
    throw GeometryError("prefix table does not match the partition grid");
  SliceTimeTable out;
  out.slice_times_us.assign(p.slices.size(), 0.0);
  for (const RectSlice& s : p.slices)
    out.slice_times_us[static_cast<std::size_t>(s.id)] = table.rect_sum(s.x0, s.y0, s.w, s.h);
  out.max_us = out.slice_times_us.front();
  for (std::size_t j = 0; j < out.slice_times_us.size(); ++j) {
    out.total_us += out.slice_times_us[j];
    if (out.slice_times_us[j] > out.max_us) {
      out.max_us = out.slice_times_us[j];
      out.argmax = j;
    }
  }
  return out;
}

SliceTimeTable partition_time(const CostMap& costs, const Partition& p) {
  return b200::partition_time(b200::default_context(), costs, p);
}

// ---- search.hpp ----------------------------------------------------------------
std::string to_string(CandidateFamily family) {
  return family == CandidateFamily::UniformOnly ? "UniformOnly" : "ColumnSplit";
}

CandidateFamily candidate_family_from_string(const std::string& s) {
  if (s == "ColumnSplit") return CandidateFamily::ColumnSplit;
  if (s == "UniformOnly") return CandidateFamily::UniformOnly;
  throw FormatError("unknown candidate family: " + s);
}

void SearchConfig::check() const {
  const sc_search_cfg c = b200::to_c(*this);
  b200::check(sc_search_cfg_check(&c));
}

// The device-materialised stream (enumerate.cu), paged 64 Ki candidates at a
// time, converted to Partitions in enumeration order on the caller's thread.
void for_each_candidate(const CtuGrid& grid, const SearchConfig& cfg,
                        const std::function<void(const Partition&)>& sink) {
  const sc_grid g = b200::to_c(grid);
  const sc_search_cfg c = b200::to_c(cfg);
  b200::Context& ctx = b200::default_context();
  constexpr uint64_t kPage = 1 << 16;
  std::vector<sc_layout> buf(kPage);
  uint64_t first = 0, total = 0;
  do {
    uint64_t n = 0;
    b200::check(sc_enumerate_candidates(ctx.get(), &g, &c, first, kPage, buf.data(), &n, &total));
    for (uint64_t i = 0; i < n; ++i)
      sink(buf[i].n_cols == 0 ? b200::uniform_partition(grid, cfg.n_slices)
                              : b200::to_partition(grid, buf[i]));
    if (n == 0) break;
    first += n;
  } while (first < total);
}

std::vector<Partition> enumerate_candidates(const CtuGrid& grid, const SearchConfig& cfg) {
  std::vector<Partition> out;
  for_each_candidate(grid, cfg, [&](const Partition& p) { out.push_back(p); });
  return out;
}

std::pair<double, Partition> min_time_search(const CostMap& est, const SearchConfig& cfg) {
  return b200::min_time_search(b200::default_context(), est, cfg, b200::default_mode());
}

SearchOutcome constrained_clustering_search(const CostMap& est, const TextureStats& stats,
                                            double t_min_us, const SearchConfig& cfg) {
  return b200::constrained_clustering_search(b200::default_context(), est, stats, t_min_us, cfg,
                                             b200::default_mode());
}

SearchOutcome two_step_partition(const CostHistory& history, const TextureStats& stats, int poc,
                                 const SearchConfig& cfg) {
  return b200::two_step_partition(b200::default_context(), history, stats, poc, cfg,
                                  b200::default_mode());
}

}  // namespace slicecraft
