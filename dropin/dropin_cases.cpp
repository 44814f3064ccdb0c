// Drop-in check: one caller program written against the reference partitioner
// API (proj/include/slicecraft) and nothing else, built twice:
//   dropin/cases_ref   linked against the UNMODIFIED reference (oracle/_ref,
//                      test infrastructure; only where /root/reference exists)
//   dropin/cases_b200  linked against libslicecraft_dropin.so +
//                      libslicecraft_b200.so only (no reference code at all)
// Each prints a canonical transcript of every API call (doubles as %a, so
// equal text means bit-equal values; exceptions by class and message).  With
// a transcript path argument the program compares its own transcript with it
// line by line and prints DROPIN OK / DROPIN FAILED; tests/golden/dropin_ref.txt
// is cases_ref's transcript (tests/test_gpu_dropin.py).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "slicecraft/cost.hpp"
#include "slicecraft/errors.hpp"
#include "slicecraft/grid.hpp"
#include "slicecraft/search.hpp"
#include "slicecraft/texture.hpp"

using namespace slicecraft;

static std::ostringstream out;

static void line(const std::string& s) { out << s << '\n'; }
static std::string hx(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}
static std::string u(uint64_t v) { return std::to_string(v); }

static const char* class_of(const Error& e) {
  if (dynamic_cast<const GeometryError*>(&e)) return "GeometryError";
  if (dynamic_cast<const OverlapError*>(&e)) return "OverlapError";
  if (dynamic_cast<const CoverageError*>(&e)) return "CoverageError";
  if (dynamic_cast<const StructureError*>(&e)) return "StructureError";
  if (dynamic_cast<const IoError*>(&e)) return "IoError";
  if (dynamic_cast<const RangeError*>(&e)) return "RangeError";
  if (dynamic_cast<const FormatError*>(&e)) return "FormatError";
  if (dynamic_cast<const ConfigError*>(&e)) return "ConfigError";
  if (dynamic_cast<const TraceError*>(&e)) return "TraceError";
  if (dynamic_cast<const NoCandidateError*>(&e)) return "NoCandidateError";
  if (dynamic_cast<const SizeError*>(&e)) return "SizeError";
  if (dynamic_cast<const UsageError*>(&e)) return "UsageError";
  return "Error";
}
// Runs fn; prints "<tag> ok" or "<tag> throws <Class>: <message>".
static void guard(const std::string& tag, const std::function<void()>& fn,
                  bool message = true) {
  try {
    fn();
    line(tag + " ok");
  } catch (const Error& e) {
    line(tag + " throws " + class_of(e) + (message ? std::string(": ") + e.what() : ""));
  }
}

static uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) h = (h ^ ((v >> (8 * i)) & 0xff)) * 0x100000001b3ull;
  return h;
}
static std::string slices(const Partition& p) {
  std::string s = to_string(p.origin) + " tiles";
  for (int w : p.tiles.col_widths) s += " " + std::to_string(w);
  s += " /";
  for (int h : p.tiles.row_heights) s += " " + std::to_string(h);
  s += " |";
  for (const RectSlice& r : p.slices)
    s += " " + std::to_string(r.x0) + "," + std::to_string(r.y0) + "," + std::to_string(r.w) +
         "x" + std::to_string(r.h) + "#" + std::to_string(r.id);
  return s;
}

static LumaPlane make_plane(int w, int h, int depth, unsigned seed) {
  LumaPlane p;
  p.width = w;
  p.height = h;
  p.bit_depth = depth;
  p.samples.resize((size_t)w * h);
  uint64_t s = seed * 0x9e3779b97f4a7c15ull + 1;
  const unsigned M = (1u << depth) - 1;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      const bool noise = ((x / 128 + 3 * (y / 128) + seed) % 4) == 0;
      p.samples[(size_t)y * w + x] =
          (uint16_t)(noise ? (s >> 33) % (M + 1) : ((x + 2 * y) * M) / (w + 2 * h));
    }
  return p;
}

static CostMap make_map(const CtuGrid& g, int poc, int tl, unsigned seed) {
  CostMap m;
  m.grid = g;
  m.poc = poc;
  m.temporal_layer = tl;
  m.qp = 22 + poc % 5;
  m.times_us.resize((size_t)g.cell_count());
  uint64_t s = seed + 77;
  for (double& t : m.times_us) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    t = 0.25 + (double)((s >> 40) % 100000) / 7919.0;
  }
  return m;
}

static void outcome(const std::string& tag, const SearchOutcome& o) {
  line(tag + " t_min " + hx(o.t_min_us) + " t_best " + hx(o.t_best_us) + " sse " +
       hx(o.sse_best) + " counts " + u(o.candidates_step1) + " " + u(o.candidates_step2) + " " +
       u(o.candidates_evaluated) + " est " + to_string(o.est_source) + " " +
       std::to_string(o.est_source_poc));
  line(tag + " best " + slices(o.best));
}

static void run() {
  // ---- grid ------------------------------------------------------------------------
  for (auto d : {std::vector<int>{1920, 1080, 128}, {3840, 2160, 128}, {1000, 700, 64},
                 {33, 1, 32}})
    guard("grid " + std::to_string(d[0]) + "x" + std::to_string(d[1]), [&] {
      const CtuGrid g = CtuGrid::make(d[0], d[1], d[2]);
      line("grid " + std::to_string(g.cols) + "x" + std::to_string(g.rows) + " cell(last) " +
           std::to_string(g.cell_width(g.cols - 1)) + "x" + std::to_string(g.cell_height(g.rows - 1)) +
           " px " + std::to_string(g.cell_pixels(g.cols - 1, g.rows - 1)));
    });
  guard("grid ctu48", [] { CtuGrid::make(640, 480, 48); });
  guard("grid zero", [] { CtuGrid::make(0, 480, 64); });
  for (int t : {7, 12, 13})
    for (int p : {1, 2, 3, 4, 5}) line("split_even " + std::to_string(t) + "/" + std::to_string(p) +
                                        [&] {
                                          std::string s;
                                          for (int v : split_even(t, p)) s += " " + std::to_string(v);
                                          return s;
                                        }());
  for (int poc = 0; poc <= 17; ++poc)
    line("tl " + std::to_string(poc) + " " + std::to_string(temporal_layer_of_poc(poc, 16)) + " " +
         std::to_string(temporal_layer_of_poc(poc, 4)));
  guard("tl gop12", [] { temporal_layer_of_poc(3, 12); });
  guard("tl negative", [] { temporal_layer_of_poc(-1, 16); });
  line("names " + to_string(PartitionOrigin::Uniform) + " " + to_string(CostSource::MostRecentAny) +
       " " + to_string(CandidateFamily::UniformOnly) + " " +
       to_string(partition_origin_from_string("Proposed")) + " " +
       to_string(candidate_family_from_string("ColumnSplit")));
  guard("origin bad", [] { partition_origin_from_string("proposed"); });
  guard("family bad", [] { candidate_family_from_string("Uniform"); });

  // ---- uniform partitions, validate_partition ------------------------------------
  const CtuGrid g1080 = CtuGrid::make(1920, 1080, 128);
  for (int n : {1, 2, 4, 6, 7, 13, 17, 64, 135})
    guard("uniform n" + std::to_string(n), [&] {
      const Partition p = uniform_partition(g1080, n);
      line("uniform n" + std::to_string(n) + " " + slices(p) + " ratio " + hx(area_ratio(p)));
      if (n == 7) out << render_ascii(p);
      const Partition v = validate_partition(g1080, p.tiles, p.slices, p.origin);
      line("revalidated " + std::to_string(v == p));
    });
  guard("uniform n136", [&] { uniform_partition(g1080, 136); });
  {
    const TileGrid t{{5, 10}, {9}};
    std::vector<RectSlice> ok = {{0, 0, 5, 4, 0}, {0, 4, 5, 5, 2}, {5, 0, 10, 9, 1}};
    guard("validate ok", [&] { validate_partition(g1080, t, ok); });
    auto mut = [&](const std::string& tag, std::function<void(TileGrid&, std::vector<RectSlice>&)> f) {
      TileGrid t2 = t;
      std::vector<RectSlice> s2 = ok;
      f(t2, s2);
      guard("validate " + tag, [&] { validate_partition(g1080, t2, s2); });
    };
    mut("overlap", [](TileGrid&, std::vector<RectSlice>& s) { s[1].y0 = 3; s[1].h = 6; });
    mut("coverage", [](TileGrid&, std::vector<RectSlice>& s) { s[1].h = 4; });
    mut("structure", [](TileGrid& t2, std::vector<RectSlice>&) { t2.col_widths = {3, 12}; });
    mut("tiles", [](TileGrid& t2, std::vector<RectSlice>&) { t2.col_widths = {5, 9}; });
    mut("bounds", [](TileGrid&, std::vector<RectSlice>& s) { s[2].w = 11; });
    mut("ids", [](TileGrid&, std::vector<RectSlice>& s) { s[2].id = 0; });
    mut("empty", [](TileGrid&, std::vector<RectSlice>& s) { s.clear(); });
    mut("tilerows", [](TileGrid& t2, std::vector<RectSlice>&) { t2.row_heights = {4, 5}; });
  }

  // ---- texture map, moments ------------------------------------------------------
  struct Plane { int w, h, depth; unsigned seed; };
  std::vector<TextureStats> stats;
  for (const Plane& pl : {Plane{1920, 1080, 10, 1}, Plane{1000, 700, 8, 2}, Plane{3840, 2160, 10, 3}}) {
    const CtuGrid g = CtuGrid::make(pl.w, pl.h, pl.w == 1000 ? 64 : 128);
    const TextureStats st = ctu_stats(make_plane(pl.w, pl.h, pl.depth, pl.seed), g, 5);
    uint64_t h = 1469598103934665603ull;
    for (const CtuRecord& r : st.records()) h = fnv(fnv(fnv(h, r.count), r.sum), r.sumsq);
    line("ctu_stats " + std::to_string(pl.w) + "x" + std::to_string(pl.h) + " poc " +
         std::to_string(st.poc()) + " hash " + u(h) + " rec0 " + u(st.record(0, 0).sum) + " " +
         u(st.record(0, 0).sumsq));
    for (auto q : {std::vector<int>{0, 0, 1, 1}, {1, 2, 3, 4}, {0, 0, g.cols, g.rows},
                   {g.cols - 1, g.rows - 1, 1, 1}, {2, 0, 0, 3}}) {
      const SliceMoments m = st.rect_moments(q[0], q[1], q[2], q[3]);
      line("rect_moments " + u(m.count) + " " + u(m.sum) + " " + u(m.sumsq) + " sse " + hx(m.sse()));
    }
    stats.push_back(st);
  }
  guard("ctu_stats mismatch", [&] { ctu_stats(make_plane(64, 64, 8, 1), g1080, 0); });
  guard("stats count", [&] { TextureStats(g1080, std::vector<CtuRecord>(3), 0); });
  guard("stats pixels", [&] {
    std::vector<CtuRecord> r = stats[0].records();
    r[4].count += 1;
    TextureStats(g1080, r, 0);
  });
  guard("stats moments", [&] {
    std::vector<CtuRecord> r = stats[0].records();
    r[9].sumsq = 0;
    TextureStats(g1080, r, 0);
  });
  line("sse edge " + hx(SliceMoments{0, 0, 0}.sse()) + " " + hx(SliceMoments{3, 1, 1ull << 63}.sse()) +
       " " + hx(SliceMoments{~0ull, ~0ull, ~0ull}.sse()));

  // ---- YUV ingest ------------------------------------------------------------------
  {
    const std::string path = "/tmp/slicecraft_dropin_cases.yuv";
    std::ofstream f(path, std::ios::binary);
    for (int i = 0; i < 3 * (64 * 48 * 3 / 2) * 2; ++i) f.put((char)((i * 7 + i / 5) & 0xff));
    f.close();
    line("yuv frames " + std::to_string(yuv_frame_count(path, 64, 48, 10)) + " " +
         std::to_string(yuv_frame_count(path, 64, 48, 8)));
    const LumaPlane p = load_yuv_frame(path, 64, 48, 2, 10);
    uint64_t h = 1469598103934665603ull;
    for (uint16_t v : p.samples) h = fnv(h, v);
    line("yuv plane " + u(h) + " " + std::to_string(p.at(5, 7)));
    guard("yuv range", [&] { load_yuv_frame(path, 64, 48, 3, 10); });
    guard("yuv format", [&] { yuv_frame_count(path, 63, 48, 10); });
    guard("yuv depth", [&] { yuv_frame_count(path, 64, 48, 12); });
    guard("yuv io", [&] { yuv_frame_count("/nonexistent/x.yuv", 64, 48, 8); }, false);
  }

  // ---- cost model --------------------------------------------------------------------
  CostHistory hist(g1080, 16);
  hist.append(make_map(g1080, 0, 0, 1));
  hist.append(make_map(g1080, 16, 0, 2));
  hist.append(make_map(g1080, 8, 1, 3));
  hist.append(make_map(g1080, 4, 2, 4));
  guard("append dup", [&] { hist.append(make_map(g1080, 8, 1, 5)); });
  guard("append grid", [&] { hist.append(make_map(CtuGrid::make(1280, 720, 128), 9, 4, 5)); });
  guard("append size", [&] {
    CostMap m = make_map(g1080, 9, 4, 5);
    m.times_us.pop_back();
    hist.append(m);
  });
  guard("append negative", [&] {
    CostMap m = make_map(g1080, 9, 4, 5);
    m.times_us[3] = -1.0;
    hist.append(m);
  });
  guard("history gop", [&] { CostHistory(g1080, 10); });
  for (int poc : {24, 12, 2, 3, 32}) {
    const CostMap e = estimate_ctu_times(hist, poc);
    uint64_t h = 1469598103934665603ull;
    for (double v : e.times_us) {
      uint64_t b;
      std::memcpy(&b, &v, 8);
      h = fnv(h, b);
    }
    line("estimate " + std::to_string(poc) + " " + to_string(e.source) + " " +
         std::to_string(e.source_poc) + " tl " + std::to_string(e.temporal_layer) + " qp " +
         std::to_string(e.qp) + " hash " + u(h) + " total " + hx(e.total_us()));
  }
  {
    const CostMap e = estimate_ctu_times(CostHistory(g1080, 16), 5);
    line("estimate empty " + to_string(e.source) + " " + std::to_string(e.source_poc) + " " +
         hx(e.total_us()));
  }
  const CostMap est = estimate_ctu_times(hist, 3);
  const PrefixSumTable sat(est);
  line("sat total " + hx(sat.total()) + " " + hx(sat.rect_sum(3, 2, 4, 5)) + " " +
       hx(sat.rect_sum(14, 8, 1, 1)));
  guard("sat dims", [] { PrefixSumTable(std::vector<double>(5), 2, 3); });

  // ---- candidate stream ------------------------------------------------------------
  {
    SearchConfig cfg;
    cfg.n_slices = 4;
    cfg.max_tile_cols = 2;
    uint64_t h = 1469598103934665603ull, n = 0;
    for_each_candidate(g1080, cfg, [&](const Partition& p) {
      for (const RectSlice& r : p.slices) h = fnv(fnv(fnv(fnv(fnv(h, r.x0), r.y0), r.w), r.h), r.id);
      if (n == 0 || n == 700) line("candidate " + u(n) + " " + slices(p));
      ++n;
    });
    line("for_each_candidate n4c2 " + u(n) + " hash " + u(h));
    cfg.n_slices = 3;
    cfg.max_tile_cols = 0;
    cfg.k_area = 1.5;
    const std::vector<Partition> all = enumerate_candidates(CtuGrid::make(320, 256, 64), cfg);
    line("enumerate n3 k1.5 " + u(all.size()) + (all.empty() ? "" : " last " + slices(all.back())));
    cfg.family = CandidateFamily::UniformOnly;
    cfg.n_slices = 6;
    line("enumerate uniform " + u(enumerate_candidates(g1080, cfg).size()));
    cfg.n_slices = 200;
    cfg.family = CandidateFamily::ColumnSplit;
    guard("enumerate n>cells", [&] { enumerate_candidates(g1080, cfg); });
  }

  // ---- searches ----------------------------------------------------------------------
  struct Case { int w, h, n, cap; double lambda, k; int family; };
  for (const Case& cs : {Case{1920, 1080, 4, 2, 0.0, 3.0, 0}, Case{1920, 1080, 8, 4, 0.1, 3.0, 0},
                         Case{1000, 700, 5, 0, 0.3, 3.0, 0}, Case{1920, 1080, 6, 0, 1.0, 2.0, 0},
                         Case{1920, 1080, 6, 0, 0.1, 3.0, 1}, Case{1920, 1080, 7, 0, 0.1, 3.0, 1},
                         Case{1920, 1080, 3, 0, 0.0, 1.05, 0}}) {
    const std::string tag = "case " + std::to_string(cs.w) + "x" + std::to_string(cs.h) + " n" +
                            std::to_string(cs.n) + " c" + std::to_string(cs.cap) + " l" +
                            hx(cs.lambda) + " k" + hx(cs.k) + " f" + std::to_string(cs.family);
    const CtuGrid g = CtuGrid::make(cs.w, cs.h, 128);
    const TextureStats st = ctu_stats(make_plane(cs.w, cs.h, 10, (unsigned)cs.n), g, 3);
    CostHistory h(g, 16);
    h.append(make_map(g, 0, 0, 1));
    h.append(make_map(g, 1, 4, 2));
    h.append(make_map(g, 2, 3, 3));
    SearchConfig cfg;
    cfg.n_slices = cs.n;
    cfg.max_tile_cols = cs.cap;
    cfg.lambda = cs.lambda;
    cfg.k_area = cs.k;
    cfg.family = cs.family ? CandidateFamily::UniformOnly : CandidateFamily::ColumnSplit;
    guard(tag + " two_step", [&] { outcome(tag + " two_step", two_step_partition(h, st, 3, cfg)); });
    const CostMap e = estimate_ctu_times(h, 3);
    guard(tag + " min_time", [&] {
      const auto r = min_time_search(e, cfg);
      line(tag + " min_time " + hx(r.first) + " " + slices(r.second));
      const SliceTimeTable t1 = partition_time(e, r.second);
      const SliceTimeTable t2 = partition_time(PrefixSumTable(e), r.second);
      std::string s;
      for (double v : t1.slice_times_us) s += " " + hx(v);
      line(tag + " partition_time" + s + " max " + hx(t1.max_us) + " total " + hx(t1.total_us) +
           " argmax " + u(t1.argmax) + " same " +
           std::to_string(t1.slice_times_us == t2.slice_times_us && t1.max_us == t2.max_us &&
                          t1.total_us == t2.total_us && t1.argmax == t2.argmax));
      std::string m;
      for (const SliceMoments& q : slice_moments(st, r.second)) m += " " + u(q.sum);
      line(tag + " partition_sse " + hx(partition_sse(st, r.second)) + " moments" + m);
      const SearchOutcome o = constrained_clustering_search(e, st, r.first, cfg);
      outcome(tag + " clustering", o);
      guard(tag + " clustering tight", [&] {
        outcome(tag + " tight", constrained_clustering_search(e, st, r.first * 0.5, cfg));
      });
    });
  }
  {
    SearchConfig cfg;
    cfg.n_slices = 3;
    const CostMap e = make_map(CtuGrid::make(256, 128, 128), 0, 0, 1);
    guard("search n>cells", [&] { min_time_search(e, cfg); });
    cfg.n_slices = 1;
    cfg.k_area = 1.0;
    guard("search k<=1", [&] { min_time_search(e, cfg); });
    cfg.k_area = 3.0;
    cfg.lambda = -0.5;
    guard("search lambda<0", [&] { min_time_search(e, cfg); });
    cfg.lambda = 0.0;
    cfg.workers = 0;
    guard("search workers", [&] { cfg.check(); });
    cfg.workers = 1;
    cfg.max_tile_cols = -1;
    guard("search cap", [&] { cfg.check(); });
  }
}

int main(int argc, char** argv) {
  run();
  const std::string mine = out.str();
  if (argc < 2) {
    std::fputs(mine.c_str(), stdout);
    return 0;
  }
  std::ifstream f(argv[1]);
  std::stringstream ref;
  ref << f.rdbuf();
  std::istringstream a(mine), b(ref.str());
  std::string la, lb;
  int n = 0, bad = 0;
  while (true) {
    const bool ga = (bool)std::getline(a, la), gb = (bool)std::getline(b, lb);
    if (!ga && !gb) break;
    ++n;
    if (!ga || !gb || la != lb) {
      if (++bad <= 10)
        std::printf("line %d differs:\n  b200: %s\n  ref:  %s\n", n, ga ? la.c_str() : "<eof>",
                    gb ? lb.c_str() : "<eof>");
    }
  }
  std::printf(bad ? "DROPIN FAILED (%d of %d lines)\n" : "DROPIN OK (%d lines)\n", bad ? bad : n, n);
  return bad ? 1 : 0;
}
