// Drop-in check: the same caller code run through the unmodified reference
// library (slicecraft::*) and through the B200 binding (slicecraft::b200::*)
// on the reference's own types.  Built by `make dropin` where the reference
// headers exist; the binary runs on the GPU box (tests/test_gpu_dropin.py).
#include <cstdio>
#include <cstdlib>

#include "slicecraft_b200.hpp"

using namespace slicecraft;

static int failures = 0;
#define EXPECT(cond, what)                                  \
  do {                                                      \
    if (!(cond)) {                                          \
      std::printf("FAIL %s (line %d)\n", what, __LINE__);   \
      ++failures;                                           \
    }                                                       \
  } while (0)

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
      const bool noise = ((x / 128 + 3 * (y / 128)) % 4) == 0;
      p.samples[(size_t)y * w + x] =
          (uint16_t)(noise ? (s >> 33) % (M + 1) : ((x + y) * M) / (w + h));
    }
  return p;
}

static CostMap make_map(const CtuGrid& g, int poc, int tl, unsigned seed) {
  CostMap m;
  m.grid = g;
  m.poc = poc;
  m.temporal_layer = tl;
  m.times_us.resize((size_t)g.cell_count());
  uint64_t s = seed + 77;
  for (double& t : m.times_us) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    t = 0.25 + (double)((s >> 40) % 1000) / 250.0;
  }
  return m;
}

int main() {
  b200::Context ctx(0);
  struct Case { int w, h, n, cap; double lambda; } cases[] = {
      {1920, 1080, 4, 2, 0.0}, {1920, 1080, 8, 4, 0.1}, {1000, 700, 5, 0, 0.3}};
  for (const Case& cs : cases) {
    const CtuGrid g = CtuGrid::make(cs.w, cs.h, 128);
    const LumaPlane luma = make_plane(cs.w, cs.h, 10, (unsigned)cs.n);
    const TextureStats ref_stats = ctu_stats(luma, g, 3);
    const TextureStats gpu_stats = b200::ctu_stats(ctx, luma, g, 3);
    EXPECT(ref_stats.records() == gpu_stats.records(), "ctu_stats records");
    CostHistory hist(g, 16);
    hist.append(make_map(g, 0, 0, 1));
    hist.append(make_map(g, 1, 4, 2));
    hist.append(make_map(g, 2, 3, 3));
    SearchConfig cfg;
    cfg.n_slices = cs.n;
    cfg.max_tile_cols = cs.cap;
    cfg.lambda = cs.lambda;
    const SearchOutcome ref = two_step_partition(hist, ref_stats, 3, cfg);
    for (int mode = 0; mode < 2; ++mode) {
      const SearchOutcome got = b200::two_step_partition(ctx, hist, gpu_stats, 3, cfg, mode);
      EXPECT(got.best == ref.best, "best partition");
      EXPECT(got.t_min_us == ref.t_min_us, "t_min_us");
      EXPECT(got.t_best_us == ref.t_best_us, "t_best_us");
      EXPECT(got.sse_best == ref.sse_best, "sse_best");
      EXPECT(got.candidates_step1 == ref.candidates_step1, "candidates_step1");
      EXPECT(got.candidates_step2 == ref.candidates_step2, "candidates_step2");
      EXPECT(got.est_source == ref.est_source && got.est_source_poc == ref.est_source_poc,
             "estimate source");
    }
    const CostMap est = estimate_ctu_times(hist, 3);
    const auto r1 = min_time_search(est, cfg);
    const auto g1 = b200::min_time_search(ctx, est, cfg);
    EXPECT(r1.first == g1.first && r1.second == g1.second, "min_time_search");
    std::printf("case %dx%d n=%d: t_min=%.17g sse=%.17g candidates=%llu\n", cs.w, cs.h, cs.n,
                ref.t_min_us, ref.sse_best, (unsigned long long)ref.candidates_evaluated);
  }
  // UniformOnly family, uniform_partition, partition_time / partition_sse
  for (int n : {1, 4, 6, 7, 13}) {
    const CtuGrid g = CtuGrid::make(1920, 1080, 128);
    const LumaPlane luma = make_plane(1920, 1080, 10, (unsigned)(40 + n));
    const TextureStats stats = ctu_stats(luma, g, 3);
    CostHistory hist(g, 16);
    hist.append(make_map(g, 0, 0, 9 + n));
    SearchConfig cfg;
    cfg.n_slices = n;
    cfg.family = CandidateFamily::UniformOnly;
    cfg.lambda = 0.1;
    const Partition up = uniform_partition(g, n);
    EXPECT(b200::uniform_partition(g, n) == up, "uniform_partition");
    const CostMap est = estimate_ctu_times(hist, 3);
    const SliceTimeTable rt = partition_time(est, up);
    const SliceTimeTable gt = b200::partition_time(ctx, est, up);
    EXPECT(rt.slice_times_us == gt.slice_times_us && rt.max_us == gt.max_us &&
               rt.total_us == gt.total_us && rt.argmax == gt.argmax,
           "partition_time");
    EXPECT(partition_sse(stats, up) == b200::partition_sse(ctx, stats, up), "partition_sse");
    bool ref_threw = false, gpu_threw = false;
    SearchOutcome ro, go;
    try { ro = two_step_partition(hist, stats, 3, cfg); } catch (const NoCandidateError&) { ref_threw = true; }
    try { go = b200::two_step_partition(ctx, hist, stats, 3, cfg); } catch (const NoCandidateError&) { gpu_threw = true; }
    EXPECT(ref_threw == gpu_threw, "UniformOnly NoCandidateError");
    if (!ref_threw) {
      EXPECT(go.best == ro.best, "UniformOnly best partition");
      EXPECT(go.t_min_us == ro.t_min_us && go.t_best_us == ro.t_best_us &&
                 go.sse_best == ro.sse_best,
             "UniformOnly values");
      EXPECT(go.candidates_step1 == ro.candidates_step1 &&
                 go.candidates_step2 == ro.candidates_step2 &&
                 go.candidates_evaluated == ro.candidates_evaluated,
             "UniformOnly counts");
    }
  }
  // exception classes cross the boundary unchanged
  {
    const CtuGrid g = CtuGrid::make(256, 128, 128);
    CostMap est = make_map(g, 0, 0, 5);
    SearchConfig cfg;
    cfg.n_slices = 3;
    bool caught = false;
    try {
      b200::min_time_search(ctx, est, cfg);
    } catch (const GeometryError&) {
      caught = true;
    }
    EXPECT(caught, "GeometryError for n > cells");
    cfg.n_slices = 1;
    cfg.k_area = 1.0;
    caught = false;
    try {
      b200::min_time_search(ctx, est, cfg);
    } catch (const ConfigError&) {
      caught = true;
    }
    EXPECT(caught, "ConfigError for k <= 1");
  }
  std::printf(failures ? "DROPIN FAILED (%d)\n" : "DROPIN OK\n", failures);
  return failures ? 1 : 0;
}
