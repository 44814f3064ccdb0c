// TEST-ONLY host emulator of the K4/K5 search kernels.
//
// Compiles the very same walk code the GPU runs (csrc/search_walk.cuh, the
// body of k_search) for the host and executes it lane by lane: `warps`
// emulated warps take the work items round-robin (increasing per warp, like
// the kernel's atomic counter), every lane keeps its first-in-order best, and
// the per-frame reduction mirrors k_finalize.  Used by the CPU test suite to
// check the kernel LOGIC against the oracle without a GPU; never part of the
// product library.
#include <cmath>
#include <cstring>
#include <vector>

#include "search_walk.cuh"

using namespace scb;

extern "C" int emu_search(int cols, int rows, int n, double k, int max_tile_cols, int coverage,
                          int step, int prune, int frames, const double* rect_time /*[F][NR]*/,
                          const double* rect_sse /*[F][NR] or NULL*/, const double* budget,
                          int warps, size_t item_target, int item_offset, int item_stride,
                          double* out_t, double* out_sse, uint64_t* out_count,
                          uint8_t* out_snap /*[F][96]*/, int* out_found, uint64_t* out_item,
                          uint64_t* out_ord, int order_mode, int split_g, int split_depth,
                          void (*seed_allreduce)(uint64_t* inc, int n)) {
  // order_mode (exhaustive step 1 only, like api.cu's cost schedule): 0 the
  // enumeration order, 1 reversed, 2 a fixed pseudo-random permutation
  if (frames < 1 || frames > 32) return 1;
  int fpw = 1;
  while (fpw < frames) fpw <<= 1;
  const int eff = max_tile_cols > 0 ? max_tile_cols : n;
  const int maxc = std::min(std::min(n, eff), cols);
  const std::vector<WorkItem> items = make_items(cols, maxc, coverage == 1, item_target);
  std::vector<int32_t> tab;
  const bool patho = make_area_tables(cols, rows, k, tab);
  const int A = cols * rows + 1;
  const int rstride = std::min(n, rows) + 1;
  std::vector<int32_t> ilo((size_t)(cols + 1) * rstride, 0);
  std::vector<uint64_t> magic(cols + 1, 0);
  for (int w = 1; w <= cols; ++w) {
    for (int r = 1; r < rstride; ++r) ilo[w * rstride + r] = tab[A + w * ((rows + r - 1) / r)];
    magic[w] = div_magic(w);
  }
  const int nyh = rows * (rows + 1) / 2;
  std::vector<int32_t> ybase(rows + 1), sfx(rows + 1), rq(rows + 1, 0);
  for (int r = 1; r <= rows; ++r) rq[r] = rows / r;
  for (int y = 0; y <= rows; ++y) {
    ybase[y] = yh_of(rows, y, 1);
    sfx[y] = y < rows ? yh_of(rows, y, rows - y) : 0;
  }
  const size_t nr = (size_t)cols * (cols + 1) / 2 * nyh;
  // time keys: per-frame exact ranks of the clamped rectangle times (api.cu
  // ranks on the device); vals[f] maps a rank back to its time bits
  std::vector<tkey> rt(nr * fpw, 0);
  std::vector<double> rs(nr * fpw, 0.0);
  std::vector<std::vector<uint64_t>> vals(fpw);
  for (int f = 0; f < frames; ++f) {
    std::vector<uint64_t> bits(nr);
    for (size_t r = 0; r < nr; ++r) {
      const double t = rect_time[(size_t)f * nr + r];
      uint64_t b;
      std::memcpy(&b, &t, 8);
      bits[r] = (t > 0.0) ? b : 0;
      if (rect_sse) rs[r * fpw + f] = rect_sse[(size_t)f * nr + r];
    }
    vals[f] = bits;
    std::sort(vals[f].begin(), vals[f].end());
    vals[f].erase(std::unique(vals[f].begin(), vals[f].end()), vals[f].end());
    for (size_t r = 0; r < nr; ++r)
      rt[r * fpw + f] =
          (tkey)(std::lower_bound(vals[f].begin(), vals[f].end(), bits[r]) - vals[f].begin());
  }
  // pruned mode: per-frame column lower bounds, shared incumbents
  const int nxw = cols * (cols + 1) / 2;
  std::vector<tkey> lbr((size_t)nxw * rstride * fpw, 0), lbm((size_t)nxw * rstride * fpw, 0);
  std::vector<uint64_t> inc(fpw, ~0ull);
  if (prune)
    for (int xw = 0; xw < nxw; ++xw)
      for (int f = 0; f < frames; ++f) {
        const size_t off = (size_t)xw * rstride * fpw + f;
        column_bounds(rt.data(), fpw, f, rows, xw * nyh, rstride - 1, lbr.data() + off,
                      lbm.data() + off, (size_t)fpw);
      }
  // split table (tables.cu k_split_table): max(run, forced rest of the column)
  std::vector<tkey> rts(nr * fpw, 0);
  for (int xw = 0; xw < cols * (cols + 1) / 2; ++xw)
    for (int y0 = 0; y0 < rows; ++y0)
      for (int h = 1; y0 + h < rows; ++h)
        for (int f = 0; f < fpw; ++f) {
          const size_t r1 = (size_t)xw * nyh + yh_of(rows, y0, h);
          const size_t r2 = (size_t)xw * nyh + yh_of(rows, y0 + h, rows - y0 - h);
          rts[r1 * fpw + f] = std::max(rt[r1 * fpw + f], rt[r2 * fpw + f]);
        }
  WalkEnv e;
  e.cols = cols;
  e.rows = rows;
  e.n = n;
  e.nyh = nyh;
  e.max_area = cols * rows;
  e.coverage = coverage;
  e.patho = patho ? 1 : 0;
  e.prune = prune;
  e.rstride = rstride;
  e.bmax = tab.data();
  e.aneed = tab.data() + A;
  e.mstar = tab.data() + 2 * A;
  e.ilo = ilo.data();
  e.magic = magic.data();
  e.rq = rq.data();
  e.rt = rt.data();
  e.rts = rts.data();
  e.rs = rs.data();
  e.lbr = lbr.data();
  e.lbm = lbm.data();
  e.inc = inc.data();
  e.seed_inc = nullptr;
  std::vector<uint64_t> sse_inc(fpw, ~0ull);  // pruned step 2: shared SSE incumbent
  e.sse_inc = (prune && step == 2) ? sse_inc.data() : nullptr;
  std::vector<uint64_t> frozen(fpw, ~0ull);
  // seeded pruned step 1 like api.cu: phase A = the first seed_items items
  size_t seed_items = 0;
  for (const WorkItem& wi : items) {
    if (wi.c > 1) break;
    ++seed_items;
  }

  std::vector<LaneState> st((size_t)warps * 32);
  std::vector<uint8_t> snaps((size_t)warps * 32 * kSnap, 0);
  for (int wp = 0; wp < warps; ++wp)
    for (int l = 0; l < 32; ++l) {
      LaneState& s = st[(size_t)wp * 32 + l];
      s.best_t = kKeyInf;
      s.best_item = ~0ull;
      s.best_ord = ~0ull;
      s.best_sse = INFINITY;
      s.count = 0;
      s.scored = 0;
      s.inc = ~0ull;
      s.sbound = INFINITY;
      s.snap = &snaps[((size_t)wp * 32 + l) * kSnap];
      s.budget = -1;
      if (step == 2 && (l % fpw) < frames) {  // largest key whose time is <= budget
        const double b = budget[l % fpw];
        s.budget = -1;  // nothing feasible (negative or NaN budget)
        if (b >= 0.0) {
          uint64_t bits;
          std::memcpy(&bits, &b, 8);
          const auto& v = vals[l % fpw];
          s.budget = (int64_t)(std::upper_bound(v.begin(), v.end(), bits) - v.begin()) - 1;
        }
      }
    }
  size_t kk = 0;
  const size_t mine = items.size() > (size_t)item_offset
                          ? (items.size() - item_offset + item_stride - 1) / item_stride
                          : 0;
  const size_t seed_local = (prune && step == 1) ? std::min(mine, seed_items) : 0;
  std::vector<size_t> seq;
  for (size_t it = (size_t)item_offset; it < items.size(); it += (size_t)item_stride) seq.push_back(it);
  if (step == 1 && !prune && order_mode == 1) std::reverse(seq.begin(), seq.end());
  if (step == 1 && !prune && order_mode == 2) {
    uint64_t z = 0x9e3779b97f4a7c15ull;
    for (size_t i = seq.size(); i > 1; --i) {
      z = z * 6364136223846793005ull + 1442695040888963407ull;
      std::swap(seq[i - 1], seq[(size_t)((z >> 33) % i)]);
    }
  }
  // pruned mode: split_g units per item (api.cu / k_search), dealt round-robin
  const int G = prune ? (split_g > 1 ? split_g : 1) : 1;
  e.split_g = G;
  e.split_depth = split_depth;
  for (size_t su = 0; su < seq.size() * (size_t)G; ++su, ++kk) {
    const size_t it = seq[su / (size_t)G];
    const int part = (int)(su % (size_t)G);
    if (prune && step == 1 && kk == seed_local * (size_t)G && seed_local > 0) {  // phase B
      frozen = inc;
      // shards (api.cu sc_comm_*): the frozen incumbent is the global minimum
      if (seed_allreduce) seed_allreduce(frozen.data(), fpw);
      e.seed_inc = frozen.data();
    }
    const int wp = (int)(kk % (size_t)warps);
    for (int l = 0; l < 32; ++l) {
      LaneState& s = st[(size_t)wp * 32 + l];
      switch (fpw * 10 + step) {
#define CASE(F)                                                                   \
  case F * 10 + 1:                                                                \
    if (prune) walk_item<F, 1, true>(e, it, items[it], l % F, l / F, s, part);    \
    else walk_item<F, 1, false>(e, it, items[it], l % F, l / F, s);               \
    break;                                                                        \
  case F * 10 + 2:                                                                \
    if (prune) walk_item<F, 2, true>(e, it, items[it], l % F, l / F, s, part);    \
    else walk_item<F, 2, false>(e, it, items[it], l % F, l / F, s);               \
    break;
        CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
        default: return 2;
      }
    }
  }
  for (int f = 0; f < frames; ++f) {
    int win = -1;
    for (int i = 0; i < warps * 32; ++i) {
      if (i % 32 % fpw != f) continue;
      const LaneState& s = st[i];
      if (s.best_item == ~0ull) continue;
      if (win < 0) { win = i; continue; }
      const LaneState& b = st[win];
      bool less;
      if (step == 2 && s.best_sse != b.best_sse) less = s.best_sse < b.best_sse;
      else if (s.best_t != b.best_t) less = s.best_t < b.best_t;
      else if (s.best_item != b.best_item) less = s.best_item < b.best_item;
      else {  // position inside the item: the layout, lexicographically (k_finalize)
        less = false;
        for (int j = 0; j < 2 * 16 + n; ++j)
          if (s.snap[j] != b.snap[j]) {
            less = s.snap[j] < b.snap[j];
            break;
          }
      }
      if (less) win = i;
    }
    out_found[f] = win >= 0;
    uint64_t cnt = 0;
    for (int wp = 0; wp < warps; ++wp) cnt += st[(size_t)wp * 32].count;
    if (prune) {  // pruned walks: the exact DP count (api.cu does the same)
      cnt = (uint64_t)count_candidates_dp(cols, rows, n, maxc, coverage == 1, tab, 1);
    }
    out_count[f] = cnt;
    if (win >= 0) {
      std::memcpy(&out_t[f], &vals[f][st[win].best_t], 8);
      out_sse[f] = st[win].best_sse;
      std::memcpy(out_snap + (size_t)f * kSnap, st[win].snap, kSnap);
      out_item[f] = st[win].best_item;
      out_ord[f] = st[win].best_ord;
    }
  }
  return 0;
}

// The exhaustive step 1 through the candidate trace (csrc/trace.cuh): the host
// build of the same generator and a scalar interpreter (one frame at a time,
// exact doubles instead of rank keys; max / < on doubles equal max / < on
// the keys), plus the layout rebuilt from the winning ordinal.  Work items
// are split in `item_target`-sized prefixes like api.cu's plan, processed in
// order, so any item-boundary mistake shows up as a different candidate set.
#include "trace.cuh"
extern "C" int emu_trace_search(int cols, int rows, int n, double k, int max_tile_cols,
                                int coverage, int frames, const double* rect_time /*[F][NR]*/,
                                size_t item_target, double* out_t, uint64_t* out_count,
                                uint64_t* out_ord, uint8_t* out_snap /*[F][96]*/, int* out_found,
                                uint64_t* out_ops) {
  const int eff = max_tile_cols > 0 ? max_tile_cols : n;
  const int maxc = std::min(std::min(n, eff), cols);
  const std::vector<WorkItem> items = make_items(cols, maxc, coverage == 1, item_target);
  std::vector<uint32_t> ops;
  std::vector<uint32_t> skel_pos;
  std::vector<uint64_t> skel_ord;
  uint64_t cand = 0;
  for (const WorkItem& wi : items) {
    TraceCount c;
    trace_item(wi, cols, rows, n, k, coverage, c);
    const size_t o0 = ops.size(), s0 = skel_pos.size();
    ops.resize(o0 + c.ops);
    skel_pos.resize(s0 + c.skels);
    skel_ord.resize(s0 + c.skels);
    TraceWrite w;
    w.ops = ops.data() + o0;
    w.op_base = o0;
    w.cand = cand;
    w.skel_pos = skel_pos.data() + s0;
    w.skel_ord = skel_ord.data() + s0;
    trace_item(wi, cols, rows, n, k, coverage, w);
    if (w.pos != c.ops || w.cand - cand != c.cands || w.nsk != c.skels) return 3;
    cand = w.cand;
  }
  skel_pos.push_back((uint32_t)ops.size());
  skel_ord.push_back(cand);
  *out_ops = ops.size();
  const int nyh = rows * (rows + 1) / 2;
  const size_t nr = (size_t)cols * (cols + 1) / 2 * nyh;
  for (int f = 0; f < frames; ++f) {
    const double* T = rect_time + (size_t)f * nr;
    auto clamp = [](double t) { return t > 0.0 ? t : 0.0; };  // layout_time's max from 0.0
    auto tsplit = [&](uint32_t idx) {  // run + forced rest of its column
      const int xw = (int)(idx / (uint32_t)nyh), yh = (int)(idx % (uint32_t)nyh);
      int y0 = 0;
      while (tr_yh(rows, y0 + 1, 1) <= yh && y0 + 1 < rows) ++y0;
      const int h = yh - tr_yh(rows, y0, 1) + 1;
      const double a = clamp(T[idx]);
      if (y0 + h >= rows) return a;
      const double b = clamp(T[(size_t)xw * nyh + tr_yh(rows, y0 + h, rows - y0 - h)]);
      return a > b ? a : b;
    };
    std::vector<double> P(n + 2, 0.0);
    double best = INFINITY;
    uint64_t best_ord = ~0ull, ord = 0;
    int ld = 0;
    for (size_t p = 0; p < ops.size(); ++p) {
      const uint32_t op = ops[p], code = tr_code(op);
      if (tr_is_push(op)) {
        const int d = tr_small_of(op);
        const uint32_t kidx = tr_kidx(op);
        const double v = kidx >= nr ? tsplit(kidx - (uint32_t)nr) : clamp(T[kidx]);
        P[d + 1] = P[d] > v ? P[d] : v;
      } else if (code == kOpLeaf) {
        const int cnt = tr_leaf_cnt(op);
        if (cnt == 0) {
          if (P[ld] < best) best = P[ld], best_ord = ord;
          ord += 1;
          continue;
        }
        const uint32_t idx = tr_kidx(op) - (uint32_t)nr;
        for (int h = 0; h < cnt; ++h) {
          const double v = tsplit(idx + (uint32_t)h);
          const double t = P[ld] > v ? P[ld] : v;
          if (t < best) best = t, best_ord = ord + (uint64_t)h;
        }
        ord += (uint64_t)cnt;
      } else if (tr_is_fix(op)) {
        const double v = clamp(T[tr_kidx(op)]);
        P[0] = P[0] > v ? P[0] : v;
      } else {
        ld = tr_skel_ld(op);
        P[0] = 0.0;
      }
    }
    out_count[f] = ord;
    out_found[f] = best_ord != ~0ull;
    out_t[f] = best;
    out_ord[f] = best_ord;
    if (best_ord != ~0ull) {
      size_t s = std::upper_bound(skel_ord.begin(), skel_ord.end(), best_ord) - skel_ord.begin() - 1;
      if (!trace_layout(ops.data() + skel_pos[s], skel_pos[s + 1] - skel_pos[s],
                        best_ord - skel_ord[s], cols, rows, n, out_snap + (size_t)f * kSnap))
        return 4;
    }
  }
  return 0;
}

// Step 2 through the trace (scalar, one frame at a time): every candidate
// with time <= budget gets its SSE folded in slice order -- leading one-run
// columns at the skeleton start, each multi-run column's runs, its forced
// rest, then the one-run columns after it (FIX tags) -- and the (sse, t,
// order) minimum is kept.  Mirrors k_trace_walk2 (csrc/trace.cu).
extern "C" int emu_trace_step2(int cols, int rows, int n, double k, int max_tile_cols,
                               int coverage, int frames, const double* rect_time,
                               const double* rect_sse, const double* budget, size_t item_target,
                               double* out_t, double* out_sse, uint64_t* out_ord,
                               uint8_t* out_snap, int* out_found) {
  const int eff = max_tile_cols > 0 ? max_tile_cols : n;
  const int maxc = std::min(std::min(n, eff), cols);
  const std::vector<WorkItem> items = make_items(cols, maxc, coverage == 1, item_target);
  std::vector<uint32_t> ops, skel_pos;
  std::vector<uint64_t> skel_ord;
  uint64_t cand = 0;
  for (const WorkItem& wi : items) {
    TraceCount c;
    trace_item(wi, cols, rows, n, k, coverage, c);
    const size_t o0 = ops.size(), s0 = skel_pos.size();
    ops.resize(o0 + c.ops);
    skel_pos.resize(s0 + c.skels);
    skel_ord.resize(s0 + c.skels);
    TraceWrite w;
    w.ops = ops.data() + o0;
    w.op_base = o0;
    w.cand = cand;
    w.skel_pos = skel_pos.data() + s0;
    w.skel_ord = skel_ord.data() + s0;
    trace_item(wi, cols, rows, n, k, coverage, w);
    cand = w.cand;
  }
  skel_pos.push_back((uint32_t)ops.size());
  skel_ord.push_back(cand);
  const int nyh = rows * (rows + 1) / 2;
  const size_t nr = (size_t)cols * (cols + 1) / 2 * nyh;
  auto rest_of = [&](uint32_t idx) {
    const int xw = (int)(idx / (uint32_t)nyh), yh = (int)(idx % (uint32_t)nyh);
    int y0 = 0;
    while (y0 + 1 < rows && tr_yh(rows, y0 + 1, 1) <= yh) ++y0;
    const int h = yh - tr_yh(rows, y0, 1) + 1;
    return (uint32_t)(xw * nyh + tr_yh(rows, y0 + h, rows - y0 - h));
  };
  for (int f = 0; f < frames; ++f) {
    const double* T = rect_time + (size_t)f * nr;
    const double* S = rect_sse + (size_t)f * nr;
    auto clamp = [](double t) { return t > 0.0 ? t : 0.0; };
    auto tkey = [&](uint32_t idx, bool split) {
      const double a = clamp(T[idx]);
      if (!split) return a;
      const double b = clamp(T[rest_of(idx)]);
      return a > b ? a : b;
    };
    std::vector<double> P(n + 2, 0.0), SS(n + 2, 0.0);
    std::vector<int> Cc(n + 2, 0);
    uint32_t fxi[SC_MAX_COLS];
    int fxt[SC_MAX_COLS], nfx = 0, ld = 0;
    double bs = INFINITY, bt = INFINITY;
    uint64_t bo = ~0ull, ord = 0;
    size_t bpos = 0;
    int bhit = 0;
    const double B = budget[f];
    auto fold_fix = [&](double s, int tag) {
      for (int j = 0; j < nfx; ++j)
        if (fxt[j] == tag) s = s + S[fxi[j]];
      return s;
    };
    auto offer = [&](double t, double sse, uint64_t o, size_t pos, int hit) {
      if (!(t <= B)) return;
      if (sse < bs || (sse == bs && (t < bt || (t == bt && o < bo)))) {
        bs = sse, bt = t, bo = o, bpos = pos, bhit = hit;
      }
    };
    for (size_t p = 0; p < ops.size(); ++p) {
      const uint32_t op = ops[p], code = tr_code(op);
      if (tr_is_push(op)) {
        const int d = tr_small_of(op);
        const uint32_t kidx = tr_kidx(op);
        const bool split = kidx >= nr;
        const uint32_t idx = split ? kidx - (uint32_t)nr : kidx;
        const double v = tkey(idx, split);
        P[d + 1] = P[d] > v ? P[d] : v;
        double s = SS[d] + S[idx];
        int c = Cc[d];
        if (split) {
          s = s + S[rest_of(idx)];
          ++c;
          s = fold_fix(s, c);
        }
        SS[d + 1] = s;
        Cc[d + 1] = c;
      } else if (code == kOpLeaf) {
        const int cnt = tr_leaf_cnt(op);
        if (cnt == 0) {
          offer(P[ld], SS[ld], ord, p, 0);
          ord += 1;
          continue;
        }
        const uint32_t idx = tr_kidx(op) - (uint32_t)nr;
        for (int h = 0; h < cnt; ++h) {
          const double v = tkey(idx + (uint32_t)h, true);
          const double t = P[ld] > v ? P[ld] : v;
          if (!(t <= B)) continue;
          double s = SS[ld] + S[idx + (uint32_t)h];
          s = s + S[rest_of(idx + (uint32_t)h)];
          s = fold_fix(s, Cc[ld] + 1);
          offer(t, s, ord + (uint64_t)h, p, h);
        }
        ord += (uint64_t)cnt;
      } else if (tr_is_fix(op)) {
        const uint32_t idx = tr_kidx(op);
        const int tag = tr_small_of(op);
        const double v = clamp(T[idx]);
        P[0] = P[0] > v ? P[0] : v;
        if (tag == 0) SS[0] = SS[0] + S[idx];
        else fxi[nfx] = idx, fxt[nfx] = tag, ++nfx;
      } else {
        ld = tr_skel_ld(op);
        P[0] = 0.0, SS[0] = 0.0, Cc[0] = 0, nfx = 0;
      }
    }
    out_found[f] = bo != ~0ull;
    out_t[f] = bt;
    out_sse[f] = bs;
    out_ord[f] = bo;
    if (bo != ~0ull) {
      size_t s = std::upper_bound(skel_ord.begin(), skel_ord.end(), bo) - skel_ord.begin() - 1;
      if (!trace_layout(ops.data() + skel_pos[s], skel_pos[s + 1] - skel_pos[s], bo - skel_ord[s],
                        cols, rows, n, out_snap + (size_t)f * kSnap))
        return 4;
      (void)bpos;
      (void)bhit;
    }
  }
  return 0;
}

// tr_unrank (csrc/trace.cuh: closed form + fix-up) against the defining
// search, for every (origin, extent) of an axis of n cells; returns the
// number of mismatches.
extern "C" int emu_unrank_check(int n) {
  int bad = 0;
  for (int a0 = 0; a0 < n; ++a0)
    for (int e0 = 1; e0 <= n - a0; ++e0) {
      const int v = tr_xw(n, a0, e0);
      int a = -1, e = -1;
      tr_unrank(n, v, a, e);
      bad += (a != a0 || e != e0) ? 1 : 0;
    }
  return bad;
}

// Trace encoding round trip (csrc/trace.cuh): every field of every op kind.
extern "C" int emu_trace_encoding_check() {
  int bad = 0;
  for (int d = 0; d < 64; ++d)
    for (uint32_t kidx : {0u, 1u, 12345u, kTrKeyMask}) {
      for (int tl = 0; tl < 2; ++tl) {
        const uint32_t op = op_push(d, kidx, tl != 0);
        bad += !(tr_is_push(op) && tr_code(op) == (tl ? kOpPushL : kOpPush) &&
                 tr_small_of(op) == d && tr_kidx(op) == kidx && tr_koff32(op) == kidx * 32u);
      }
      if (kidx <= kTrIdxMask) {
        const uint32_t fx = op_fix(kidx, d);
        bad += !(tr_code(fx) == kOpSkel && tr_is_fix(fx) && !tr_is_push(fx) &&
                 tr_small_of(fx) == d && tr_kidx(fx) == kidx);
      }
    }
  for (int cnt = 0; cnt <= kTrLeafMax; ++cnt)
    for (uint32_t kidx : {0u, 777u, kTrKeyMask}) {
      const uint32_t op = op_leaf(kidx, cnt);
      bad += !(tr_code(op) == kOpLeaf && !tr_is_push(op) && !tr_is_fix(op) &&
               tr_leaf_cnt(op) == cnt && tr_kidx(op) == kidx);
    }
  for (int ld = 0; ld < 64; ++ld) {
    const uint32_t op = op_skel(ld);
    bad += !(tr_code(op) == kOpSkel && !tr_is_fix(op) && tr_skel_ld(op) == ld);
  }
  return bad;
}
