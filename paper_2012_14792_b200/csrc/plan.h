// Frame-independent search plan (host C++, no CUDA): the work items that tile
// the reference's enumeration order and the integer area tables.  Shared by
// api.cu and the test-only host emulator (tests/emu).
#pragma once

#include <stdint.h>

#include <algorithm>
#include <vector>

namespace scb {

// A work item is a lex-ordered prefix (c, w_0..w_{d-1}) of the ColumnSplit
// enumeration (search.cpp:120-143); the items, in index order, tile the
// reference's enumeration order exactly.
struct WorkItem {
  uint8_t c, d, pad0, pad1;
  uint8_t w[12];
};
static_assert(sizeof(WorkItem) == 16, "WorkItem is one uint4");

// All width prefixes of depth d for c columns, in lex order (rec_widths,
// search.cpp:133-143: w_i in [1, cols_left - (c - i - 1)]).
inline void gen_prefixes(int cols, int c, int d, bool covering, std::vector<WorkItem>& out) {
  int w[16] = {0};
  int cl[17];
  int i = 0;
  cl[0] = cols;
  w[0] = 0;
  if (d == 0) {
    WorkItem it{};
    it.c = (uint8_t)c;
    out.push_back(it);
    return;
  }
  while (i >= 0) {
    const int maxw = cl[i] - (c - i - 1);
    if (++w[i] > maxw) {
      --i;
      continue;
    }
    if (i == d - 1) {
      if (covering && d == c && cl[i] - w[i] != 0) continue;
      WorkItem it{};
      it.c = (uint8_t)c;
      it.d = (uint8_t)d;
      for (int j = 0; j < d; ++j) it.w[j] = (uint8_t)w[j];
      out.push_back(it);
      continue;
    }
    cl[i + 1] = cl[i] - w[i];
    ++i;
    w[i] = 0;
  }
}

// Work items: width prefixes of depth min(c, D), D grown until there are at
// least `target` items (or every width is fixed).
inline std::vector<WorkItem> make_items(int cols, int maxc, bool covering, size_t target) {
  std::vector<WorkItem> items;
  for (int D = 1; D <= 12; ++D) {
    items.clear();
    for (int c = 1; c <= maxc; ++c) gen_prefixes(cols, c, std::min(c, D), covering, items);
    if (items.size() >= target || D >= maxc || items.size() > (1u << 22)) break;
  }
  return items;
}

// Area tables (the admissibility test k*(double)amin > (double)amax of
// search.cpp:182-183, tabulated so the kernels compare integers only), laid
// out bmax[A] | aneed[A] | mstar[(cols+1)*(rows+1)], A = cols*rows + 1:
//   bmax[a]      largest B in [0, max_area] with k*(double)a > (double)B (-1: none)
//   aneed[B]     smallest a >= 1 with bmax[a] >= B (max_area+1: none)
//   mstar[w][rl] smallest m in [1, rl/2] with w*(rl-m) <= bmax[w*m]
//                (rl/2+1: none) -- the two-run split admissibility bound
// Returns true when some single area a fails the test (k barely above 1).
inline bool make_area_tables(int cols, int rows, double k, std::vector<int32_t>& t) {
  const int max_area = cols * rows;
  const int A = max_area + 1;
  t.assign((size_t)2 * A + (size_t)(cols + 1) * (rows + 1), 0);
  int32_t* bm = t.data();
  int32_t* an = bm + A;
  int32_t* ms = an + A;
  int b = -1;
  bool pathological = false;
  for (int a = 0; a <= max_area; ++a) {
    // k*a is non-decreasing in a, so b only moves up
    while (b + 1 <= max_area && k * (double)a > (double)(b + 1)) ++b;
    bm[a] = b;
    if (a >= 1 && b < a) pathological = true;
  }
  int a_cur = 1;
  for (int B = 0; B <= max_area; ++B) {
    while (a_cur <= max_area && bm[a_cur] < B) ++a_cur;
    an[B] = a_cur;
  }
  for (int w = 1; w <= cols; ++w)
    for (int rl = 0; rl <= rows; ++rl) {
      int m = 1;
      while (m <= rl / 2 && !((int64_t)w * (rl - m) <= bm[w * m])) ++m;
      ms[w * (rows + 1) + rl] = (rl >= 2) ? m : rl / 2 + 1;
    }
  return pathological;
}

// uniform_partition (grid.cpp:186-262): the best r x c factorization of n by
// its largest slice area (ties toward more columns), tiles from split_even
// (grid.cpp:53-61), slices row-major; when no factorization fits, c =
// min(n, cols) columns each cut into near-equal runs.  Returns false if n is
// outside [1, cols * rows] (the reference's GeometryError).  Slices as
// {x0, y0, w, h} in id order.
struct UniformPartition {
  std::vector<int> tile_cols, tile_rows;
  std::vector<int> rects;  // 4 ints per slice
};
inline std::vector<int> split_even(int total, int parts) {
  std::vector<int> out((size_t)parts);
  for (int i = 0; i < parts; ++i) out[(size_t)i] = total / parts + (i < total % parts ? 1 : 0);
  return out;
}
inline bool uniform_partition(int cols, int rows, int n, UniformPartition& p) {
  if (n < 1 || (int64_t)n > (int64_t)cols * rows) return false;
  int best_c = -1, best_r = -1;
  int64_t best_area = -1;
  for (int c = 1; c <= std::min(n, cols); ++c) {
    if (n % c != 0) continue;
    const int r = n / c;
    if (r > rows) continue;
    const int64_t a = (int64_t)((cols + c - 1) / c) * ((rows + r - 1) / r);
    if (best_area < 0 || a < best_area || (a == best_area && c > best_c)) {
      best_area = a;
      best_c = c;
      best_r = r;
    }
  }
  p.rects.clear();
  if (best_c > 0) {
    p.tile_cols = split_even(cols, best_c);
    p.tile_rows = split_even(rows, best_r);
    for (int r = 0, y = 0; r < best_r; y += p.tile_rows[(size_t)r], ++r)
      for (int c = 0, x = 0; c < best_c; x += p.tile_cols[(size_t)c], ++c)
        p.rects.insert(p.rects.end(), {x, y, p.tile_cols[(size_t)c], p.tile_rows[(size_t)r]});
    return true;
  }
  const int c = std::min(n, cols);
  p.tile_cols = split_even(cols, c);
  p.tile_rows = {rows};
  const std::vector<int> counts = split_even(n, c);
  for (int col = 0, x = 0; col < c; x += p.tile_cols[(size_t)col], ++col) {
    int y = 0;
    for (int h : split_even(rows, counts[(size_t)col])) {
      p.rects.insert(p.rects.end(), {x, y, p.tile_cols[(size_t)col], h});
      y += h;
    }
  }
  return true;
}

}  // namespace scb

#include <thread>

namespace scb {

// Exact candidate count of the ColumnSplit family (what for_each_candidate
// would enumerate, search.cpp:302-319) without enumerating it.
//
// A candidate is admissible iff all its slice areas lie in one window
// [a, bmax[a]] (a = its smallest area).  So
//     count = sum_a  N(a, bmax[a]) - N(a+1, bmax[a])
// where N(lo, hi) counts candidates whose areas all lie in [lo, hi].  N
// factorises over columns: a column of width w with r runs contributes the
// number of compositions of `rows` into r parts in [ceil(lo/w), floor(hi/w)],
// and a DP over (columns, width used, runs used) sums the products.  Only
// a <= cells / n can be a smallest area (n disjoint slices of area >= a).
// Counts are exact in 128 bits (cfg5: ~6.1e29 < 2^100).
using u128 = unsigned __int128;

inline u128 count_candidates_dp(int cols, int rows, int n, int maxc, bool covering,
                                const std::vector<int32_t>& tab, int threads = 0) {
  const int max_area = cols * rows;
  const int32_t* bm = tab.data();
  const int rmax = std::min(n, rows);
  // comp[hl][hh][r]: compositions of rows into r parts, each in [hl, hh]
  const int R1 = rows + 1;
  std::vector<u128> comp((size_t)R1 * R1 * (rmax + 1), 0);
  for (int hl = 1; hl <= rows; ++hl)
    for (int hh = hl; hh <= rows; ++hh) {
      std::vector<u128> f((size_t)(rmax + 1) * R1, 0);  // f[r][sum]
      f[0] = 1;
      for (int r = 1; r <= rmax; ++r)
        for (int sum = 0; sum <= rows; ++sum) {
          u128 v = 0;
          for (int h = hl; h <= hh && h <= sum; ++h) v += f[(size_t)(r - 1) * R1 + sum - h];
          f[(size_t)r * R1 + sum] = v;
        }
      for (int r = 1; r <= rmax; ++r) comp[((size_t)hl * R1 + hh) * (rmax + 1) + r] = f[(size_t)r * R1 + rows];
    }
  auto N = [&](int lo, int hi) -> u128 {
    if (lo > hi) return 0;
    // nonzero column options (w, r, ways)
    struct Opt { int w, r; u128 ways; };
    std::vector<Opt> opts;
    for (int w = 1; w <= cols; ++w) {
      const int hl = std::max(1, (lo + w - 1) / w), hh = std::min(rows, hi / w);
      if (hl > hh) continue;
      for (int r = 1; r <= rmax; ++r) {
        const u128 v = comp[((size_t)hl * R1 + hh) * (rmax + 1) + r];
        if (v) opts.push_back({w, r, v});
      }
    }
    if (opts.empty()) return 0;
    // D[x][s] for j columns, rolled over j
    const size_t S = (size_t)n + 1;
    std::vector<u128> D((size_t)(cols + 1) * S, 0), E((size_t)(cols + 1) * S, 0);
    D[0] = 1;
    u128 total = 0;
    for (int j = 1; j <= maxc; ++j) {
      std::fill(E.begin(), E.end(), (u128)0);
      for (int x = 0; x < cols; ++x)
        for (int s = 0; s < n; ++s) {
          const u128 d = D[(size_t)x * S + s];
          if (!d) continue;
          for (const Opt& o : opts) {
            if (x + o.w > cols || s + o.r > n) continue;
            E[(size_t)(x + o.w) * S + s + o.r] += d * o.ways;
          }
        }
      std::swap(D, E);
      for (int x = covering ? cols : 1; x <= cols; ++x) total += D[(size_t)x * S + n];
    }
    return total;
  };
  const int amax_min = max_area / std::max(n, 1);
  if (threads <= 0) threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<u128> part((size_t)threads, 0);
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&, t] {
      for (int a = 1 + t; a <= amax_min; a += threads) {
        const int B = bm[a];
        if (B < a) continue;
        part[t] += N(a, B) - N(a + 1, B);
      }
    });
  for (auto& x : th) x.join();
  u128 tot = 0;
  for (u128 v : part) tot += v;
  return tot;
}

}  // namespace scb
