// K4/K5 — exhaustive ColumnSplit search, step 1 (min time) and step 2
// (min SSE under the time budget).  Replaces ColumnSplitGenerator +
// run_blocked + layout_time/layout_sse + the two reductions
// (search.cpp:110-298, 334-405).
//
// Execution model:
//  * The candidate order of the reference is lexicographic in
//    (c, widths, runs, heights) (search.cpp:120-190).  The host cuts it into
//    work items = width prefixes (c, w_0..w_{d-1}); item index order equals
//    the reference's enumeration order.
//  * One warp walks one item at a time, fetched from a global atomic counter
//    (so a warp's items are increasing).  The walk is WARP-UNIFORM: every lane
//    executes the same DFS, because the candidate set and order do not depend
//    on the frame.  Lanes differ only by the frame they score
//    (f = lane % FPW) and, when fewer than 32 frames share the warp, by the
//    slot (lane / FPW) of the innermost height loop they take.
//  * Columns with one run are fixed by the skeleton and folded up front; the
//    heights DFS runs over the multi-run columns only, and its deepest level
//    (second-to-last run of the last multi-run column, whose last run is
//    forced) is the leaf loop.
//  * A lane keeps its first-in-order best with a strict comparison (its
//    candidates arrive in increasing (item, ordinal) order); finalize
//    reduces lanes by (key, item, ordinal), which is exactly the reference's
//    "first in enumeration order" tie-break.
//  * Times are compared as the u64 bit patterns of non-negative doubles
//    (monotone), SSE sums are accumulated in slice order with __dadd_rn.
#include <algorithm>

#include "common.cuh"

namespace scb {

constexpr int kMaxLevels = SC_MAX_SLICES;
constexpr int kBigArea = 1 << 20;  // "no slice yet" sentinel for amin

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// Area thresholds of a partial candidate ("admissible
// height intervals").  With bmax[] the tabulated admissibility test of
// search.cpp:182-183, a further slice of area x keeps the candidate
// admissible iff  T2 <= x <= T1  (and x <= bmax[x]), where
//   T1 = bmax[amin]   (+inf before the first slice)
//   T2 = aneed[amax]  (the smallest a with bmax[a] >= amax).
struct Thr {
  int t1, t2;
};
__device__ __forceinline__ Thr thresholds(const int32_t* s_bmax, const int32_t* s_aneed, int amin,
                                          int amax) {
  Thr t;
  t.t1 = amin >= kBigArea ? kBigArea : s_bmax[amin];
  t.t2 = s_aneed[amax];
  return t;
}

// Admissible heights of a run of width w starting with rl rows left in its
// column and runs_left runs (this one included).  runs_left == 2 means the
// next run is forced to take the rest (rl - h); then both areas w*h and
// w*(rl-h) must pass, which is the symmetric interval [m, rl-m] with
// m = max(ceil(T2/w), rl - floor(T1/w), mstar[w][rl]).  Otherwise the
// interval also encodes a look-ahead: the rl - h rows left must still split
// into runs_left-1 runs of admissible height (thresholds only tighten).
__device__ __forceinline__ int2 height_interval(const int32_t* s_mstar, int rows1, Thr t, int w,
                                                int rl, int runs_left) {
  const int hmin_a = max(1, (t.t2 + w - 1) / w);
  const int hmax_a = t.t1 < 0 ? 0 : t.t1 / w;
  if (runs_left == 2) {
    int m = max(hmin_a, rl - hmax_a);
    m = max(m, s_mstar[w * rows1 + rl]);
    return make_int2(m, rl - m);
  }
  const int k = runs_left - 1;
  int lo = max(hmin_a, rl - k * hmax_a);
  int hi = min(rl - k * hmin_a, hmax_a);
  return make_int2(lo, hi);
}

template <int FPW, int STEP>
__global__ void __launch_bounds__(256) k_search(SearchArgs a) {
  extern __shared__ int32_t s_tab[];
  const int A = a.max_area + 1;
  const int rows1 = a.rows + 1;
  const int ntab = 2 * A + (a.cols + 1) * rows1;
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) s_tab[i] = a.bmax[i];
  __syncthreads();
  const int32_t* s_bmax = s_tab;
  const int32_t* s_aneed = s_tab + A;
  const int32_t* s_mstar = s_tab + 2 * A;
  // column windows I(w, r) lower ends, ilo[w * rstride + r] (r <= min(n, rows))
  const int rstride = min(a.n, a.rows) + 1;
  int32_t* s_ilo = s_tab + ntab;
  for (int i = threadIdx.x; i < (a.cols + 1) * rstride; i += blockDim.x) {
    const int w = i / rstride, r = i % rstride;
    s_ilo[i] = (w >= 1 && r >= 1) ? s_aneed[w * ((a.rows + r - 1) / r)] : 0;
  }
  __syncthreads();

  constexpr int J = 32 / FPW;
  const int lane = threadIdx.x & 31;
  const int f = lane % FPW;
  const int slot = lane / FPW;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int rows = a.rows, cols = a.cols, nyh = a.nyh;
  const bool patho = a.pathological != 0;
  const uint64_t* __restrict__ rt = a.rt;
  const double* __restrict__ rs = a.rs;

  uint64_t best_t = ~0ull, best_item = ~0ull, best_ord = ~0ull;
  double best_sse = __longlong_as_double(0x7ff0000000000000ll);
  uint64_t budget = 0;
  if (STEP == 2) budget = a.budget[f];
  unsigned long long count = 0;
  uint8_t* snap = a.snaps + ((size_t)gwarp * 32 + lane) * kSnapBytes;

  // warp-uniform DFS state (identical in every lane)
  int W[SC_MAX_COLS], R[SC_MAX_COLS], X0[SC_MAX_COLS + 1], RS0[SC_MAX_COLS];
  uint8_t curH[SC_MAX_SLICES];
  uint8_t Lcol[kMaxLevels], Lrun[kMaxLevels], Ly0[kMaxLevels], Lh[kMaxLevels], Lhi[kMaxLevels];
  int32_t Amin[kMaxLevels], Amax[kMaxLevels];
  uint64_t Pin[kMaxLevels];

  auto rect = [&](int x0, int w, int y0, int h) -> int {
    return xw_index(cols, x0, w) * nyh + yh_index(rows, y0, h);
  };

  // Every multi-run column from `from` on can still be filled with runs of
  // admissible height (necessary condition; prunes dead subtrees early).
  auto columns_feasible = [&](int from, int c, Thr t) -> bool {
    for (int i = from; i < c; ++i) {
      if (R[i] < 2) continue;
      const int w = W[i];
      const int hmin_a = max(1, (t.t2 + w - 1) / w);
      const int hmax_a = t.t1 < 0 ? 0 : t.t1 / w;
      if (R[i] * hmin_a > rows || R[i] * hmax_a < rows) return false;
    }
    return true;
  };

  // snapshot of the current candidate; the leaf run `lr` takes height lh
  // and the forced run lr+1 the rest of its column (lr < 0: no leaf loop).
  auto take_snapshot = [&](int c, int lr, int lh, int lrest) {
    for (int i = 0; i < SC_MAX_COLS; ++i) {
      snap[i] = (uint8_t)(i < c ? W[i] : 0);
      snap[SC_MAX_COLS + i] = (uint8_t)(i < c ? R[i] : 0);
    }
    for (int i = 0; i < a.n; ++i) {
      uint8_t v = curH[i];
      if (i == lr) v = (uint8_t)lh;
      if (i == lr + 1 && lr >= 0) v = (uint8_t)lrest;
      snap[2 * SC_MAX_COLS + i] = v;
    }
  };

  // step-2 objective: sum of slice SSEs in slice order (search.cpp:85-91)
  auto layout_sse = [&](int c, int lr, int lh, int lrest) -> double {
    double tot = 0.0;
    int run = 0;
    for (int i = 0; i < c; ++i) {
      int y = 0;
      const int base = xw_index(cols, X0[i], W[i]) * nyh;
      for (int j = 0; j < R[i]; ++j, ++run) {
        int hh = curH[run];
        if (run == lr) hh = lh;
        else if (lr >= 0 && run == lr + 1) hh = lrest;
        tot = __dadd_rn(tot, rs[(size_t)(base + yh_index(rows, y, hh)) * FPW + f]);
        y += hh;
      }
    }
    return tot;
  };

  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(a.counter, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= a.n_items) break;
    const uint64_t item = (uint64_t)a.item_offset + (uint64_t)k * a.item_stride;
    const WorkItem wi = a.items[item];
    const int c = wi.c, d = wi.d;
    uint64_t ord = 0;  // ordinal of the next candidate inside this item

    // ---- widths DFS over positions d..c-1 (lex, search.cpp:133-143).  A
    //      width w can only host windows a in the hull of its column
    //      intervals [ilo(w, r_max), w*rows] (r <= n-c+1): prefixes whose hulls
    //      do not intersect cannot complete and are skipped.
    const int rmax_c = min(a.n - c + 1, rows);
    int WL[SC_MAX_COLS + 1], WH[SC_MAX_COLS + 1];
    X0[0] = 0;
    WL[0] = 1;
    WH[0] = a.max_area;
    bool ok = (a.n >= c) && (a.n <= c * rows);
    for (int i = 0; i < d && ok; ++i) {
      W[i] = wi.w[i];
      X0[i + 1] = X0[i] + W[i];
      WL[i + 1] = max(WL[i], s_ilo[W[i] * rstride + rmax_c]);
      WH[i + 1] = min(WH[i], W[i] * rows);
      ok = WL[i + 1] <= WH[i + 1];
    }
    int pos = d;
    bool have_widths = ok && d == c;  // item fixes every width
    if (ok && d < c) W[pos] = 0;
    while (ok) {
      if (!have_widths) {
        // advance the widths DFS to the next complete, hull-feasible vector
        bool got = false;
        while (true) {
          const int maxw = cols - X0[pos] - (c - pos - 1);
          int wv;
          if (a.coverage && pos == c - 1) wv = (W[pos] == 0) ? maxw : maxw + 1;
          else wv = W[pos] + 1;
          if (wv > maxw) {
            if (pos == d) break;
            --pos;
            continue;
          }
          W[pos] = wv;
          const int nL = max(WL[pos], s_ilo[wv * rstride + rmax_c]);
          const int nH = min(WH[pos], wv * rows);
          if (nL > nH) continue;
          X0[pos + 1] = X0[pos] + wv;
          WL[pos + 1] = nL;
          WH[pos + 1] = nH;
          if (pos == c - 1) {
            got = true;
            break;
          }
          ++pos;
          W[pos] = 0;
        }
        if (!got) break;
      }
      // ---- runs DFS (lex, search.cpp:145-161).  The skeleton (widths, runs)
      //      has an admissible completion iff the column windows
      //      I(w_i, r_i) = [aneed[w*ceil(rows/r)], w*floor(rows/r)] intersect
      //      (DESIGN.md §Search); I slides down as r grows, so each position's
      //      feasible r form one contiguous range.
      {
        int RL[SC_MAX_COLS], RH[SC_MAX_COLS], SL[SC_MAX_COLS];
        int rp = 0;
        RL[0] = 1;
        RH[0] = a.max_area;
        SL[0] = a.n;
        R[0] = max(1, a.n - (c - 1) * rows) - 1;
        while (true) {
          const int after = c - 1 - rp;
          const int rhi = min(rows, SL[rp] - after);
          const int w = W[rp];
          int r = R[rp] + 1, lo = 0, hi = 0;
          bool found = false;
          for (; r <= rhi; ++r) {
            lo = s_ilo[w * rstride + r];
            hi = w * (rows / r);
            if (hi < RL[rp]) break;  // every larger r is lower still
            if (lo <= RH[rp]) {
              found = true;
              break;
            }
          }
          if (!found) {
            if (rp == 0) break;
            --rp;
            continue;
          }
          R[rp] = r;
          const int nL = max(RL[rp], lo), nH = min(RH[rp], hi);
          if (nL > nH) continue;
          if (rp < c - 1) {
            SL[rp + 1] = SL[rp] - r;
            RL[rp + 1] = nL;
            RH[rp + 1] = nH;
            ++rp;
            R[rp] = max(1, SL[rp] - (c - 1 - rp) * rows) - 1;
            continue;
          }
          // ---- one live skeleton (c, widths, runs); window a in [nL, nH]
          const int win_lo = nL, win_hi = s_bmax[nH];
          // thresholds of a partial candidate, tightened by the skeleton window:
          // every area lies in [win_lo, bmax[win_hi]]
          auto thr = [&](int amn, int amx) -> Thr {
            Thr t = thresholds(s_bmax, s_aneed, amn, amx);
            t.t2 = max(t.t2, win_lo);
            t.t1 = min(t.t1, win_hi);
            return t;
          };
          // fold the one-run columns (fixed by the skeleton)
          int amin = kBigArea, amax = 0;
          int run = 0, nl = 0;
          for (int i = 0; i < c; ++i) {
            RS0[i] = run;
            if (R[i] == 1) {
              const int ar = W[i] * rows;
              amin = min(amin, ar);
              amax = max(amax, ar);
              curH[run] = (uint8_t)rows;
            } else {
              for (int j = 0; j < R[i] - 1; ++j, ++nl) {
                Lcol[nl] = (uint8_t)i;
                Lrun[nl] = (uint8_t)j;
              }
            }
            run += R[i];
          }
          uint64_t P = 0;
          for (int i = 0; i < c; ++i)
            if (R[i] == 1) P = umax64(P, rt[(size_t)rect(X0[i], W[i], 0, rows) * FPW + f]);

          if (nl == 0) {
            // the skeleton is a single candidate
            if (slot == 0) {
              const uint64_t t = P;
              if (STEP == 1) {
                if (t < best_t) {
                  best_t = t; best_item = item; best_ord = ord;
                  take_snapshot(c, -1, 0, 0);
                }
              } else if (t <= budget) {
                const double e = layout_sse(c, -1, 0, 0);
                if (e < best_sse || (e == best_sse && t < best_t)) {
                  best_sse = e; best_t = t; best_item = item; best_ord = ord;
                  take_snapshot(c, -1, 0, 0);
                }
              }
            }
            ord += 1;
            continue;
          }
          // ---- heights DFS over the multi-run columns (search.cpp:163-190)
          int l = 0;
          const bool leaf_now = (nl == 1);
          if (!leaf_now) {
            const int i = Lcol[0];
            const int2 iv = height_interval(s_mstar, rows1, thr(amin, amax), W[i], rows, R[i]);
            Lh[0] = (uint8_t)(iv.x - 1);
            Lhi[0] = (uint8_t)max(iv.y, 0);
            Pin[0] = P;
            Amin[0] = amin;
            Amax[0] = amax;
            Ly0[0] = 0;
          }
          while (true) {
            int lv;  // level whose state feeds the leaf loop
            uint64_t Pl;
            int amin_l, amax_l, y0l;
            if (leaf_now) {
              lv = 0; Pl = P; amin_l = amin; amax_l = amax; y0l = 0;
            } else {
              // advance level l to its next admissible height
              const int i = Lcol[l], j = Lrun[l];
              const int w = W[i], y0 = Ly0[l];
              const int rows_left = rows - y0;
              const bool forced = (R[i] - j) == 2;
              int h = Lh[l] + 1;
              const int hhi = Lhi[l];
              if (patho && !forced)
                while (h <= hhi && !(w * h <= s_bmax[w * h])) ++h;
              if (h > hhi) {
                if (l == 0) break;
                --l;
                continue;
              }
              Lh[l] = (uint8_t)h;
              const int a1 = w * h;
              int na = min(Amin[l], a1), nx = max(Amax[l], a1);
              const int ridx = RS0[i] + j;
              curH[ridx] = (uint8_t)h;
              uint64_t Pn = umax64(Pin[l], rt[(size_t)rect(X0[i], w, y0, h) * FPW + f]);
              if (forced) {
                const int a2 = w * (rows_left - h);
                na = min(na, a2);
                nx = max(nx, a2);
                curH[ridx + 1] = (uint8_t)(rows_left - h);
                Pn = umax64(Pn, rt[(size_t)rect(X0[i], w, y0 + h, rows_left - h) * FPW + f]);
              }
              const int nxt = l + 1;
              const bool new_col = Lrun[nxt] == 0;
              const int y0n = new_col ? 0 : y0 + h;
              const Thr tn = thr(na, nx);
              if (new_col && !columns_feasible(Lcol[nxt], c, tn)) continue;
              if (nxt < nl - 1) {
                const int i2 = Lcol[nxt];
                const int2 iv = height_interval(s_mstar, rows1, tn, W[i2], rows - y0n,
                                                R[i2] - Lrun[nxt]);
                if (iv.x > iv.y) continue;
                l = nxt;
                Lh[l] = (uint8_t)(iv.x - 1);
                Lhi[l] = (uint8_t)iv.y;
                Pin[l] = Pn;
                Amin[l] = na;
                Amax[l] = nx;
                Ly0[l] = (uint8_t)y0n;
                continue;
              }
              lv = nxt; Pl = Pn; amin_l = na; amax_l = nx; y0l = y0n;
            }
            // ---- leaf loop: run Lrun[lv] of column Lcol[lv] takes every
            //      admissible height; the column's last run is forced.
            {
              const int i = Lcol[lv];
              const int w = W[i];
              const int rows_left = rows - y0l;
              const int2 iv = height_interval(s_mstar, rows1, thr(amin_l, amax_l), w, rows_left, 2);
              const int lr = RS0[i] + Lrun[lv];
              const int xwb = xw_index(cols, X0[i], w) * nyh;
              const int ybase = yh_index(rows, y0l, 1);
              for (int h0 = iv.x; h0 <= iv.y; h0 += J) {
                const int h = h0 + slot;
                if (h <= iv.y) {
                  const uint64_t my_ord = ord + (uint64_t)(h - iv.x);
                  const int y1 = y0l + h, h2 = rows_left - h;
                  const uint64_t v1 = rt[(size_t)(xwb + ybase + h - 1) * FPW + f];
                  const uint64_t v2 = rt[(size_t)(xwb + yh_index(rows, y1, h2)) * FPW + f];
                  const uint64_t t = umax64(Pl, umax64(v1, v2));
                  if (STEP == 1) {
                    if (t < best_t) {
                      best_t = t; best_item = item; best_ord = my_ord;
                      take_snapshot(c, lr, h, h2);
                    }
                  } else if (t <= budget) {
                    const double e = layout_sse(c, lr, h, h2);
                    if (e < best_sse || (e == best_sse && t < best_t)) {
                      best_sse = e; best_t = t; best_item = item; best_ord = my_ord;
                      take_snapshot(c, lr, h, h2);
                    }
                  }
                }
              }
              if (iv.y >= iv.x) ord += (uint64_t)(iv.y - iv.x + 1);
            }
            if (leaf_now) break;
          }
        }
      }
      if (have_widths) break;
    }
    count += ord;
  }

  LaneBest lb;
  lb.t = best_t;
  lb.sse = best_sse;
  lb.item = best_item;
  lb.ord = best_ord;
  a.lanes[(size_t)gwarp * 32 + lane] = lb;
  if (lane == 0 && count) atomicAdd(a.count_out, count);
}

// ---- finalize: per frame, reduce all lanes of that frame ---------------------
__device__ __forceinline__ bool key_less(int step, const LaneBest& x, const LaneBest& y) {
  if (step == 2) {
    if (x.sse < y.sse) return true;
    if (x.sse > y.sse) return false;
  }
  if (x.t != y.t) return x.t < y.t;
  if (x.item != y.item) return x.item < y.item;
  return x.ord < y.ord;
}

__global__ void k_finalize(int step, int fpw, int frames_in_group, uint32_t n_warps,
                           const LaneBest* __restrict__ lanes, const uint8_t* __restrict__ snaps,
                           const unsigned long long* count, double lambda,
                           FrameBest* __restrict__ out, uint64_t* __restrict__ budget_out) {
  const int f = blockIdx.x;
  if (f >= frames_in_group) return;
  __shared__ LaneBest sb[256];
  __shared__ uint32_t si[256];
  LaneBest best;
  best.t = ~0ull; best.sse = __longlong_as_double(0x7ff0000000000000ll);
  best.item = ~0ull; best.ord = ~0ull;
  uint32_t bi = 0xffffffffu;
  const uint32_t n_lanes = n_warps * 32;
  for (uint32_t li = threadIdx.x * fpw + f; li < n_lanes; li += blockDim.x * fpw) {
    const LaneBest x = lanes[li];
    if (x.item != ~0ull && key_less(step, x, best)) { best = x; bi = li; }
  }
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const LaneBest y = sb[threadIdx.x + o];
      if (si[threadIdx.x + o] != 0xffffffffu &&
          (si[threadIdx.x] == 0xffffffffu || key_less(step, y, sb[threadIdx.x]))) {
        sb[threadIdx.x] = y;
        si[threadIdx.x] = si[threadIdx.x + o];
      }
    }
    __syncthreads();
  }
  __shared__ uint32_t win;
  if (threadIdx.x == 0) win = si[0];
  __syncthreads();
  FrameBest* o = out + f;
  if (threadIdx.x == 0) {
    o->t = sb[0].t;
    o->sse = sb[0].sse;
    o->item = sb[0].item;
    o->ord = sb[0].ord;
    o->count = *count;
    o->found = (win == 0xffffffffu) ? 0 : 1;
    if (budget_out && step == 1) {
      // budget = t_min * (1.0 + lambda)   (search.cpp:344)
      const double tmin = __longlong_as_double((long long)sb[0].t);
      const double b = __dmul_rn(tmin, __dadd_rn(1.0, lambda));
      budget_out[f] = (b > 0.0) ? (uint64_t)__double_as_longlong(b) : 0ull;
    }
  }
  if (win != 0xffffffffu)
    for (int i = threadIdx.x; i < kSnapBytes; i += blockDim.x)
      o->snap[i] = snaps[(size_t)win * kSnapBytes + i];
}

// ---- host launchers ------------------------------------------------------------
template <int FPW, int STEP>
static void launch_fpw(const SearchArgs& a, int blocks, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    SCB_CUDA(cudaFuncSetAttribute(k_search<FPW, STEP>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  k_search<FPW, STEP><<<blocks, 256, smem, st>>>(a);
}

int search_blocks_per_sm(int fpw, int step) {
  int nb = 0;
  const size_t smem = 16 * 1024;
#define OCC(F)                                                                               \
  if (fpw == F) {                                                                            \
    if (step == 1)                                                                           \
      SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_search<F, 1>, 256, smem)); \
    else                                                                                     \
      SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_search<F, 2>, 256, smem)); \
  }
  OCC(1) OCC(2) OCC(4) OCC(8) OCC(16) OCC(32)
#undef OCC
  return nb < 1 ? 1 : nb;
}

void search_launch(int fpw, int step, const SearchArgs& a, int blocks, cudaStream_t st) {
  const size_t smem = ((size_t)2 * (a.max_area + 1) + (size_t)(a.cols + 1) * (a.rows + 1) +
                       (size_t)(a.cols + 1) * (std::min(a.n, a.rows) + 1)) *
                      sizeof(int32_t);
  if (smem > 64 * 1024) fail(SC_ERR_SIZE, "CTU grid too large for the area tables");
  switch (fpw * 10 + step) {
    case 11: launch_fpw<1, 1>(a, blocks, smem, st); break;
    case 12: launch_fpw<1, 2>(a, blocks, smem, st); break;
    case 21: launch_fpw<2, 1>(a, blocks, smem, st); break;
    case 22: launch_fpw<2, 2>(a, blocks, smem, st); break;
    case 41: launch_fpw<4, 1>(a, blocks, smem, st); break;
    case 42: launch_fpw<4, 2>(a, blocks, smem, st); break;
    case 81: launch_fpw<8, 1>(a, blocks, smem, st); break;
    case 82: launch_fpw<8, 2>(a, blocks, smem, st); break;
    case 161: launch_fpw<16, 1>(a, blocks, smem, st); break;
    case 162: launch_fpw<16, 2>(a, blocks, smem, st); break;
    case 321: launch_fpw<32, 1>(a, blocks, smem, st); break;
    case 322: launch_fpw<32, 2>(a, blocks, smem, st); break;
    default: fail(SC_ERR_INTERNAL, "bad frames-per-warp");
  }
  SCB_CUDA(cudaGetLastError());
}

void finalize_launch(int step, int fpw, int frames_in_group, uint32_t n_warps,
                     const LaneBest* lanes, const uint8_t* snaps,
                     const unsigned long long* count, double lambda, FrameBest* out,
                     uint64_t* budget_out, cudaStream_t st) {
  k_finalize<<<frames_in_group, 256, 0, st>>>(step, fpw, frames_in_group, n_warps, lanes, snaps,
                                              count, lambda, out, budget_out);
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
