// The warp-uniform walk of one work item — the body of the K4/K5 search
// kernels (search.cu).  Written as a __host__ __device__ function so that
// the test-only host emulator (tests/emu) executes the very same code lane
// by lane on the CPU; the product path only ever runs it on the GPU.
//
// Replaces ColumnSplitGenerator + layout_time/layout_sse + the step-1/step-2
// reductions (search.cpp:77-91, 110-196, 280-289, 375-394).
#pragma once

#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "plan.h"
#include "slicecraft_b200.h"

#ifdef __CUDACC__
#define SCB_HD __host__ __device__ __forceinline__
#else
#define SCB_HD inline
#endif

namespace scb {

#if defined(SCB_STATS) && !defined(__CUDA_ARCH__)
struct WalkStats {
  uint64_t widths, runs_steps, skeletons, levels, leaf_calls, leaves, levels_leafcol, leafr[65];
  uint64_t width_steps, items;
};
inline WalkStats g_stats;
#define SCB_STAT(x) (++g_stats.x)
#elif defined(SCB_COUNT_STEPS) && defined(__CUDA_ARCH__)
#define SCB_STAT(x) (++st.scored)  // diagnostics build: DFS steps in `scored`
#else
#define SCB_STAT(x) ((void)0)
#endif

// ---- portable intrinsics -------------------------------------------------------
#ifdef __CUDA_ARCH__
#define SCB_SYNCWARP() __syncwarp()
#else
#define SCB_SYNCWARP() ((void)0)
#endif
SCB_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
SCB_HD double dadd_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;  // no contraction possible: a plain add
  return r;
#endif
}
SCB_HD int imin(int a, int b) { return a < b ? a : b; }
SCB_HD int imax(int a, int b) { return a > b ? a : b; }
SCB_HD uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// Time key: the exact per-frame RANK of a (clamped) time among all rectangle
// times of that frame.  Ranks are an injective, order-preserving image of the
// doubles, so max / < / <= on keys equal max / < / <= on the times
// (DESIGN.md §Search); 32 bits instead of 64 halve the table traffic.
typedef uint32_t tkey;
constexpr tkey kKeyInf = 0xffffffffu;
SCB_HD tkey kmax(tkey a, tkey b) { return a > b ? a : b; }
SCB_HD tkey kmin(tkey a, tkey b) { return a < b ? a : b; }
SCB_HD tkey umin3(tkey a, tkey b, tkey c) {
  const tkey m = a < b ? a : b;
  return m < c ? m : c;
}

// Warp-uniform DFS arrays of the exhaustive walk, one copy per warp in shared
// memory on the GPU (int offsets; curH bytes at kUniH).
constexpr int kUniW = 0, kUniR = 16, kUniX0 = 32, kUniWL = 49, kUniWH = 66, kUniRL = 83,
              kUniRH = 99, kUniSL = 115, kUniH = 131, kUniSMN = 147, kUniSMX = 164,
              kUniCR1 = 184, kUniCR2 = 200, kUniInts = 216;  // 864 B

// one 16-byte record of the heights DFS (a single 128-bit local access)
struct alignas(16) Lvl {
  int32_t a, b, c, d;
};

SCB_HD int xw_of(int cols, int x0, int w) { return x0 * cols - (x0 * (x0 - 1)) / 2 + (w - 1); }
SCB_HD int yh_of(int rows, int y0, int h) { return y0 * rows - (y0 * (y0 - 1)) / 2 + (h - 1); }

constexpr int kMaxLevels = SC_MAX_SLICES;
constexpr int kBigArea = 1 << 20;  // "no slice yet" sentinel for amin
constexpr int kSnap = 96;          // snapshot bytes: W[16] R[16] H[64]

// Table access.  On the GPU the small tables are static shared arrays and the
// area tables sit at the start of dynamic shared memory, bmax/aneed
// interleaved, so every table address is a compile-time constant plus the
// index (no base pointers to keep live or rematerialise in the register-bound
// walk).  The host build (tests/emu) reads the same tables through WalkEnv.
constexpr int kTabDim = 256;  // grid cols and rows are <= 255 (api.cu check_cfg)
#ifdef __CUDACC__
__shared__ uint64_t g_magic[kTabDim];
__shared__ int32_t g_rq[kTabDim];
extern __shared__ int32_t g_dyn[];  // [2A] bmax|aneed interleaved, mstar, ilo
#endif
#ifdef __CUDA_ARCH__
#define SCB_BMAX(a) (g_dyn[2 * (a)])
#define SCB_ANEED(a) (g_dyn[2 * (a) + 1])
#define SCB_MSTAR(i) (g_dyn[e.mstar_off + (i)])
#define SCB_ILO(i) (g_dyn[e.ilo_off + (i)])
#define SCB_MAGIC(w) (g_magic[w])
#define SCB_RQ(r) (g_rq[r])
#else
#define SCB_BMAX(a) (e.bmax[a])
#define SCB_ANEED(a) (e.aneed[a])
#define SCB_MSTAR(i) (e.mstar[i])
#define SCB_ILO(i) (e.ilo[i])
#define SCB_MAGIC(w) (e.magic[w])
#define SCB_RQ(r) (e.rq[r])
#endif

// yh(y, 1) = y*rows - y*(y-1)/2, the first rectangle starting at row y:
// computed (4 ALU operations) rather than loaded, off the shared-memory
// latency chain of the walk's address computations
#define SCB_YBASE(y) ((y) * e.rows - (((y) * ((y) - 1)) >> 1))

// Read-only walk environment (tables live in shared memory on the GPU).
struct WalkEnv {
  int cols, rows, n, nyh, max_area, coverage, patho, rstride;
  int prune;  // exact branch-and-bound (SC_MODE_PRUNED): skip subtrees that
              // cannot strictly improve this lane's best (step 1) or that
              // exceed the budget (step 2); ordinals are then not dense
  const int32_t* bmax;    // [max_area + 1]
  const int32_t* aneed;   // [max_area + 1]
  const int32_t* mstar;   // [(cols+1) * (rows+1)]
  const int32_t* ilo;     // [(cols+1) * rstride]: lower end of window I(w, r)
  const uint64_t* magic;  // [cols+1]: division by w (div_magic)
  const int32_t* rq;      // [rows+1]: rows / r (no integer division in the runs DFS)
  int mstar_off, ilo_off;  // GPU: offsets of mstar / ilo in dynamic shared memory
  // GPU, exhaustive walks: this warp's heights-DFS level records in shared
  // memory (LS = lvl[0, lvl_cap), D = lvl[lvl_cap, 2 lvl_cap)).  The walk is
  // warp-uniform, so one copy per warp replaces 32 per-thread copies in local
  // memory (which crowded L1); only the per-frame Pin stays per lane.
  Lvl* lvl;
  tkey* pin;  // this lane's Pin slots: pin[l * 32]
  int* uni;   // this warp's uniform DFS arrays (kUni* offsets)
  int lvl_cap;
  // pruned mode: split_g warps share each work item; the subtrees below
  // level split_depth of the heights DFS (or a whole skeleton, if it has
  // fewer levels) are dealt to them by a hash of their identity
  int split_g, split_depth;
  const tkey* rt;         // [NR][FPW] time key of every rectangle
  const tkey* rts;        // [NR][FPW] split table: at rect(x0,w,y0,h) with y0+h < rows,
                          // max(time(y0,h), time(y0+h, rows-y0-h)) -- a run plus the
                          // forced rest of its column in one load
  const double* rs;       // [NR][FPW] SSE of every rectangle (step 2)
  // pruned mode only: per-frame lower bounds on a column's slowest slice,
  // lbr[(xw*rstride + r)*FPW + f] for exactly r runs and lbm[...] for any
  // r' <= r (prefix minimum); inc[f] is the shared step-1 incumbent, packed
  // (time key << 32 | work item) so that ties are ordered by item.
  const tkey* lbr;
  const tkey* lbm;
  uint64_t* inc;
  // incumbent frozen after the seed phase (or nullptr): its candidate precedes
  // every item still to walk, so a tie with it can never win
  const uint64_t* seed_inc;
  // pruned step 2: shared per-frame SSE incumbent (f64 bits; SSEs are >= 0,
  // so the bit patterns order like the values), or nullptr
  uint64_t* sse_inc;
};

// One lane's running first-in-order best and its candidate snapshot.
struct LaneState {
  tkey best_t;
  uint64_t best_item, best_ord;
  double best_sse;
  int64_t budget;   // step 2: largest key whose time is <= t_min * (1 + lambda), -1: none
  uint64_t count;   // candidates enumerated (uniform over the warp)
  uint64_t scored;  // candidates this lane actually scored
  uint64_t inc;     // last seen shared incumbent (pruned step 1), packed as EnvWalk::inc
  double sbound;    // pruned step 2: min(own best SSE, last seen shared SSE incumbent)
  tkey bcmp;        // exhaustive step 1: a candidate wins iff t < bcmp (see walk_item)
  bool tie;         // pruned, shared items: this item part may precede the best's layout
  uint8_t* snap;
};

// Shared incumbent (t << 32 | item): a candidate with time t exists in work
// item `item` of this frame, so no slower candidate can win, and an equal one
// only from an item not after it (positions inside one item are unknown).
// A subtree of item X with lower bound P can still win iff (P << 32 | X) <= inc.
SCB_HD uint64_t inc_pack(tkey t, uint64_t item) { return ((uint64_t)t << 32) | (uint32_t)item; }
SCB_HD uint64_t incumbent_load(uint64_t* p) {
#ifdef __CUDA_ARCH__
  return *(volatile uint64_t*)p;
#else
  return *p;
#endif
}
SCB_HD double sse_incumbent(const uint64_t* p) {
  uint64_t b = incumbent_load(const_cast<uint64_t*>(p));
  double d;
  memcpy(&d, &b, 8);
  return d;
}
SCB_HD void incumbent_offer(uint64_t* p, uint64_t v) {
#ifdef __CUDA_ARCH__
  atomicMin((unsigned long long*)p, (unsigned long long)v);
#else
  if (v < *p) *p = v;
#endif
}

// Lower bound on the slowest slice of a column (x0, w) cut into exactly r
// runs, for every r <= rmax: min over all compositions (area constraint
// relaxed) of the max run time, by a DP over rows.  lbr/lbm are written at
// [r * stride] (lbm: prefix minimum over r).  Keys are ranks, so max / min
// are exact.
SCB_HD void column_bounds(const tkey* rt, int fpw, int f, int rows, int base, int rmax,
                          tkey* lbr, tkey* lbm, size_t stride) {
  tkey prev[256], cur[256];
  const tkey INF = kKeyInf;
  for (int y = 0; y <= rows; ++y) prev[y] = y == 0 ? 0 : INF;
  tkey run_min = INF;
  lbr[0] = INF;
  lbm[0] = INF;
  for (int r = 1; r <= rmax; ++r) {
    for (int y = 0; y <= rows; ++y) {
      tkey best = INF;
      for (int y0 = r - 1; y0 < y; ++y0) {
        if (prev[y0] == INF) continue;
        const tkey v = rt[(size_t)(base + yh_of(rows, y0, y - y0)) * fpw + f];
        const tkey m = prev[y0] > v ? prev[y0] : v;
        if (m < best) best = m;
      }
      cur[y] = best;
    }
    lbr[(size_t)r * stride] = cur[rows];
    run_min = cur[rows] < run_min ? cur[rows] : run_min;
    lbm[(size_t)r * stride] = run_min;
    for (int y = 0; y <= rows; ++y) prev[y] = cur[y];
  }
}

// Area thresholds of a partial candidate: a further slice of area x keeps it
// admissible iff T2 <= x <= T1 (and x <= bmax[x]); T1 = bmax[amin] (+inf
// before the first slice), T2 = aneed[amax].
struct Thr {
  int t1, t2;
};

// floor(x / w) for 0 <= x <= 2^20, 1 <= w <= 2^11 with the 33-bit magic
// floor(2^32/w)+1: one wide multiply, exact because x * w < 2^32.
SCB_HD int div_w(int x, uint64_t magic) { return (int)(((uint64_t)(uint32_t)x * magic) >> 32); }
SCB_HD uint64_t div_magic(int w) { return 0x100000000ull / (uint64_t)w + 1ull; }

// Admissible heights of a run of width w with rl rows left in its column and
// runs_left runs (this one included).  runs_left == 2: the next run is forced
// to rl - h, both areas must pass -> symmetric [m, rl - m] with
// m = max(ceil(T2/w), rl - floor(T1/w), mstar[w][rl]).  Otherwise the
// interval includes a look-ahead: rl - h rows must still split into
// runs_left - 1 runs of admissible height (thresholds only tighten).
SCB_HD void height_interval(const WalkEnv& e, Thr t, int w, int rl, int runs_left, int& lo,
                            int& hi) {
  const uint64_t mg = SCB_MAGIC(w);
  const int hmin_a = imax(1, div_w(t.t2 + w - 1, mg));
  const int hmax_a = t.t1 < 0 ? 0 : div_w(t.t1, mg);
  if (runs_left == 2) {
    int m = imax(hmin_a, rl - hmax_a);
    m = imax(m, SCB_MSTAR(w * (e.rows + 1) + rl));
    lo = m;
    hi = rl - m;
    return;
  }
  const int k = runs_left - 1;
  lo = imax(hmin_a, rl - k * hmax_a);
  hi = imin(rl - k * hmin_a, hmax_a);
}

// Walk work item `item` (prefix wi) for frame slot f and leaf slot `slot`
// (J = 32 / FPW lanes share a frame and split the innermost height loop).
// Owner (0..g-1) of a subtree of the pruned walk: a hash of the skeleton and
// of the heights fixed above the split level.  It depends only on the
// subtree's identity, never on what a warp pruned before reaching it, so every
// subtree has exactly one owner among the warps sharing its work item.
SCB_HD uint32_t split_owner(uint64_t key, int g) {
  key ^= key >> 31;
  key *= 0x9e3779b97f4a7c15ull;
  key ^= key >> 29;
  return (uint32_t)((key >> 32) % (uint64_t)g);
}

template <int FPW, int STEP, bool PRUNE>
SCB_HD void walk_item(const WalkEnv& e, uint64_t item, const WorkItem& wi, int f, int slot,
                      LaneState& st, int split_r = 0) {
  constexpr int J = 32 / FPW;
  const int rows = e.rows, cols = e.cols, nyh = e.nyh;
  const tkey* rt = e.rt;
  const double* rs = e.rs;
  const int c = wi.c, d = wi.d;
  uint64_t ord = 0;  // ordinal of the next candidate inside this item
  // Exhaustive step 1 may take items in any order (api.cu schedules them by
  // measured cost): a candidate beats the lane's best iff its time is lower,
  // or equal with an earlier item; inside an item candidates come in order,
  // so after the first update the comparison is strict again.
  if (STEP == 1 && !PRUNE)
    st.bcmp = (st.best_t != kKeyInf && item < st.best_item) ? st.best_t + 1 : st.best_t;
  // Pruned mode with shared items: another part of this same item may have
  // produced the lane's best, and this part's subtrees can precede it, so ties
  // with the best are decided by the layouts (enumeration order).
  if (PRUNE) st.tie = e.split_g > 1 && item == st.best_item;

  // warp-uniform DFS state (identical in every lane of the warp)
  int W_[SC_MAX_COLS], R_[SC_MAX_COLS], X0_[SC_MAX_COLS + 1], RS0[SC_MAX_COLS];
  int WL_[SC_MAX_COLS + 1], WH_[SC_MAX_COLS + 1], RL_[SC_MAX_COLS], RH_[SC_MAX_COLS],
      SL_[SC_MAX_COLS], SMN_[SC_MAX_COLS + 1], SMX_[SC_MAX_COLS + 1], CR1_[SC_MAX_COLS],
      CR2_[SC_MAX_COLS];
  uint8_t curH_[SC_MAX_SLICES];
  // exhaustive walks on the GPU: these warp-uniform DFS arrays live once per
  // warp in shared memory (WalkEnv::uni, layout kUni*); pruned walks and the
  // host emulator keep them per lane
#ifdef __CUDA_ARCH__
  constexpr bool kUniform = !PRUNE;
#else
  constexpr bool kUniform = false;
#endif
  int* const W = kUniform ? e.uni + kUniW : W_;
  int* const R = kUniform ? e.uni + kUniR : R_;
  int* const X0 = kUniform ? e.uni + kUniX0 : X0_;
  int* const WL = kUniform ? e.uni + kUniWL : WL_;
  int* const WH = kUniform ? e.uni + kUniWH : WH_;
  int* const RL = kUniform ? e.uni + kUniRL : RL_;
  int* const RH = kUniform ? e.uni + kUniRH : RH_;
  int* const SL = kUniform ? e.uni + kUniSL : SL_;
  uint8_t* const curH = kUniform ? reinterpret_cast<uint8_t*>(e.uni + kUniH) : curH_;
  int* const SMN = kUniform ? e.uni + kUniSMN : SMN_;
  int* const SMX = kUniform ? e.uni + kUniSMX : SMX_;
  int* const CR1 = kUniform ? e.uni + kUniCR1 : CR1_;  // per column: run counts whose
  int* const CR2 = kUniform ? e.uni + kUniCR2 : CR2_;  // window meets the widths hull
  // pruned walks: heights-DFS state per level in local arrays
  uint8_t Lcol[kMaxLevels], Lrun[kMaxLevels], Ly0[kMaxLevels], Lh[kMaxLevels], Lhi[kMaxLevels];
  int32_t Amin[kMaxLevels], Amax[kMaxLevels], Lbase[kMaxLevels];
  tkey Pin[kMaxLevels];
  double Sp[STEP == 2 && PRUNE ? kMaxLevels : 1];  // pruned step 2: SSE prefix per level
  // heights-DFS levels: LS static (w | runs left << 8 | run << 16 | column << 24,
  // column rectangle base, suffix fillability bounds), D the spilled state of
  // the levels above the current one (h | hhi << 8 | y0 << 16, -, Amin, Amax; Pin
  // per lane in PIN)
#ifdef __CUDA_ARCH__
  // exhaustive walks: the level records are warp-uniform, one copy per warp
  // in shared memory; the fixed-slice maximum Pin of a level depends on the
  // lane's frame, so it has its own lane-interleaved array (PIN[l * 32])
  Lvl* const LS = e.lvl;
  Lvl* const D = e.lvl + e.lvl_cap;
  tkey* const PIN = e.pin;
  constexpr int PS = 32;
#else
  Lvl LSa[kMaxLevels], Da[kMaxLevels];
  tkey PINa[kMaxLevels];
  Lvl* const LS = LSa;
  Lvl* const D = Da;
  tkey* const PIN = PINa;
  constexpr int PS = 1;
#endif

  auto thresholds = [&](int amin, int amax, int win_lo, int win_hi) -> Thr {
    Thr t;
    t.t1 = amin >= kBigArea ? kBigArea : SCB_BMAX(amin);
    t.t2 = SCB_ANEED(amax);
    t.t2 = imax(t.t2, win_lo);
    t.t1 = imin(t.t1, win_hi);
    return t;
  };
  auto rt_at = [&](int x0, int w, int y0, int h) -> tkey {
    return rt[(size_t)(xw_of(cols, x0, w) * nyh + yh_of(rows, y0, h)) * FPW + f];
  };
  // Every multi-run column from `from` on can still be filled with runs of
  // admissible height (necessary condition; prunes dead subtrees early).
  auto columns_feasible = [&](int from, Thr t) -> bool {
    for (int i = from; i < c; ++i) {
      if (R[i] < 2) continue;
      const int w = W[i];
      const uint64_t mg = SCB_MAGIC(w);
      const int hmin_a = imax(1, div_w(t.t2 + w - 1, mg));
      const int hmax_a = t.t1 < 0 ? 0 : div_w(t.t1, mg);
      if (R[i] * hmin_a > rows || R[i] * hmax_a < rows) return false;
    }
    return true;
  };
  // snapshot of the current candidate; run `lr` takes height lh and the
  // forced run lr+1 the rest of its column (lr < 0: no leaf loop).
  // (rolled loops: constant indices would pull W and R into 32 registers)
  auto take_snapshot = [&](int lr, int lh, int lrest) {
#pragma unroll 1
    for (int i = 0; i < c; ++i) {
      st.snap[i] = (uint8_t)W[i];
      st.snap[SC_MAX_COLS + i] = (uint8_t)R[i];
    }
#pragma unroll 1
    for (int i = c; i < SC_MAX_COLS; ++i) {
      st.snap[i] = 0;
      st.snap[SC_MAX_COLS + i] = 0;
    }
#pragma unroll 1
    for (int i = 0; i < e.n; ++i) {
      uint8_t v = curH[i];
      if (i == lr) v = (uint8_t)lh;
      if (i == lr + 1 && lr >= 0) v = (uint8_t)lrest;
      st.snap[2 * SC_MAX_COLS + i] = v;
    }
  };
  // step-2 objective: slice SSEs summed in slice order (search.cpp:85-91)
  auto layout_sse = [&](int lr, int lh, int lrest) -> double {
    double tot = 0.0;
    int run = 0;
    for (int i = 0; i < c; ++i) {
      int y = 0;
      const int base = xw_of(cols, X0[i], W[i]) * nyh;
      for (int j = 0; j < R[i]; ++j, ++run) {
        int hh = curH[run];
        if (run == lr) hh = lh;
        else if (lr >= 0 && run == lr + 1) hh = lrest;
        tot = dadd_rn(tot, rs[(size_t)(base + yh_of(rows, y, hh)) * FPW + f]);
        y += hh;
      }
    }
    return tot;
  };
  // can a subtree whose fixed slices already reach time P still win?
  const uint64_t seed_inc = (STEP == 1 && PRUNE && e.seed_inc) ? e.seed_inc[f] : ~0ull;
  const uint64_t item32 = (uint32_t)item;
  auto viable = [&](tkey P) -> bool {
    return !PRUNE ||
           (STEP == 1 ? ((P < st.best_t || (st.tie && P == st.best_t)) &&
                         (((uint64_t)P << 32) | item32) <= st.inc &&
                         (((uint64_t)P << 32) | item32) < seed_inc)
                      : ((int64_t)P <= st.budget));
  };
  // does the current candidate precede the lane's best in enumeration order?
  // (same item: compare the layouts lexicographically, as k_finalize does)
  auto precedes_best = [&](int lr, int lh, int lrest) -> bool {
    for (int i = 0; i < SC_MAX_COLS; ++i) {
      const int v = i < c ? W[i] : 0;
      if (v != st.snap[i]) return v < st.snap[i];
    }
    for (int i = 0; i < SC_MAX_COLS; ++i) {
      const int v = i < c ? R[i] : 0;
      if (v != st.snap[SC_MAX_COLS + i]) return v < st.snap[SC_MAX_COLS + i];
    }
    for (int i = 0; i < e.n; ++i) {
      int v = curH[i];
      if (i == lr) v = lh;
      if (i == lr + 1 && lr >= 0) v = lrest;
      if (v != st.snap[2 * SC_MAX_COLS + i]) return v < st.snap[2 * SC_MAX_COLS + i];
    }
    return false;
  };
  if (STEP == 1 && PRUNE) st.inc = incumbent_load(e.inc + f);
  // lower bound of column (x0, w) with r runs (exact r) / any r' <= r
  auto lb_r = [&](int x0, int w, int r) -> tkey {
    return e.lbr[((size_t)xw_of(cols, x0, w) * e.rstride + r) * FPW + f];
  };
  auto lb_m = [&](int x0, int w, int r) -> tkey {
    return e.lbm[((size_t)xw_of(cols, x0, w) * e.rstride + r) * FPW + f];
  };
  // score one candidate (strict comparisons keep the first in order)
  // sse_pre >= 0: the candidate's SSE, already folded in slice order by the
  // caller (pruned step 2); otherwise layout_sse computes it
  auto score = [&](tkey t, uint64_t o, int lr, int lh, int lrest, double sse_pre = -1.0) {
    if (PRUNE) ++st.scored;
    if (STEP == 1) {
      if (t < (PRUNE ? st.best_t : st.bcmp) ||
          (PRUNE && st.tie && t == st.best_t && precedes_best(lr, lh, lrest))) {
        st.best_t = t;
        st.bcmp = t;
        st.best_item = item;
        st.best_ord = o;
        take_snapshot(lr, lh, lrest);
        if (PRUNE) {
          st.tie = false;  // the rest of this part comes after it
          incumbent_offer(e.inc + f, inc_pack(t, item));
        }
      }
    } else if ((int64_t)t <= st.budget) {
      const double s = sse_pre >= 0.0 ? sse_pre : layout_sse(lr, lh, lrest);
      if (s < st.best_sse ||
          (s == st.best_sse && (t < st.best_t || (PRUNE && st.tie && t == st.best_t &&
                                                  precedes_best(lr, lh, lrest))))) {
        st.best_sse = s;
        st.best_t = t;
        st.best_item = item;
        st.best_ord = o;
        take_snapshot(lr, lh, lrest);
        if (PRUNE) {
          st.tie = false;
          st.sbound = s < st.sbound ? s : st.sbound;
          if (e.sse_inc) {
            uint64_t b;
            memcpy(&b, &s, 8);
            incumbent_offer(e.sse_inc + f, b);
          }
        }
      }
    }
  };

  // ---- widths DFS over positions d..c-1 (lex, search.cpp:133-143).  A width
  //      w can only host windows a in the hull [ilo(w, r_max), w*rows] of its
  //      column windows (r <= n-c+1): prefixes whose hulls do not intersect
  //      cannot complete and are skipped.
  const int rmax_c = imin(e.n - c + 1, rows);
  tkey PW[SC_MAX_COLS + 1];  // pruned mode: max of the columns' lower bounds
  X0[0] = 0;
  WL[0] = 1;
  WH[0] = e.max_area;
  PW[0] = 0;
  bool ok = (e.n >= c) && (e.n <= c * rows);
  for (int i = 0; i < d && ok; ++i) {
    W[i] = wi.w[i];
    X0[i + 1] = X0[i] + W[i];
    WL[i + 1] = imax(WL[i], SCB_ILO(W[i] * e.rstride + rmax_c));
    WH[i + 1] = imin(WH[i], W[i] * rows);
    ok = WL[i + 1] <= WH[i + 1];
    if (PRUNE) {
      PW[i + 1] = kmax(PW[i], lb_m(X0[i], W[i], rmax_c));
      ok = ok && viable(PW[i + 1]);
    }
  }
  int pos = d;
  const bool fixed_widths = d == c;
  if (ok && !fixed_widths) W[pos] = 0;
  while (ok) {
    if (!fixed_widths) {
      bool got = false;
      while (true) {
        // uniform arrays: no lane may still read the previous skeleton's
        // state (a best update's snapshot) when they change
        if (kUniform) SCB_SYNCWARP();
        const int maxw = cols - X0[pos] - (c - pos - 1);
        int wv;
        if (e.coverage && pos == c - 1) wv = (W[pos] == 0) ? maxw : maxw + 1;
        else wv = W[pos] + 1;
        if (wv > maxw) {
          if (pos == d) break;
          --pos;
          continue;
        }
        W[pos] = wv;
        SCB_STAT(width_steps);
        const int nL = imax(WL[pos], SCB_ILO(wv * e.rstride + rmax_c));
        const int nH = imin(WH[pos], wv * rows);
        if (nL > nH) continue;
        if (PRUNE) {
          PW[pos + 1] = kmax(PW[pos], lb_m(X0[pos], wv, rmax_c));
          if (!viable(PW[pos + 1])) continue;
        }
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
    SCB_STAT(widths);
    if (STEP == 1 && PRUNE) st.inc = incumbent_load(e.inc + f);
    // ---- runs DFS (lex, search.cpp:145-161).  The skeleton (widths, runs)
    //      has an admissible completion iff the column windows
    //      I(w, r) = [aneed[w*ceil(rows/r)], w*floor(rows/r)] intersect; I
    //      slides down as r grows, so the feasible r of a position form one
    //      contiguous range.
    //      Suffix run-count bounds: column j can only take r runs whose
    //      window meets the widths hull [WL[c], WH[c]] (r in [r1_j, r2_j],
    //      the window only shrinks from there), so position rp only tries r
    //      with SL - r in [SMN[rp+1], SMX[rp+1]] (sums of r1 / r2 over the
    //      columns after it); a width vector whose sums miss n has no
    //      skeleton.  Skipped r lead to no skeleton: the walk is unchanged.
    bool dead = false;
    SMN[c] = 0;
    SMX[c] = 0;
#pragma unroll 1
    for (int j = c - 1; j >= 0 && !dead; --j) {
      const int w = W[j];
      int r1 = 0, r2 = 0;
#pragma unroll 1
      for (int r = 1; r <= rmax_c; ++r) {
        if (w * SCB_RQ(r) < WL[c]) break;  // every larger r is lower still
        if (SCB_ILO(w * e.rstride + r) <= WH[c]) {
          if (!r1) r1 = r;
          r2 = r;
        }
      }
      dead = r1 == 0;
      CR1[j] = r1;
      CR2[j] = r2;
      SMN[j] = SMN[j + 1] + r1;
      SMX[j] = SMX[j + 1] + r2;
    }
    dead = dead || SMN[0] > e.n || SMX[0] < e.n;
    tkey PR[SC_MAX_COLS + 1];  // pruned mode: widths bound, tightened per exact r
    PR[0] = PRUNE ? PW[c] : 0;
    int rp = 0;
    RL[0] = 1;
    RH[0] = e.max_area;
    SL[0] = e.n;
    R[0] = dead ? rows : imax(1, e.n - (c - 1) * rows) - 1;  // dead: the loop ends at once
    while (true) {
      if (kUniform) SCB_SYNCWARP();
      SCB_STAT(runs_steps);
      const int rhi = imin(CR2[rp], SL[rp] - SMN[rp + 1]);
      const int w = W[rp];
      int r = imax(imax(R[rp] + 1, CR1[rp]), SL[rp] - SMX[rp + 1]), lo = 0, hi = 0;
      bool found = false;
      for (; r <= rhi; ++r) {
        lo = SCB_ILO(w * e.rstride + r);
        hi = w * SCB_RQ(r);
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
      const int nL = imax(RL[rp], lo), nH = imin(RH[rp], hi);
      if (nL > nH) continue;
      if (PRUNE) {
        PR[rp + 1] = kmax(PR[rp], lb_r(X0[rp], W[rp], r));
        if (!viable(PR[rp + 1])) continue;
      }
      if (rp < c - 1) {
        SL[rp + 1] = SL[rp] - r;
        RL[rp + 1] = nL;
        RH[rp + 1] = nH;
        ++rp;
        R[rp] = imax(1, SL[rp] - (c - 1 - rp) * rows) - 1;
        continue;
      }
      if constexpr (PRUNE) {
        // pruned walks diverge per frame: the DFS state stays in per-level
        // local arrays, which keeps the lanes of a warp reconverging at every
        // step of the loop (measured 1.6x fewer warp instructions than the
        // register-resident walk below on cfg5)
        // ---- one live skeleton (c, widths, runs); every area lies in
        //      [win_lo, bmax[nH]] for a window a in [nL, nH]
        const int win_lo = nL, win_hi = SCB_BMAX(nH);
        SCB_STAT(skeletons);
        if (STEP == 1 && PRUNE) st.inc = incumbent_load(e.inc + f);
        int amin = kBigArea, amax = 0;
        int run = 0, nl = 0;
        for (int i = 0; i < c; ++i) {
          RS0[i] = run;
          if (R[i] == 1) {  // one-run columns are fixed by the skeleton
            const int ar = W[i] * rows;
            amin = imin(amin, ar);
            amax = imax(amax, ar);
            curH[run] = (uint8_t)rows;
          } else {
            const int base = xw_of(cols, X0[i], W[i]) * nyh;
            for (int j = 0; j < R[i] - 1; ++j, ++nl) {
              Lcol[nl] = (uint8_t)i;
              Lrun[nl] = (uint8_t)j;
              Lbase[nl] = base;
            }
          }
          run += R[i];
        }
        tkey P = 0;
        for (int i = 0; i < c; ++i)
          if (R[i] == 1) P = kmax(P, rt_at(X0[i], W[i], 0, rows));
        // pruned mode, shared items: identity of this skeleton
        const bool split = PRUNE && e.split_g > 1;
        uint64_t skey = 0;
        int lsplit = -1;  // heights level whose values are dealt to the warps
        if (split) {
          skey = (uint64_t)c;
          for (int i = 0; i < c; ++i) skey = skey * 0x100000001b3ull ^ (uint64_t)(W[i] | (R[i] << 8));
          if (nl >= 2) lsplit = imin(e.split_depth, nl - 2);
          else if (split_owner(skey, e.split_g) != (uint32_t)split_r) {
            ord += 1;
            continue;
          }
        }
        if (nl == 0) {  // the skeleton is a single candidate
          if (slot == 0 && viable(P)) score(P, ord, -1, 0, 0);
          ord += 1;
          continue;
        }
        // pruned mode: every column's bound (PR) floors the whole subtree
        const tkey colfloor = PRUNE ? kmax(P, PR[c]) : P;
        if (!viable(colfloor)) continue;
        // step 2: SSE prefix in slice order (the left fold of layout_sse,
        // search.cpp:85-91).  Slice SSEs are >= 0, so a prefix above the
        // lane's best SSE already loses (strictly): the subtree is skipped.
        // Sp[l] = the fold of every slice before level l's run; one-run
        // columns enter at their positions.
        auto sse_at = [&](int lb, int y0, int h) -> double {
          return rs[(size_t)(lb + SCB_YBASE(y0) + h - 1) * FPW + f];
        };
        auto fold_one_run = [&](double acc, int from, int to) -> double {
          for (int i = from; i < to; ++i)
            if (R[i] == 1)
              acc = dadd_rn(acc, rs[(size_t)(xw_of(cols, X0[i], W[i]) * nyh +
                                             yh_of(rows, 0, rows)) * FPW + f]);
          return acc;
        };
        if (STEP == 2) {
          // bound: the lane's own best, or a better one another warp found
          if (e.sse_inc) {
            const double sh = sse_incumbent(e.sse_inc + f);
            st.sbound = sh < st.best_sse ? sh : st.best_sse;
          } else {
            st.sbound = st.best_sse;
          }
          Sp[0] = fold_one_run(0.0, 0, Lcol[0]);
          if (Sp[0] > st.sbound) continue;
        }
        // ---- heights DFS over the multi-run columns (search.cpp:163-190)
        int l = 0;
        const bool leaf_now = (nl == 1);
        if (!leaf_now) {
          const int i = Lcol[0];
          int lo0, hi0;
          height_interval(e, thresholds(amin, amax, win_lo, win_hi), W[i], rows, R[i], lo0, hi0);
          Lh[0] = (uint8_t)(lo0 - 1);
          Lhi[0] = (uint8_t)imax(hi0, 0);
          Pin[0] = P;
          Amin[0] = amin;
          Amax[0] = amax;
          Ly0[0] = 0;
        }
        while (true) {
          int lv;  // level whose state feeds the leaf loop
          tkey Pl;
          int amin_l, amax_l, y0l;
          double Sl = 0.0;  // step 2: SSE fold before the leaf run
          if (leaf_now) {
            lv = 0;
            Pl = P;
            amin_l = amin;
            amax_l = amax;
            y0l = 0;
            if (STEP == 2) Sl = Sp[0];
          } else {
            // advance level l to its next admissible height
            SCB_STAT(levels);
            const int i = Lcol[l], j = Lrun[l];
  #if defined(SCB_STATS) && !defined(__CUDA_ARCH__)
            if (i == Lcol[nl - 1]) ++g_stats.levels_leafcol;
  #endif
            const int w = W[i], y0 = Ly0[l];
            const int rows_left = rows - y0;
            const bool forced = (R[i] - j) == 2;
            int h = Lh[l] + 1;
            const int hhi = Lhi[l];
            if (e.patho && !forced)
              while (h <= hhi && !(w * h <= SCB_BMAX(w * h))) ++h;
            if (h > hhi) {
              if (l == 0) break;
              --l;
              continue;
            }
            Lh[l] = (uint8_t)h;
            if (split && l == lsplit) {  // deal this subtree to one warp of the item
              uint64_t k = skey;
              for (int q = 0; q <= l; ++q) k = k * 0x100000001b3ull ^ (uint64_t)(Lh[q] + 1);
              if (split_owner(k, e.split_g) != (uint32_t)split_r) continue;
            }
            const int a1 = w * h;
            int na = imin(Amin[l], a1), nx = imax(Amax[l], a1);
            const int ridx = RS0[i] + j;
            curH[ridx] = (uint8_t)h;
            const int lb = Lbase[l];
            const size_t ri = (size_t)(lb + SCB_YBASE(y0) + h - 1) * FPW + f;
            tkey Pn;
            if (forced) {
              const int a2 = w * (rows_left - h);
              na = imin(na, a2);
              nx = imax(nx, a2);
              curH[ridx + 1] = (uint8_t)(rows_left - h);
              Pn = kmax(Pin[l], e.rts[ri]);
            } else {
              Pn = kmax(Pin[l], rt[ri]);
            }
            if (!viable(PRUNE ? kmax(Pn, colfloor) : Pn)) continue;
            const int nxt = l + 1;
            const bool new_col = Lrun[nxt] == 0;
            const int y0n = new_col ? 0 : y0 + h;
            double Sn = 0.0;
            if (STEP == 2) {
              Sn = dadd_rn(Sp[l], sse_at(lb, y0, h));
              if (forced) {
                Sn = dadd_rn(Sn, sse_at(lb, y0 + h, rows_left - h));
                Sn = fold_one_run(Sn, i + 1, Lcol[nxt]);
              }
              if (Sn > st.sbound) continue;
            }
            const Thr tn = thresholds(na, nx, win_lo, win_hi);
            if (new_col && !columns_feasible(Lcol[nxt], tn)) continue;
            if (nxt < nl - 1) {
              const int i2 = Lcol[nxt];
              int lo2, hi2;
              height_interval(e, tn, W[i2], rows - y0n, R[i2] - Lrun[nxt], lo2, hi2);
              if (lo2 > hi2) continue;
              l = nxt;
              Lh[l] = (uint8_t)(lo2 - 1);
              Lhi[l] = (uint8_t)hi2;
              Pin[l] = Pn;
              if (STEP == 2) Sp[l] = Sn;
              Amin[l] = na;
              Amax[l] = nx;
              Ly0[l] = (uint8_t)y0n;
              continue;
            }
            lv = nxt;
            Pl = Pn;
            amin_l = na;
            amax_l = nx;
            y0l = y0n;
            Sl = Sn;
          }
          // ---- leaf loop: run Lrun[lv] of column Lcol[lv] takes every
          //      admissible height; the column's last run is forced.
          {
            const int i = Lcol[lv];
            const int w = W[i];
            const int rows_left = rows - y0l;
            int lo, hi;
            height_interval(e, thresholds(amin_l, amax_l, win_lo, win_hi), w, rows_left, 2, lo, hi);
            const int lr = RS0[i] + Lrun[lv];
            const int xwb = Lbase[lv];
            SCB_STAT(leaf_calls);
  #if defined(SCB_STATS) && !defined(__CUDA_ARCH__)
            ++g_stats.leafr[R[i]];
  #endif
            if (lo + slot <= hi && viable(PRUNE ? kmax(Pl, colfloor) : Pl) &&
                !(STEP == 2 && Sl > st.sbound)) {
              // the split table holds max(run h, forced rest) at the run's own
              // rectangle index, which advances by +1 per h; lanes step h by J.
              int h = lo + slot;
              const tkey* p = e.rts + (size_t)(xwb + SCB_YBASE(y0l) + h - 1) * FPW + f;
              tkey v = *p;
              while (true) {
                const int hn = h + J;
                const bool more = hn <= hi;
                const tkey vn = more ? p[J * FPW] : 0;  // prefetch the next height
                double sc = -1.0;
                if (STEP == 2 && (int64_t)kmax(Pl, v) <= st.budget) {
                  // the candidate's SSE: the prefix, the leaf run, its forced
                  // rest, then the one-run columns after the leaf column
                  sc = dadd_rn(dadd_rn(Sl, sse_at(xwb, y0l, h)), sse_at(xwb, y0l + h, rows_left - h));
                  sc = fold_one_run(sc, i + 1, c);
                }
                score(kmax(Pl, v), ord + (uint64_t)(h - lo), lr, h, rows_left - h, sc);
                if (!more) break;
                h = hn;
                p += J * FPW;
                v = vn;
              }
            }
            if (hi >= lo) ord += (uint64_t)(hi - lo + 1);
          }
          if (leaf_now) break;
        }
      } else {
        // ---- one live skeleton (c, widths, runs); every area lies in
        //      [win_lo, bmax[nH]] for a window a in [nL, nH]
        const int win_lo = nL, win_hi = SCB_BMAX(nH);
        SCB_STAT(skeletons);
        if (STEP == 1 && PRUNE) st.inc = incumbent_load(e.inc + f);
        // Levels of the heights DFS: every run of a multi-run column but its
        // last (forced) one, column by column.  Static per-level facts go to
        // LS[] once per skeleton; the DFS keeps its current level in registers
        // and spills a level's state to D[] only when it descends.
        int amin = kBigArea, amax = 0;
        int nl = 0;
        tkey P = 0;
        {
          int run = 0;
  #pragma unroll 1
          for (int i = 0; i < c; ++i) {
            if (R[i] == 1) {  // one-run columns are fixed by the skeleton
              const int ar = W[i] * rows;
              amin = imin(amin, ar);
              amax = imax(amax, ar);
              curH[run] = (uint8_t)rows;
              P = kmax(P, rt_at(X0[i], W[i], 0, rows));
            } else {
              nl += R[i] - 1;
            }
            run += R[i];
          }
        }
        // pruned mode, shared items: identity of this skeleton
        const bool split = PRUNE && e.split_g > 1;
        uint64_t skey = 0;
        int lsplit = -1;  // heights level whose values are dealt to the warps
        if (split) {
          skey = (uint64_t)c;
          for (int i = 0; i < c; ++i) skey = skey * 0x100000001b3ull ^ (uint64_t)(W[i] | (R[i] << 8));
          if (nl >= 2) lsplit = imin(e.split_depth, nl - 2);
          else if (split_owner(skey, e.split_g) != (uint32_t)split_r) {
            ord += 1;
            continue;
          }
        }
        if (nl == 0) {  // the skeleton is a single candidate
          if (slot == 0 && viable(P)) score(P, ord, -1, 0, 0);
          ord += 1;
          continue;
        }
        // pruned mode: every column's bound (PR) floors the whole subtree
        const tkey colfloor = PRUNE ? kmax(P, PR[c]) : P;
        if (!viable(colfloor)) continue;
        SCB_SYNCWARP();  // every lane is done with the previous skeleton's records
        {
          // level records, built from the last column backwards: a multi-run
          // column stays fillable iff t2 <= w*floor(rows/R) and
          // t1 >= w*ceil(rows/R) (the columns_feasible test), so each level
          // carries the suffix bounds over the columns from its own on
          int sLo = 0, sHi = kBigArea, lvl = nl, rr = e.n;
  #pragma unroll 1
          for (int i = c - 1; i >= 0; --i) {
            rr -= R[i];  // first run of column i
            if (R[i] < 2) continue;
            sLo = imax(sLo, W[i] * ((rows + R[i] - 1) / R[i]));
            sHi = imin(sHi, W[i] * SCB_RQ(R[i]));
            const int base = xw_of(cols, X0[i], W[i]) * nyh;
  #pragma unroll 1
            for (int j = R[i] - 2; j >= 0; --j)
              LS[--lvl] = Lvl{W[i] | ((R[i] - j) << 8) | ((rr + j) << 16) | (i << 24), base, sLo, sHi};
          }
        }

        // current level (registers): static facts, height h in (.., hhi],
        // first row y0, fixed-slice maximum Pin and areas Amin / Amax
        int l = 0, cw = 0, crl = 0, h = 0, hhi = 0, y0 = 0, cAmin = amin, cAmax = amax;
        int cridx = 0, clbase = 0;
        int crow = 0;  // rectangle index of the current level's run at h = 0
        tkey cPin = P;
        auto load_static = [&](const Lvl& s) {
          cw = s.a & 255;
          crl = (s.a >> 8) & 255;
          cridx = (s.a >> 16) & 255;
          clbase = s.b;
        };
        // curH holds the heights of the levels above the current one (written
        // when the DFS descends past them); the current level's own run (and its
        // forced rest) is written only before a score that may read it
        auto sync_heights = [&]() {
          if (l < 0) return;
          curH[cridx] = (uint8_t)h;
          if (crl == 2) curH[cridx + 1] = (uint8_t)(rows - y0 - h);
        };
        // ---- leaf: run `lr` of the last multi-run column takes every
        //      admissible height; the column's last run is forced.
        const Lvl LL = LS[nl - 1];
        const int lw = LL.a & 255, lr = (LL.a >> 16) & 255, lxwb = LL.b;
        const uint64_t lmg = SCB_MAGIC(lw);
        const int lms = lw * (e.rows + 1);
        // t: the area thresholds after every slice fixed above the leaf
        // candidates counted by the leaves since the last flush into `ord`: a
        // 32-bit add per leaf (a level has at most 255 heights of at most 255
        // candidates each between flushes)
        uint32_t ordl = 0;
        auto leaf = [&](tkey Pl, Thr t, int y0l) {
          SCB_STAT(leaf_calls);
          const int rows_left = rows - y0l;
          const int hmin_a = imax(1, div_w(t.t2 + lw - 1, lmg));
          const int hmax_a = t.t1 < 0 ? 0 : div_w(t.t1, lmg);
          const int lo = imax(imax(hmin_a, rows_left - hmax_a), SCB_MSTAR(lms + rows_left));
          const int hi = rows_left - lo;
          if (lo + slot <= hi && viable(PRUNE ? kmax(Pl, colfloor) : Pl)) {
            // the split table holds max(run h, forced rest) at the run's own
            // rectangle index, which advances by +1 per h; lanes step h by J
            // (J * FPW = 32 keys between consecutive heights of a lane)
            const tkey* p0 = e.rts + (size_t)(lxwb + SCB_YBASE(y0l) + lo + slot - 1) * FPW + f;
            if (STEP == 1 && !PRUNE) {
              // every candidate's time max(Pl, v_h) is evaluated as one
              // min-reduction; only a chunk that can beat the lane's best
              // replays its heights in order through score()
              const int nh = (hi - lo - slot) / J + 1;
              // first four heights outside the loop (most leaves have <= 4)
              tkey m = umin3(p0[0], nh > 1 ? p0[32] : kKeyInf, nh > 2 ? p0[64] : kKeyInf);
              m = nh > 3 ? kmin(m, p0[96]) : m;
              const tkey* p = p0 + 4 * 32;
  #pragma unroll 1
              for (int k = 4; k < nh; k += 4, p += 4 * 32) {
                const tkey v0 = p[0];
                const tkey v1 = k + 1 < nh ? p[32] : kKeyInf;
                const tkey v2 = k + 2 < nh ? p[64] : kKeyInf;
                const tkey v3 = k + 3 < nh ? p[96] : kKeyInf;
                m = umin3(m, umin3(v0, v1, v2), v3);
              }
              const tkey thr = st.bcmp;
              if (kmax(Pl, m) < thr) {
                sync_heights();
                const tkey* q = p0;
  #pragma unroll 1
                for (int hh = lo + slot; hh <= hi; hh += J, q += 32)
                  score(kmax(Pl, *q), ord + (uint64_t)(ordl + (uint32_t)(hh - lo)), lr, hh, rows_left - hh);
              }
            } else {  // pruned walks and step 2: leaves are few, winners common
              sync_heights();
              int hh = lo + slot;
              const tkey* q = p0;
              tkey v = *q;
              while (true) {
                const int hn = hh + J;
                const bool more = hn <= hi;
                const tkey vn = more ? q[32] : 0;  // prefetch the next height
                score(kmax(Pl, v), ord + (uint64_t)(ordl + (uint32_t)(hh - lo)), lr, hh, rows_left - hh);
                if (!more) break;
                hh = hn;
                q += 32;
                v = vn;
              }
            }
          }
          if (hi >= lo) ordl += (uint32_t)(hi - lo + 1);
        };
        if (nl == 1) {
          l = -1;  // no level above the leaf
          leaf(P, thresholds(amin, amax, win_lo, win_hi), 0);
          ord += ordl;
          continue;
        }
        // ---- heights DFS over the levels above the leaf (search.cpp:163-190)
        load_static(LS[0]);
        {
          int lo0, hi0;
          height_interval(e, thresholds(amin, amax, win_lo, win_hi), cw, rows, crl, lo0, hi0);
          h = lo0 - 1;
          hhi = imax(hi0, 0);
          crow = clbase - 1;  // y0 = 0: ybase(0) = 0
        }
        // the leaf's parent level runs in the leaf's own column (the column has
        // three or more runs): its heights go straight into the leaf from a
        // tight loop -- never forced, no column change, nothing to push
        const bool tail_fused = nl >= 2 && (LS[nl - 2].a >> 24) == (LS[nl - 1].a >> 24);
        while (true) {
          SCB_STAT(levels);
          // the level records are written by every lane with the same value;
          // a lane may only overwrite one after all lanes finished reading it
          SCB_SYNCWARP();
          const bool forced = crl == 2;
          if (tail_fused && l == nl - 2) {
            while (true) {
              ++h;
              if (e.patho)
                while (h <= hhi && !(cw * h <= SCB_BMAX(cw * h))) ++h;
              if (h > hhi) break;
              const int a1 = cw * h;
              const tkey Pn = kmax(cPin, rt[(size_t)(crow + h) * FPW + f]);
              leaf(Pn, thresholds(imin(cAmin, a1), imax(cAmax, a1), win_lo, win_hi), y0 + h);
              SCB_SYNCWARP();
            }
            ord += ordl;
            ordl = 0;
          } else if (forced && l == nl - 2) {
            // the leaf's parent closes its column (forced rest): the leaf
            // starts the next column at row 0, whose fillability bounds are
            // fixed for the loop
            const Lvl sn = LS[nl - 1];
            while (true) {
              ++h;
              if (h > hhi) break;
              const int a1 = cw * h, a2 = cw * (rows - y0 - h);
              const int na = imin(imin(cAmin, a1), a2), nx = imax(imax(cAmax, a1), a2);
              const tkey Pn = kmax(cPin, e.rts[(size_t)(crow + h) * FPW + f]);
              const Thr tn = thresholds(na, nx, win_lo, win_hi);
              if (tn.t2 > sn.d || tn.t1 < sn.c) continue;
              leaf(Pn, tn, 0);
              SCB_SYNCWARP();
            }
            ord += ordl;
            ordl = 0;
          } else {
            ++h;
            if (e.patho && !forced)
              while (h <= hhi && !(cw * h <= SCB_BMAX(cw * h))) ++h;
          }
          if (h > hhi) {
            if (l == 0) break;
            --l;
            load_static(LS[l]);
            const Lvl dl = D[l];
            h = dl.a & 255;
            hhi = (dl.a >> 8) & 255;
            y0 = (dl.a >> 16) & 255;
            cPin = PIN[l * PS];
            cAmin = dl.c;
            cAmax = dl.d;
            crow = clbase + SCB_YBASE(y0) - 1;
            continue;
          }
          if (split && l == lsplit) {  // deal this subtree to one warp of the item
            uint64_t k = skey;
            for (int q = 0; q < l; ++q) k = k * 0x100000001b3ull ^ (uint64_t)((D[q].a & 255) + 1);
            k = k * 0x100000001b3ull ^ (uint64_t)(h + 1);
            if (split_owner(k, e.split_g) != (uint32_t)split_r) continue;
          }
          const int a1 = cw * h;
          int na = imin(cAmin, a1), nx = imax(cAmax, a1);
          const size_t ri = (size_t)(crow + h) * FPW + f;
          tkey Pn;
          if (forced) {
            const int a2 = cw * (rows - y0 - h);
            na = imin(na, a2);
            nx = imax(nx, a2);
            Pn = kmax(cPin, e.rts[ri]);
          } else {
            Pn = kmax(cPin, rt[ri]);
          }
          if (!viable(PRUNE ? kmax(Pn, colfloor) : Pn)) continue;
          const int nxt = l + 1;
          const int y0n = forced ? 0 : y0 + h;
          const Thr tn = thresholds(na, nx, win_lo, win_hi);
          const Lvl sn = LS[nxt];
          // a new column: every multi-run column from it on must stay fillable
          if (forced && (tn.t2 > sn.d || tn.t1 < sn.c)) continue;
          if (nxt < nl - 1) {
            int lo2, hi2;
            height_interval(e, tn, sn.a & 255, rows - y0n, (sn.a >> 8) & 255, lo2, hi2);
            if (lo2 > hi2) continue;
            D[l] = Lvl{h | (hhi << 8) | (y0 << 16), 0, cAmin, cAmax};
          PIN[l * PS] = cPin;
            sync_heights();
            l = nxt;
            load_static(sn);
            h = lo2 - 1;
            hhi = hi2;
            y0 = y0n;
            cPin = Pn;
            cAmin = na;
            cAmax = nx;
            crow = clbase + SCB_YBASE(y0) - 1;
            continue;
          }
          leaf(Pn, tn, y0n);
          ord += ordl;
          ordl = 0;
        }
      }
    }
    if (fixed_widths) break;
  }
  st.count += ord;
}

}  // namespace scb
