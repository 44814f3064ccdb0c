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
#include "common.cuh"

namespace scb {

constexpr int kMaxLevels = SC_MAX_SLICES;

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

template <int FPW, int STEP>
__global__ void __launch_bounds__(256) k_search(SearchArgs a) {
  extern __shared__ int32_t s_bmax[];
  for (int i = threadIdx.x; i <= a.max_area; i += blockDim.x) s_bmax[i] = a.bmax[i];
  __syncthreads();

  constexpr int J = 32 / FPW;
  const int lane = threadIdx.x & 31;
  const int f = lane % FPW;
  const int slot = lane / FPW;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int rows = a.rows, cols = a.cols, nyh = a.nyh;
  const uint64_t* __restrict__ rt = a.rt;
  const double* __restrict__ rs = a.rs;
  const uint32_t below_mask = (slot * FPW) >= 32 ? 0xffffffffu : ((1u << (slot * FPW)) - 1u);

  uint64_t best_t = ~0ull, best_item = ~0ull, best_ord = ~0ull;
  double best_sse = __longlong_as_double(0x7ff0000000000000ll);
  uint64_t budget = 0;
  if (STEP == 2) budget = a.budget[f];
  unsigned long long count = 0;
  uint8_t* snap = a.snaps + ((size_t)gwarp * 32 + lane) * kSnapBytes;

  // warp-uniform DFS state (identical in every lane)
  int W[SC_MAX_COLS], R[SC_MAX_COLS], X0[SC_MAX_COLS + 1], RS0[SC_MAX_COLS];
  uint8_t curH[SC_MAX_SLICES];
  uint8_t Lcol[kMaxLevels], Lrun[kMaxLevels], Ly0[kMaxLevels], Lh[kMaxLevels];
  int32_t Amin[kMaxLevels], Amax[kMaxLevels];
  uint64_t Pin[kMaxLevels];

  auto rect = [&](int x0, int w, int y0, int h) -> int {
    return xw_index(cols, x0, w) * nyh + yh_index(rows, y0, h);
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

    int used = 0;
    for (int i = 0; i < d; ++i) {
      W[i] = wi.w[i];
      used += W[i];
    }
    for (int i = d; i < c; ++i) W[i] = 1;
    if (a.coverage && d < c) W[c - 1] = cols - (used + (c - 1 - d));
    const bool runs_possible = (a.n >= c) && (a.n <= c * rows);

    bool more_widths = runs_possible;
    while (more_widths) {
      X0[0] = 0;
      for (int i = 0; i < c; ++i) X0[i + 1] = X0[i] + W[i];
      // ---- runs: lexicographic compositions of n (search.cpp:145-161)
      {
        int s = a.n;
        for (int i = 0; i < c; ++i) {
          const int after = c - 1 - i;
          int lo = s - after * rows;
          if (lo < 1) lo = 1;
          R[i] = lo;
          s -= lo;
        }
      }
      bool more_runs = true;
      while (more_runs) {
        // ---- one skeleton (c, widths, runs)
        int amin = 0x7fffffff, amax = 0;
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
        if (amin == 0x7fffffff || amax <= s_bmax[amin]) {
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
          } else {
            // ---- heights DFS over the multi-run columns (search.cpp:163-190)
            int l = 0;
            Lh[0] = 0;
            Pin[0] = P;
            Amin[0] = amin;
            Amax[0] = amax;
            Ly0[0] = 0;
            bool leaf_now = (nl == 1);
            while (true) {
              int lv;          // level whose state feeds the leaf loop
              uint64_t Pl;
              int amin_l, amax_l, y0l;
              if (leaf_now) {
                // nl == 1: the only level is the leaf level
                lv = 0; Pl = P; amin_l = amin; amax_l = amax; y0l = 0;
              } else {
                // advance level l to its next admissible height
                const int i = Lcol[l], j = Lrun[l];
                const int w = W[i], y0 = Ly0[l];
                const int rows_left = rows - y0, runs_left = R[i] - j;
                const bool forced = runs_left == 2;
                const int hmax = rows_left - (runs_left - 1);
                const int ain = Amin[l], xin = Amax[l];
                int h = Lh[l] + 1;
                int na = 0, nx = 0;
                for (; h <= hmax; ++h) {
                  const int a1 = w * h;
                  na = min(ain, a1);
                  nx = max(xin, a1);
                  if (forced) {
                    const int a2 = w * (rows_left - h);
                    na = min(na, a2);
                    nx = max(nx, a2);
                  }
                  if (nx <= s_bmax[na]) break;
                }
                if (h > hmax) {
                  if (l == 0) break;
                  --l;
                  continue;
                }
                Lh[l] = (uint8_t)h;
                const int ridx = RS0[i] + j;
                curH[ridx] = (uint8_t)h;
                uint64_t Pn = umax64(Pin[l], rt[(size_t)rect(X0[i], w, y0, h) * FPW + f]);
                if (forced) {
                  curH[ridx + 1] = (uint8_t)(rows_left - h);
                  Pn = umax64(Pn, rt[(size_t)rect(X0[i], w, y0 + h, rows_left - h) * FPW + f]);
                }
                const int nxt = l + 1;
                const int y0n = (Lrun[nxt] == 0) ? 0 : y0 + h;
                if (nxt < nl - 1) {
                  l = nxt;
                  Lh[l] = 0;
                  Pin[l] = Pn;
                  Amin[l] = na;
                  Amax[l] = nx;
                  Ly0[l] = (uint8_t)y0n;
                  continue;
                }
                lv = nxt; Pl = Pn; amin_l = na; amax_l = nx; y0l = y0n;
              }
              // ---- leaf loop: run Lrun[lv] of column Lcol[lv] varies, the
              //      next (last) run of that column is forced.
              {
                const int i = Lcol[lv];
                const int w = W[i];
                const int rows_left = rows - y0l;
                const int hmax = rows_left - 1;
                const int lr = RS0[i] + Lrun[lv];
                const int xwb = xw_index(cols, X0[i], w) * nyh;
                const int wrl = w * rows_left;
                const int ybase = yh_index(rows, y0l, 1);
                for (int h0 = 1; h0 <= hmax; h0 += J) {
                  const int h = h0 + slot;
                  bool adm = false;
                  if (h <= hmax) {
                    const int a1 = w * h, a2 = wrl - a1;
                    const int na = min(amin_l, min(a1, a2));
                    const int nx = max(amax_l, max(a1, a2));
                    adm = nx <= s_bmax[na];
                  }
                  const uint32_t bal = __ballot_sync(0xffffffffu, adm);
                  if (adm) {
                    const uint64_t my_ord = ord + (uint64_t)(__popc(bal & below_mask) / FPW);
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
                  ord += (uint64_t)(__popc(bal) / FPW);
                }
              }
              if (leaf_now) break;
            }
          }
        }
        // ---- next runs composition (lex)
        more_runs = false;
        {
          int pre = 0;
          int s_at[SC_MAX_COLS];
          for (int i = 0; i < c; ++i) {
            s_at[i] = a.n - pre;
            pre += R[i];
          }
          for (int i = c - 2; i >= 0; --i) {
            const int after = c - 1 - i;
            const int hi = min(rows, s_at[i] - after);
            if (R[i] < hi) {
              R[i] += 1;
              int s = s_at[i] - R[i];
              for (int jj = i + 1; jj < c; ++jj) {
                const int aft = c - 1 - jj;
                int lo = s - aft * rows;
                if (lo < 1) lo = 1;
                R[jj] = lo;
                s -= lo;
              }
              more_runs = true;
              break;
            }
          }
        }
      }
      // ---- next widths (lex, search.cpp:133-143)
      more_widths = false;
      if (!a.coverage) {
        for (int i = c - 1; i >= d; --i) {
          const int maxw = (cols - X0[i]) - (c - i - 1);
          if (W[i] < maxw) {
            W[i] += 1;
            for (int jj = i + 1; jj < c; ++jj) W[jj] = 1;
            more_widths = true;
            break;
          }
        }
      } else {
        for (int i = c - 2; i >= d; --i) {
          const int maxw = (cols - X0[i]) - (c - i - 1);
          if (W[i] < maxw) {
            W[i] += 1;
            for (int jj = i + 1; jj < c - 1; ++jj) W[jj] = 1;
            W[c - 1] = cols - (X0[i] + W[i] + (c - 2 - i));
            more_widths = true;
            break;
          }
        }
      }
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
  const size_t smem = (size_t)(a.max_area + 1) * sizeof(int32_t);
  if (smem > 64 * 1024) fail(SC_ERR_SIZE, "CTU grid too large for the area table");
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
