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

#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "search_walk.cuh"

namespace scb {

#ifndef SCB_SEARCH_MINB
#define SCB_SEARCH_MINB 2
#endif
#ifndef SCB_SEARCH_BLOCK
#define SCB_SEARCH_BLOCK 256
#endif
// Exhaustive step 1 (the headline walk, warp-uniform): 128-thread blocks under
// a register cap (__maxnreg__) instead of a blocks-per-SM launch bound; the
// cap keeps ptxas at <= 96 registers (86 used), so the register file holds 20
// warps/SM.  Measured on cfg3, step-1 ms: block 128 / 160 /
// 320 (5 / 4 / 2 blocks): 4.31; 64 (10 blocks, twice the per-block table
// copies in shared memory, less L1): 4.39; 192 (3 blocks, 18 warps): 4.56.
// Cap -> registers (64-thread blocks): 96 -> 89: 4.47, 100 -> 92: 4.49,
// uncapped -> 102 (fewer warps): 4.79.
#ifndef SCB_SEARCH_BLOCK1
#define SCB_SEARCH_BLOCK1 128
#endif
#ifndef SCB_SEARCH_REGS1
#define SCB_SEARCH_REGS1 96
#endif
template <int STEP, bool PRUNE>
struct SearchShape {
  static constexpr bool kHead = STEP == 1 && !PRUNE;
  static constexpr int kBlock = kHead ? SCB_SEARCH_BLOCK1 : SCB_SEARCH_BLOCK;
};
int search_block_threads(int step, bool prune) {
  return (step == 1 && !prune) ? SCB_SEARCH_BLOCK1 : SCB_SEARCH_BLOCK;
}
// dynamic shared memory of the search kernels: bmax|aneed [2A], mstar, ilo
// (int32), then, for the warp-uniform exhaustive walks, 2 * n level records
// (16 B) per warp (search_walk.cuh WalkEnv::lvl)
size_t search_tables_bytes(int cols, int rows, int n) {
  return ((size_t)2 * (cols * rows + 1) + (size_t)(cols + 1) * (rows + 1) +
          (size_t)(cols + 1) * (std::min(n, rows) + 1)) *
         sizeof(int32_t);
}
size_t search_smem_bytes(int cols, int rows, int n, int step, bool prune) {
  size_t b = search_tables_bytes(cols, rows, n);
  // per warp: 2 * n level records, 32 lanes x n Pin keys, the uniform arrays
  if (!prune)
    b = (b + 15) / 16 * 16 +
        (size_t)(search_block_threads(step, prune) / 32) *
            ((size_t)std::max(n, 1) * (2 * sizeof(Lvl) + 32 * sizeof(uint32_t)) +
             kUniInts * sizeof(int));
  return b;
}

template <int FPW, int STEP, bool PRUNE>
__device__ __forceinline__ void search_body(const SearchArgs& a) {
  // shared-memory tables (search_walk.cuh): g_dyn = bmax|aneed interleaved
  // [2A], mstar [(cols+1)(rows+1)], ilo [(cols+1) * rstride]; static magic,
  // rq
  const int A = a.max_area + 1;
  const int nms = (a.cols + 1) * (a.rows + 1);
  const int rstride = min(a.n, a.rows) + 1;
  for (int i = threadIdx.x; i < A; i += blockDim.x) {
    g_dyn[2 * i] = a.bmax[i];
    g_dyn[2 * i + 1] = a.bmax[A + i];
  }
  for (int i = threadIdx.x; i < nms; i += blockDim.x) g_dyn[2 * A + i] = a.bmax[2 * A + i];
  __syncthreads();
  const int ilo_off = 2 * A + nms;
  for (int i = threadIdx.x; i < (a.cols + 1) * rstride; i += blockDim.x) {
    const int w = i / rstride, r = i % rstride;
    g_dyn[ilo_off + i] = (w >= 1 && r >= 1) ? g_dyn[2 * (w * ((a.rows + r - 1) / r)) + 1] : 0;
  }
  for (int w = threadIdx.x; w < kTabDim; w += blockDim.x)
    g_magic[w] = (w >= 1 && w <= a.cols) ? div_magic(w) : 0ull;
  for (int y = threadIdx.x; y < kTabDim; y += blockDim.x) {
    g_rq[y] = (y >= 1 && y <= a.rows) ? a.rows / y : 0;
  }
  __syncthreads();
  WalkEnv e;
  e.cols = a.cols;
  e.rows = a.rows;
  e.n = a.n;
  e.nyh = a.nyh;
  e.max_area = a.max_area;
  e.coverage = a.coverage;
  e.patho = a.pathological;
  e.prune = a.prune;
  e.rstride = rstride;
  e.split_g = (PRUNE && a.split_g > 1) ? a.split_g : 1;
  e.split_depth = a.split_depth;
  e.mstar_off = 2 * A;
  e.ilo_off = ilo_off;
  if (!PRUNE) {
    const int tab_words = ilo_off + (a.cols + 1) * rstride;
    const int lvl_cap = max(a.n, 1);
    Lvl* const lvl0 = reinterpret_cast<Lvl*>(g_dyn + (tab_words + 3) / 4 * 4);
    const int nwarps = blockDim.x >> 5, wib = threadIdx.x >> 5;
    e.lvl = lvl0 + (size_t)wib * 2 * lvl_cap;
    tkey* const pin0 = reinterpret_cast<tkey*>(lvl0 + (size_t)nwarps * 2 * lvl_cap);
    e.pin = pin0 + (size_t)wib * 32 * lvl_cap + (threadIdx.x & 31);
    e.uni = reinterpret_cast<int*>(pin0 + (size_t)nwarps * 32 * lvl_cap) + (size_t)wib * kUniInts;
    e.lvl_cap = lvl_cap;
  } else {
    e.lvl = nullptr;
    e.pin = nullptr;
    e.uni = nullptr;
    e.lvl_cap = 0;
  }
  e.rt = a.rt;
  e.rts = a.rts;
  e.rs = a.rs;
  e.lbr = a.lbr;
  e.lbm = a.lbm;
  e.inc = a.inc;
  e.seed_inc = a.seed_inc;
  e.sse_inc = (PRUNE && STEP == 2) ? a.sse_inc : nullptr;

  const int lane = threadIdx.x & 31;
  const int f = lane % FPW;
  const int slot = lane / FPW;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  LaneState st;
  st.best_t = kKeyInf;
  st.best_item = ~0ull;
  st.best_ord = ~0ull;
  st.best_sse = __longlong_as_double(0x7ff0000000000000ll);
  if (a.resume) {  // second phase of a seeded launch: keep this lane's best
    const LaneBest prev = a.lanes[(size_t)gwarp * 32 + lane];
    st.best_t = (tkey)prev.t;
    st.best_item = prev.item;
    st.best_ord = prev.ord;
    st.best_sse = prev.sse;
  }
  st.budget = STEP == 2 ? a.budget[f] : -1;
  st.count = 0;
  st.scored = 0;
  st.inc = ~0ull;
  st.sbound = __longlong_as_double(0x7ff0000000000000ll);
  st.snap = a.snaps + ((size_t)gwarp * 32 + lane) * kSnapBytes;
  const uint32_t n_items = a.n_items_dev ? *a.n_items_dev * (uint32_t)e.split_g : a.n_items;
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = a.k_begin + atomicAdd(a.counter, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= n_items) break;
    // pruned mode: split_g consecutive counter values share one work item
    const uint32_t kk = k / (uint32_t)e.split_g, part = k % (uint32_t)e.split_g;
    const uint64_t item =
        a.order ? (uint64_t)a.order[kk] : (uint64_t)a.item_offset + (uint64_t)kk * a.item_stride;
    const WorkItem wi = a.items[item];
    const long long c0 = a.cost ? clock64() : 0;
    walk_item<FPW, STEP, PRUNE>(e, item, wi, f, slot, st, (int)part);
    __syncwarp();
    if (a.cost && lane == 0) a.cost[item] = (uint32_t)min((clock64() - c0) >> 6, 0xffffffffll);
  }
  LaneBest lb;
  lb.t = st.best_t == kKeyInf ? ~0ull : (uint64_t)st.best_t;
  lb.sse = st.best_sse;
  lb.item = st.best_item;
  lb.ord = st.best_ord;
  a.lanes[(size_t)gwarp * 32 + lane] = lb;
  if (lane == 0 && st.count) atomicAdd(a.count_out, (unsigned long long)st.count);
  unsigned long long sc = st.scored;
  for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
  if (lane == 0 && sc) atomicAdd(a.scored_out, sc);
}

// The headline walk (exhaustive step 1) under a register cap (5 blocks of 4
// warps resident per SM); the other walks under a plain launch bound.
template <int FPW>
__global__ void __maxnreg__(SCB_SEARCH_REGS1)
    k_search_head(SearchArgs a) {
  search_body<FPW, 1, false>(a);
}
template <int FPW, int STEP, bool PRUNE>
__global__ void __launch_bounds__(SCB_SEARCH_BLOCK, SCB_SEARCH_MINB) k_search(SearchArgs a) {
  search_body<FPW, STEP, PRUNE>(a);
}
template <int FPW, int STEP, bool PRUNE>
constexpr void (*search_kernel())(SearchArgs) {
  if constexpr (STEP == 1 && !PRUNE) return k_search_head<FPW>;
  else return k_search<FPW, STEP, PRUNE>;
}

// ---- pruned mode: per-frame column lower bounds (search_walk.cuh) -------------
__global__ void k_column_bounds(const uint32_t* __restrict__ rt, int fpw, int frames_in_group,
                                int cols, int rows, int rmax, int rstride, uint32_t* lbr,
                                uint32_t* lbm) {
  const int nxw = cols * (cols + 1) / 2;
  const int nyh = rows * (rows + 1) / 2;
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nxw * fpw) return;
  const int xw = id / fpw, f = id % fpw;
  if (f >= frames_in_group) return;
  const size_t off = (size_t)xw * rstride * fpw + f;
  column_bounds(rt, fpw, f, rows, xw * nyh, rmax, lbr + off, lbm + off, (size_t)fpw);
}

// One block per column (x0, w): the column's rectangle keys of every frame of
// the group are staged in shared memory ([yh][fpw], coalesced) and the DP over
// rows runs with one thread per (row end y, frame), a barrier per run count r
// -- the same recurrence as column_bounds() (search_walk.cuh), parallel over y.
__global__ void k_column_bounds_blk(const uint32_t* __restrict__ rt, int fpw, int frames_in_group,
                                   int rows, int rmax, int rstride, uint32_t* lbr,
                                   uint32_t* lbm) {
  extern __shared__ uint32_t cb_sm[];
  const int xw = blockIdx.x;
  const int nyh = rows * (rows + 1) / 2;
  const int ny = (rows + 1) * fpw;
  uint32_t* tab = cb_sm;          // [nyh][fpw]
  uint32_t* prev = tab + (size_t)nyh * fpw;  // [rows + 1][fpw]
  uint32_t* cur = prev + ny;
  uint32_t* rmin = cur + ny;      // [fpw] running minimum over r
  const uint32_t INF = kKeyInf;
  const uint32_t* src = rt + (size_t)xw * nyh * fpw;
  for (int i = threadIdx.x; i < nyh * fpw; i += blockDim.x) tab[i] = src[i];
  for (int i = threadIdx.x; i < ny; i += blockDim.x) prev[i] = i < fpw ? 0u : INF;
  for (int i = threadIdx.x; i < fpw; i += blockDim.x) rmin[i] = INF;
  __syncthreads();
  const size_t out0 = (size_t)xw * rstride * fpw;
  for (int i = threadIdx.x; i < frames_in_group; i += blockDim.x) {
    lbr[out0 + i] = INF;
    lbm[out0 + i] = INF;
  }
  for (int r = 1; r <= rmax; ++r) {
    for (int i = threadIdx.x; i < ny; i += blockDim.x) {
      const int y = i / fpw, f = i - y * fpw;
      uint32_t best = INF;
      for (int y0 = r - 1; y0 < y; ++y0) {
        const uint32_t p = prev[y0 * fpw + f];
        if (p == INF) continue;
        const uint32_t v = tab[yh_of(rows, y0, y - y0) * fpw + f];
        const uint32_t m = p > v ? p : v;
        best = m < best ? m : best;
      }
      cur[i] = best;
    }
    __syncthreads();
    for (int f = threadIdx.x; f < frames_in_group; f += blockDim.x) {
      const uint32_t c = cur[rows * fpw + f];
      const uint32_t m = c < rmin[f] ? c : rmin[f];
      rmin[f] = m;
      lbr[out0 + (size_t)r * fpw + f] = c;
      lbm[out0 + (size_t)r * fpw + f] = m;
    }
    uint32_t* t = prev;
    prev = cur;
    cur = t;
    __syncthreads();
  }
}

void column_bounds_launch(const uint32_t* rt, int fpw, int frames_in_group, int cols, int rows,
                          int rmax, int rstride, uint32_t* lbr, uint32_t* lbm, cudaStream_t st) {
  const int nxw = cols * (cols + 1) / 2;
  const size_t nyh = (size_t)rows * (rows + 1) / 2;
  const size_t smem = (nyh * fpw + 2 * (size_t)(rows + 1) * fpw + fpw) * sizeof(uint32_t);
  if (smem <= 96 * 1024) {
    once_per_device((const void*)k_column_bounds_blk, [] {
      SCB_CUDA(cudaFuncSetAttribute(k_column_bounds_blk,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    });
    SCB_LAUNCH(k_column_bounds_blk<<<nxw, 256, smem, st>>>(rt, fpw, frames_in_group, rows, rmax, rstride,
                                                lbr, lbm));
  } else {  // tall grids: one thread per (column, frame)
    const int threads = 128, total = nxw * fpw;
    SCB_LAUNCH(k_column_bounds<<<(total + threads - 1) / threads, threads, 0, st>>>(
        rt, fpw, frames_in_group, cols, rows, rmax, rstride, lbr, lbm));
  }
  SCB_CUDA(cudaGetLastError());
}

// ---- finalize: per frame, reduce all lanes of that frame ---------------------
// Order: step key ((t) or (sse, t)), then work item, then the candidate's
// position inside the item, read from the snapshots: widths, runs, heights
// compared lexicographically -- the reference's enumeration order.  (Ordinals
// are not dense under pruning, so the layout itself is the position.)
__device__ __forceinline__ bool lane_less(int step, int n, const LaneBest& x, uint32_t xi,
                                          const LaneBest& y, uint32_t yi,
                                          const uint8_t* __restrict__ snaps) {
  if (step == 2) {
    if (x.sse < y.sse) return true;
    if (x.sse > y.sse) return false;
  }
  if (x.t != y.t) return x.t < y.t;
  if (x.item != y.item) return x.item < y.item;
  const uint8_t* a = snaps + (size_t)xi * kSnapBytes;
  const uint8_t* b = snaps + (size_t)yi * kSnapBytes;
  const int len = 2 * SC_MAX_COLS + n;
  for (int i = 0; i < len; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return xi < yi;
}

__device__ __forceinline__ int64_t budget_key_f(const uint64_t* vals, uint32_t n, double b) {
  if (!(b >= 0.0)) return -1;
  const uint64_t bits = (uint64_t)__double_as_longlong(b);
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (vals[mid] <= bits) lo = mid + 1;
    else hi = mid;
  }
  return (int64_t)lo - 1;
}

// Block minimum (lane_less order) of the lanes a block's threads scanned;
// thread 0 ends with it in sb[0] / si[0] (si: the lane, 0xffffffff: none).
__device__ __forceinline__ void finalize_block_min(int step, int n, LaneBest best, uint32_t bi,
                                                   const uint8_t* __restrict__ snaps,
                                                   LaneBest* sb, uint32_t* si) {
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const uint32_t yi = si[threadIdx.x + o];
      if (yi != 0xffffffffu &&
          (si[threadIdx.x] == 0xffffffffu ||
           lane_less(step, n, sb[threadIdx.x + o], yi, sb[threadIdx.x], si[threadIdx.x], snaps))) {
        sb[threadIdx.x] = sb[threadIdx.x + o];
        si[threadIdx.x] = yi;
      }
    }
    __syncthreads();
  }
}

// First level of the per-frame reduction: part p of frame f's lanes
// (blockIdx = (p, f)) -> its minimum and that lane's index.  Spreads the
// scan of the persistent grid's ~10^5 lanes over many blocks (one block per
// frame took ~100 us).
__global__ void k_finalize_part(int step, int n, int fpw, uint32_t n_warps,
                                const LaneBest* __restrict__ lanes,
                                const uint8_t* __restrict__ snaps, LaneBest* part_best,
                                uint32_t* part_lane) {
  const int f = blockIdx.y, parts = gridDim.x;
  __shared__ LaneBest sb[256];
  __shared__ uint32_t si[256];
  LaneBest best;
  best.t = ~0ull; best.sse = __longlong_as_double(0x7ff0000000000000ll);
  best.item = ~0ull; best.ord = ~0ull;
  uint32_t bi = 0xffffffffu;
  const uint32_t n_lanes = n_warps * 32;
  for (uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) * fpw + f; li < n_lanes;
       li += (uint32_t)parts * blockDim.x * fpw) {
    const LaneBest x = lanes[li];
    if (x.item == ~0ull) continue;
    if (bi == 0xffffffffu || lane_less(step, n, x, li, best, bi, snaps)) { best = x; bi = li; }
  }
  finalize_block_min(step, n, best, bi, snaps, sb, si);
  if (threadIdx.x == 0) {
    part_best[(size_t)f * parts + blockIdx.x] = sb[0];
    part_lane[(size_t)f * parts + blockIdx.x] = si[0];
  }
}

__global__ void k_finalize(int step, int n, int parts, int frames_in_group,
                           const LaneBest* __restrict__ part_best,
                           const uint32_t* __restrict__ part_lane, const uint8_t* __restrict__ snaps,
                           const unsigned long long* count, const unsigned long long* scored,
                           double lambda, const uint64_t* __restrict__ vals,
                           const uint32_t* __restrict__ nvals, size_t nr,
                           FrameBest* __restrict__ out, int64_t* __restrict__ budget_out) {
  const int f = blockIdx.x;
  if (f >= frames_in_group) return;
  __shared__ LaneBest sb[256];
  __shared__ uint32_t si[256];
  LaneBest best;
  best.t = ~0ull; best.sse = __longlong_as_double(0x7ff0000000000000ll);
  best.item = ~0ull; best.ord = ~0ull;
  uint32_t bi = 0xffffffffu;
  for (int pi = threadIdx.x; pi < parts; pi += blockDim.x) {
    const uint32_t li = part_lane[(size_t)f * parts + pi];
    if (li == 0xffffffffu) continue;
    const LaneBest x = part_best[(size_t)f * parts + pi];
    if (bi == 0xffffffffu || lane_less(step, n, x, li, best, bi, snaps)) { best = x; bi = li; }
  }
  finalize_block_min(step, n, best, bi, snaps, sb, si);
  __shared__ uint32_t win;
  const uint64_t* fv = vals + (size_t)f * nr;  // this frame's key -> time bits
  if (threadIdx.x == 0) {
    win = si[0];
    // step 1 keeps `t < best_t` from best_t = +inf (search.cpp:277-285): a
    // family whose every time is +inf has no argmin (NoCandidateError)
    if (step == 1 && win != 0xffffffffu && fv[sb[0].t] == 0x7ff0000000000000ull)
      win = 0xffffffffu;
  }
  __syncthreads();
  FrameBest* o = out + f;
  if (threadIdx.x == 0) {
    o->t = win == 0xffffffffu ? ~0ull : fv[sb[0].t];
    o->sse = sb[0].sse;
    o->item = sb[0].item;
    o->ord = sb[0].ord;
    o->count = *count;
    o->scored = *scored;
    o->found = (win == 0xffffffffu) ? 0 : 1;
    if (budget_out && step == 1 && win != 0xffffffffu) {
      // budget = t_min * (1.0 + lambda)   (search.cpp:344), as a time key
      const double tmin = __longlong_as_double((long long)fv[sb[0].t]);
      const double b = __dmul_rn(tmin, __dadd_rn(1.0, lambda));
      budget_out[f] = budget_key_f(fv, nvals[f], b);
    }
  }
  if (win != 0xffffffffu)
    for (int i = threadIdx.x; i < kSnapBytes; i += blockDim.x)
      o->snap[i] = snaps[(size_t)win * kSnapBytes + i];
}

// ---- host launchers ------------------------------------------------------------
// The walks may use the device's whole opt-in shared memory (per device).
template <int FPW, int STEP>
static void set_search_attrs() {
  once_per_device((const void*)search_kernel<FPW, STEP, false>(), [] {
    for (const void* k : {(const void*)search_kernel<FPW, STEP, false>(),
                          (const void*)search_kernel<FPW, STEP, true>()})
      SCB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    max_dynamic_smem(k)));
  });
}

template <int FPW, int STEP>
static void launch_fpw(const SearchArgs& a, int blocks, size_t smem, cudaStream_t st) {
  set_search_attrs<FPW, STEP>();
  if (a.prune)
    SCB_LAUNCH(search_kernel<FPW, STEP, true>()<<<blocks, SearchShape<STEP, true>::kBlock, smem, st>>>(a));
  else
    SCB_LAUNCH(search_kernel<FPW, STEP, false>()<<<blocks, SearchShape<STEP, false>::kBlock, smem, st>>>(a));
}

int search_blocks_per_sm(int fpw, int step, bool prune, size_t smem) {
  int nb = 0;
#define OCC1(F, S, P)                                                                        \
  set_search_attrs<F, S>();                                                                  \
  SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, search_kernel<F, S, P>(),           \
                                                         SearchShape<S, P>::kBlock, smem))
#define OCC(F)                                                                               \
  if (fpw == F) {                                                                            \
    if (step == 1) {                                                                         \
      if (prune) { OCC1(F, 1, true); }                                                       \
      else { OCC1(F, 1, false); }                                                            \
    } else {                                                                                 \
      if (prune) { OCC1(F, 2, true); }                                                       \
      else { OCC1(F, 2, false); }                                                            \
    }                                                                                        \
  }
  OCC(1) OCC(2) OCC(4) OCC(8) OCC(16) OCC(32)
#undef OCC
#undef OCC1
  return nb < 1 ? 1 : nb;
}

void search_launch(int fpw, int step, const SearchArgs& a, int blocks, cudaStream_t st) {
  const size_t smem = search_smem_bytes(a.cols, a.rows, a.n, step, a.prune != 0);
  if (search_tables_bytes(a.cols, a.rows, a.n) > 64 * 1024)
    fail(SC_ERR_SIZE, "CTU grid too large for the area tables");
  if (smem > (size_t)max_dynamic_smem((const void*)search_kernel<1, 1, false>()))
    fail(SC_ERR_SIZE, "search walk state (" + std::to_string(smem) +
                          " B of shared memory per block) exceeds the device limit");
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

// ---- pruned mode: work-item prefilter ---------------------------------------
// The walk's first test (walk_item, search_walk.cuh) is on the item's fixed
// width prefix alone: the window hulls must intersect and, for some frame of
// the group, the prefix's column bounds must pass the incumbent (step 1:
// (P << 32 | item) <= inc and < the frozen seed incumbent) or the budget
// (step 2: P <= budget).  An item that fails for every frame is skipped by
// every lane with no candidate scored, so dropping it before the launch
// changes nothing but the launch's per-item overhead.  The survivors keep
// their order (DeviceSelect is stable), so each warp's items still increase.
__global__ void k_item_filter(const WorkItem* __restrict__ items, uint32_t k0, uint32_t k1,
                              uint32_t offset, uint32_t stride, int cols, int rows, int n,
                              int max_area, int rstride, const int32_t* __restrict__ tab,
                              const uint32_t* __restrict__ lbm, int fpw, int frames, int step,
                              const uint64_t* inc, const uint64_t* seed_inc,
                              const int64_t* budget, uint32_t* idx, uint8_t* flag) {
  const uint32_t k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  const uint32_t item = offset + k * stride;
  const WorkItem wi = items[item];
  const int c = wi.c, d = wi.d;
  const int A = max_area + 1;
  const int rmax_c = min(n - c + 1, rows);
  bool ok = (n >= c) && (n <= c * rows);
  int x0 = 0, wl = 1, wh = max_area;
  const uint32_t* lb[SC_MAX_COLS];
  for (int i = 0; i < d && ok; ++i) {
    const int w = wi.w[i];
    wl = max(wl, tab[A + w * ((rows + rmax_c - 1) / rmax_c)]);  // ilo(w, rmax_c)
    wh = min(wh, w * rows);
    ok = wl <= wh;
    lb[i] = lbm + ((size_t)xw_of(cols, x0, w) * rstride + rmax_c) * fpw;
    x0 += w;
  }
  bool any = false;
  for (int f = 0; f < frames && ok && !any; ++f) {
    uint32_t P = 0;
    for (int i = 0; i < d; ++i) P = max(P, lb[i][f]);
    if (step == 1) {
      const uint64_t key = ((uint64_t)P << 32) | (uint32_t)item;
      any = key <= inc[f] && key < seed_inc[f];
    } else {
      any = (int64_t)P <= budget[f];
    }
  }
  idx[k - k0] = item;
  flag[k - k0] = any ? 1 : 0;
}

// Survivors of units [k0, k1) of this shard into `list` (in order) and their
// number into *count, all on the stream.
void item_filter_launch(sc_ctx* ctx, const SearchArgs& a, uint32_t k0, uint32_t k1, int fpw,
                        int frames, int step, const uint64_t* seed_inc, uint32_t* list,
                        uint32_t* count, cudaStream_t st) {
  const uint32_t m = k1 > k0 ? k1 - k0 : 0;
  ctx->flt_idx.ensure((size_t)(m + 1) * sizeof(uint32_t));
  ctx->flt_flag.ensure((size_t)(m + 1));
  const int rstride = std::min(a.n, a.rows) + 1;
  if (m) {
    SCB_LAUNCH(k_item_filter<<<(m + 255) / 256, 256, 0, st>>>(
        a.items, k0, k1, a.item_offset, a.item_stride, a.cols, a.rows, a.n, a.max_area, rstride,
        a.bmax, a.lbm, fpw, frames, step, a.inc, seed_inc, a.budget, ctx->flt_idx.as<uint32_t>(),
        ctx->flt_flag.as<uint8_t>()));
    SCB_CUDA(cudaGetLastError());
  }
  size_t tb = 0;
  SCB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ctx->flt_idx.as<uint32_t>(),
                                      ctx->flt_flag.as<uint8_t>(), list, count, (int)m, st));
  ctx->flt_temp.ensure(tb + 16);
  SCB_CUDA(cub::DeviceSelect::Flagged(ctx->flt_temp.p, tb, ctx->flt_idx.as<uint32_t>(),
                                      ctx->flt_flag.as<uint8_t>(), list, count, (int)m, st));
  count_launches(2);  // CUB select: init + sweep
}

void finalize_launch(int step, int n, int fpw, int frames_in_group, uint32_t n_warps,
                     const LaneBest* lanes, const uint8_t* snaps,
                     const unsigned long long* count, const unsigned long long* scored,
                     double lambda, const uint64_t* vals, const uint32_t* nvals, size_t nr,
                     FrameBest* out, int64_t* budget_out, DevBuf& scratch, cudaStream_t st) {
  // ~2 blocks' worth of lanes per part
  const int parts = (int)std::max<uint32_t>(1, std::min<uint32_t>(256, n_warps * 32 / fpw / 512));
  scratch.ensure((size_t)frames_in_group * parts * (sizeof(LaneBest) + sizeof(uint32_t)));
  LaneBest* pb = scratch.as<LaneBest>();
  uint32_t* pl = reinterpret_cast<uint32_t*>(pb + (size_t)frames_in_group * parts);
  SCB_LAUNCH(k_finalize_part<<<dim3(parts, frames_in_group), 256, 0, st>>>(step, n, fpw, n_warps, lanes, snaps,
                                                                pb, pl));
  SCB_CUDA(cudaGetLastError());
  SCB_LAUNCH(k_finalize<<<frames_in_group, 256, 0, st>>>(step, n, parts, frames_in_group, pb, pl, snaps, count,
                                              scored, lambda, vals, nvals, nr, out, budget_out));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
