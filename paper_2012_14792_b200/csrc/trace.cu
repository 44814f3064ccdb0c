// K4 (exhaustive step 1) as an interpreter of the plan's candidate trace
// (trace.cuh): build the trace once per plan, then every call streams it.
//
// Build (first call of a plan): one thread per work item runs the reference
// enumeration below its width prefix twice -- counting ops, candidates and
// skeletons, then writing them at scanned offsets -- and the trace is cut into
// chunks at SKEL ops and depth-0 pushes (k_trace_cuts / k_trace_chunks), each
// with the global ordinal of its first candidate; the rectangles the ops read
// are listed for the per-call ranking (k_trace_mark).
//
// Walk (every call): persistent 32-warp blocks take striped groups of
// adjacent chunks, then single chunks from an atomic counter; the 32 lanes of
// a warp are frames (lanes = FPW frames x J slots), so every op is
// warp-uniform: a warp fetches 32 ops with one coalesced load and broadcasts
// them with shuffles.  Per lane: the running maxima P[depth] (shared memory,
// [depth][lane]; P[0] and the stack top in registers), the best (time key,
// ordinal) and the tie threshold.  A PUSHL is handled together with its LEAF;
// a LEAF evaluates its candidates' times as one min-reduction over
// consecutive split-table keys; only a leaf that beats the lane's best is
// replayed in order.  Every candidate's time key is loaded; the candidate
// set, order, ordinals and first-in-order tie rule are the reference's
// (search.cpp:257-298).
//
// Finalize: per frame, the lexicographic minimum of (time key, ordinal) over
// the lanes; the winner's layout is rebuilt from its skeleton's ops
// (trace_layout) into the same FrameBest record the walk kernels produce.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"
#include "search_walk.cuh"
#include "trace.cuh"

namespace scb {

// ---- build -----------------------------------------------------------------------
__global__ void k_trace_count(const WorkItem* __restrict__ items, uint32_t n_items, int cols,
                              int rows, int n, double k, int covering, uint64_t* ops,
                              uint64_t* cands, uint64_t* skels) {
  const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  TraceCount c;
  trace_item(items[it], cols, rows, n, k, covering, c);
  ops[it] = c.ops;
  cands[it] = c.cands;
  skels[it] = c.skels;
}

__global__ void k_trace_emit(const WorkItem* __restrict__ items, uint32_t n_items, int cols,
                             int rows, int n, double k, int covering,
                             const uint64_t* __restrict__ op_off, const uint64_t* __restrict__ cand_off,
                             const uint64_t* __restrict__ skel_off, uint32_t* ops,
                             uint32_t* skel_pos, uint64_t* skel_ord) {
  const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  TraceWrite w;
  w.ops = ops + op_off[it];
  w.op_base = op_off[it];
  w.cand = cand_off[it];
  w.skel_pos = skel_pos + skel_off[it];
  w.skel_ord = skel_ord + skel_off[it];
  trace_item(items[it], cols, rows, n, k, covering, w);
}

// Chunks may start at a skeleton's SKEL op or, inside a skeleton, at any push
// of depth 0 (the path below it is empty: the state a walker needs there is
// the skeleton's SKEL + FIX prologue and the candidate ordinal).  Long
// skeletons (cfg3: up to 4,178 ops) are thus split over many warps instead of
// setting a one-warp critical path.
// cut[p] = 1 for a SKEL op or a depth-0 push; cnt[p] = candidates of a LEAF
__global__ void k_trace_cuts(const uint32_t* __restrict__ ops, uint64_t nops,
                             uint8_t* __restrict__ cut, uint32_t* __restrict__ cnt) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nops;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t op = ops[p];
    const uint32_t code = tr_code(op);
    cut[p] = (tr_is_push(op) && tr_small_of(op) == 0) || (code == kOpSkel && !tr_is_fix(op));
    cnt[p] = code == kOpLeaf ? (tr_leaf_cnt(op) ? (uint32_t)tr_leaf_cnt(op) : 1u) : 0u;
  }
}

// chunk c = {first op, end op, its skeleton's SKEL op, ordinal of its first
// candidate}: it starts at the first cut at or after c * size; record
// n_chunks is the sentinel {nops, nops, -, all candidates}
__global__ void k_trace_chunks(const uint32_t* __restrict__ cutpos, uint32_t ncut,
                               const uint32_t* __restrict__ ordp, const uint32_t* __restrict__ skel_pos,
                               uint32_t nskel, uint32_t nops, uint32_t ncands, uint32_t n_chunks,
                               uint32_t size, uint4* __restrict__ chunks) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_chunks) return;
  auto first_cut = [&](uint32_t cc) -> uint32_t {
    if (cc >= n_chunks) return nops;
    const uint64_t target = (uint64_t)cc * size;
    uint32_t lo = 0, hi = ncut;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (cutpos[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    return lo < ncut ? cutpos[lo] : nops;
  };
  const uint32_t start = first_cut(c), end = first_cut(c + 1);
  uint4 r = make_uint4(start, end, start, ncands);
  if (start < nops) {
    uint32_t lo = 0, hi = nskel;  // the last skeleton starting at or before `start`
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (skel_pos[mid] <= start) lo = mid + 1;
      else hi = mid;
    }
    r.z = skel_pos[lo - 1];
    r.w = ordp[start];
  }
  chunks[c] = r;
}

// ---- walk ------------------------------------------------------------------------
__device__ __noinline__ void trace_finalize_frame(const FinArgs& a, int f);
__device__ __noinline__ void trace_finalize2_frame(const FinArgs& a, int f);

struct TraceArgs {
  const uint32_t* ops;
  const uint4* chunks;        // [n_chunks + 1] {first op, end op, SKEL op, first ordinal}
  uint32_t n_chunks;
  uint32_t chunk_offset, chunk_stride;  // shard: chunks offset, offset + stride, ...
  uint32_t n_mine;            // chunks of this shard
  uint32_t groups_static;     // per block: groups of (warps per block) adjacent chunks taken in
  uint32_t k_static;          // stripes (= groups_static * blocks * warps); the rest dynamically
  uint32_t sm_major;
  uint32_t sm_count;          // blocks b, b + sm_count, ... (one SM's, in the first wave) take
                              // adjacent groups
  uint32_t* counter;
  const uint32_t* keys;       // [2][NR][FPW] time keys | split table of this frame group
  uint32_t nr;
  int depth_cap;              // P stack entries per lane
  uint64_t* lanes;            // [warps * 32] x {time key (u64), ordinal}
  uint32_t* done;             // fused finalize (one frame): blocks finished so far, or nullptr
  FinArgs fin;
};

// keys + off as one IMAD.WIDE (off = an op's pre-scaled key offset)
__device__ __forceinline__ const uint32_t* key_at(const uint32_t* base, uint32_t off) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(r) : "r"(off), "l"(base));
  return reinterpret_cast<const uint32_t*>(r);
}

// min over `cnt` consecutive split-table keys of one lane (stride FPW words)
template <int FPW>
__device__ __forceinline__ tkey leaf_min(const uint32_t* __restrict__ pv, int cnt) {
#define LD(i) __ldg(pv + (i) * FPW)
  // most leaves hold <= 8 heights: a three-level branch tree (warp-uniform)
  // into straight-line loads
  if (cnt <= 4) {
    if (cnt <= 2) {
      if (cnt == 1) return LD(0);
      return kmin(LD(0), LD(1));
    }
    if (cnt == 3) return umin3(LD(0), LD(1), LD(2));
    return kmin(umin3(LD(0), LD(1), LD(2)), LD(3));
  }
  if (cnt <= 6) {
    if (cnt == 5) return umin3(umin3(LD(0), LD(1), LD(2)), LD(3), LD(4));
    return kmin(umin3(LD(0), LD(1), LD(2)), umin3(LD(3), LD(4), LD(5)));
  }
  if (cnt == 7) return umin3(umin3(LD(0), LD(1), LD(2)), umin3(LD(3), LD(4), LD(5)), LD(6));
  tkey m = umin3(umin3(LD(0), LD(1), LD(2)), umin3(LD(3), LD(4), LD(5)), kmin(LD(6), LD(7)));
#pragma unroll 1
  for (int h = 8; h < cnt; ++h) m = kmin(m, LD(h));
  return m;
#undef LD
}

// Chunks reach the warps in two phases.  First each block walks its own
// stripes of the chunk sequence -- groups of (warps per block) ADJACENT
// chunks, handed to its warps through a shared-memory ticket: adjacent chunks
// share their columns' rectangles, so the warps of an SM hit each other's key
// lines in L1.  The last ~40 % of the chunks are taken one by one from a
// global counter (the dynamic tail that evens out the blocks).
// FUSE: a single-frame call (FPW 1) whose last block also finalizes.
template <int FPW, bool FUSE>
__global__ void __launch_bounds__(1024, 2) k_trace_walk(TraceArgs a) {
  constexpr int J = 32 / FPW;
  constexpr int SH = FPW == 32 ? 0 : FPW == 16 ? 1 : FPW == 8 ? 2 : FPW == 4 ? 3 : FPW == 2 ? 4 : 5;
  extern __shared__ uint32_t tr_sm[];
  __shared__ uint32_t s_ticket;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int f = lane % FPW, slot = lane / FPW;
  const int prow = a.depth_cap < 4 ? 4 : a.depth_cap;  // the records of the reduction fit
  uint32_t* P = tr_sm + (size_t)wib * prow * 32 + lane;  // P[d] at P[d * 32]
  // the best's LEAF op and height (rare writes)
  uint32_t* s_pos = tr_sm + (size_t)nw * prow * 32;
  uint32_t* s_hit = s_pos + blockDim.x;
  if (threadIdx.x == 0) s_ticket = 0;
  __syncthreads();
  // rt | rts of this lane's frame: an op's key is keys[(its offset field) >> SH]
  const uint32_t* __restrict__ keys = a.keys + f;
  asm volatile("" : "+l"(keys));  // keep the per-lane base in registers (no re-derivation per op)
  // lane state in registers: best key, its global ordinal (the trace holds
  // < 2^31 candidates) and the tie threshold; the best's op position and
  // height go to shared memory only when the best changes
  tkey best = kKeyInf;
  uint32_t best_ord = 0xffffffffu;
  while (true) {
    uint32_t k = 0;
    if (lane == 0) {
      const uint32_t t = atomicAdd(&s_ticket, 1u);
      const uint32_t g = t / (uint32_t)nw;
      // stripe position of this block: SM-major, so the blocks of one SM are neighbours
      const uint32_t bps = (gridDim.x + a.sm_count - 1) / a.sm_count;
      uint32_t bpos = (blockIdx.x % a.sm_count) * bps + blockIdx.x / a.sm_count;
      if (gridDim.x % a.sm_count || a.sm_major == 0) bpos = blockIdx.x;  // partial waves: plain order
      k = g < a.groups_static ? (g * gridDim.x + bpos) * (uint32_t)nw + t % (uint32_t)nw
                              : a.k_static + atomicAdd(a.counter, 1u);
    }
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= a.n_mine) break;
    const uint4 rec = __ldg(a.chunks + a.chunk_offset + k * a.chunk_stride);
    const uint32_t b = rec.x, e = rec.y;
    if (b >= e) continue;
    uint32_t ord = rec.w;  // global ordinal of the next candidate
    // ties: a candidate of this chunk precedes the lane's best iff the best
    // comes from a later ordinal; inside the chunk ordinals only grow
    tkey bcmp = (best != kKeyInf && best_ord > ord) ? best + 1 : best;
    // P[0] and P[ld] of the current path live in registers (P0, Pt): a PUSHL
    // reads P[ld - 1] (at Pl1) and leaves P[ld] in Pt for its LEAF(s)
    tkey P0 = 0, Pt = 0;
    const uint32_t* Pl1 = P;
    int nbw = 32;
    if (rec.z != b) {
      // the chunk starts inside a skeleton (at a depth-0 push): its SKEL + FIX
      // prologue (at most 1 + 16 ops) gives the leaf depth and P[0]
      const uint32_t pro = __ldg(a.ops + rec.z + lane);
      const int npro = __ffs(~__ballot_sync(0xffffffffu, tr_code(pro) == kOpSkel)) - 1;
      const int ld = tr_skel_ld(__shfl_sync(0xffffffffu, pro, 0));
      Pl1 = P + (ld > 0 ? ld - 1 : 0) * 32;
      for (int q = 1; q < npro; ++q)
        P0 = kmax(P0, __ldg(key_at(keys, tr_koff32(__shfl_sync(0xffffffffu, pro, q)) >> SH)));
      Pt = P0;
      P[0] = P0;
    }
    // a leaf's minimum against the lane's best; a winner is replayed in order
    // (the first minimum wins)
    auto leaf_tail = [&](tkey m, int cnt, const uint32_t* pv, uint32_t pos) {
      const tkey t = kmax(Pt, m);
      if (t < bcmp) {
        int hit = slot;
        for (int h = slot; h < cnt; h += J)
          if (kmax(Pt, __ldg(pv + h * FPW)) == t) {
            hit = h;
            break;
          }
        best = t;
        bcmp = t;
        best_ord = ord + (uint32_t)hit;
        s_pos[threadIdx.x] = pos;
        s_hit[threadIdx.x] = (uint32_t)hit;
      }
      ord += (uint32_t)cnt;
    };
    for (uint32_t p0 = b; p0 < e; p0 += (uint32_t)nbw) {
      const uint32_t mine = p0 + lane < e ? __ldg(a.ops + p0 + lane) : 0u;
      int nb = (int)min(32u, e - p0);
      // a PUSHL and its LEAF (the next op) stay in one fetch: a window that
      // would end on a PUSHL ends one op earlier
      if (tr_code(__shfl_sync(0xffffffffu, mine, nb - 1)) == kOpPushL) --nb;
      nbw = nb;
#pragma unroll 1
      for (int q = 0; q < nb; ++q) {
        uint32_t op = __shfl_sync(0xffffffffu, mine, q);
        uint32_t code = tr_code(op);
        if (__builtin_expect(code == kOpPushL, 1)) {
          // fused PUSHL + LEAF (the next op, in this fetch): the push's key
          // and the leaf's keys are all requested before any is consumed
          const tkey v = __ldg(key_at(keys, tr_koff32(op) >> SH));
          const tkey pl = *Pl1;
          op = __shfl_sync(0xffffffffu, mine, ++q);
          const int cnt = tr_leaf_cnt(op);  // >= 1 below a PUSHL
          const uint32_t* pv = key_at(keys, tr_koff32(op) >> SH);
          tkey m;
          if (J == 1) {
            m = leaf_min<FPW>(pv, cnt);
          } else {
            m = kKeyInf;
            for (int h = slot; h < cnt; h += J) m = kmin(m, __ldg(pv + h * FPW));
          }
          Pt = kmax(pl, v);
          leaf_tail(m, cnt, pv, p0 + q);
          continue;
        }
        if (code == kOpLeaf) {
          const int cnt = tr_leaf_cnt(op);
          if (cnt == 0) {  // the skeleton's single candidate
            if (slot == 0 && Pt < bcmp) {
              best = Pt;
              bcmp = Pt;
              best_ord = ord;
              s_pos[threadIdx.x] = p0 + q;
              s_hit[threadIdx.x] = 0;
            }
            ord += 1;
            continue;
          }
          const uint32_t* pv = key_at(keys, tr_koff32(op) >> SH);
          tkey m;
          if (J == 1) {
            m = leaf_min<FPW>(pv, cnt);
          } else {
            m = kKeyInf;
            for (int h = slot; h < cnt; h += J) m = kmin(m, __ldg(pv + h * FPW));
          }
          leaf_tail(m, cnt, pv, p0 + q);
        } else if (code == kOpPush) {
          const uint32_t d = (uint32_t)tr_small_of(op);
          P[(d + 1) * 32] = kmax(P[d * 32], __ldg(key_at(keys, tr_koff32(op) >> SH)));
        } else if (tr_is_fix(op)) {
          P0 = kmax(P0, __ldg(key_at(keys, tr_koff32(op) >> SH)));
          Pt = P0;
          P[0] = P0;
        } else {  // SKEL
          const int ld = tr_skel_ld(op);
          Pl1 = P + (ld > 0 ? ld - 1 : 0) * 32;
          P0 = 0;
          Pt = 0;
          P[0] = 0;
        }
      }
    }
  }
  // block-level reduction of the warps' lanes with the same lane index (same
  // frame and slot): {key << 32 | LEAF op, height << 32 | ordinal}; the
  // records take the place of the (now dead) P stacks
  __syncthreads();
  uint64_t* s_red0 = reinterpret_cast<uint64_t*>(tr_sm);
  uint64_t* s_red1 = s_red0 + blockDim.x;
  s_red0[threadIdx.x] = best == kKeyInf ? ~0ull : ((uint64_t)best << 32) | s_pos[threadIdx.x];
  s_red1[threadIdx.x] = best == kKeyInf ? ~0ull : ((uint64_t)s_hit[threadIdx.x] << 32) | best_ord;
  __syncthreads();
  if (wib == 0) {
    uint64_t k0 = s_red0[lane], k1 = s_red1[lane];
    for (int w = 1; w < nw; ++w) {
      const uint64_t a0 = s_red0[w * 32 + lane], a1 = s_red1[w * 32 + lane];
      if ((a0 >> 32) < (k0 >> 32) || ((a0 >> 32) == (k0 >> 32) && (uint32_t)a1 < (uint32_t)k1))
        k0 = a0, k1 = a1;
    }
    a.lanes[2 * ((size_t)blockIdx.x * 32 + lane)] = k0;
    a.lanes[2 * ((size_t)blockIdx.x * 32 + lane) + 1] = k1;
  }
  if constexpr (FUSE) {
    // single-frame call: the last block to finish reduces the blocks'
    // records and rebuilds the winner (no separate finalize launch)
    __shared__ uint32_t s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (s_last) {
      __threadfence();
      trace_finalize_frame(a.fin, 0);
    }
  }
}

// Largest index with vals[i] <= bits(b), -1 when none: a warp-wide 32-ary
// search (three rounds of independent loads instead of ~17 dependent ones).
// Called by one full warp; every lane returns the result.
__device__ __forceinline__ int64_t budget_key_warp(const uint64_t* __restrict__ vals, uint32_t n,
                                                   double b) {
  if (!(b >= 0.0)) return -1;
  const int lane = threadIdx.x & 31;
  const uint64_t bits = (uint64_t)__double_as_longlong(b);
  uint32_t lo = 0, hi = n;  // the first index with vals > bits lies in [lo, hi]
  while (hi - lo > 0) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t probe = lo + (uint32_t)lane * step;
    const bool le = probe < hi && vals[probe] <= bits;
    const uint32_t m = __ballot_sync(0xffffffffu, le);
    if (m == 0) {  // vals[lo] > bits
      hi = lo;
      break;
    }
    const int last = 31 - __clz(m);  // the last probe with vals <= bits
    const uint32_t nlo = lo + (uint32_t)last * step + 1;
    hi = min(hi, lo + (uint32_t)(last + 1) * step);
    lo = nlo;
  }
  return (int64_t)lo - 1;
}

// Warp-cooperative rebuild of the layout of the candidate at height
// `leafoff` of the LEAF op at `leafpos` (called by one full warp): its
// skeleton (32-ary search of the skeleton starts), the last PUSH of every
// depth before the LEAF (lane d owns depths d and d + 32) and the one-run
// columns (the FIX ops after the SKEL); lane 0 writes the snapshot.
__device__ void trace_rebuild(const uint32_t* __restrict__ ops, const uint32_t* __restrict__ skel_pos,
                              uint32_t nskel, uint32_t nr, int cols, int rows, uint32_t leafpos,
                              uint32_t leafoff, uint32_t* path, uint32_t* fixes, uint8_t* snap) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = nskel;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t probe = lo + (uint32_t)lane * step;
    const bool le = probe < hi && skel_pos[probe] <= leafpos;
    const uint32_t m = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(m);  // lane 0 always qualifies (skel_pos[lo] <= leafpos)
    const uint32_t nlo = lo + (uint32_t)last * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  const uint32_t b = skel_pos[lo];
  const int ld = tr_skel_ld(ops[b]);
  // The path's entry at depth d is the LAST push of depth d before the LEAF
  // (a LEAF is only emitted after every shallower depth was pushed again), so
  // the ops are scanned backwards from the LEAF, 32 at a time, until every
  // depth below ld is found -- a few windows, however long the skeleton is.
  uint32_t my0 = ~0u, my1 = ~0u;
  bool f0 = lane >= ld, f1 = lane + 32 >= ld;  // depths this lane still looks for
  for (uint32_t hi_p = leafpos; hi_p > b;) {
    const uint32_t lo_p = hi_p - b > 32u ? hi_p - 32u : b;
    const uint32_t mine = lo_p + lane < hi_p ? ops[lo_p + lane] : ~0u;
    const int nb = (int)(hi_p - lo_p);
    for (int q = nb - 1; q >= 0; --q) {
      const uint32_t op = __shfl_sync(0xffffffffu, mine, q);
      if (tr_is_push(op)) {
        const int d = tr_small_of(op);
        const uint32_t kidx = tr_kidx(op);
        const uint32_t idx = kidx >= nr ? kidx - nr : kidx;
        if (d == lane && !f0) my0 = idx, f0 = true;
        if (d == lane + 32 && !f1) my1 = idx, f1 = true;
      }
    }
    if (__all_sync(0xffffffffu, f0 && f1)) break;
    hi_p = lo_p;
  }
  path[lane] = my0;
  path[lane + 32] = my1;
  const uint32_t fop = b + 1 + lane < leafpos && lane < SC_MAX_COLS ? ops[b + 1 + lane] : 0u;
  const bool isfix = tr_is_fix(fop);
  const uint32_t fm = __ballot_sync(0xffffffffu, isfix);
  const int nfix = __ffs(~fm) - 1;       // consecutive FIXes from the start
  if (lane < nfix) fixes[lane] = tr_kidx(fop);
  __syncwarp();
  if (lane == 0) {
    const uint32_t lop = ops[leafpos];
    const int cnt = tr_leaf_cnt(lop);
    trace_snapshot(fixes, nfix, path, ld, cnt ? tr_kidx(lop) - nr + leafoff : ~0u, cols, rows,
                   snap);
  }
  __syncwarp();
}

// Per frame: min (key, ordinal) over the blocks' records of frame f; then
// warp 0 rebuilds the winner's layout: its skeleton (32-ary search of the
// skeleton starts for the LEAF op the walk recorded), the last PUSH of every
// depth before that LEAF (lane d owns depths d and d + 32) and the one-run
// columns (the FIX ops after the SKEL).  The step-2 budget as in k_finalize.
__device__ __noinline__ void trace_finalize_frame(const FinArgs& a, int f) {
  __shared__ uint64_t skey[256], sord[256];
  __shared__ uint32_t path[64], fixes[SC_MAX_COLS];
  const int fpw = a.fpw;
  uint64_t bk = ~0ull, bo = ~0ull;
  // (__ldcg: inside the walk kernel the records were written by other blocks)
  for (uint32_t li = threadIdx.x * fpw + f; li < a.n_lanes; li += blockDim.x * fpw) {
    const uint64_t k = __ldcg(a.lanes + 2 * li), o = __ldcg(a.lanes + 2 * li + 1);
    if ((k >> 32) < (bk >> 32) || ((k >> 32) == (bk >> 32) && (uint32_t)o < (uint32_t)bo))
      bk = k, bo = o;
  }
  skey[threadIdx.x] = bk;
  sord[threadIdx.x] = bo;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const uint64_t k = skey[threadIdx.x + s], o = sord[threadIdx.x + s];
      if ((k >> 32) < (skey[threadIdx.x] >> 32) ||
          ((k >> 32) == (skey[threadIdx.x] >> 32) && (uint32_t)o < (uint32_t)sord[threadIdx.x]))
        skey[threadIdx.x] = k, sord[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x >= 64) return;
  const int lane = threadIdx.x & 31;
  FrameBest* o = a.out + f;
  const uint64_t* fv = a.vals + (size_t)f * a.nr_vals;
  bk = skey[0];
  bo = sord[0];
  // step 1 keeps `t < best_t` from best_t = +inf (search.cpp:277-285)
  const bool found = bk != ~0ull && fv[bk >> 32] != 0x7ff0000000000000ull;
  if (threadIdx.x >= 32) {  // warp 1: step 2's budget, beside warp 0's layout rebuild
    if (found && a.budget_out) {
      const double tmin = __longlong_as_double((long long)fv[bk >> 32]);
      const int64_t bkey =
          budget_key_warp(fv, a.nvals[f], __dmul_rn(tmin, __dadd_rn(1.0, a.lambda)));
      if (lane == 0) a.budget_out[f] = bkey;
    }
    return;
  }
  if (lane == 0) {
    o->t = found ? fv[bk >> 32] : ~0ull;
    o->sse = __longlong_as_double(0x7ff0000000000000ll);
    o->item = found ? (uint32_t)bo : ~0ull;  // the global ordinal (shard merge orders by it)
    o->ord = 0;
    o->count = a.count;
    o->scored = a.count * (uint64_t)fpw;
    o->found = found ? 1 : 0;
  }
  if (!found) return;
  const uint32_t leafpos = (uint32_t)bk, leafoff = (uint32_t)(bo >> 32);
  trace_rebuild(a.ops, a.skel_pos, a.nskel, a.nr, a.cols, a.rows, leafpos, leafoff, path, fixes,
                o->snap);
}

__global__ void k_trace_finalize(FinArgs a) {
  if ((int)blockIdx.x < a.frames_in_group) trace_finalize_frame(a, (int)blockIdx.x);
}

// ---- step 2 ---------------------------------------------------------------------
// Subtree ends for the step-2 walk: skip[p] for a PUSH at p = the next op of
// depth <= its own (or the skeleton's end); for a SKEL = the skeleton's end.
// One thread per skeleton, a depth stack over its ops (once per plan).
__global__ void k_trace_skips(const uint32_t* __restrict__ ops, const uint32_t* __restrict__ skel_pos,
                              uint32_t nskel, uint32_t* __restrict__ skip) {
  const uint32_t sk = blockIdx.x * blockDim.x + threadIdx.x;
  if (sk >= nskel) return;
  const uint32_t b = skel_pos[sk], e = skel_pos[sk + 1];
  uint32_t open_pos[64];
  int open_d[64], top = 0;
  skip[b] = e;
  for (uint32_t p = b + 1; p < e; ++p) {
    const uint32_t op = ops[p];
    if (tr_is_push(op)) {
      const int d = tr_small_of(op);
      while (top > 0 && open_d[top - 1] >= d) skip[open_pos[--top]] = p;
      open_pos[top] = p;
      open_d[top++] = d;
    } else {
      skip[p] = p + 1;
    }
  }
  while (top > 0) skip[open_pos[--top]] = e;
}

struct Trace2Args {
  const uint32_t* ops;
  const uint32_t* skip;
  const uint4* chunks;       // [n_chunks + 1] {first op, end op, SKEL op, first ordinal}
  uint32_t n_chunks, chunk_offset, chunk_stride, n_mine;
  uint32_t* counter;
  const uint32_t* keys;      // [2][NR][FPW] time keys | split table of this frame group
  const double2* rsp;        // [NR][FPW] {slice SSE, SSE of the run's forced rest} (per call)
  const int64_t* budget;     // [FPW] largest key with time <= t_min * (1 + lambda), -1: none
  uint32_t nr;
  int depth_cap;
  uint64_t* lanes;           // per block lane: {sse bits, key << 32 | op, height << 32 | ordinal}
  uint32_t* done;            // fused finalize (one frame): blocks finished so far
  FinArgs fin;
};

// Step 2 (constrained_clustering_search, search.cpp:334-405) through the
// trace: per lane (frame), the running maxima P and the SSE prefix S of the
// current path (S folds the slices in slice order: leading one-run columns,
// then each multi-run column's runs and forced rest followed by the one-run
// columns right of it -- the FIX tags), and the (sse, t, ordinal) minimum
// over the candidates with t <= budget.  A subtree whose fixed slices already
// exceed every lane's budget is skipped through the skip table.
//
// Like the step-1 walk, the top of the stacks (P[ld], S[ld]) lives in
// registers and a PUSHL is processed together with its LEAF.  The tagged
// one-run columns' SSEs sit at the top end of the S stack (the path needs
// nl - 1 entries, the skeleton has n - nl - nmulti one-run columns: both fit
// depth_cap = n), their tags in a 64-bit uniform register (4 bits each); a
// candidate's loads ({key}, {sse, rest sse} as one 128-bit load) are issued
// unconditionally, two heights at a time, so dead lanes only predicate the
// offer.
template <int FPW, bool FUSE>
__global__ void __launch_bounds__(256) k_trace_walk2(Trace2Args a) {
  constexpr int J = 32 / FPW;
  constexpr int SH = FPW == 32 ? 0 : FPW == 16 ? 1 : FPW == 8 ? 2 : FPW == 4 ? 3 : FPW == 2 ? 4 : 5;
  extern __shared__ __align__(16) uint8_t tr2_sm[];
  __shared__ uint32_t s_pos[256], s_hit[256];
  __shared__ uint32_t s_cc[8][SC_MAX_SLICES];  // closed multi-run columns above each depth (uniform)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int f = lane % FPW, slot = lane / FPW;
  const size_t dstride = (size_t)a.depth_cap * 32;
  const int nw = blockDim.x >> 5;
  double* S = reinterpret_cast<double*>(tr2_sm) + (size_t)wib * dstride + lane;
  uint32_t* P = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(tr2_sm) + nw * dstride) +
                (size_t)wib * dstride + lane;
  double* Sfix = S + (size_t)(a.depth_cap - 1) * 32;  // tagged fix j at Sfix[-j * 32]
  uint32_t* Cc = s_cc[wib];
  const uint32_t* __restrict__ keys = a.keys + f;
  const double2* __restrict__ rsp = a.rsp + f;
  asm volatile("" : "+l"(keys));
  asm volatile("" : "+l"(rsp));
  const uint32_t nrf = a.nr * FPW;  // element offset of the split table
  const int64_t budget = a.budget[f];
  const uint32_t bp1 = budget < 0 ? 0u : (uint32_t)budget + 1u;  // live iff key < bp1
  double best_sse = __longlong_as_double(0x7ff0000000000000ll);
  tkey best_t = kKeyInf;
  uint32_t best_ord = 0xffffffffu;
  auto offer = [&](tkey t, double sse, uint32_t o, uint32_t pos, int hit) {
    if (sse < best_sse || (sse == best_sse && (t < best_t || (t == best_t && o < best_ord)))) {
      best_sse = sse;
      best_t = t;
      best_ord = o;
      s_pos[threadIdx.x] = pos;
      s_hit[threadIdx.x] = (uint32_t)hit;
    }
  };
  while (true) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(a.counter, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= a.n_mine) break;
    const uint4 rec = __ldg(a.chunks + a.chunk_offset + k * a.chunk_stride);
    const uint32_t b = rec.x, e = rec.y;
    if (b >= e) continue;
    uint32_t ord = rec.w;
    // a chunk that starts inside a skeleton (at a depth-0 push) first runs the
    // skeleton's SKEL + FIX prologue, then jumps to its first op
    bool pro = rec.z != b;
    // path state: P[0] / S[0] and the top P[ld] / S[ld] in registers
    tkey P0 = 0, Pt = 0;
    double S0 = 0.0, St = 0.0;
    int ld = 0;
    uint32_t ctop = 0;        // closed multi-run columns above the leaf depth
    uint64_t fxt = 0;         // tags of the tagged one-run columns, 4 bits each
    int nfx = 0, jl = 0;      // their number; first one with the highest tag so far
    uint32_t lasttag = 0;
    uint32_t base = rec.z - 32u, mine = 0;
    auto fetch = [&](uint32_t pp) {
      if (pp - base >= 32u) {
        base = pp;
        mine = pp + lane < e ? __ldg(a.ops + pp + lane) : 0u;
      }
      return __shfl_sync(0xffffffffu, mine, pp - base);
    };
    auto fold_fix = [&](double sv, uint32_t tag) {
      for (int j = 0; j < nfx; ++j)
        if (((uint32_t)(fxt >> (4 * j)) & 15u) == tag) sv = __dadd_rn(sv, Sfix[-j * 32]);
      return sv;
    };
    // the candidates of one LEAF op (cnt >= 1) under the path state above
    auto leaf = [&](uint32_t op, uint32_t pos) {
      const int cnt = tr_leaf_cnt(op);
      if (__any_sync(0xffffffffu, Pt < bp1)) {
        const uint32_t off = tr_koff32(op) >> SH;
        const uint32_t* pk = key_at(keys, off);
        const double2* pp = rsp + (off - nrf);
        // the one-run columns right of the last multi-run column
        const int j0 = lasttag == ctop + 1u ? jl : nfx;
        for (int h = slot; h < cnt; h += 2 * J) {
          const bool two = h + J < cnt;
          const tkey k0 = __ldg(pk + h * FPW);
          const double2 a0 = __ldg(pp + h * FPW);
          const tkey k1 = two ? __ldg(pk + (h + J) * FPW) : kKeyInf;
          const double2 a1 = two ? __ldg(pp + (h + J) * FPW) : make_double2(0.0, 0.0);
          double sv0 = __dadd_rn(__dadd_rn(St, a0.x), a0.y);
          double sv1 = __dadd_rn(__dadd_rn(St, a1.x), a1.y);
          for (int j = j0; j < nfx; ++j) {
            const double fv = Sfix[-j * 32];
            sv0 = __dadd_rn(sv0, fv);
            sv1 = __dadd_rn(sv1, fv);
          }
          const tkey t0 = kmax(Pt, k0), t1 = kmax(Pt, k1);
          if (t0 < bp1 && sv0 <= best_sse) offer(t0, sv0, ord + (uint32_t)h, pos, h);
          if (t1 < bp1 && sv1 <= best_sse) offer(t1, sv1, ord + (uint32_t)(h + J), pos, h + J);
        }
      }
      ord += (uint32_t)cnt;
    };
    uint32_t p = rec.z;
    while (p < e) {
      const uint32_t op = fetch(p);
      if (tr_is_push(op)) {
        const uint32_t d = (uint32_t)tr_small_of(op);
        const uint32_t off = tr_koff32(op) >> SH;
        const bool split = off >= nrf;  // the column's second-to-last run: its rest follows
        const tkey v = __ldg(key_at(keys, off));
        const double2* pr = rsp + (split ? off - nrf : off);
        const double r0 = __ldg(&pr->x);
        const double r1 = split ? __ldg(&pr->y) : 0.0;
        const uint32_t c = Cc[d] + (split ? 1u : 0u);
        const tkey Pn = kmax(P[d * 32], v);
        double sv = __dadd_rn(S[d * 32], r0);
        if (split) sv = fold_fix(__dadd_rn(sv, r1), c);
        if (tr_code(op) == kOpPushL) {  // stays in registers; its LEAF is the next op
          Pt = Pn;
          St = sv;
          ctop = c;
          leaf(fetch(p + 1), p + 1);
          p += 2;
          continue;
        }
        P[(d + 1) * 32] = Pn;
        S[(d + 1) * 32] = sv;
        Cc[d + 1] = c;  // one word per warp: every lane writes the same value
        __syncwarp();
        // no lane can meet its budget below: skip the subtree
        p = (a.skip && !__any_sync(0xffffffffu, Pn < bp1)) ? __ldg(a.skip + p) : p + 1;
        continue;
      }
      if (tr_code(op) == kOpLeaf) {
        if (tr_leaf_cnt(op) == 0) {  // the skeleton's single candidate
          if (slot == 0 && Pt < bp1) offer(Pt, St, ord, p, 0);
          ord += 1;
        } else {
          leaf(op, p);
        }
      } else if (tr_is_fix(op)) {
        const uint32_t off = tr_koff32(op) >> SH;
        const uint32_t tag = (uint32_t)tr_small_of(op);
        P0 = kmax(P0, __ldg(key_at(keys, off)));
        const double r0 = __ldg(&(rsp + off)->x);
        if (tag == 0) {
          S0 = __dadd_rn(S0, r0);
        } else {
          Sfix[-nfx * 32] = r0;
          fxt |= (uint64_t)tag << (4 * nfx);
          if (tag != lasttag) jl = nfx, lasttag = tag;
          ++nfx;
        }
        P[0] = P0;
        S[0] = S0;
        Pt = P0;
        St = S0;
      } else {  // SKEL
        ld = tr_skel_ld(op);
        P0 = 0, Pt = 0;
        S0 = 0.0, St = 0.0;
        P[0] = 0;
        S[0] = 0.0;
        Cc[0] = 0;
        __syncwarp();
        ctop = 0;
        fxt = 0;
        nfx = 0, jl = 0;
        lasttag = 0;
      }
      ++p;
      if (pro && tr_code(fetch(p)) != kOpSkel) {  // end of the prologue
        p = b;
        pro = false;
      }
    }
    (void)ld;
  }
  // block-level reduction of the warps' lanes with the same lane index (the
  // stacks are dead: their shared memory holds the records)
  __syncthreads();
  double* s_rsse = reinterpret_cast<double*>(tr2_sm);
  uint64_t* s_rk = reinterpret_cast<uint64_t*>(tr2_sm) + blockDim.x;
  uint64_t* s_ro = s_rk + blockDim.x;
  s_rsse[threadIdx.x] = best_sse;
  s_rk[threadIdx.x] = best_t == kKeyInf ? ~0ull : ((uint64_t)best_t << 32) | s_pos[threadIdx.x];
  s_ro[threadIdx.x] = best_t == kKeyInf ? ~0ull : ((uint64_t)s_hit[threadIdx.x] << 32) | best_ord;
  __syncthreads();
  if (wib == 0) {
    double bs = s_rsse[lane];
    uint64_t k0 = s_rk[lane], k1 = s_ro[lane];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      const double as = s_rsse[w * 32 + lane];
      const uint64_t a0 = s_rk[w * 32 + lane], a1 = s_ro[w * 32 + lane];
      if (a0 == ~0ull) continue;
      if (k0 == ~0ull || as < bs ||
          (as == bs && ((a0 >> 32) < (k0 >> 32) ||
                        ((a0 >> 32) == (k0 >> 32) && (uint32_t)a1 < (uint32_t)k1))))
        bs = as, k0 = a0, k1 = a1;
    }
    uint64_t* out = a.lanes + 3 * ((size_t)blockIdx.x * 32 + lane);
    out[0] = (uint64_t)__double_as_longlong(bs);
    out[1] = k0;
    out[2] = k1;
  }
  if constexpr (FUSE) {  // single-frame call: the last block to finish also finalizes
    __shared__ uint32_t s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (s_last) {
      __threadfence();
      trace_finalize2_frame(a.fin, 0);
    }
  }
}

// rsp[r][f] = {rs[r][f], rs[rest_of[r]][f]}: a run's SSE and the SSE of its
// forced rest side by side, so the step-2 walk reads both with one load.
__global__ void k_rest_sse(const double* __restrict__ rs, const uint32_t* __restrict__ rest_of,
                           size_t nr, int fpw, double2* __restrict__ rsp) {
  const size_t total = nr * (size_t)fpw;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / fpw, f = i % fpw;
    rsp[i] = make_double2(rs[i], rs[(size_t)rest_of[r] * fpw + f]);
  }
}

// Per frame: min (sse, key, ordinal) over the blocks' records, then the
// winner's layout (trace_rebuild).
__device__ __noinline__ void trace_finalize2_frame(const FinArgs& a, int f) {
  __shared__ double ssse[256];
  __shared__ uint64_t skey[256], sord[256];
  __shared__ uint32_t path[64], fixes[SC_MAX_COLS];
  const int fpw = a.fpw;
  auto less = [](double as, uint64_t a0, uint64_t a1, double bs, uint64_t b0, uint64_t b1) {
    if (a0 == ~0ull) return false;
    if (b0 == ~0ull) return true;
    if (as != bs) return as < bs;
    if ((a0 >> 32) != (b0 >> 32)) return (a0 >> 32) < (b0 >> 32);
    return (uint32_t)a1 < (uint32_t)b1;
  };
  double bs = 0.0;
  uint64_t bk = ~0ull, bo = ~0ull;
  // (__ldcg: inside the walk kernel the records were written by other blocks)
  for (uint32_t li = threadIdx.x * fpw + f; li < a.n_lanes; li += blockDim.x * fpw) {
    const uint64_t* r = a.lanes + 3 * (size_t)li;
    const uint64_t r0 = __ldcg(r), r1 = __ldcg(r + 1), r2 = __ldcg(r + 2);
    const double as = __longlong_as_double((long long)r0);
    if (less(as, r1, r2, bs, bk, bo)) bs = as, bk = r1, bo = r2;
  }
  ssse[threadIdx.x] = bs;
  skey[threadIdx.x] = bk;
  sord[threadIdx.x] = bo;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s &&
        less(ssse[threadIdx.x + s], skey[threadIdx.x + s], sord[threadIdx.x + s], ssse[threadIdx.x],
             skey[threadIdx.x], sord[threadIdx.x])) {
      ssse[threadIdx.x] = ssse[threadIdx.x + s];
      skey[threadIdx.x] = skey[threadIdx.x + s];
      sord[threadIdx.x] = sord[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  FrameBest* o = a.out + f;
  bs = ssse[0];
  bk = skey[0];
  bo = sord[0];
  const bool found = bk != ~0ull;
  if (lane == 0) {
    o->t = found ? a.vals[(size_t)f * a.nr_vals + (bk >> 32)] : ~0ull;
    o->sse = bs;
    o->item = found ? (uint32_t)bo : ~0ull;
    o->ord = 0;
    o->count = a.count;
    o->scored = a.count * (uint64_t)fpw;
    o->found = found ? 1 : 0;
  }
  if (!found) return;
  trace_rebuild(a.ops, a.skel_pos, a.nskel, a.nr, a.cols, a.rows, (uint32_t)bk,
                (uint32_t)(bo >> 32), path, fixes, o->snap);
}

__global__ void k_trace_finalize2(FinArgs a) {
  if ((int)blockIdx.x < a.frames_in_group) trace_finalize2_frame(a, (int)blockIdx.x);
}

// ---- host side -------------------------------------------------------------------

// Builds the trace into the plan's buffers.  Returns false (and builds
// nothing) when it would exceed `max_ops`.
bool trace_build_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                        double k, int covering, uint64_t max_ops, DevBuf& ops, DevBuf& skel_pos,
                        DevBuf& skel_ord, DevBuf& chunks, DevBuf& scratch, DevBuf& temp,
                        int sm_count, TraceHost* out, cudaStream_t st) {
  scratch.ensure((size_t)n_items * 6 * sizeof(uint64_t) + 64);
  uint64_t* c_ops = scratch.as<uint64_t>();
  uint64_t* c_cand = c_ops + n_items;
  uint64_t* c_skel = c_cand + n_items;
  uint64_t* o_ops = c_skel + n_items;
  uint64_t* o_cand = o_ops + n_items;
  uint64_t* o_skel = o_cand + n_items;
  const unsigned blocks = (n_items + 127) / 128;
  SCB_LAUNCH(k_trace_count<<<blocks, 128, 0, st>>>(d_items, n_items, cols, rows, n, k, covering, c_ops, c_cand,
                                        c_skel));
  SCB_CUDA(cudaGetLastError());
  size_t tb = 0;
  SCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, c_ops, o_ops, (int)n_items, st));
  temp.ensure(tb + 16);
  for (int i = 0; i < 3; ++i)
    SCB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, c_ops + (size_t)i * n_items,
                                           o_ops + (size_t)i * n_items, (int)n_items, st));
  count_launches(6);  // CUB scan: init + scan, three times
  uint64_t last[6];
  for (int i = 0; i < 3; ++i) {
    SCB_CUDA(cudaMemcpyAsync(&last[i], c_ops + (size_t)i * n_items + n_items - 1, 8,
                             cudaMemcpyDeviceToHost, st));
    SCB_CUDA(cudaMemcpyAsync(&last[3 + i], o_ops + (size_t)i * n_items + n_items - 1, 8,
                             cudaMemcpyDeviceToHost, st));
  }
  SCB_CUDA(cudaStreamSynchronize(st));
  const uint64_t tot_ops = last[0] + last[3], tot_cand = last[1] + last[4],
                 tot_skel = last[2] + last[5];
  if (tot_ops > max_ops || tot_ops >= (1ull << 32) || tot_skel >= (1ull << 32)) return false;
  ops.ensure(tot_ops * sizeof(uint32_t) + 128);
  skel_pos.ensure((tot_skel + 1) * sizeof(uint32_t));
  skel_ord.ensure((tot_skel + 1) * sizeof(uint64_t));
  SCB_LAUNCH(k_trace_emit<<<blocks, 128, 0, st>>>(d_items, n_items, cols, rows, n, k, covering, o_ops,
                                       o_cand, o_skel, ops.as<uint32_t>(), skel_pos.as<uint32_t>(),
                                       skel_ord.as<uint64_t>()));
  SCB_CUDA(cudaGetLastError());
  const uint32_t tail_pos = (uint32_t)tot_ops;
  SCB_CUDA(cudaMemcpyAsync(skel_pos.as<uint32_t>() + tot_skel, &tail_pos, 4, cudaMemcpyHostToDevice,
                           st));
  SCB_CUDA(cudaMemcpyAsync(skel_ord.as<uint64_t>() + tot_skel, &tot_cand, 8, cudaMemcpyHostToDevice,
                           st));
  // ~1024 chunks per SM (persistent warps take them dynamically: ~16 per
  // warp, so the kernel's tail is a small share of a warp's work), 16..8192
  // ops: small spaces get short chunks, so their few ops run on many warps
  // instead of one warp's serial chain of dependent loads
  uint64_t per_sm = 1024;
  if (const char* v = getenv("SLICECRAFT_B200_TRACE_CHUNKS")) per_sm = std::max(1, atoi(v));
  const uint64_t chunk_ops = std::min<uint64_t>(
      8192, std::max<uint64_t>(16, (tot_ops + (uint64_t)sm_count * per_sm - 1) /
                                       ((uint64_t)sm_count * per_sm)));
  const uint32_t n_chunks = (uint32_t)std::max<uint64_t>(1, (tot_ops + chunk_ops - 1) / chunk_ops);
  chunks.ensure(((size_t)n_chunks + 1) * sizeof(uint4));
  {
    // cut points (SKEL ops and depth-0 pushes), the ordinal of every op (a
    // scan of the LEAF counts; the trace holds < 2^31 candidates), the chunks
    DevBuf cutb, cntb, ordb, cutpos;
    cutb.ensure(tot_ops + 16);
    cntb.ensure(tot_ops * sizeof(uint32_t) + 16);
    ordb.ensure(tot_ops * sizeof(uint32_t) + 16);
    cutpos.ensure(tot_ops * sizeof(uint32_t) + 16);
    SCB_LAUNCH(k_trace_cuts<<<sm_count * 8, 256, 0, st>>>(ops.as<uint32_t>(), tot_ops,
                                                          cutb.as<uint8_t>(), cntb.as<uint32_t>()));
    SCB_CUDA(cudaGetLastError());
    size_t t1 = 0, t2 = 0;
    cub::CountingInputIterator<uint32_t> iota(0);
    uint32_t* d_ncut = cutpos.as<uint32_t>() + tot_ops;
    SCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, cntb.as<uint32_t>(), ordb.as<uint32_t>(),
                                           (int)tot_ops, st));
    SCB_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, iota, cutb.as<uint8_t>(),
                                        cutpos.as<uint32_t>(), d_ncut, (int)tot_ops, st));
    temp.ensure(std::max(t1, t2) + 16);
    SCB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, t1, cntb.as<uint32_t>(), ordb.as<uint32_t>(),
                                           (int)tot_ops, st));
    SCB_CUDA(cub::DeviceSelect::Flagged(temp.p, t2, iota, cutb.as<uint8_t>(),
                                        cutpos.as<uint32_t>(), d_ncut, (int)tot_ops, st));
    count_launches(4);
    uint32_t ncut = 0;
    SCB_CUDA(cudaMemcpyAsync(&ncut, d_ncut, 4, cudaMemcpyDeviceToHost, st));
    SCB_CUDA(cudaStreamSynchronize(st));
    SCB_LAUNCH(k_trace_chunks<<<(n_chunks + 1 + 255) / 256, 256, 0, st>>>(
        cutpos.as<uint32_t>(), ncut, ordb.as<uint32_t>(), skel_pos.as<uint32_t>(),
        (uint32_t)tot_skel, (uint32_t)tot_ops, (uint32_t)tot_cand, n_chunks, (uint32_t)chunk_ops,
        chunks.as<uint4>()));
    SCB_CUDA(cudaGetLastError());
    SCB_CUDA(cudaStreamSynchronize(st));
    cutb.release();
    cntb.release();
    ordb.release();
    cutpos.release();
  }
  SCB_CUDA(cudaStreamSynchronize(st));  // tail_pos / tot_cand live on this stack frame
  out->ops = tot_ops;
  out->cands = tot_cand;
  out->nskel = (uint32_t)tot_skel;
  out->n_chunks = n_chunks;
  return true;
}

// per warp: the P stack (>= 4 rows: the reduction's records reuse it) and the
// best's position / height words
size_t trace_smem_bytes(int depth_cap, int warps) {
  return (size_t)warps * (std::max(depth_cap, 4) * 32 + 64) * sizeof(uint32_t);
}

// Warps per block of the step-1 walk: 32 when the space gives every SM a few
// groups of 32 adjacent chunks (key lines shared in L1), else 8; fewer when
// deep stacks would not fit shared memory.  SLICECRAFT_B200_TRACE_WARPS
// overrides (A/B runs).
int trace_warps(int depth_cap, uint64_t chunks, int sm_count) {
  int nw = chunks >= (uint64_t)sm_count * 64 * 4 ? 32 : 8;
  if (const char* v = getenv("SLICECRAFT_B200_TRACE_WARPS")) {
    const int x = atoi(v);
    if (x == 1 || x == 2 || x == 4 || x == 8 || x == 16 || x == 32) nw = x;
  }
  const size_t lim = (size_t)max_dynamic_smem((const void*)k_trace_walk<32, false>);
  while (nw > 1 && trace_smem_bytes(depth_cap, nw) > lim) nw >>= 1;
  return nw;
}

// deep skeletons (n up to 64) need more than the 48 KB default per block
template <int F>
static void trace_attrs() {
  once_per_device((const void*)k_trace_walk<F, false>, [] {
    SCB_CUDA(cudaFuncSetAttribute(k_trace_walk<F, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dynamic_smem((const void*)k_trace_walk<F, false>)));
  });
}

int trace_blocks_per_sm(int fpw, int depth_cap, int warps) {
  int nb = 0;
  const size_t smem = trace_smem_bytes(depth_cap, warps);
#define OCC(F)                                                                                  \
  if (fpw == F) {                                                                               \
    trace_attrs<F>();                                                                           \
    SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_trace_walk<F, false>, 32 * warps,    \
                                                           smem));                              \
  }
  OCC(1) OCC(2) OCC(4) OCC(8) OCC(16) OCC(32)
#undef OCC
  return nb < 1 ? 1 : nb;
}

// fin / done: when given, the last block to finish runs the finalize of the
// call's single frame (blocks of 256 threads only; *done zeroed by the caller)
void trace_walk_launch(int fpw, int blocks, int warps, int sm_count, const uint32_t* ops,
                       const uint4* chunks, uint32_t n_chunks,
                       uint32_t rank, uint32_t world, uint32_t* counter, const uint32_t* keys,
                       uint32_t nr, int depth_cap, uint64_t* lanes, const FinArgs* fin,
                       uint32_t* done, cudaStream_t st) {
  TraceArgs a;
  if (fpw != 1 || warps != 8) fin = nullptr;  // the fused kernel: one frame, 256-thread blocks
  a.done = fin ? done : nullptr;
  if (fin) a.fin = *fin;
  else a.fin = FinArgs{};
  a.ops = ops;
  a.chunks = chunks;
  a.n_chunks = n_chunks;
  a.chunk_offset = rank;
  a.chunk_stride = world;
  a.n_mine = n_chunks > rank ? (n_chunks - rank + world - 1) / world : 0;
  // striped groups for the first ~60 % of the chunks, the rest dynamically
  const uint64_t per_round = (uint64_t)blocks * warps;
  int pct = 60;  // measured on cfg3 (profiles/ab_warps.sh): 88 -> 970 us, 70 -> 940, 60 -> 926, 50 -> 925
  if (const char* v = getenv("SLICECRAFT_B200_TRACE_STATIC")) pct = std::max(0, std::min(100, atoi(v)));
  a.sm_count = (uint32_t)sm_count;
  a.sm_major = 0;
  if (const char* v = getenv("SLICECRAFT_B200_TRACE_SMMAJOR")) a.sm_major = atoi(v);
  a.groups_static = (uint32_t)((uint64_t)a.n_mine * pct / 100 / per_round);
  a.k_static = (uint32_t)(a.groups_static * per_round);
  a.counter = counter;
  a.keys = keys;
  a.nr = nr;
  a.depth_cap = depth_cap;
  a.lanes = lanes;
  const size_t smem = trace_smem_bytes(depth_cap, warps);
  switch (fpw) {
#define L(F) \
  case F: SCB_LAUNCH(k_trace_walk<F, false><<<blocks, 32 * warps, smem, st>>>(a)); break;
    L(2) L(4) L(8) L(16) L(32)
#undef L
    case 1:
      if (a.done) {
        once_per_device((const void*)k_trace_walk<1, true>, [] {
          SCB_CUDA(cudaFuncSetAttribute(k_trace_walk<1, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        max_dynamic_smem((const void*)k_trace_walk<1, true>)));
        });
        SCB_LAUNCH(k_trace_walk<1, true><<<blocks, 32 * warps, smem, st>>>(a));
      } else {
        SCB_LAUNCH(k_trace_walk<1, false><<<blocks, 32 * warps, smem, st>>>(a));
      }
      break;
    default: fail(SC_ERR_INTERNAL, "bad frames-per-warp");
  }
  SCB_CUDA(cudaGetLastError());
}

void trace_finalize_launch(const FinArgs& fa, cudaStream_t st) {
  SCB_LAUNCH(k_trace_finalize<<<fa.frames_in_group, 256, 0, st>>>(fa));
  SCB_CUDA(cudaGetLastError());
}

// ---- the rectangles a plan's candidates use ---------------------------------------
// Every rectangle that is a slice of some candidate: the keys the ops read
// (rt entries directly; a split-table entry stands for the run and its forced
// rest).  Under the area test most rectangles of a grid are never a slice
// (cfg3: 32 % are), so the per-call time-key ranking (rank.cu) only ranks
// these; the others keep the key "infinite", which no candidate reads.
__global__ void k_trace_mark(const uint32_t* __restrict__ ops, uint64_t nops, uint32_t nr,
                             uint8_t* __restrict__ used_rt, uint8_t* __restrict__ used_rts) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nops;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t op = ops[p];
    const uint32_t kidx = tr_kidx(op);
    if (tr_is_push(op)) {
      if (kidx >= nr) used_rts[kidx - nr] = 1;
      else used_rt[kidx] = 1;
    } else if (tr_code(op) == kOpLeaf) {
      const int cnt = tr_leaf_cnt(op);
      for (int i = 0; i < cnt; ++i) used_rts[kidx - nr + i] = 1;
    } else if (tr_is_fix(op)) {
      used_rt[kidx] = 1;
    }
  }
}

__global__ void k_trace_used_close(int rows, uint32_t nr, uint8_t* __restrict__ used_rt,
                                   const uint8_t* __restrict__ used_rts) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr || !used_rts[idx]) return;
  const int nyh = rows * (rows + 1) / 2;
  const int xw = (int)(idx / (uint32_t)nyh), yh = (int)(idx % (uint32_t)nyh);
  int y0 = 0;
  while (y0 + 1 < rows && tr_yh(rows, y0 + 1, 1) <= yh) ++y0;
  const int h = yh - tr_yh(rows, y0, 1) + 1;
  used_rt[idx] = 1;
  if (y0 + h < rows) used_rt[(uint32_t)(xw * nyh + tr_yh(rows, y0 + h, rows - y0 - h))] = 1;
}

// The ascending lists of used rectangle indices and of the rectangles whose
// split-table entry is read (once per plan); returns the first list's length,
// the second's in *n_split.
uint32_t trace_used_device(const uint32_t* ops, uint64_t nops, int rows, uint32_t nr, DevBuf& used,
                           DevBuf& used_split, uint32_t* n_split, DevBuf& scratch, DevBuf& temp,
                           int sm_count, cudaStream_t st) {
  scratch.ensure((size_t)nr * 2 + 16);
  uint8_t* f_rt = scratch.as<uint8_t>();
  uint8_t* f_rts = f_rt + nr;
  SCB_CUDA(cudaMemsetAsync(f_rt, 0, (size_t)nr * 2, st));
  SCB_LAUNCH(k_trace_mark<<<sm_count * 8, 256, 0, st>>>(ops, nops, nr, f_rt, f_rts));
  SCB_CUDA(cudaGetLastError());
  SCB_LAUNCH(k_trace_used_close<<<(nr + 255) / 256, 256, 0, st>>>(rows, nr, f_rt, f_rts));
  SCB_CUDA(cudaGetLastError());
  used.ensure((size_t)nr * sizeof(uint32_t) + 16);
  uint32_t* d_count = used.as<uint32_t>() + nr;
  size_t tb = 0;
  cub::CountingInputIterator<uint32_t> iota(0);
  SCB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, f_rt, used.as<uint32_t>(), d_count,
                                      (int)nr, st));
  temp.ensure(tb + 16);
  SCB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, iota, f_rt, used.as<uint32_t>(), d_count,
                                      (int)nr, st));
  count_launches(2);  // CUB select: init + sweep
  used_split.ensure((size_t)nr * sizeof(uint32_t) + 16);
  uint32_t* d_count2 = used_split.as<uint32_t>() + nr;
  SCB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, iota, f_rts, used_split.as<uint32_t>(), d_count2,
                                      (int)nr, st));
  count_launches(2);
  uint32_t n = 0;
  SCB_CUDA(cudaMemcpyAsync(&n, d_count, 4, cudaMemcpyDeviceToHost, st));
  SCB_CUDA(cudaMemcpyAsync(n_split, d_count2, 4, cudaMemcpyDeviceToHost, st));
  SCB_CUDA(cudaStreamSynchronize(st));
  return n;
}

// ---- step 2 host side --------------------------------------------------------------
void trace_skips_device(const uint32_t* ops, const uint32_t* skel_pos, uint32_t nskel,
                        uint32_t* skip, cudaStream_t st) {
  if (nskel == 0) return;
  SCB_LAUNCH(k_trace_skips<<<(nskel + 127) / 128, 128, 0, st>>>(ops, skel_pos, nskel, skip));
  SCB_CUDA(cudaGetLastError());
}

// Per-warp stacks (S doubles, P and C words) of depth_cap entries x 32 lanes;
// deep plans (n up to 64) run fewer warps per block to fit shared memory.
size_t trace2_warp_bytes(int depth_cap) {
  return (size_t)depth_cap * 32 * (sizeof(double) + sizeof(uint32_t));
}
int trace2_warps(int depth_cap) {
  const int lim = max_dynamic_smem((const void*)k_trace_walk2<32, false>);
  return std::max(1, std::min(8, (int)(lim / trace2_warp_bytes(depth_cap))));
}
size_t trace2_smem_bytes(int depth_cap) {
  return (size_t)trace2_warps(depth_cap) * trace2_warp_bytes(depth_cap);
}

template <int F>
static void trace2_attrs() {
  once_per_device((const void*)k_trace_walk2<F, false>, [] {
    SCB_CUDA(cudaFuncSetAttribute(k_trace_walk2<F, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dynamic_smem((const void*)k_trace_walk2<F, false>)));
  });
}

int trace2_blocks_per_sm(int fpw, int depth_cap) {
  int nb = 0;
  const size_t smem = trace2_smem_bytes(depth_cap);
#define OCC(F)                                                                                   \
  if (fpw == F) {                                                                                \
    trace2_attrs<F>();                                                                           \
    SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_trace_walk2<F, false>,              \
                                                           32 * trace2_warps(depth_cap), smem)); \
  }
  OCC(1) OCC(2) OCC(4) OCC(8) OCC(16) OCC(32)
#undef OCC
  return nb < 1 ? 1 : nb;
}

// rss = {sse, sse of the forced rest} pairs of one frame group (k_rest_sse)
void rest_pairs_device(const double* rs, const uint32_t* rest_of, uint32_t nr, int fpw, double* rss,
                       int sm_count, cudaStream_t st) {
  const size_t total = (size_t)nr * fpw;
  const unsigned gb = (unsigned)std::min<size_t>((total + 255) / 256, (size_t)sm_count * 8);
  SCB_LAUNCH(k_rest_sse<<<gb, 256, 0, st>>>(rs, rest_of, nr, fpw, reinterpret_cast<double2*>(rss)));
  SCB_CUDA(cudaGetLastError());
}

void trace_walk2_launch(int fpw, int blocks, const uint32_t* ops, const uint32_t* skip,
                        const uint4* chunks, uint32_t n_chunks, uint32_t rank,
                        uint32_t world, uint32_t* counter, const uint32_t* keys, const double* rs,
                        const uint32_t* rest_of, double* rss, const int64_t* budget, uint32_t nr,
                        int depth_cap, uint64_t* lanes, int sm_count, bool gather,
                        const FinArgs* fin, uint32_t* done, cudaStream_t st) {
  if (gather) rest_pairs_device(rs, rest_of, nr, fpw, rss, sm_count, st);
  Trace2Args a;
  a.ops = ops;
  a.skip = skip;
  a.chunks = chunks;
  a.n_chunks = n_chunks;
  a.chunk_offset = rank;
  a.chunk_stride = world;
  a.n_mine = n_chunks > rank ? (n_chunks - rank + world - 1) / world : 0;
  a.counter = counter;
  a.keys = keys;
  a.rsp = reinterpret_cast<const double2*>(rss);
  a.budget = budget;
  a.nr = nr;
  a.depth_cap = depth_cap;
  a.lanes = lanes;
  const size_t smem = trace2_smem_bytes(depth_cap);
  const int threads = 32 * trace2_warps(depth_cap);
  if (fpw != 1 || threads != 256) fin = nullptr;  // the fused kernel: one frame, 256-thread blocks
  a.done = fin ? done : nullptr;
  a.fin = fin ? *fin : FinArgs{};
  switch (fpw) {
#define L(F) \
  case F: SCB_LAUNCH(k_trace_walk2<F, false><<<blocks, threads, smem, st>>>(a)); break;
    L(2) L(4) L(8) L(16) L(32)
#undef L
    case 1:
      if (fin) {
        once_per_device((const void*)k_trace_walk2<1, true>, [] {
          SCB_CUDA(cudaFuncSetAttribute(k_trace_walk2<1, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        max_dynamic_smem((const void*)k_trace_walk2<1, true>)));
        });
        SCB_LAUNCH(k_trace_walk2<1, true><<<blocks, threads, smem, st>>>(a));
      } else {
        SCB_LAUNCH(k_trace_walk2<1, false><<<blocks, threads, smem, st>>>(a));
      }
      break;
    default: fail(SC_ERR_INTERNAL, "bad frames-per-warp");
  }
  SCB_CUDA(cudaGetLastError());
}

// true when trace_walk2_launch will run the fused (walk + finalize) kernel
bool trace_walk2_fuses(int fpw, int depth_cap) {
  return fpw == 1 && 32 * trace2_warps(depth_cap) == 256;
}

void trace_finalize2_launch(const FinArgs& fa, cudaStream_t st) {
  SCB_LAUNCH(k_trace_finalize2<<<fa.frames_in_group, 256, 0, st>>>(fa));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
