// Shared declarations of the B200 TRS partitioner core (C-ABI implementation).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "plan.h"
#include "slicecraft_b200.h"

namespace scb {

// ---- errors ----------------------------------------------------------------
// Exceptions never cross the C ABI: every entry point catches scb::Fail and
// maps it to its sc_status plus the thread-local message (sc_last_error).
struct Fail {
  sc_status status;
  std::string msg;
};
[[noreturn]] inline void fail(sc_status s, const std::string& m) { throw Fail{s, m}; }

#define SCB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      ::scb::fail(SC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---- kernel-launch accounting ---------------------------------------------------
// Every kernel launch of the library goes through SCB_LAUNCH, which counts it
// (sc_kernel_launches).  CUB calls add their kernels by count_launches(n); a
// CUDA-graph replay adds the launches counted while the graph was captured.
uint64_t& launch_counter();  // process-wide (api.cu); host-side, one writer per stream of calls
inline void count_launches(uint64_t n) { launch_counter() += n; }
#define SCB_LAUNCH(...)          \
  do {                           \
    ::scb::count_launches(1);    \
    __VA_ARGS__;                 \
  } while (0)

// ---- per-device kernel attributes ---------------------------------------------
// cudaFuncSetAttribute acts on the current device only, so an opt-in (e.g. the
// dynamic shared-memory limit) is applied once per (device, kernel), under a
// lock: a process may drive several GPUs from several host threads.
template <typename F>
void once_per_device(const void* kernel, F&& set) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  SCB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kernel})) return;
  set();
  done.insert({dev, kernel});
}
// The device's opt-in shared-memory limit per block (227 KB on B200).
inline int smem_optin_bytes() {
  int dev = 0, v = 0;
  SCB_CUDA(cudaGetDevice(&dev));
  SCB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return v;
}
// The most dynamic shared memory a kernel may opt into: the opt-in limit
// minus its static shared memory.
inline int max_dynamic_smem(const void* kernel) {
  cudaFuncAttributes fa;
  SCB_CUDA(cudaFuncGetAttributes(&fa, kernel));
  return smem_optin_bytes() - (int)fa.sharedSizeBytes;
}

// ---- geometry --------------------------------------------------------------
inline int cell_w(const sc_grid& g, int x) {
  int r = g.frame_width - x * g.ctu_size;
  return r < g.ctu_size ? r : g.ctu_size;
}
inline int cell_h(const sc_grid& g, int y) {
  int r = g.frame_height - y * g.ctu_size;
  return r < g.ctu_size ? r : g.ctu_size;
}
// Rectangle numbering shared by every table:
//   rect(x0,w,y0,h) = xw(x0,w) * NYH + yh(y0,h)
__host__ __device__ inline int xw_index(int cols, int x0, int w) {
  return x0 * cols - (x0 * (x0 - 1)) / 2 + (w - 1);
}
__host__ __device__ inline int yh_index(int rows, int y0, int h) {
  return y0 * rows - (y0 * (y0 - 1)) / 2 + (h - 1);
}
inline int n_xw(int cols) { return cols * (cols + 1) / 2; }
inline int n_yh(int rows) { return rows * (rows + 1) / 2; }

// ---- device buffers ----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    SCB_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    SCB_CUDA(cudaMallocHost(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ---- search plan (frame-independent; cached per grid+config) ----------------

struct PlanKey {
  int cols, rows, n, maxc, coverage;
  double k;
  bool operator==(const PlanKey& o) const {
    return cols == o.cols && rows == o.rows && n == o.n && maxc == o.maxc &&
           coverage == o.coverage && k == o.k;
  }
};

struct Plan {
  PlanKey key{};
  std::vector<WorkItem> items;
  std::vector<int32_t> bmax;  // bmax | aneed | mstar tables (api.cu get_plan)
  bool pathological = false;  // some single area fails the test (k ~ 1)
  uint32_t seed_items = 0;    // pruned mode: items of the seeding phase
  bool have_count = false;    // exact DP count computed (pruned mode)
  // exhaustive step 1 schedule: the first call measures each item's walk
  // cost, later calls take the items in decreasing cost (shorter tail)
  int order_state = 0;        // 0: measure, 1: measured (copy pending), 2: ordered
  uint32_t order_rank = 0, order_world = 1;  // the shard the order belongs to
  DevBuf d_order, d_cost;
  unsigned __int128 count = 0;
  DevBuf d_items, d_bmax;
  bool uploaded = false;
  // exhaustive step 1 as a trace interpreter (trace.cu): the family's
  // candidate trace, its skeleton starts (op index, first ordinal) and chunks
  int trace_state = 0;  // 0: not built, 1: built, -1: not used for this plan
  uint64_t trace_ops = 0, trace_cands = 0;
  uint32_t trace_nskel = 0, trace_chunks = 0;
  uint64_t trace_shard_key = ~0ull, trace_shard_cands = 0;  // candidates of one shard
  DevBuf tr_ops, tr_skel_pos, tr_skel_ord;
  DevBuf tr_chunks;       // uint4 {first op, end op, SKEL op, first ordinal} per chunk + sentinel
  DevBuf tr_skip;         // step 2: subtree ends (trace.cu k_trace_skips)
  DevBuf tr_used;         // ascending indices of the rectangles the candidates use
  uint32_t n_used = 0;    // (0: unknown -- every rectangle is ranked)
  DevBuf tr_used_split;   // the rectangles whose split-table entry the candidates read
  uint32_t n_used_split = 0;
  bool have_skip = false;
  // step 2's walk per lambda, measured on the first call (api.cu enqueue_step)
  std::vector<std::pair<double, int>> step2_choice;
  // candidate stream (enumerate.cu): per-item counts, their offsets, total
  DevBuf d_enum_counts, d_enum_offsets;
  bool have_enum = false;
  uint64_t enum_total = 0;
};

// Per-lane best record written by the search kernels (one per lane of every
// persistent warp); reduced per frame by the finalize kernel.
struct LaneBest {
  uint64_t t;      // f64 bits of the best time (non-negative => monotone)
  double sse;      // step 2 key
  uint64_t item;   // work-item index
  uint64_t ord;    // ordinal of the candidate inside the item
};
constexpr int kSnapBytes = 96;  // W[16] R[16] H[64], bytes

// Arguments of the search kernels (search.cu), filled by api.cu.
struct SearchArgs {
  int cols, rows, n, nyh, max_area, coverage, pathological, prune;
  const WorkItem* items;
  uint32_t n_items;       // items of this shard: k in [k_begin, n_items)
  uint32_t k_begin;       // first local item index of this launch
  int resume;             // lanes continue from the LaneBest left by a previous launch
  uint32_t item_offset;   // global index = offset + k * stride
  uint32_t item_stride;
  uint32_t* counter;
  const int32_t* bmax;    // bmax[A] | aneed[A] | mstar[(cols+1)*(rows+1)], A = max_area+1
  const uint32_t* rt;     // [NR][FPW] time keys (rank.cu), this frame group
  const uint32_t* rts;    // [NR][FPW] split table (run + forced rest of its column)
  const double* rs;       // [NR][FPW] SSE (step 2)
  const int64_t* budget;  // [FPW] step-2 budget keys (-1: nothing feasible)
  LaneBest* lanes;        // [warps * 32]
  uint8_t* snaps;         // [warps * 32][kSnapBytes]
  unsigned long long* count_out;
  unsigned long long* scored_out;  // candidate-frame scores actually evaluated
  const uint32_t* lbr;             // pruned mode: column lower bounds (search_walk.cuh)
  const uint32_t* lbm;
  uint64_t* inc;                   // pruned mode: shared step-1 incumbent [FPW] (t << 32 | item)
  const uint64_t* seed_inc;        // pruned mode, phase B: incumbent frozen after phase A
  uint64_t* sse_inc;               // pruned step 2: shared SSE incumbent [FPW] (f64 bits)
  const uint32_t* order;           // exhaustive step 1: item k -> work item (or nullptr)
  int split_g, split_depth;        // pruned mode: warps per work item (WalkEnv)
  uint32_t* cost;                  // per work item: walk cycles / 64 (or nullptr)
  const uint32_t* n_items_dev;     // pruned mode: surviving items in `order` (device count;
                                   // n_items = count * split_g, k from 0), or nullptr
};

// Device-side per-frame result written by finalize.
struct FrameBest {
  uint64_t t;
  double sse;
  uint64_t item;
  uint64_t ord;
  uint64_t count;
  uint64_t scored;
  uint8_t snap[kSnapBytes];
  int32_t found;
  int32_t pad;
};

// What the per-frame finalize needs (k_trace_finalize); a single-frame call
// runs it inside the walk kernel, in the last block to finish.
struct FinArgs {
  int fpw, frames_in_group;
  uint32_t n_lanes;
  const uint64_t* lanes;
  const uint32_t* ops;
  const uint32_t* skel_pos;
  uint32_t nskel, nr;
  int cols, rows;
  uint64_t count;
  double lambda;
  const uint64_t* vals;
  const uint32_t* nvals;
  size_t nr_vals;
  FrameBest* out;
  int64_t* budget_out;
};
// Size of a plan's candidate trace (trace.cu).
struct TraceHost {
  uint64_t ops = 0, cands = 0;
  uint32_t nskel = 0, n_chunks = 0;
};

// Verdict of the device post-check of one partition (validate.cu).
struct VCheck {
  int32_t status;  // SC_OK, SC_ERR_OVERLAP, SC_ERR_COVERAGE, SC_ERR_STRUCTURE
                   // (SC_ERR_GEOMETRY: a result snapshot that does not decode)
  int32_t a, b;    // overlap: owner id, claiming id; structure: slice id
  int32_t x, y;    // overlap / coverage: the cell
};

}  // namespace scb

// The opaque context behind sc_ctx*.
struct sc_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;
  cudaStream_t user_stream = nullptr;
  cudaEvent_t ev[11] = {};  // [10]: the side stream's join point
  cudaEvent_t ev_s2[3] = {};   // step-2 walk timing on the first call of a (plan, lambda)
  bool s2_pending = false;
  double s2_lambda = 0.0;
  scb::Plan* s2_plan = nullptr;
  double timings[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int shard_rank = 0, shard_world = 1;
  // the exchange between shards when the library owns it (sc_comm_init_*):
  // 0 none (per-shard results, merged by the caller), 1 NCCL, 2 host callback
  int comm_kind = 0;
  void* nccl_comm = nullptr;  // ncclComm_t
  sc_allgather_fn comm_fn = nullptr;
  void* comm_user = nullptr;
  scb::DevBuf comm_buf, gtmin;
  // staging / tables
  scb::DevBuf luma, records, est, sat, rect_t, rect_s, rt_search, rs_search, usat;
  // rt_search: the time keys [groups][rt | rts][rect][fpw] (rank.cu, split table)
  scb::DevBuf lanes, snaps, frame_best, counter, budget, scratch, dec, lbr, lbm, inc, seed_inc;
  scb::DevBuf sse_inc;
  // the time-table phase (K2 + K3 + ranks + split table, ~20 launches) as a
  // CUDA graph, replayed while the call shape and buffers repeat (api.cu)
  std::vector<uintptr_t> tt_key, tt_prev_key;
  cudaGraphExec_t tt_exec = nullptr;
  uint64_t tt_launches = 0;  // kernels in the captured time-table phase
  bool pairs_on_side = false;  // this call: the side stream gathers the step-2 trace walk's pairs
  // the key table whose unused rectangles currently hold the "infinite" key (rank.cu)
  const void* rk_inf_keys = nullptr;
  const void* rk_inf_used = nullptr;
  size_t rk_inf_nu = 0, rk_inf_words = 0;
  scb::DevBuf rt_bits, vals, nvals, budget_f64;                       // time keys (rank.cu)
  scb::DevBuf rk_idx, rk_sorted, rk_flags, rk_offsets, rk_temp, rk_bits_c;  // rank.cu scratch
  scb::DevBuf flt_idx, flt_flag, flt_list, flt_count, flt_temp;      // item filter (search.cu)
  // device post-check of the returned partitions (validate.cu): CTU -> slice
  // id maps [2][frames][cells] of the last search, owner scratch, verdicts
  scb::DevBuf slice_maps, owner, vcheck, val_in, enum_out, enum_temp;
  scb::DevBuf rest_of;  // [NR] forced rest of each run, per decode-table grid (step-2 trace)
  scb::DevBuf rss;      // [NR][FPW] SSE of each run's forced rest (step-2 trace, per group)
  scb::DevBuf fin_scratch;  // two-level finalize partials (search.cu)
  scb::HostBuf h_vcheck;
  int maps_frames[2] = {0, 0};
  size_t maps_cells = 0;
  int dec_cols = -1, dec_rows = -1;
  scb::HostBuf h_stage, h_records, h_frame_best, h_budget, h_luma;  // h_luma: YUV reads
  std::vector<scb::Plan*> plans;
  // last step results (for shard export)
  std::vector<scb::FrameBest> last_best[2];
  uint64_t last_leaves[2] = {0, 0};
  bool last_pruned = false;  // last search ran in SC_MODE_PRUNED (DP counts)
  int last_fpw = 1;          // frames per warp of the last search (leaf counters)
  uint64_t last_count_hi[2] = {0, 0};  // high bits of this shard's DP count per step
  int diag_step = 0;         // diagnostics builds only
  ~sc_ctx();
};
