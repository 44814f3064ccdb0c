// C-ABI entry points (include/slicecraft_b200.h) and the host-side planner.
//
// Host work here is O(cells) or O(items) bookkeeping — geometry, validation,
// the frame-independent work-item plan, the area-threshold table — plus the
// CUDA launches.  No candidate is scored on the host.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "common.cuh"

namespace scb {
uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}
}  // namespace scb

namespace scb {
// kernels (texture.cu, tables.cu, search.cu)
void texture_moments_device(const void* d_luma, int bps, int W, int H, size_t pitch,
                            size_t fstride, int ctu, int frames, int cols, int rows,
                            sc_ctu_record* d_out, cudaStream_t st);
void split_table_device(uint32_t* d_keys, int cols, int rows, int groups, int fpw, int sm_count,
                        const uint32_t* list, size_t nl, cudaStream_t st);
uint32_t trace_used_device(const uint32_t* ops, uint64_t nops, int rows, uint32_t nr, DevBuf& used,
                           DevBuf& used_split, uint32_t* n_split, DevBuf& scratch, DevBuf& temp,
                           int sm_count, cudaStream_t st);
void rank_times_device(sc_ctx* ctx, const uint64_t* bits_fm, size_t nr, int frames, int fpw,
                       uint32_t* keys, uint64_t* vals, uint32_t* nvals, const uint32_t* used,
                       size_t nu, size_t groups, cudaStream_t st);
void budget_keys_device(const double* d_budgets, const uint64_t* vals, const uint32_t* nvals,
                        size_t nr, int frames, int64_t* out, cudaStream_t st);
void grid_sat_device(const double* d_est, const sc_ctu_record* d_rec, int cols, int rows,
                     int frames, double* d_sat, uint64_t* d_usat, cudaStream_t st);
void rect_tables_device(const double* d_sat, const uint64_t* d_usat, const int16_t* d_dec,
                        int cols, int rows, int frames, int fpw, double* d_rect_t,
                        double* d_rect_s, uint64_t* d_rt, double* d_rs, int sm_count,
                        cudaStream_t st);
void search_launch(int fpw, int step, const SearchArgs& a, int blocks, cudaStream_t st);
int search_blocks_per_sm(int fpw, int step, bool prune, size_t smem);
size_t search_smem_bytes(int cols, int rows, int n, int step, bool prune);
void item_filter_launch(sc_ctx* ctx, const SearchArgs& a, uint32_t k0, uint32_t k1, int fpw,
                        int frames, int step, const uint64_t* seed_inc, uint32_t* list,
                        uint32_t* count, cudaStream_t st);
int search_block_threads(int step, bool prune);
void column_bounds_launch(const uint32_t* rt, int fpw, int frames_in_group, int cols, int rows,
                          int rmax, int rstride, uint32_t* lbr, uint32_t* lbm, cudaStream_t st);
void partition_eval_device(const double* d_sat, const uint64_t* d_usat, const int* d_rects, int n,
                           int cols, int rows, int frames, sc_partition_stats* d_out,
                           double* d_slice_times, sc_ctu_record* d_slice_mom, cudaStream_t st);
int yuv_bytes_per_sample(int bit_depth);
int yuv_frame_count(const char* path, int w, int h, int bit_depth);
void yuv_read_luma(const char* path, int w, int h, int bit_depth, int first, int n, void* dst);
void finalize_launch(int step, int n, int fpw, int frames_in_group, uint32_t n_warps,
                     const LaneBest* lanes, const uint8_t* snaps,
                     const unsigned long long* count, const unsigned long long* scored,
                     double lambda, const uint64_t* vals, const uint32_t* nvals, size_t nr,
                     FrameBest* out, int64_t* budget_out, DevBuf& scratch, cudaStream_t st);
bool small_tables_device(const double* d_est, int cols, int rows, int frames, int fpw,
                         const int16_t* d_dec, uint32_t* keys, uint64_t* vals, uint32_t* nvals,
                         cudaStream_t st);
// device post-check and candidate stream (validate.cu, enumerate.cu)
void validate_device(int n, const int* d_rects, int nbx, const int* d_bx, int nby, const int* d_by,
                     int cols, int rows, int* d_owner, int32_t* d_map, VCheck* d_out,
                     cudaStream_t st);
void result_maps_device(const FrameBest* d_fb, size_t fb_stride, int frames, int first_step,
                        int steps, int n, int cols, int rows, int* d_owner, int32_t* d_maps,
                        VCheck* d_out, FrameBest* h_fb, cudaStream_t st);
void enumerate_count_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                            double k, int covering, uint64_t* d_counts, uint64_t* d_offsets,
                            DevBuf& temp, cudaStream_t st);
void enumerate_emit_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                           double k, int covering, const uint64_t* d_counts,
                           const uint64_t* d_offsets, uint64_t first, uint64_t limit,
                           uint8_t* d_out, cudaStream_t st);
// exhaustive step 1 as a trace interpreter (trace.cu)
bool trace_build_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                        double k, int covering, uint64_t max_ops, DevBuf& ops, DevBuf& skel_pos,
                        DevBuf& skel_ord, DevBuf& chunks, DevBuf& scratch, DevBuf& temp,
                        int sm_count, TraceHost* out, cudaStream_t st);
size_t trace_smem_bytes(int depth_cap, int warps);
int trace_warps(int depth_cap, uint64_t chunks, int sm_count);
int trace_blocks_per_sm(int fpw, int depth_cap, int warps);
void trace_walk_launch(int fpw, int blocks, int warps, int sm_count, const uint32_t* ops,
                       const uint4* chunks, uint32_t n_chunks,
                       uint32_t rank, uint32_t world, uint32_t* counter, const uint32_t* keys,
                       uint32_t nr, int depth_cap, uint64_t* lanes, const FinArgs* fin,
                       uint32_t* done, cudaStream_t st);
void trace_finalize_launch(const FinArgs& fa, cudaStream_t st);
void trace_skips_device(const uint32_t* ops, const uint32_t* skel_pos, uint32_t nskel,
                        uint32_t* skip, cudaStream_t st);
int trace2_blocks_per_sm(int fpw, int depth_cap);
void rest_pairs_device(const double* rs, const uint32_t* rest_of, uint32_t nr, int fpw, double* rss,
                       int sm_count, cudaStream_t st);
void trace_walk2_launch(int fpw, int blocks, const uint32_t* ops, const uint32_t* skip,
                        const uint4* chunks, uint32_t n_chunks, uint32_t rank,
                        uint32_t world, uint32_t* counter, const uint32_t* keys, const double* rs,
                        const uint32_t* rest_of, double* rss, const int64_t* budget, uint32_t nr,
                        int depth_cap, uint64_t* lanes, int sm_count, bool gather,
                        const FinArgs* fin, uint32_t* done, cudaStream_t st);
void trace_finalize2_launch(const FinArgs& fa, cudaStream_t st);
bool trace_walk2_fuses(int fpw, int depth_cap);
}  // namespace scb

namespace scb {
thread_local std::string g_last_error;
// shared with host.cpp: the thread's sc_last_error() message
sc_status set_last_error(sc_status s, const char* msg) {
  g_last_error = msg;
  return s;
}
}  // namespace scb

using namespace scb;

namespace {

void export_shards(sc_ctx* ctx, int step, int frames, sc_shard_best* out);
void merge_shards(int step, int world, int frames, const sc_shard_best* gathered,
                  sc_search_result* inout);

// ---- the library-owned exchange of candidate-space shards ---------------------
// NCCL is opened at run time (dlopen), so the library has no link-time NCCL
// dependency and shares the process's libnccl (e.g. torch's) when one is
// loaded.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.allGather &&
           a.errorString;
    return a;
  }();
  if (!api.ok) fail(SC_ERR_CUDA, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SC_ERR_CUDA, std::string(what) + ": " + nccl().errorString(r));
}

bool has_comm(const sc_ctx* ctx) { return ctx->comm_kind != 0; }

// Element-wise global minimum of n u64 on the device (in place, on st).
void comm_min_u64(sc_ctx* ctx, uint64_t* d, size_t n, cudaStream_t st) {
  if (ctx->comm_kind == 1) {
    nccl_check(nccl().allReduce(d, d, n, ncclUint64, ncclMin, (ncclComm_t)ctx->nccl_comm, st),
               "ncclAllReduce");
    return;
  }
  // host transport: the caller's all-gather between the ranks
  const int W = ctx->shard_world;
  std::vector<uint64_t> mine(n), all(n * (size_t)W);
  SCB_CUDA(cudaMemcpyAsync(mine.data(), d, n * 8, cudaMemcpyDeviceToHost, st));
  SCB_CUDA(cudaStreamSynchronize(st));
  if (ctx->comm_fn(ctx->comm_user, mine.data(), n * 8, all.data()) != 0)
    fail(SC_ERR_INTERNAL, "the all-gather callback failed");
  for (int r = 0; r < W; ++r)
    for (size_t i = 0; i < n; ++i) mine[i] = std::min(mine[i], all[(size_t)r * n + i]);
  SCB_CUDA(cudaMemcpyAsync(d, mine.data(), n * 8, cudaMemcpyHostToDevice, st));
  SCB_CUDA(cudaStreamSynchronize(st));
}

// All-gather of `bytes` host bytes per rank into recv (world * bytes).
void comm_allgather_host(sc_ctx* ctx, const void* send, size_t bytes, void* recv,
                         cudaStream_t st) {
  if (ctx->comm_kind == 1) {
    const int W = ctx->shard_world;
    ctx->comm_buf.ensure(bytes * (size_t)(W + 1));
    uint8_t* d = ctx->comm_buf.as<uint8_t>();
    SCB_CUDA(cudaMemcpyAsync(d, send, bytes, cudaMemcpyHostToDevice, st));
    nccl_check(nccl().allGather(d, d + bytes, bytes, ncclUint8, (ncclComm_t)ctx->nccl_comm, st),
               "ncclAllGather");
    SCB_CUDA(cudaMemcpyAsync(recv, d + bytes, bytes * (size_t)W, cudaMemcpyDeviceToHost, st));
    SCB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (ctx->comm_fn(ctx->comm_user, send, bytes, recv) != 0)
    fail(SC_ERR_INTERNAL, "the all-gather callback failed");
}

sc_status set_error(sc_status s, const std::string& m) {
  g_last_error = m;
  return s;
}

template <typename F>
sc_status guarded(F&& fn) {
  try {
    fn();
    g_last_error.clear();
    return SC_OK;
  } catch (const Fail& f) {
    return set_error(f.status, f.msg);
  } catch (const std::bad_alloc&) {
    return set_error(SC_ERR_INTERNAL, "host allocation failed");
  } catch (const std::exception& e) {
    return set_error(SC_ERR_INTERNAL, e.what());
  }
}

// CtuGrid::make (grid.cpp:9-24)
sc_grid make_grid(int w, int h, int ctu) {
  if (ctu != 32 && ctu != 64 && ctu != 128)
    fail(SC_ERR_GEOMETRY, "ctu_size must be one of {32, 64, 128}, got " + std::to_string(ctu));
  if (w < 1 || h < 1) fail(SC_ERR_GEOMETRY, "frame dimensions must be positive");
  sc_grid g;
  g.frame_width = w;
  g.frame_height = h;
  g.ctu_size = ctu;
  g.cols = (w + ctu - 1) / ctu;
  g.rows = (h + ctu - 1) / ctu;
  return g;
}

void check_grid(const sc_grid* g) {
  if (!g) fail(SC_ERR_USAGE, "grid is NULL");
  sc_grid m = make_grid(g->frame_width, g->frame_height, g->ctu_size);
  if (m.cols != g->cols || m.rows != g->rows)
    fail(SC_ERR_GEOMETRY, "grid cols/rows inconsistent with frame and CTU size");
}

// SearchConfig::check (search.cpp:28-36), same order and messages.
void check_cfg_fields(const sc_search_cfg* c) {
  if (!c) fail(SC_ERR_USAGE, "cfg is NULL");
  if (c->n_slices < 1) fail(SC_ERR_CONFIG, "n_slices must be >= 1");
  if (!(c->k_area > 1.0)) fail(SC_ERR_CONFIG, "k_area must be > 1");
  if (!(c->lambda >= 0.0) || !std::isfinite(c->lambda))
    fail(SC_ERR_CONFIG, "lambda must be finite and >= 0");
  if (c->workers < 1) fail(SC_ERR_CONFIG, "workers must be >= 1");
  if (c->max_tile_cols < 0) fail(SC_ERR_CONFIG, "max_tile_cols must be >= 0");
}

// SearchConfig::check + the B200 fields and the kernels' compiled limits.
int check_cfg(const sc_grid& g, const sc_search_cfg* c) {
  check_cfg_fields(c);
  if (c->family != SC_FAMILY_COLUMN_SPLIT && c->family != SC_FAMILY_UNIFORM_ONLY)
    fail(SC_ERR_CONFIG, "unknown candidate family");
  if (c->coverage != SC_COVERAGE_REFERENCE && c->coverage != SC_COVERAGE_COVERING)
    fail(SC_ERR_CONFIG, "unknown coverage");
  if (c->mode != SC_MODE_EXHAUSTIVE && c->mode != SC_MODE_PRUNED)
    fail(SC_ERR_CONFIG, "unknown search mode");
  // run_step1 / for_each_candidate (search.cpp:260-262, 305-307)
  if (c->n_slices > g.cols * g.rows) fail(SC_ERR_GEOMETRY, "n_slices exceeds the CTU cell count");
  const int eff = c->max_tile_cols > 0 ? c->max_tile_cols : c->n_slices;
  const int maxc = std::min({c->n_slices, eff, g.cols});
  if (c->n_slices > SC_MAX_SLICES)
    fail(SC_ERR_SIZE, "n_slices exceeds the compiled limit SC_MAX_SLICES");
  if (c->family == SC_FAMILY_COLUMN_SPLIT && maxc > SC_MAX_COLS)
    fail(SC_ERR_SIZE, "tile-column count exceeds SC_MAX_COLS");
  if (g.rows > 255) fail(SC_ERR_SIZE, "more than 255 CTU rows");
  if (g.cols > 255) fail(SC_ERR_SIZE, "more than 255 CTU columns");
  return maxc;
}

// TextureStats ctor validation (texture.cpp:90-111).
void validate_records(const sc_grid& g, const sc_ctu_record* r) {
  for (int y = 0; y < g.rows; ++y)
    for (int x = 0; x < g.cols; ++x) {
      const sc_ctu_record& c = r[(size_t)y * g.cols + x];
      if (c.count != (uint64_t)cell_w(g, x) * (uint64_t)cell_h(g, y))
        fail(SC_ERR_FORMAT, "CTU pixel count mismatch at (" + std::to_string(x) + "," +
                                std::to_string(y) + ")");
      const unsigned __int128 lhs = (unsigned __int128)c.count * c.sumsq;
      const unsigned __int128 rhs = (unsigned __int128)c.sum * c.sum;
      if (lhs < rhs)
        fail(SC_ERR_FORMAT, "CTU statistics violate count*sumsq >= sum^2 at (" +
                                std::to_string(x) + "," + std::to_string(y) + ")");
    }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// ---- planner (plan.h) ------------------------------------------------------
// Exact candidate count of the plan's family (computed once, cached).
unsigned __int128 plan_count(Plan* p, const sc_grid& g, const sc_search_cfg& cfg) {
  if (!p->have_count) {
    p->count = count_candidates_dp(g.cols, g.rows, cfg.n_slices, p->key.maxc,
                                   cfg.coverage == SC_COVERAGE_COVERING, p->bmax);
    p->have_count = true;
  }
  return p->count;
}

Plan* get_plan(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, int maxc) {
  PlanKey key{g.cols, g.rows, cfg.n_slices, maxc, cfg.coverage, cfg.k_area};
  for (Plan* p : ctx->plans)
    if (p->key == key) return p;
  Plan* p = new Plan();
  p->key = key;
  const bool covering = cfg.coverage == SC_COVERAGE_COVERING;
  // work-item granularity: at least SLICECRAFT_B200_ITEMS_PER_SM (512) width
  // prefixes per SM (make_items deepens the prefixes until there are)
  const char* ips = getenv("SLICECRAFT_B200_ITEMS_PER_SM");
  const size_t per_sm = ips ? (size_t)std::max(1, atoi(ips)) : 512;
  p->items = make_items(g.cols, maxc, covering, (size_t)ctx->sm_count * per_sm);
  // seed phase of the pruned mode: the items of the smallest column count(s)
  p->seed_items = 0;
  for (const WorkItem& it : p->items) {
    if (it.c > 1) break;
    ++p->seed_items;
  }
  p->pathological = make_area_tables(g.cols, g.rows, cfg.k_area, p->bmax);
  ctx->plans.push_back(p);
  return p;
}

void upload_plan(sc_ctx* ctx, Plan* p) {
  if (p->uploaded) return;
  p->d_items.ensure(p->items.size() * sizeof(WorkItem));
  SCB_CUDA(cudaMemcpy(p->d_items.p, p->items.data(), p->items.size() * sizeof(WorkItem),
                      cudaMemcpyHostToDevice));
  p->d_bmax.ensure(p->bmax.size() * sizeof(int32_t));
  SCB_CUDA(cudaMemcpy(p->d_bmax.p, p->bmax.data(), p->bmax.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice));
  p->uploaded = true;
  (void)ctx;
}

void layout_from_snap(const FrameBest& fb, int n, sc_layout* L) {
  std::memset(L, 0, sizeof(*L));
  int c = 0;
  while (c < SC_MAX_COLS && fb.snap[c] != 0) ++c;
  L->n_cols = c;
  L->n_slices = n;
  for (int i = 0; i < c; ++i) {
    L->col_widths[i] = fb.snap[i];
    L->runs_per_col[i] = fb.snap[SC_MAX_COLS + i];
  }
  for (int i = 0; i < n; ++i) L->run_heights[i] = fb.snap[2 * SC_MAX_COLS + i];
}


cudaStream_t main_stream(sc_ctx* ctx) { return ctx->user_stream ? ctx->user_stream : ctx->stream; }

struct Layouts {
  int frames = 0, fpw = 1, groups = 1;
  size_t nr = 0;
  int nsat = 0;
};

Layouts layouts_for(const sc_grid& g, int frames) {
  Layouts L;
  L.frames = frames;
  L.fpw = std::min(32, next_pow2(frames));
  L.groups = (frames + L.fpw - 1) / L.fpw;
  L.nr = (size_t)n_xw(g.cols) * n_yh(g.rows);
  L.nsat = (g.cols + 1) * (g.rows + 1);
  return L;
}

// Time keys of frame group gi: [groups][rt | rts][rect][fpw] in ctx->rt_search
// (rank.cu writes rt, the split table rts).
uint32_t* rt_of(sc_ctx* ctx, const Layouts& L, int gi) {
  return ctx->rt_search.as<uint32_t>() + (size_t)gi * 2 * L.nr * L.fpw;
}
uint32_t* rts_of(sc_ctx* ctx, const Layouts& L, int gi) { return rt_of(ctx, L, gi) + L.nr * L.fpw; }

// Rectangle decode table (xw -> x0,w ; yh -> y0,h), cached per grid.
const int16_t* decode_table(sc_ctx* ctx, const sc_grid& g) {
  if (ctx->dec_cols == g.cols && ctx->dec_rows == g.rows) return ctx->dec.as<int16_t>();
  const int nxw = n_xw(g.cols), nyh = n_yh(g.rows);
  std::vector<int16_t> dec((size_t)2 * nxw + 2 * nyh);
  for (int x0 = 0; x0 < g.cols; ++x0)
    for (int w = 1; w <= g.cols - x0; ++w) {
      const int i = xw_index(g.cols, x0, w);
      dec[i] = (int16_t)x0;
      dec[nxw + i] = (int16_t)w;
    }
  for (int y0 = 0; y0 < g.rows; ++y0)
    for (int h = 1; h <= g.rows - y0; ++h) {
      const int i = yh_index(g.rows, y0, h);
      dec[2 * nxw + i] = (int16_t)y0;
      dec[2 * nxw + nyh + i] = (int16_t)h;
    }
  ctx->dec.ensure(dec.size() * sizeof(int16_t));
  SCB_CUDA(cudaMemcpy(ctx->dec.p, dec.data(), dec.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
  // the forced rest (x0, w, y0 + h, rows - y0 - h) of every run that leaves
  // rows below it (step-2 trace walk)
  std::vector<uint32_t> rest((size_t)nxw * nyh, 0);
  for (int xw = 0; xw < nxw; ++xw)
    for (int y0 = 0; y0 < g.rows; ++y0)
      for (int h = 1; y0 + h < g.rows; ++h)
        rest[(size_t)xw * nyh + yh_index(g.rows, y0, h)] =
            (uint32_t)((size_t)xw * nyh + yh_index(g.rows, y0 + h, g.rows - y0 - h));
  ctx->rest_of.ensure(rest.size() * sizeof(uint32_t));
  SCB_CUDA(cudaMemcpy(ctx->rest_of.p, rest.data(), rest.size() * sizeof(uint32_t),
                      cudaMemcpyHostToDevice));
  ctx->dec_cols = g.cols;
  ctx->dec_rows = g.rows;
  return ctx->dec.as<int16_t>();
}

// CUDA graphs for the time-table phase (SLICECRAFT_B200_GRAPHS=0: plain launches).
bool graphs_enabled() {
  const char* v = getenv("SLICECRAFT_B200_GRAPHS");
  return !(v && v[0] == '0');
}

void enqueue_time_tables_body(sc_ctx* ctx, const sc_grid& g, const Layouts& L, bool raw,
                              const int16_t* dec, const uint32_t* used, size_t nu,
                              const uint32_t* usplit, size_t nus, cudaStream_t st);

// SLICECRAFT_B200_RANK_USED=0: rank every rectangle even when the plan knows
// which ones its candidates use
bool rank_used_enabled() {
  const char* v = getenv("SLICECRAFT_B200_RANK_USED");
  return !(v && v[0] == '0');
}

// K2 (f64 SAT) + K3 (time tables) from ctx->est.  The ~20 short launches of
// this phase leave the device waiting on the host's launch rate, so when a
// call repeats the previous call's shape and buffers (the steady state of a
// frame pipeline) the phase is captured once into a CUDA graph and replayed.
void enqueue_time_tables(sc_ctx* ctx, const sc_grid& g, const Layouts& L, bool raw,
                         const uint32_t* used, size_t nu, const uint32_t* usplit, size_t nus,
                         cudaStream_t st) {
  const int16_t* dec = decode_table(ctx, g);
  if (!rank_used_enabled() || nu == 0 || nu >= L.nr) used = nullptr, nu = 0;
  if (!used) usplit = nullptr, nus = 0;
  ctx->sat.ensure((size_t)L.frames * L.nsat * sizeof(double));
  ctx->rt_bits.ensure((size_t)L.frames * L.nr * sizeof(uint64_t));
  ctx->rt_search.ensure((size_t)L.groups * 2 * L.fpw * L.nr * sizeof(uint32_t));
  ctx->vals.ensure((size_t)L.frames * L.nr * sizeof(uint64_t));
  ctx->nvals.ensure((size_t)L.frames * sizeof(uint32_t));
  if (raw) ctx->rect_t.ensure((size_t)L.frames * L.nr * sizeof(double));
  if (used) {
    ctx->rk_bits_c.ensure(nu * (size_t)L.frames * sizeof(uint64_t));
    // the rectangles outside the used list keep the key "infinite": written
    // once per (key table, used list) and outside the replayed graph -- later
    // calls only rewrite the used entries, and the split table of an infinite
    // key stays infinite
    const size_t words = (size_t)L.groups * 2 * L.nr * L.fpw;
    if (ctx->rk_inf_keys != ctx->rt_search.p || ctx->rk_inf_used != used ||
        ctx->rk_inf_nu != nu || ctx->rk_inf_words != words) {
      SCB_CUDA(cudaMemsetAsync(ctx->rt_search.p, 0xff, words * sizeof(uint32_t), st));
      ctx->rk_inf_keys = ctx->rt_search.p;
      ctx->rk_inf_used = used;
      ctx->rk_inf_nu = nu;
      ctx->rk_inf_words = words;
    }
  } else {
    ctx->rk_inf_keys = nullptr;  // every entry is rewritten: no "infinite" filler left
  }
  if (!graphs_enabled()) {
    enqueue_time_tables_body(ctx, g, L, raw, dec, used, nu, usplit, nus, st);
    return;
  }
  // everything a replay depends on: shape and every buffer address
  std::vector<uintptr_t> key = {
      (uintptr_t)g.cols, (uintptr_t)g.rows, (uintptr_t)L.frames, (uintptr_t)L.fpw,
      (uintptr_t)L.groups, (uintptr_t)L.nr, (uintptr_t)raw, (uintptr_t)st, (uintptr_t)dec,
      (uintptr_t)ctx->est.p, (uintptr_t)ctx->sat.p, (uintptr_t)ctx->rt_bits.p,
      (uintptr_t)ctx->rt_search.p, (uintptr_t)ctx->vals.p, (uintptr_t)ctx->nvals.p,
      (uintptr_t)ctx->rect_t.p, (uintptr_t)ctx->rk_idx.p,
      (uintptr_t)ctx->rk_sorted.p, (uintptr_t)ctx->rk_flags.p, (uintptr_t)ctx->rk_temp.p,
      (uintptr_t)ctx->rk_temp.bytes, (uintptr_t)used, (uintptr_t)nu, (uintptr_t)ctx->rk_bits_c.p,
      (uintptr_t)usplit, (uintptr_t)nus};
  if (ctx->tt_exec && key == ctx->tt_key) {
    SCB_CUDA(cudaGraphLaunch(ctx->tt_exec, st));
    count_launches(ctx->tt_launches);  // the kernels of the captured phase
    return;
  }
  if (ctx->tt_exec) {
    cudaGraphExecDestroy(ctx->tt_exec);
    ctx->tt_exec = nullptr;
  }
  if (key != ctx->tt_prev_key) {
    // first call of this shape: plain launches (they size the scratch buffers)
    enqueue_time_tables_body(ctx, g, L, raw, dec, used, nu, usplit, nus, st);
    ctx->tt_prev_key = key;
    return;
  }
  // second call of the same shape: capture, instantiate, launch
  cudaGraph_t graph = nullptr;
  const uint64_t launches_before = launch_counter();
  SCB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_time_tables_body(ctx, g, L, raw, dec, used, nu, usplit, nus, st);
  } catch (...) {  // leave the stream out of capture mode before reporting
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    ctx->tt_prev_key.clear();
    throw;
  }
  SCB_CUDA(cudaStreamEndCapture(st, &graph));
  SCB_CUDA(cudaGraphInstantiate(&ctx->tt_exec, graph, 0));
  cudaGraphDestroy(graph);
  ctx->tt_key = key;
  ctx->tt_launches = launch_counter() - launches_before;
  SCB_CUDA(cudaGraphLaunch(ctx->tt_exec, st));
}

void enqueue_time_tables_body(sc_ctx* ctx, const sc_grid& g, const Layouts& L, bool raw,
                              const int16_t* dec, const uint32_t* used, size_t nu,
                              const uint32_t* usplit, size_t nus, cudaStream_t st) {
  // small grids: the whole phase in one CTA per frame (small_tables.cu);
  // SLICECRAFT_B200_SMALL_TABLES=0 keeps the general pipeline
  const char* sv = getenv("SLICECRAFT_B200_SMALL_TABLES");
  if (!raw && !(sv && sv[0] == '0') &&
      small_tables_device(ctx->est.as<double>(), g.cols, g.rows, L.frames, L.fpw, dec,
                          ctx->rt_search.as<uint32_t>(), ctx->vals.as<uint64_t>(),
                          ctx->nvals.as<uint32_t>(), st))
    return;
  grid_sat_device(ctx->est.as<double>(), nullptr, g.cols, g.rows, L.frames, ctx->sat.as<double>(),
                  nullptr, st);
  rect_tables_device(ctx->sat.as<double>(), nullptr, dec, g.cols, g.rows, L.frames, L.fpw,
                     raw ? ctx->rect_t.as<double>() : nullptr, nullptr,
                     ctx->rt_bits.as<uint64_t>(), nullptr, ctx->sm_count, st);
  // exact per-frame ranks of the times (rank.cu) -> 32-bit search keys
  rank_times_device(ctx, ctx->rt_bits.as<uint64_t>(), L.nr, L.frames, L.fpw,
                    ctx->rt_search.as<uint32_t>(), ctx->vals.as<uint64_t>(),
                    ctx->nvals.as<uint32_t>(), used, nu, (size_t)L.groups, st);
  split_table_device(ctx->rt_search.as<uint32_t>(), g.cols, g.rows, L.groups, L.fpw, ctx->sm_count,
                     usplit, nus, st);
}

// K2 (u64 SATs) + K3 (SSE tables) from ctx->records.
void enqueue_moment_tables(sc_ctx* ctx, const sc_grid& g, const Layouts& L, bool raw,
                           cudaStream_t st) {
  const int16_t* dec = decode_table(ctx, g);
  ctx->usat.ensure((size_t)L.frames * 3 * L.nsat * sizeof(uint64_t));
  ctx->rs_search.ensure((size_t)L.groups * L.fpw * L.nr * sizeof(double));
  if (raw) ctx->rect_s.ensure((size_t)L.frames * L.nr * sizeof(double));
  grid_sat_device(nullptr, ctx->records.as<sc_ctu_record>(), g.cols, g.rows, L.frames, nullptr,
                  ctx->usat.as<uint64_t>(), st);
  rect_tables_device(nullptr, ctx->usat.as<uint64_t>(), dec, g.cols, g.rows, L.frames, L.fpw,
                     nullptr, raw ? ctx->rect_s.as<double>() : nullptr, nullptr,
                     ctx->rs_search.as<double>(), ctx->sm_count, st);
}

// Exhaustive mode, step 2: walk only the subtrees whose partial time can still
// meet the budget.  Exact: a subtree whose fixed slices already exceed the
// budget holds no feasible candidate, and step 1 evaluated the time of every
// candidate of the family.  SLICECRAFT_B200_STEP2_BOUND=0 walks them all.
// SLICECRAFT_B200_SIDE_BOUNDS=0: step 2 computes its column bounds itself
bool side_bounds_enabled() {
  const char* v = getenv("SLICECRAFT_B200_SIDE_BOUNDS");
  return !(v && v[0] == '0');
}

// SLICECRAFT_B200_FUSE_FIN=0: single-frame calls launch their finalize kernels separately
bool fuse_finalize_enabled() {
  const char* v = getenv("SLICECRAFT_B200_FUSE_FIN");
  return !(v && v[0] == '0');
}

bool step2_bounded(const sc_search_cfg& cfg) {
  if (cfg.mode != SC_MODE_EXHAUSTIVE) return false;
  const char* v = getenv("SLICECRAFT_B200_STEP2_BOUND");
  return !(v && v[0] == '0');
}

// Cost-ordered schedule of the exhaustive step-1 walk (Plan::order_state);
// SLICECRAFT_B200_SCHEDULE=0 keeps the enumeration order.
// exhaustive mode's budget-bounded step 2 (SLICECRAFT_B200_SPLIT2 overrides)
constexpr int kBoundedStep2Split = 16;
constexpr int kSplitDepth1 = 8;

// Pruned walks: warps sharing one work item and the heights level whose
// subtrees they deal out.  Sharing costs every warp of an item the walk down
// to the split level; since the item prefilter (k_item_filter) drops the
// items that die at their prefix, only surviving items pay it, and the
// survivors are few and heavy.  Measured on B200 (profiles/r01_split_sweep.md)
// 16 ways is best or even on configs 3-5 in both steps, 64 for cfg5's step 2.
// SLICECRAFT_B200_SPLIT / SLICECRAFT_B200_SPLIT2 (step 2) override.
int split_ways(int step, int n, bool pruned_mode) {
  const char* v = getenv(step == 1 ? "SLICECRAFT_B200_SPLIT" : "SLICECRAFT_B200_SPLIT2");
  // n >= 24 (cfg5): step 2 spreads its few deep items over 64 warps (4.7 ->
  // 4.2 ms on cfg5, with depth 2 below); 16 elsewhere
  int g = v ? atoi(v)
            : (!pruned_mode ? kBoundedStep2Split : (step == 2 && n >= 24 ? 64 : 16));
  return g < 1 ? 1 : (g > 64 ? 64 : g);
}
// Heights level whose subtrees the warps of a shared item deal out.  Step 1
// (SLICECRAFT_B200_SPLIT_DEPTH): deep, so the seed phase's few long
// single-column walks spread over all the item's warps; step 2
// (SLICECRAFT_B200_SPLIT_DEPTH2): shallow, its leaves are expensive and a
// deep split repeats the walk above it in every warp
// (profiles/r01_split_sweep.md).
int split_depth(int step, int n) {
  const char* v = getenv(step == 1 ? "SLICECRAFT_B200_SPLIT_DEPTH" : "SLICECRAFT_B200_SPLIT_DEPTH2");
  // measured: depth 8 takes cfg5 (n = 32) step 1 from 4.8 to 3.6 ms, but
  // costs cfg3 (n = 8) 13 %; cfg4 (n = 16) is even.  Step 2: depth 2 for n >= 24
  const int d = v ? atoi(v) : (n >= 24 ? (step == 1 ? kSplitDepth1 : 2) : 1);
  return d < 0 ? 0 : (d > 62 ? 62 : d);
}

// Pruned walks: drop the items whose prefix fails every frame before the
// launch (SLICECRAFT_B200_FILTER=0 keeps every item).
bool item_filter_enabled() {
  const char* v = getenv("SLICECRAFT_B200_FILTER");
  return !(v && v[0] == '0');
}

// Device post-check of returned partitions (SLICECRAFT_B200_POSTCHECK=0: off).
bool postcheck_enabled() {
  const char* v = getenv("SLICECRAFT_B200_POSTCHECK");
  return !(v && v[0] == '0');
}

bool schedule_enabled() {
  const char* v = getenv("SLICECRAFT_B200_SCHEDULE");
  return !(v && v[0] == '0');
}

// After a measuring call: items by decreasing measured walk cost (ties by
// index), uploaded for the next calls.
// (A shard orders its own items, rank, rank + world, ...: LPT per rank.)
void finish_schedule(Plan* p) {
  if (p->order_state != 1) return;
  const size_t n = p->items.size();
  const uint32_t rank = p->order_rank, world = p->order_world;
  std::vector<uint32_t> cost(n), order;
  SCB_CUDA(cudaMemcpy(cost.data(), p->d_cost.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  for (size_t i = rank; i < n; i += world) order.push_back((uint32_t)i);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
  p->d_order.ensure(std::max<size_t>(1, order.size()) * sizeof(uint32_t));
  if (!order.empty())
    SCB_CUDA(cudaMemcpy(p->d_order.p, order.data(), order.size() * sizeof(uint32_t),
                        cudaMemcpyHostToDevice));
  p->order_state = 2;
}

// Exhaustive step 1 through the candidate trace (trace.cuh): on by default
// for families up to kTraceMaxCands candidates (the build runs the
// enumeration once per plan); SLICECRAFT_B200_TRACE=0 keeps the DFS walk.
constexpr double kTraceMaxCands = 2e9;  // < 2^31: 32-bit ordinals in the walk
constexpr uint64_t kTraceMaxOps = 1ull << 28;  // 1 GiB of ops
bool trace_enabled() {
  const char* v = getenv("SLICECRAFT_B200_TRACE");
  return !(v && v[0] == '0');
}

// Builds the plan's trace on first use; false when the plan does not use one.
bool ensure_trace(sc_ctx* ctx, Plan* p, const sc_grid& g, const sc_search_cfg& cfg,
                  cudaStream_t st) {
  if (p->trace_state != 0) return p->trace_state == 1;
  p->trace_state = -1;
  if ((double)plan_count(p, g, cfg) > kTraceMaxCands) return false;
  if ((size_t)n_xw(g.cols) * n_yh(g.rows) > ((size_t)1 << 22)) return false;
  TraceHost th;
  DevBuf scratch, temp;
  const bool ok = trace_build_device(p->d_items.as<WorkItem>(), (uint32_t)p->items.size(), g.cols,
                                     g.rows, cfg.n_slices, cfg.k_area, cfg.coverage, kTraceMaxOps,
                                     p->tr_ops, p->tr_skel_pos, p->tr_skel_ord, p->tr_chunks,
                                     scratch, temp, ctx->sm_count, &th, st);
  scratch.release();
  temp.release();
  if (!ok) {
    p->tr_ops.release();
    p->tr_skel_pos.release();
    p->tr_skel_ord.release();
    p->tr_chunks.release();
    return false;
  }
  if ((unsigned __int128)th.cands != plan_count(p, g, cfg))
    fail(SC_ERR_INTERNAL, "candidate trace count differs from the counting DP");
  p->trace_ops = th.ops;
  p->trace_cands = th.cands;
  p->trace_nskel = th.nskel;
  p->trace_chunks = th.n_chunks;
  p->trace_state = 1;
  {  // the rectangles the candidates use (later calls rank only these)
    DevBuf sc2, tmp2;
    p->n_used = trace_used_device(p->tr_ops.as<uint32_t>(), th.ops, g.rows,
                                  (uint32_t)((size_t)n_xw(g.cols) * n_yh(g.rows)), p->tr_used,
                                  p->tr_used_split, &p->n_used_split, sc2, tmp2, ctx->sm_count,
                                  st);
    sc2.release();
    tmp2.release();
  }
  return true;
}

// Step 2 of the exhaustive mode has two exact walks: the budget-bounded DFS
// walk (per-lane pruning; fast when few candidates fit the budget, e.g. the
// reference family at small lambda) and the trace interpreter (fast when
// many do, e.g. the covering family at lambda 0.3, where the DFS walk's
// per-lane divergence costs 10x).  The first call of a (plan, lambda) runs
// both, timed with events, and later calls take the faster (results are
// identical).  SLICECRAFT_B200_TRACE2=0 / =1 forces the DFS walk / the trace.
int trace2_mode() {
  const char* v = getenv("SLICECRAFT_B200_TRACE2");
  if (!trace_enabled() || (v && v[0] == '0')) return 1;
  if (v && v[0] == '1') return 2;
  return 0;
}

// The plan's subtree-end table for the step-2 walk (built on first use).
const uint32_t* ensure_skips(Plan* p, cudaStream_t st) {
  if (!p->have_skip) {
    p->tr_skip.ensure((size_t)p->trace_ops * sizeof(uint32_t) + 4);
    trace_skips_device(p->tr_ops.as<uint32_t>(), p->tr_skel_pos.as<uint32_t>(), p->trace_nskel,
                       p->tr_skip.as<uint32_t>(), st);
    p->have_skip = true;
  }
  return p->tr_skip.as<uint32_t>();
}

// Candidates in the trace chunks of shard `rank` of `world` (all of them for
// world 1), from the chunk and skeleton tables (once per shard layout).
uint64_t trace_shard_count(Plan* p, int rank, int world) {
  if (world == 1) return p->trace_cands;
  const uint64_t key = ((uint64_t)rank << 32) | (uint32_t)world;
  if (p->trace_shard_key == key) return p->trace_shard_cands;
  // chunk records {first op, end op, SKEL op, first ordinal}; record n is the sentinel
  std::vector<uint32_t> cs(((size_t)p->trace_chunks + 1) * 4);
  SCB_CUDA(cudaMemcpy(cs.data(), p->tr_chunks.p, cs.size() * 4, cudaMemcpyDeviceToHost));
  uint64_t tot = 0;
  for (uint32_t c = (uint32_t)rank; c < p->trace_chunks; c += (uint32_t)world)
    tot += (uint64_t)(cs[4 * (size_t)(c + 1) + 3] - cs[4 * (size_t)c + 3]);
  p->trace_shard_key = key;
  p->trace_shard_cands = tot;
  return tot;
}

void enqueue_step_walks(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, Plan* plan,
                        const Layouts& L, int step, bool compute_bounds, cudaStream_t st, int s2);

// Per-frame column lower bounds (search.cu) from the time keys of every frame
// group: they depend on the time tables only, so the exhaustive mode's
// bounded step 2 can have them computed on the side stream while step 1 runs.
void enqueue_column_bounds(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg,
                           const Layouts& L, cudaStream_t st) {
  const int rstride = std::min(cfg.n_slices, g.rows) + 1;
  const size_t lb_per_group = (size_t)n_xw(g.cols) * rstride * L.fpw;
  ctx->lbr.ensure(lb_per_group * L.groups * sizeof(uint32_t));
  ctx->lbm.ensure(lb_per_group * L.groups * sizeof(uint32_t));
  for (int gi = 0; gi < L.groups; ++gi)
    column_bounds_launch(rt_of(ctx, L, gi), L.fpw, std::min(L.fpw, L.frames - gi * L.fpw), g.cols,
                         g.rows, rstride - 1, rstride,
                         ctx->lbr.as<uint32_t>() + gi * lb_per_group,
                         ctx->lbm.as<uint32_t>() + gi * lb_per_group, st);
}

// One search step over all frame groups; finalize writes FrameBest[step] and,
// after step 1, the device budgets of step 2.  No host synchronisation.
void enqueue_step(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, Plan* plan,
                  const Layouts& L, int step, bool compute_bounds, cudaStream_t st) {
  int s2 = 1;  // step 2: 1 = DFS walk, 2 = trace, 3 = both (timed, first call)
  if (step == 2 && cfg.mode == SC_MODE_EXHAUSTIVE && trace2_mode() != 1 &&
      ensure_trace(ctx, plan, g, cfg, st)) {
    s2 = trace2_mode();
    if (s2 == 0) {
      s2 = 3;
      for (const auto& c : plan->step2_choice)
        if (c.first == cfg.lambda && c.second > 0) s2 = c.second;
    }
  }
  if (s2 == 3) {
    SCB_CUDA(cudaEventRecord(ctx->ev_s2[0], st));
    enqueue_step_walks(ctx, g, cfg, plan, L, step, compute_bounds, st, 1);
    SCB_CUDA(cudaEventRecord(ctx->ev_s2[1], st));
    enqueue_step_walks(ctx, g, cfg, plan, L, step, compute_bounds, st, 2);
    SCB_CUDA(cudaEventRecord(ctx->ev_s2[2], st));
    ctx->s2_pending = true;
    ctx->s2_lambda = cfg.lambda;
    ctx->s2_plan = plan;
    return;
  }
  enqueue_step_walks(ctx, g, cfg, plan, L, step, compute_bounds, st, s2);
}

// The walks of one step (s2: step 2's walk, 1 = DFS, 2 = trace).
void enqueue_step_walks(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, Plan* plan,
                        const Layouts& L, int step, bool compute_bounds, cudaStream_t st, int s2) {
  const bool prune = cfg.mode == SC_MODE_PRUNED || (step == 2 && step2_bounded(cfg));
  if (step == 2 && s2 == 2) {
    // step 2 through the trace; SLICECRAFT_B200_STEP2_BOUND=0 walks every op
    // (no subtree skipping: the reference's full re-enumeration)
    const uint32_t* skip = ensure_skips(plan, st);
    const bool skipping = step2_bounded(cfg);
    const int depth_cap = std::max(cfg.n_slices, 2);
    // no more blocks than the shard has chunks for (small spaces: a few)
    const int blocks = std::max(
        1, (int)std::min<uint64_t>((uint64_t)ctx->sm_count * trace2_blocks_per_sm(L.fpw, depth_cap),
                                   (plan->trace_chunks / ctx->shard_world + 8) / 2));
    const uint32_t n_lanes = (uint32_t)blocks * 32;  // one record per block lane
    const size_t lane_bytes = (size_t)n_lanes * 3 * sizeof(uint64_t);
    ctx->lanes.ensure(lane_bytes * L.groups);
    ctx->counter.ensure((size_t)L.groups * 8 * sizeof(uint64_t));
    ctx->frame_best.ensure((size_t)2 * L.groups * L.fpw * sizeof(FrameBest));
    FrameBest* fb = ctx->frame_best.as<FrameBest>() + (size_t)L.groups * L.fpw;
    ctx->rss.ensure(L.nr * L.fpw * 2 * sizeof(double));  // {sse, rest sse} pairs
    for (int gi = 0; gi < L.groups; ++gi) {
      uint64_t* ctr = ctx->counter.as<uint64_t>() + 8 * gi + 4;
      SCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint64_t) * 4, st));
      uint64_t* lanes = reinterpret_cast<uint64_t*>(ctx->lanes.as<uint8_t>() + lane_bytes * gi);
      const int fig = std::min(L.fpw, L.frames - gi * L.fpw);
      FinArgs fa{};
      fa.fpw = L.fpw;
      fa.frames_in_group = fig;
      fa.n_lanes = n_lanes;
      fa.lanes = lanes;
      fa.ops = plan->tr_ops.as<uint32_t>();
      fa.skel_pos = plan->tr_skel_pos.as<uint32_t>();
      fa.nskel = plan->trace_nskel;
      fa.nr = (uint32_t)L.nr;
      fa.cols = g.cols;
      fa.rows = g.rows;
      fa.count = trace_shard_count(plan, ctx->shard_rank, ctx->shard_world);
      fa.vals = ctx->vals.as<uint64_t>() + (size_t)gi * L.fpw * L.nr;
      fa.nr_vals = L.nr;
      fa.out = fb + (size_t)gi * L.fpw;
      const bool fuse = fig == 1 && trace_walk2_fuses(L.fpw, depth_cap) && fuse_finalize_enabled();
      trace_walk2_launch(L.fpw, blocks, plan->tr_ops.as<uint32_t>(), skipping ? skip : nullptr,
                         plan->tr_chunks.as<uint4>(), plan->trace_chunks,
                         (uint32_t)ctx->shard_rank, (uint32_t)ctx->shard_world,
                         reinterpret_cast<uint32_t*>(ctr), rt_of(ctx, L, gi),
                         ctx->rs_search.as<double>() + (size_t)gi * L.nr * L.fpw,
                         ctx->rest_of.as<uint32_t>(), ctx->rss.as<double>(),
                         ctx->budget.as<int64_t>() + (size_t)gi * L.fpw, (uint32_t)L.nr, depth_cap,
                         lanes, ctx->sm_count, !ctx->pairs_on_side, fuse ? &fa : nullptr,
                         reinterpret_cast<uint32_t*>(ctr + 1), st);
      if (!fuse) trace_finalize2_launch(fa, st);
    }
    return;
  }
  if (step == 1 && !prune && trace_enabled() && ensure_trace(ctx, plan, g, cfg, st)) {
    const int depth_cap = std::max(cfg.n_slices, 2);
    // blocks per SM: the occupancy limit, or SLICECRAFT_B200_TRACE_BPS (fewer
    // leave room for the side stream's texture pass to run beside the walk)
    const int warps = trace_warps(depth_cap, plan->trace_chunks / ctx->shard_world, ctx->sm_count);
    int bps = trace_blocks_per_sm(L.fpw, depth_cap, warps);
    if (const char* v = getenv("SLICECRAFT_B200_TRACE_BPS")) bps = std::max(1, std::min(bps, atoi(v)));
    // small spaces: no more warps than half the chunks
    const int blocks = std::max(
        1, (int)std::min<uint64_t>((uint64_t)ctx->sm_count * bps,
                                   (plan->trace_chunks / ctx->shard_world * 8 / warps + 8) / 2));
    const uint32_t n_lanes = (uint32_t)blocks * 32;  // one record per block lane (trace.cu)
    const size_t lane_bytes = (size_t)n_lanes * 2 * sizeof(uint64_t);
    ctx->lanes.ensure(lane_bytes * L.groups);
    ctx->counter.ensure((size_t)L.groups * 8 * sizeof(uint64_t));
    ctx->frame_best.ensure((size_t)2 * L.groups * L.fpw * sizeof(FrameBest));
    ctx->budget.ensure((size_t)L.groups * L.fpw * sizeof(int64_t));
    for (int gi = 0; gi < L.groups; ++gi) {
      uint64_t* ctr = ctx->counter.as<uint64_t>() + 8 * gi;
      SCB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint64_t) * 4, st));
      uint64_t* lanes = reinterpret_cast<uint64_t*>(ctx->lanes.as<uint8_t>() + lane_bytes * gi);
      const int fig = std::min(L.fpw, L.frames - gi * L.fpw);
      FinArgs fa{};
      fa.fpw = L.fpw;
      fa.frames_in_group = fig;
      fa.n_lanes = n_lanes;
      fa.lanes = lanes;
      fa.ops = plan->tr_ops.as<uint32_t>();
      fa.skel_pos = plan->tr_skel_pos.as<uint32_t>();
      fa.nskel = plan->trace_nskel;
      fa.nr = (uint32_t)L.nr;
      fa.cols = g.cols;
      fa.rows = g.rows;
      fa.count = trace_shard_count(plan, ctx->shard_rank, ctx->shard_world);
      fa.lambda = cfg.lambda;
      fa.vals = ctx->vals.as<uint64_t>() + (size_t)gi * L.fpw * L.nr;
      fa.nvals = ctx->nvals.as<uint32_t>() + (size_t)gi * L.fpw;
      fa.nr_vals = L.nr;
      fa.out = ctx->frame_best.as<FrameBest>() + (size_t)gi * L.fpw;
      fa.budget_out = ctx->budget.as<int64_t>() + (size_t)gi * L.fpw;
      // a single-frame call with 256-thread blocks: the walk's last block
      // finalizes (SLICECRAFT_B200_FUSE_FIN=0: separate launch)
      const bool fuse = fig == 1 && L.fpw == 1 && warps == 8 && fuse_finalize_enabled();
      trace_walk_launch(L.fpw, blocks, warps, ctx->sm_count, plan->tr_ops.as<uint32_t>(),
                        plan->tr_chunks.as<uint4>(), plan->trace_chunks,
                        (uint32_t)ctx->shard_rank, (uint32_t)ctx->shard_world,
                        reinterpret_cast<uint32_t*>(ctr), rt_of(ctx, L, gi), (uint32_t)L.nr,
                        depth_cap, lanes, fuse ? &fa : nullptr,
                        reinterpret_cast<uint32_t*>(ctr + 1), st);
      if (!fuse) trace_finalize_launch(fa, st);
    }
    return;
  }
  const int bps =
      search_blocks_per_sm(L.fpw, step, prune,
                           search_smem_bytes(g.cols, g.rows, cfg.n_slices, step, prune));
  const int blocks = ctx->sm_count * bps;
  const uint32_t warps = (uint32_t)blocks * (search_block_threads(step, prune) / 32);
  const size_t lane_bytes = (size_t)warps * 32 * sizeof(LaneBest);
  const size_t snap_bytes = (size_t)warps * 32 * kSnapBytes;
  ctx->lanes.ensure(lane_bytes * L.groups);
  ctx->snaps.ensure(snap_bytes * L.groups);
  ctx->counter.ensure((size_t)L.groups * 8 * sizeof(uint64_t));
  ctx->frame_best.ensure((size_t)2 * L.groups * L.fpw * sizeof(FrameBest));
  ctx->budget.ensure((size_t)L.groups * L.fpw * sizeof(int64_t));
  // per group: 4 u64 per step = {item counter, candidates, scored, pad}
  uint64_t* ctr_base = ctx->counter.as<uint64_t>() + (step - 1) * 4;
  SCB_CUDA(cudaMemsetAsync(ctr_base, 0, sizeof(uint64_t) * 4, st));
  for (int gi = 1; gi < L.groups; ++gi)
    SCB_CUDA(cudaMemsetAsync(ctr_base + 8 * gi, 0, sizeof(uint64_t) * 4, st));
  const uint32_t total = (uint32_t)plan->items.size();
  const uint32_t rank = (uint32_t)ctx->shard_rank, world = (uint32_t)ctx->shard_world;
  const uint32_t mine = total > rank ? (total - rank + world - 1) / world : 0;
  FrameBest* fb = ctx->frame_best.as<FrameBest>() + (size_t)(step - 1) * L.groups * L.fpw;
  const bool sched = step == 1 && !prune && schedule_enabled();
  if (sched && plan->order_state == 2 && (plan->order_rank != rank || plan->order_world != world))
    plan->order_state = 0;  // another shard layout: measure again
  if (sched && plan->order_state != 2) {
    plan->d_cost.ensure(plan->items.size() * sizeof(uint32_t));
    plan->order_state = 1;
    plan->order_rank = rank;
    plan->order_world = world;
  }
  const int rstride = std::min(cfg.n_slices, g.rows) + 1;
  const size_t lb_per_group = (size_t)n_xw(g.cols) * rstride * L.fpw;
  if (prune) {
    ctx->inc.ensure((size_t)L.groups * L.fpw * sizeof(uint64_t));
    ctx->seed_inc.ensure((size_t)L.groups * L.fpw * sizeof(uint64_t));
    // column lower bounds from the time tables; shared incumbents to +inf
    if (compute_bounds) enqueue_column_bounds(ctx, g, cfg, L, st);
    SCB_CUDA(cudaMemsetAsync(ctx->inc.p, 0xff, (size_t)L.groups * L.fpw * sizeof(uint64_t), st));
    if (step == 2) {  // shared SSE incumbents start at "none" (all-ones bits)
      ctx->sse_inc.ensure((size_t)L.groups * L.fpw * sizeof(uint64_t));
      SCB_CUDA(cudaMemsetAsync(ctx->sse_inc.p, 0xff,
                               (size_t)L.groups * L.fpw * sizeof(uint64_t), st));
    }
  }
  for (int gi = 0; gi < L.groups; ++gi) {
    SearchArgs a{};
    a.cols = g.cols;
    a.rows = g.rows;
    a.n = cfg.n_slices;
    a.nyh = n_yh(g.rows);
    a.max_area = g.cols * g.rows;
    a.coverage = cfg.coverage;
    a.items = plan->d_items.as<WorkItem>();
    const uint32_t G =
        prune ? (uint32_t)split_ways(step, cfg.n_slices, cfg.mode == SC_MODE_PRUNED) : 1u;
    a.split_g = (int)G;
    a.split_depth = split_depth(step, cfg.n_slices);
    a.n_items = mine * G;
    a.item_offset = rank;
    a.item_stride = world;
    uint64_t* ctr = ctr_base + 8 * gi;
    a.counter = reinterpret_cast<uint32_t*>(ctr);
    a.count_out = reinterpret_cast<unsigned long long*>(ctr + 1);
    a.scored_out = reinterpret_cast<unsigned long long*>(ctr + 2);
    a.prune = prune ? 1 : 0;
    if (prune) {
      a.lbr = ctx->lbr.as<uint32_t>() + gi * lb_per_group;
      a.lbm = ctx->lbm.as<uint32_t>() + gi * lb_per_group;
      a.inc = ctx->inc.as<uint64_t>() + (size_t)gi * L.fpw;
      if (step == 2) a.sse_inc = ctx->sse_inc.as<uint64_t>() + (size_t)gi * L.fpw;
    }
    a.bmax = plan->d_bmax.as<int32_t>();
    a.pathological = plan->pathological ? 1 : 0;
    a.rt = rt_of(ctx, L, gi);
    a.rts = rts_of(ctx, L, gi);
    a.rs = step == 2 ? ctx->rs_search.as<double>() + (size_t)gi * L.nr * L.fpw : nullptr;
    a.budget = ctx->budget.as<int64_t>() + (size_t)gi * L.fpw;
    if (sched) {
      if (plan->order_state == 2) a.order = plan->d_order.as<uint32_t>();
      else a.cost = plan->d_cost.as<uint32_t>();
    }
#ifdef SCB_DIAG_COSTS  // diagnostics build: per-item walk cycles of every launch
    plan->d_cost.ensure(plan->items.size() * sizeof(uint32_t));
    a.cost = plan->d_cost.as<uint32_t>();
    ctx->diag_step = step;
#endif
    a.lanes = reinterpret_cast<LaneBest*>(ctx->lanes.as<uint8_t>() + lane_bytes * gi);
    a.snaps = ctx->snaps.as<uint8_t>() + snap_bytes * gi;
    const int fig = std::min(L.fpw, L.frames - gi * L.fpw);
    // pruned walks: the items whose width prefix already fails every frame
    // are dropped before the launch (k_item_filter); the survivors, in
    // order, are the launch's item list
    uint32_t* flt_list = nullptr;
    uint32_t* flt_count = nullptr;
    if (prune && item_filter_enabled()) {
      ctx->flt_list.ensure((size_t)(mine + 1) * sizeof(uint32_t) * L.groups);
      ctx->flt_count.ensure(sizeof(uint32_t) * 2 * L.groups);
      flt_list = ctx->flt_list.as<uint32_t>() + (size_t)gi * (mine + 1);
      flt_count = ctx->flt_count.as<uint32_t>() + 2 * gi;
    }
    if (prune && step == 1 && mine > 1) {
      // Seeded branch-and-bound: phase A walks the first items (the smallest
      // column counts, which hold the fast candidates of the family) so every
      // frame has a shared incumbent before phase B spreads the rest of the
      // space over all warps.  Both phases keep each lane's items increasing.
      const uint32_t seed_items = std::min<uint32_t>(mine, plan->seed_items);
      a.k_begin = 0;
      a.n_items = seed_items * G;
      search_launch(L.fpw, step, a, blocks, st);
      uint64_t* frozen = ctx->seed_inc.as<uint64_t>() + (size_t)gi * L.fpw;
      SCB_CUDA(cudaMemcpyAsync(frozen, a.inc, L.fpw * sizeof(uint64_t),
                               cudaMemcpyDeviceToDevice, st));
      // shards: every rank prunes phase B with the global seed incumbent
      if (has_comm(ctx)) comm_min_u64(ctx, frozen, L.fpw, st);
      a.seed_inc = frozen;
      a.k_begin = seed_items * G;
      a.n_items = mine * G;
      a.resume = 1;
      a.counter = reinterpret_cast<uint32_t*>(ctr + 3);
      if (flt_list) {
        item_filter_launch(ctx, a, seed_items, mine, L.fpw, fig, 1, frozen, flt_list, flt_count,
                           st);
        a.order = flt_list;
        a.n_items_dev = flt_count;
        a.k_begin = 0;
      }
      search_launch(L.fpw, step, a, blocks, st);
    } else {
      if (flt_list && step == 2) {
        item_filter_launch(ctx, a, 0, mine, L.fpw, fig, 2, nullptr, flt_list, flt_count, st);
        a.order = flt_list;
        a.n_items_dev = flt_count;
      }
      search_launch(L.fpw, step, a, blocks, st);
    }
    finalize_launch(step, cfg.n_slices, L.fpw, fig, warps, a.lanes, a.snaps, a.count_out,
                    a.scored_out, cfg.lambda,
                    ctx->vals.as<uint64_t>() + (size_t)gi * L.fpw * L.nr,
                    ctx->nvals.as<uint32_t>() + (size_t)gi * L.fpw, L.nr,
                    fb + (size_t)gi * L.fpw,
                    step == 1 ? ctx->budget.as<int64_t>() + (size_t)gi * L.fpw : nullptr,
                    ctx->fin_scratch, st);
  }
}

// Shards: step 1's per-frame time bits (FrameBest::t, all ones when none)
// gathered for the all-reduce, and step 2's budget keys from the global min.
__global__ void k_tmin_gather(const FrameBest* __restrict__ fb, int frames, uint64_t* t) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < frames) t[f] = fb[f].found ? fb[f].t : ~0ull;
}
__global__ void k_budget_from_tmin(const uint64_t* __restrict__ t, int frames, double lambda,
                                   const uint64_t* __restrict__ vals,
                                   const uint32_t* __restrict__ nvals, size_t nr, int fpw,
                                   int64_t* __restrict__ budget) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= frames) return;
  const int g = f / fpw, slot = f % fpw;
  int64_t key = -1;
  if (t[f] != ~0ull) {
    const double b = __dmul_rn(__longlong_as_double((long long)t[f]), __dadd_rn(1.0, lambda));
    const uint64_t bits = (uint64_t)__double_as_longlong(b);
    const uint64_t* fv = vals + ((size_t)g * fpw + slot) * nr;
    uint32_t lo = 0, hi = nvals[f];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (fv[mid] <= bits) lo = mid + 1;
      else hi = mid;
    }
    key = b >= 0.0 ? (int64_t)lo - 1 : -1;
  }
  budget[(size_t)g * fpw + slot] = key;
}

// Device budget keys from caller t_min values (constrained_clustering with a
// caller-supplied t_min; budget = t_min * (1.0 + lambda), search.cpp:344):
// the doubles are computed here, then mapped to time keys on the device.
void upload_budgets(sc_ctx* ctx, const Layouts& L, const double* t_min, double lambda,
                    cudaStream_t st) {
  ctx->h_budget.ensure((size_t)L.frames * sizeof(double));
  double* b = ctx->h_budget.as<double>();
  SCB_CUDA(cudaMemcpy(b, t_min, (size_t)L.frames * sizeof(double), cudaMemcpyDefault));
  for (int f = 0; f < L.frames; ++f) b[f] = b[f] * (1.0 + lambda);
  ctx->budget_f64.ensure((size_t)L.frames * sizeof(double));
  SCB_CUDA(cudaMemcpyAsync(ctx->budget_f64.p, b, (size_t)L.frames * sizeof(double),
                           cudaMemcpyHostToDevice, st));
  ctx->budget.ensure((size_t)L.groups * L.fpw * sizeof(int64_t));
  budget_keys_device(ctx->budget_f64.as<double>(), ctx->vals.as<uint64_t>(),
                     ctx->nvals.as<uint32_t>(), L.nr, L.frames, ctx->budget.as<int64_t>(), st);
}

double bits_to_double(uint64_t b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}


// The per-batch hot path.  luma (host or device) may be NULL when records
// are given; est / records / t_min_in are host or device pointers.
//   main stream : est -> K2/K3 time tables -> step 1 -> [join] -> step 2
//   side stream : luma H2D -> K1 -> K2/K3 moment tables          (overlaps step 1)
// The luma batch on the device: device pointers are used in place; host
// batches are copied on `s`, luma planes only (a frame stride wider than the
// plane, e.g. planar 4:2:0 frames, is skipped by a 2D copy).  Returns the
// device pointer and its frame stride.
const void* stage_luma(sc_ctx* ctx, const void* luma, int bps, int W, int H, size_t pitch,
                       size_t fstride, int frames, cudaStream_t s, size_t* d_fstride) {
  *d_fstride = fstride;
  if (is_device_ptr(luma)) return luma;
  const size_t plane = pitch * (H - 1) + (size_t)W * bps;
  if (frames > 1 && fstride > pitch * H) {
    const size_t dense = pitch * H;
    ctx->luma.ensure(dense * frames);
    SCB_CUDA(cudaMemcpy2DAsync(ctx->luma.p, dense, luma, fstride, plane, frames,
                               cudaMemcpyHostToDevice, s));
    *d_fstride = dense;
    return ctx->luma.p;
  }
  const size_t span = (size_t)(frames - 1) * fstride + plane;
  ctx->luma.ensure(span);
  SCB_CUDA(cudaMemcpyAsync(ctx->luma.p, luma, span, cudaMemcpyHostToDevice, s));
  return ctx->luma.p;
}

// Host uniform_partition (plan.h) with the reference's errors.
UniformPartition uniform_or_fail(const sc_grid& g, int n) {
  UniformPartition u;
  if (n < 1) fail(SC_ERR_GEOMETRY, "slice count must be >= 1");
  if (!uniform_partition(g.cols, g.rows, n, u))
    fail(SC_ERR_GEOMETRY, "slice count " + std::to_string(n) + " exceeds CTU cell count " +
                              std::to_string(g.cols * g.rows));
  return u;
}

// area_constraint_ok (search.cpp:93-108): k * min area > max area.
bool uniform_area_ok(const UniformPartition& u, double k) {
  int64_t amin = INT64_MAX, amax = 0;
  for (size_t i = 0; i < u.rects.size(); i += 4) {
    const int64_t a = (int64_t)u.rects[i + 2] * u.rects[i + 3];
    amin = std::min(amin, a);
    amax = std::max(amax, a);
  }
  return k * (double)amin > (double)amax;
}

// partition_time / partition_sse of `rects` (id order) on the device, from
// est (host/device, may be NULL) and records already in ctx->records (or
// `records`, host/device, may be NULL).  Results in ctx->h_stage.
const sc_partition_stats* eval_partition(sc_ctx* ctx, const sc_grid& g, const std::vector<int>& rects,
                                        const double* est, const sc_ctu_record* records,
                                        bool records_resident, int frames, cudaStream_t s,
                                        double* slice_times, sc_ctu_record* slice_mom) {
  const int n = (int)rects.size() / 4;
  const size_t cells = (size_t)g.cols * g.rows;
  const int nsat = (g.cols + 1) * (g.rows + 1);
  ctx->scratch.ensure(rects.size() * sizeof(int) + (size_t)frames * sizeof(sc_partition_stats) +
                      (size_t)frames * n * (sizeof(double) + sizeof(sc_ctu_record)) + 64);
  int* d_rects = ctx->scratch.as<int>();
  sc_partition_stats* d_out = reinterpret_cast<sc_partition_stats*>(
      ctx->scratch.as<uint8_t>() + ((rects.size() * sizeof(int) + 15) & ~size_t(15)));
  double* d_times = reinterpret_cast<double*>(d_out + frames);
  sc_ctu_record* d_mom = reinterpret_cast<sc_ctu_record*>(d_times + (size_t)frames * n);
  SCB_CUDA(cudaMemcpyAsync(d_rects, rects.data(), rects.size() * sizeof(int),
                           cudaMemcpyHostToDevice, s));
  if (est) {
    ctx->est.ensure((size_t)frames * cells * sizeof(double));
    ctx->sat.ensure((size_t)frames * nsat * sizeof(double));
    SCB_CUDA(cudaMemcpyAsync(ctx->est.p, est, (size_t)frames * cells * sizeof(double),
                             cudaMemcpyDefault, s));
    grid_sat_device(ctx->est.as<double>(), nullptr, g.cols, g.rows, frames, ctx->sat.as<double>(),
                    nullptr, s);
  }
  const bool have_rec = records || records_resident;
  if (have_rec) {
    if (!records_resident) {
      ctx->records.ensure((size_t)frames * cells * sizeof(sc_ctu_record));
      SCB_CUDA(cudaMemcpyAsync(ctx->records.p, records, (size_t)frames * cells * sizeof(sc_ctu_record),
                               cudaMemcpyDefault, s));
    }
    ctx->usat.ensure((size_t)frames * 3 * nsat * sizeof(uint64_t));
    grid_sat_device(nullptr, ctx->records.as<sc_ctu_record>(), g.cols, g.rows, frames, nullptr,
                    ctx->usat.as<uint64_t>(), s);
  }
  partition_eval_device(est ? ctx->sat.as<double>() : nullptr,
                        have_rec ? ctx->usat.as<uint64_t>() : nullptr, d_rects, n, g.cols, g.rows,
                        frames, d_out, d_times, d_mom, s);
  ctx->h_stage.ensure((size_t)frames * sizeof(sc_partition_stats));
  sc_partition_stats* h = ctx->h_stage.as<sc_partition_stats>();
  std::memset(h, 0, (size_t)frames * sizeof(sc_partition_stats));
  SCB_CUDA(cudaMemcpyAsync(h, d_out, (size_t)frames * sizeof(sc_partition_stats),
                           cudaMemcpyDeviceToHost, s));
  if (slice_times && est)
    SCB_CUDA(cudaMemcpyAsync(slice_times, d_times, (size_t)frames * n * sizeof(double),
                             cudaMemcpyDefault, s));
  if (slice_mom && have_rec)
    SCB_CUDA(cudaMemcpyAsync(slice_mom, d_mom, (size_t)frames * n * sizeof(sc_ctu_record),
                             cudaMemcpyDefault, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  return h;
}

// The UniformOnly family (search.cpp:265-275 step 1, 349-364 step 2): the one
// uniform candidate, evaluated on the device for every frame.
void run_uniform(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, int frames,
                 const void* luma, int bps, size_t pitch, size_t fstride, const double* est,
                 const sc_ctu_record* records, const double* t_min_in, bool do1, bool do2,
                 sc_search_result* out, sc_ctu_record* records_out) {
  const UniformPartition u = uniform_or_fail(g, cfg.n_slices);
  if (!uniform_area_ok(u, cfg.k_area))
    fail(SC_ERR_NO_CANDIDATE, "uniform partition violates the area constraint");
  ctx->maps_frames[0] = ctx->maps_frames[1] = 0;  // no ColumnSplit layouts returned
  cudaStream_t s = main_stream(ctx);
  cudaEvent_t* ev = ctx->ev;
  SCB_CUDA(cudaEventRecord(ev[0], s));
  const size_t cells = (size_t)g.cols * g.rows;
  bool resident = false;
  if (do2 && luma) {  // K1 on the batch
    const int W = g.frame_width, H = g.frame_height;
    size_t dfs = fstride;
    const void* d_luma = stage_luma(ctx, luma, bps, W, H, pitch, fstride, frames, s, &dfs);
    ctx->records.ensure(cells * frames * sizeof(sc_ctu_record));
    texture_moments_device(d_luma, bps, W, H, pitch, dfs, g.ctu_size, frames, g.cols, g.rows,
                           ctx->records.as<sc_ctu_record>(), s);
    resident = true;
  }
  const sc_partition_stats* h =
      eval_partition(ctx, g, u.rects, est, do2 ? records : nullptr, resident, frames, s, nullptr,
                     nullptr);
  if (records_out && resident)
    SCB_CUDA(cudaMemcpy(records_out, ctx->records.p, cells * frames * sizeof(sc_ctu_record),
                        cudaMemcpyDefault));
  SCB_CUDA(cudaEventRecord(ev[9], s));
  SCB_CUDA(cudaEventSynchronize(ev[9]));
  const double us = 1000.0 * ev_ms(ev[0], ev[9]);
  for (int i = 0; i < 8; ++i) ctx->timings[i] = 0.0;
  ctx->timings[do1 ? 2 : 3] = us;
  ctx->timings[4] = us;
  ctx->last_best[0].clear();
  ctx->last_best[1].clear();
  for (int f = 0; f < frames; ++f) {
    sc_search_result& r = out[f];
    std::memset(&r, 0, sizeof(r));
    r.origin = SC_ORIGIN_UNIFORM;
    r.argmin.n_slices = r.best.n_slices = cfg.n_slices;
    double t_min = 0.0;
    if (do1) {
      t_min = h[f].max_us;
      r.candidates_step1 = 1;
    } else {
      SCB_CUDA(cudaMemcpy(&t_min, t_min_in + f, sizeof(double), cudaMemcpyDefault));
    }
    r.t_min_us = t_min;
    if (do2) {
      const double budget = t_min * (1.0 + cfg.lambda);
      if (h[f].max_us > budget)
        fail(SC_ERR_NO_CANDIDATE, "uniform partition exceeds the time budget");
      r.t_best_us = h[f].max_us;
      r.sse_best = h[f].sse;
      r.candidates_step2 = 1;
    }
    r.candidates_evaluated = r.candidates_step1 + r.candidates_step2;
    r.time_min_step_us = ctx->timings[2] / frames;
    r.clustering_step_us = ctx->timings[3] / frames;
    r.search_time_us = us / frames;
  }
}

void run_pipeline(sc_ctx* ctx, const sc_grid& g, const sc_search_cfg& cfg, int maxc, int frames,
                  const void* luma, int bps, size_t pitch, size_t fstride, const double* est,
                  const sc_ctu_record* records, const double* t_min_in, bool do1, bool do2,
                  sc_search_result* out, sc_ctu_record* records_out) {
  if (frames < 1) fail(SC_ERR_USAGE, "n_frames must be >= 1");
  if (cfg.family == SC_FAMILY_UNIFORM_ONLY) {
    run_uniform(ctx, g, cfg, frames, luma, bps, pitch, fstride, est, records, t_min_in, do1, do2,
                out, records_out);
    return;
  }
  Plan* plan = get_plan(ctx, g, cfg, maxc);
  upload_plan(ctx, plan);
  const Layouts L = layouts_for(g, frames);
  const size_t cells = (size_t)g.cols * g.rows;
  cudaStream_t s = main_stream(ctx), s2 = ctx->stream2;
  cudaEvent_t* ev = ctx->ev;
  SCB_CUDA(cudaEventRecord(ev[0], s));
  // fork the side stream from the caller's stream
  SCB_CUDA(cudaEventRecord(ev[7], s));
  SCB_CUDA(cudaStreamWaitEvent(s2, ev[7], 0));
  // The main stream goes first: with a host luma batch its small est upload
  // must not queue behind the luma copy on the copy engine, and step 1 then
  // overlaps that copy; with device luma the high-priority time tables take
  // the SMs and K1 (low priority) fills the gaps.
  const bool need_moments = do2;
  // (SLICECRAFT_B200_K1_LATE=0: K1 first for device luma -- measured 1.6 %
  // slower on cfg3: with the main stream at high priority the time tables
  // get the SMs first either way, and K1 fills the gaps)
  const char* k1l = getenv("SLICECRAFT_B200_K1_LATE");
  const bool main_first =
      need_moments && luma && (!is_device_ptr(luma) || !(k1l && k1l[0] == '0'));
  // exhaustive mode: step 1 runs the trace walk (no bounds), the bounded step
  // 2 needs the column bounds -- computed on the side stream beside step 1
  // (only when the main stream is enqueued first: the side stream waits for
  // this call's time tables)
  const bool bounds_on_side = main_first && do1 && do2 && cfg.mode == SC_MODE_EXHAUSTIVE &&
                              step2_bounded(cfg) && side_bounds_enabled();
  // the step-2 trace walk reads {sse, rest sse} pairs gathered per call: when
  // it is known to be step 2's walk (the plan has its trace and this lambda's
  // choice was measured) and there is one frame group, the side stream gathers
  // them right after the moment tables
  ctx->pairs_on_side = false;
  if (do2 && need_moments && L.groups == 1 && cfg.mode == SC_MODE_EXHAUSTIVE &&
      plan->trace_state == 1 && ctx->rest_of.p && trace2_mode() != 1) {
    int choice = trace2_mode() == 2 ? 2 : 0;
    for (const auto& c : plan->step2_choice)
      if (c.first == cfg.lambda && choice == 0) choice = c.second;
    ctx->pairs_on_side = choice == 2;
  }
  auto enqueue_main = [&] {
    ctx->est.ensure((size_t)frames * cells * sizeof(double));
    SCB_CUDA(cudaMemcpyAsync(ctx->est.p, est, (size_t)frames * cells * sizeof(double),
                             cudaMemcpyDefault, s));
    // a plan that has its trace ranks only the rectangles its candidates use
    enqueue_time_tables(ctx, g, L, false, plan->n_used ? plan->tr_used.as<uint32_t>() : nullptr,
                        plan->n_used, plan->tr_used_split.as<uint32_t>(), plan->n_used_split, s);
    SCB_CUDA(cudaEventRecord(ev[1], s));
    if (do1) {
      enqueue_step(ctx, g, cfg, plan, L, 1, true, s);
      if (do2 && has_comm(ctx)) {  // step 2's budget from the global t_min
        ctx->gtmin.ensure((size_t)frames * sizeof(uint64_t));
        SCB_LAUNCH(k_tmin_gather<<<(frames + 127) / 128, 128, 0, s>>>(ctx->frame_best.as<FrameBest>(), frames,
                                                            ctx->gtmin.as<uint64_t>()));
        SCB_CUDA(cudaGetLastError());
        comm_min_u64(ctx, ctx->gtmin.as<uint64_t>(), (size_t)frames, s);
        SCB_LAUNCH(k_budget_from_tmin<<<(frames + 127) / 128, 128, 0, s>>>(
            ctx->gtmin.as<uint64_t>(), frames, cfg.lambda, ctx->vals.as<uint64_t>(),
            ctx->nvals.as<uint32_t>(), L.nr, L.fpw, ctx->budget.as<int64_t>()));
        SCB_CUDA(cudaGetLastError());
      }
    } else {
      upload_budgets(ctx, L, t_min_in, cfg.lambda, s);
    }
    SCB_CUDA(cudaEventRecord(ev[2], s));
  };
  auto enqueue_side = [&] {
    SCB_CUDA(cudaEventRecord(ev[4], s2));
    if (need_moments) {
      ctx->records.ensure(cells * frames * sizeof(sc_ctu_record));
      if (luma) {
        const int W = g.frame_width, H = g.frame_height;
        size_t dfs = fstride;
        const void* d_luma = stage_luma(ctx, luma, bps, W, H, pitch, fstride, frames, s2, &dfs);
        SCB_CUDA(cudaEventRecord(ev[4], s2));
        texture_moments_device(d_luma, bps, W, H, pitch, dfs, g.ctu_size, frames, g.cols, g.rows,
                               ctx->records.as<sc_ctu_record>(), s2);
      } else {
        SCB_CUDA(cudaMemcpyAsync(ctx->records.p, records, cells * frames * sizeof(sc_ctu_record),
                                 cudaMemcpyDefault, s2));
        SCB_CUDA(cudaEventRecord(ev[4], s2));
      }
    }
    SCB_CUDA(cudaEventRecord(ev[5], s2));
    if (need_moments) enqueue_moment_tables(ctx, g, L, false, s2);
    SCB_CUDA(cudaEventRecord(ev[6], s2));
    if (ctx->pairs_on_side) {  // the step-2 trace walk's {sse, rest sse} pairs, off the main stream
      ctx->rss.ensure(L.nr * L.fpw * 2 * sizeof(double));
      rest_pairs_device(ctx->rs_search.as<double>(), ctx->rest_of.as<uint32_t>(), (uint32_t)L.nr,
                        L.fpw, ctx->rss.as<double>(), ctx->sm_count, s2);
    }
    if (bounds_on_side) {  // after this call's time tables (ev[1], already recorded on s)
      SCB_CUDA(cudaStreamWaitEvent(s2, ev[1], 0));
      enqueue_column_bounds(ctx, g, cfg, L, s2);
    }
    SCB_CUDA(cudaEventRecord(ev[10], s2));
  };
  if (main_first) {
    enqueue_main();
    enqueue_side();
  } else {
    enqueue_side();
    enqueue_main();
  }
  SCB_CUDA(cudaStreamWaitEvent(s, ev[10], 0));  // join
  SCB_CUDA(cudaEventRecord(ev[8], s));
  if (do2)
    enqueue_step(ctx, g, cfg, plan, L, 2, (!do1 || step2_bounded(cfg)) && !bounds_on_side, s);
  SCB_CUDA(cudaEventRecord(ev[3], s));
  // device post-check of the partitions this call returns (validate_partition,
  // grid.cpp:86-184, over the columns the layout spans) and their CTU ->
  // slice-id maps (sc_result_slice_maps)
  const bool post = postcheck_enabled();
  const size_t vb = (size_t)frames * sizeof(VCheck);
  const size_t nfb = (size_t)2 * L.groups * L.fpw;
  ctx->h_frame_best.ensure(nfb * sizeof(FrameBest));
  if (post) {  // both steps' partitions in one launch
    ctx->slice_maps.ensure((size_t)2 * frames * cells * sizeof(int32_t));
    ctx->owner.ensure((size_t)2 * frames * cells * sizeof(int));
    ctx->h_vcheck.ensure(2 * vb);
    // the kernel writes its verdicts and the FrameBest records straight into
    // pinned host memory: no device-to-host copy on the call's critical path
    result_maps_device(ctx->frame_best.as<FrameBest>(), (size_t)L.groups * L.fpw, frames,
                       do1 ? 1 : 2, (do1 ? 1 : 0) + (do2 ? 1 : 0), cfg.n_slices, g.cols, g.rows,
                       ctx->owner.as<int>(), ctx->slice_maps.as<int32_t>(),
                       ctx->h_vcheck.as<VCheck>(), ctx->h_frame_best.as<FrameBest>(), s);
  } else {
    SCB_CUDA(cudaMemcpyAsync(ctx->h_frame_best.p, ctx->frame_best.p, nfb * sizeof(FrameBest),
                             cudaMemcpyDeviceToHost, s));
  }
  ctx->maps_cells = cells;
  ctx->maps_frames[0] = post && do1 ? frames : 0;
  ctx->maps_frames[1] = post && do2 ? frames : 0;
  if (records_out && need_moments)
    SCB_CUDA(cudaMemcpyAsync(records_out, ctx->records.p, cells * frames * sizeof(sc_ctu_record),
                             cudaMemcpyDefault, s));
  SCB_CUDA(cudaEventRecord(ev[9], s));
  SCB_CUDA(cudaStreamSynchronize(s));
  finish_schedule(plan);
  if (ctx->s2_pending) {
    // the first call of a (plan, lambda) warms both step-2 walks (their
    // first-use allocations), the second times them; later calls take the
    // faster one
    const float dfs = ev_ms(ctx->ev_s2[0], ctx->ev_s2[1]), tr = ev_ms(ctx->ev_s2[1], ctx->ev_s2[2]);
    auto& ch = ctx->s2_plan->step2_choice;
    auto it = ch.begin();
    while (it != ch.end() && it->first != ctx->s2_lambda) ++it;
    if (it == ch.end()) ch.push_back({ctx->s2_lambda, 0});  // warmed
    else it->second = tr < dfs ? 2 : 1;                     // measured
    ctx->s2_pending = false;
  }
  if (post) {
    const VCheck* vc = ctx->h_vcheck.as<VCheck>();
    for (int st = 1; st <= 2; ++st)
      for (int f = 0; f < frames && ctx->maps_frames[st - 1]; ++f) {
        const VCheck& v = vc[(size_t)(st - 1) * frames + f];
        if (v.status != SC_OK)
          fail(SC_ERR_INTERNAL, "device post-check: the step-" + std::to_string(st) +
                                    " partition of frame " + std::to_string(f) +
                                    " failed validate_partition (status " +
                                    std::to_string(v.status) + ")");
      }
  }
#ifdef SCB_DIAG_COSTS
  if (const char* path = getenv("SCB_DIAG_COSTS_OUT")) {
    std::vector<uint32_t> cost(plan->items.size());
    SCB_CUDA(cudaMemcpy(cost.data(), plan->d_cost.p, cost.size() * 4, cudaMemcpyDeviceToHost));
    if (FILE* fp = fopen(path, "wb")) {
      fwrite(cost.data(), 4, cost.size(), fp);
      fclose(fp);
    }
  }
#endif
  // timings
  ctx->timings[0] = need_moments && luma ? 1000.0 * ev_ms(ev[4], ev[5]) : 0.0;
  ctx->timings[1] = 1000.0 * (ev_ms(ev[0], ev[1]) + (need_moments ? ev_ms(ev[5], ev[6]) : 0.f));
  ctx->timings[2] = do1 ? 1000.0 * ev_ms(ev[1], ev[2]) : 0.0;
  ctx->timings[3] = do2 ? 1000.0 * ev_ms(ev[8], ev[3]) : 0.0;
  ctx->timings[4] = 1000.0 * ev_ms(ev[0], ev[9]);
  ctx->timings[5] = 1000.0 * ev_ms(ev[0], ev[1]);                        // time tables (main)
  ctx->timings[6] = need_moments ? 1000.0 * ev_ms(ev[5], ev[6]) : 0.0;   // moment tables (side)
  ctx->timings[7] = 1000.0 * ev_ms(ev[3], ev[9]);                        // post-check + copies
  // results
  const FrameBest* hb = ctx->h_frame_best.as<FrameBest>();
  const FrameBest* b1 = hb;
  const FrameBest* b2 = hb + (size_t)L.groups * L.fpw;
  ctx->last_best[0].assign(b1, b1 + frames);
  ctx->last_best[1].assign(b2, b2 + frames);
  ctx->last_pruned = cfg.mode == SC_MODE_PRUNED;
  ctx->last_fpw = L.fpw;
  // walks that skip subtrees report the family's exact DP count (plan.h);
  // shards export it from rank 0 only
  const bool dp1 = cfg.mode == SC_MODE_PRUNED;
  const bool dp2 = dp1 || (do2 && step2_bounded(cfg));
  ctx->last_count_hi[0] = ctx->last_count_hi[1] = 0;
  if (dp1 || dp2) {
    const unsigned __int128 cnt = plan_count(plan, g, cfg);
    for (int s2 = 0; s2 < 2; ++s2)
      if (s2 == 0 ? dp1 : dp2)
        for (auto& fbv : ctx->last_best[s2]) fbv.count = ctx->shard_rank == 0 ? (uint64_t)cnt : 0;
    for (int s2 = 0; s2 < 2; ++s2)
      ctx->last_count_hi[s2] =
          ((s2 == 0 ? dp1 : dp2) && ctx->shard_rank == 0) ? (uint64_t)(cnt >> 64) : 0;
  }
  const bool whole = ctx->shard_world == 1;  // false: per-shard results, merged later
  for (int f = 0; f < frames; ++f) {
    sc_search_result& r = out[f];
    std::memset(&r, 0, sizeof(r));
    if (do1) {
      // a shard may hold no candidate of a frame: sc_shard_merge decides
      if (!b1[f].found && whole)
        fail(SC_ERR_NO_CANDIDATE, "area constraint admits no candidate partition");
      r.t_min_us = bits_to_double(b1[f].t);
      r.candidates_step1 = b1[f].count;
      r.leaves_scored_step1 = b1[f].scored / (uint64_t)L.fpw;
      layout_from_snap(b1[f], cfg.n_slices, &r.argmin);
    } else if (t_min_in) {
      double tm;
      SCB_CUDA(cudaMemcpy(&tm, t_min_in + f, sizeof(double), cudaMemcpyDefault));
      r.t_min_us = tm;
    }
    if (do2) {
      if (!b2[f].found && whole) fail(SC_ERR_NO_CANDIDATE, "no candidate within the time budget");
      r.t_best_us = bits_to_double(b2[f].t);
      r.sse_best = b2[f].sse;
      r.candidates_step2 = b2[f].count;
      r.leaves_scored_step2 = b2[f].scored / (uint64_t)L.fpw;
      layout_from_snap(b2[f], cfg.n_slices, &r.best);
    }
    if (dp1 || dp2) {
      // walks that skip subtrees do not enumerate every candidate: the
      // counters come from the exact DP (plan.h count_candidates_dp) -- the
      // reference's values
      const unsigned __int128 cnt = plan_count(plan, g, cfg);
      if (do1 && dp1) {
        r.candidates_step1 = (uint64_t)cnt;
        r.candidates_step1_hi = (uint64_t)(cnt >> 64);
      }
      if (do2 && dp2) {
        r.candidates_step2 = (uint64_t)cnt;
        r.candidates_step2_hi = (uint64_t)(cnt >> 64);
      }
    }
    r.candidates_evaluated = r.candidates_step1 + r.candidates_step2;
    r.time_min_step_us = ctx->timings[2] / frames;
    r.clustering_step_us = ctx->timings[3] / frames;
    r.search_time_us = (ctx->timings[2] + ctx->timings[3]) / frames;
  }
  if (has_comm(ctx)) {  // the library's exchange: every rank returns the merged results
    const int W = ctx->shard_world;
    std::vector<sc_shard_best> mine(frames), all((size_t)W * frames);
    for (int st = 1; st <= 2; ++st) {
      if (st == 1 ? !do1 : !do2) continue;
      export_shards(ctx, st, frames, mine.data());
      comm_allgather_host(ctx, mine.data(), mine.size() * sizeof(sc_shard_best), all.data(), s);
      merge_shards(st, W, frames, all.data(), out);
    }
  }
}

}  // namespace

sc_ctx::~sc_ctx() {
  if (tt_exec) cudaGraphExecDestroy(tt_exec);
  for (auto* b : {&luma, &records, &est, &sat, &rect_t, &rect_s, &rt_search, &rs_search, &usat,
                  &lanes, &snaps, &frame_best, &counter, &budget, &scratch, &dec, &lbr, &lbm, &inc, &seed_inc, &rt_bits, &vals, &nvals, &budget_f64, &rk_idx, &rk_sorted,
                  &rk_flags, &rk_offsets, &rk_temp, &rk_bits_c, &sse_inc, &flt_idx, &flt_flag, &flt_list,
                  &flt_count, &flt_temp, &slice_maps, &owner, &vcheck, &val_in, &enum_out,
                  &enum_temp, &rest_of, &rss, &fin_scratch})
    b->release();
  h_vcheck.release();
  h_stage.release();
  h_luma.release();
  h_records.release();
  h_frame_best.release();
  h_budget.release();
  for (Plan* p : plans) {
    p->d_items.release();
    p->d_bmax.release();
    p->d_order.release();
    p->d_cost.release();
    p->d_enum_counts.release();
    p->d_enum_offsets.release();
    for (auto* b : {&p->tr_ops, &p->tr_skel_pos, &p->tr_skel_ord, &p->tr_chunks, &p->tr_skip,
                    &p->tr_used, &p->tr_used_split})
      b->release();
    delete p;
  }
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_s2)
    if (e) cudaEventDestroy(e);
  if (comm_kind == 1 && nccl_comm) nccl().commDestroy((ncclComm_t)nccl_comm);
  comm_buf.release();
  gtmin.release();
  if (stream) cudaStreamDestroy(stream);
  if (stream2) cudaStreamDestroy(stream2);
}

// Lexicographic (widths, runs, heights) order of two layouts of one work
// item: the reference's enumeration order (search.cpp:120-190).
bool layout_less(const sc_layout& a, const sc_layout& b) {
  for (int i = 0; i < SC_MAX_COLS; ++i)
    if (a.col_widths[i] != b.col_widths[i]) return a.col_widths[i] < b.col_widths[i];
  for (int i = 0; i < SC_MAX_COLS; ++i)
    if (a.runs_per_col[i] != b.runs_per_col[i]) return a.runs_per_col[i] < b.runs_per_col[i];
  for (int i = 0; i < SC_MAX_SLICES; ++i)
    if (a.run_heights[i] != b.run_heights[i]) return a.run_heights[i] < b.run_heights[i];
  return false;
}

extern "C" {

uint64_t sc_kernel_launches(void) { return scb::launch_counter(); }

const char* sc_last_error(void) { return g_last_error.c_str(); }
int sc_abi_version(void) { return SC_ABI_VERSION; }

sc_status sc_grid_make(int32_t w, int32_t h, int32_t ctu, sc_grid* out) {
  return guarded([&] {
    if (!out) fail(SC_ERR_USAGE, "out is NULL");
    *out = make_grid(w, h, ctu);
  });
}

// temporal_layer_of_poc (cost.cpp:28-38)
sc_status sc_temporal_layer(int32_t poc, int32_t gop, int32_t* out) {
  return guarded([&] {
    if (gop < 1 || (gop & (gop - 1)) != 0)
      fail(SC_ERR_CONFIG, "gop size must be a power of two, got " + std::to_string(gop));
    if (poc < 0) fail(SC_ERR_CONFIG, "poc must be >= 0");
    const unsigned rem = (unsigned)poc % (unsigned)gop;
    *out = rem == 0 ? 0 : (__builtin_ctz((unsigned)gop) - __builtin_ctz(rem));
  });
}

sc_status sc_search_cfg_check(const sc_search_cfg* cfg) {
  return guarded([&] { check_cfg_fields(cfg); });
}

sc_status sc_ctx_create(int32_t device, sc_ctx** out) {
  return guarded([&] {
    if (!out) fail(SC_ERR_USAGE, "out is NULL");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(SC_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= n) fail(SC_ERR_CUDA, "device index out of range");
    SCB_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    SCB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      fail(SC_ERR_CUDA, std::string("device is not sm_100-class: ") + prop.name);
    sc_ctx* c = new sc_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    // the side stream (K1 + moment tables, overlapping the time tables and
    // step 1) runs at low priority: as SM slots free up the block scheduler
    // prefers the critical-path kernels of the main stream
    int prio_lo = 0, prio_hi = 0;
    SCB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SCB_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
    SCB_CUDA(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_lo));
    for (auto& e : c->ev) SCB_CUDA(cudaEventCreate(&e));
    for (auto& e : c->ev_s2) SCB_CUDA(cudaEventCreate(&e));
    *out = c;
  });
}

sc_status sc_ctx_destroy(sc_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
  });
}

sc_status sc_ctx_set_shard(sc_ctx* ctx, int32_t rank, int32_t world) {
  return guarded([&] {
    if (!ctx) fail(SC_ERR_USAGE, "ctx is NULL");
    if (world < 1 || rank < 0 || rank >= world) fail(SC_ERR_CONFIG, "bad shard rank/world");
    ctx->shard_rank = rank;
    ctx->shard_world = world;
  });
}

sc_status sc_texture_validate(const sc_grid* grid, const sc_ctu_record* records) {
  return guarded([&] {
    check_grid(grid);
    if (!records) fail(SC_ERR_USAGE, "records is NULL");
    validate_records(*grid, records);
  });
}

sc_status sc_ctx_set_stream(sc_ctx* ctx, void* cuda_stream) {
  return guarded([&] {
    if (!ctx) fail(SC_ERR_USAGE, "ctx is NULL");
    ctx->user_stream = static_cast<cudaStream_t>(cuda_stream);
  });
}

sc_status sc_ctx_timings(sc_ctx* ctx, double out[5]) {
  return guarded([&] {
    if (!ctx || !out) fail(SC_ERR_USAGE, "NULL argument");
    for (int i = 0; i < 5; ++i) out[i] = ctx->timings[i];
  });
}

sc_status sc_ctx_timings_ex(sc_ctx* ctx, int32_t n, double* out) {
  return guarded([&] {
    if (!ctx || !out || n < 0) fail(SC_ERR_USAGE, "bad argument");
    for (int i = 0; i < n; ++i) out[i] = i < 8 ? ctx->timings[i] : 0.0;
  });
}

sc_status sc_texture_moments(sc_ctx* ctx, const void* luma, int32_t bps, int32_t width,
                             int32_t height, size_t pitch, size_t fstride, int32_t ctu,
                             int32_t frames, sc_ctu_record* out) {
  return guarded([&] {
    if (!ctx || !luma || !out) fail(SC_ERR_USAGE, "NULL argument");
    SCB_CUDA(cudaSetDevice(ctx->device));
    sc_grid g = make_grid(width, height, ctu);
    if (bps != 1 && bps != 2) fail(SC_ERR_FORMAT, "bytes_per_sample must be 1 or 2");
    if (frames < 1) fail(SC_ERR_USAGE, "n_frames must be >= 1");
    if (pitch < (size_t)width * bps) fail(SC_ERR_GEOMETRY, "pitch smaller than a row");
    if (frames > 1 && fstride < pitch * height) fail(SC_ERR_GEOMETRY, "frame stride too small");
    cudaStream_t s = main_stream(ctx);
    size_t dfs = fstride;
    const void* d_luma = stage_luma(ctx, luma, bps, width, height, pitch, fstride, frames, s, &dfs);
    const size_t cells = (size_t)g.cols * g.rows;
    sc_ctu_record* d_out = out;
    const bool out_dev = is_device_ptr(out);
    if (!out_dev) {
      ctx->records.ensure(cells * frames * sizeof(sc_ctu_record));
      d_out = ctx->records.as<sc_ctu_record>();
    }
    SCB_CUDA(cudaEventRecord(ctx->ev[4], s));
    texture_moments_device(d_luma, bps, width, height, pitch, dfs, ctu, frames, g.cols, g.rows,
                           d_out, s);
    SCB_CUDA(cudaEventRecord(ctx->ev[5], s));
    if (!out_dev)
      SCB_CUDA(cudaMemcpyAsync(out, d_out, cells * frames * sizeof(sc_ctu_record),
                               cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    ctx->timings[0] = 1000.0 * ev_ms(ctx->ev[4], ctx->ev[5]);
  });
}

sc_status sc_grid_tables(sc_ctx* ctx, const sc_grid* grid, const double* est,
                         const sc_ctu_record* records, int32_t frames, double* rect_time,
                         double* rect_sse, double* sat) {
  return guarded([&] {
    if (!ctx || !est) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    if (frames < 1) fail(SC_ERR_USAGE, "n_frames must be >= 1");
    SCB_CUDA(cudaSetDevice(ctx->device));
    const sc_grid& g = *grid;
    const size_t cells = (size_t)g.cols * g.rows;
    if (records && !is_device_ptr(records))
      for (int f = 0; f < frames; ++f) validate_records(g, records + f * cells);
    const Layouts L = layouts_for(g, frames);
    cudaStream_t s = main_stream(ctx);
    ctx->est.ensure((size_t)frames * cells * sizeof(double));
    SCB_CUDA(cudaMemcpyAsync(ctx->est.p, est, (size_t)frames * cells * sizeof(double),
                             cudaMemcpyDefault, s));
    enqueue_time_tables(ctx, g, L, true, nullptr, 0, nullptr, 0, s);
    if (records) {
      ctx->records.ensure(cells * frames * sizeof(sc_ctu_record));
      SCB_CUDA(cudaMemcpyAsync(ctx->records.p, records, cells * frames * sizeof(sc_ctu_record),
                               cudaMemcpyDefault, s));
      enqueue_moment_tables(ctx, g, L, true, s);
    }
    if (sat)
      SCB_CUDA(cudaMemcpyAsync(sat, ctx->sat.p, (size_t)frames * L.nsat * sizeof(double),
                               cudaMemcpyDefault, s));
    if (rect_time)
      SCB_CUDA(cudaMemcpyAsync(rect_time, ctx->rect_t.p, (size_t)frames * L.nr * sizeof(double),
                               cudaMemcpyDefault, s));
    if (rect_sse && records)
      SCB_CUDA(cudaMemcpyAsync(rect_sse, ctx->rect_s.p, (size_t)frames * L.nr * sizeof(double),
                               cudaMemcpyDefault, s));
    SCB_CUDA(cudaStreamSynchronize(s));
  });
}

sc_status sc_min_time_search(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                             const double* est, int32_t frames, sc_search_result* out) {
  return guarded([&] {
    if (!ctx || !est || !out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    SCB_CUDA(cudaSetDevice(ctx->device));
    run_pipeline(ctx, *grid, *cfg, maxc, frames, nullptr, 0, 0, 0, est, nullptr, nullptr, true,
                 false, out, nullptr);
  });
}

sc_status sc_constrained_clustering(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                                    const double* est, const sc_ctu_record* records,
                                    const double* t_min, int32_t frames, sc_search_result* out) {
  return guarded([&] {
    if (!ctx || !est || !records || !t_min || !out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    SCB_CUDA(cudaSetDevice(ctx->device));
    const size_t cells = (size_t)grid->cols * grid->rows;
    if (!is_device_ptr(records))
      for (int f = 0; f < frames; ++f) validate_records(*grid, records + f * cells);
    run_pipeline(ctx, *grid, *cfg, maxc, frames, nullptr, 0, 0, 0, est, records, t_min, false,
                 true, out, nullptr);
  });
}

sc_status sc_two_step(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                      const double* est, const sc_ctu_record* records, int32_t frames,
                      sc_search_result* out) {
  return guarded([&] {
    if (!ctx || !est || !records || !out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    SCB_CUDA(cudaSetDevice(ctx->device));
    const size_t cells = (size_t)grid->cols * grid->rows;
    if (!is_device_ptr(records))
      for (int f = 0; f < frames; ++f) validate_records(*grid, records + f * cells);
    run_pipeline(ctx, *grid, *cfg, maxc, frames, nullptr, 0, 0, 0, est, records, nullptr, true,
                 true, out, nullptr);
  });
}

sc_status sc_partition_frames(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                              const void* luma, int32_t bps, size_t pitch, size_t fstride,
                              const double* est, int32_t frames, sc_ctu_record* records_out,
                              sc_search_result* out) {
  return guarded([&] {
    if (!ctx || !luma || !est || !out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    SCB_CUDA(cudaSetDevice(ctx->device));
    if (bps != 1 && bps != 2) fail(SC_ERR_FORMAT, "bytes_per_sample must be 1 or 2");
    if (pitch < (size_t)grid->frame_width * bps) fail(SC_ERR_GEOMETRY, "pitch smaller than a row");
    if (frames > 1 && fstride < pitch * grid->frame_height)
      fail(SC_ERR_GEOMETRY, "frame stride too small");
    run_pipeline(ctx, *grid, *cfg, maxc, frames, luma, bps, pitch, fstride, est, nullptr, nullptr,
                 true, true, out, records_out);
  });
}

sc_status sc_count_candidates(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                              uint64_t* count) {
  return guarded([&] {
    if (!ctx || !count) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    SCB_CUDA(cudaSetDevice(ctx->device));
    const size_t cells = (size_t)grid->cols * grid->rows;
    std::vector<double> ones(cells, 1.0);
    sc_search_result r;
    if (cfg->family == SC_FAMILY_UNIFORM_ONLY) {  // for_each_candidate (search.cpp:308-312)
      *count = uniform_area_ok(uniform_or_fail(*grid, cfg->n_slices), cfg->k_area) ? 1 : 0;
      return;
    }
    run_pipeline(ctx, *grid, *cfg, maxc, 1, nullptr, 0, 0, 0, ones.data(), nullptr, nullptr, true,
                 false, &r, nullptr);
    *count = r.candidates_step1;
  });
}

sc_status sc_yuv_frame_count(const char* path, int32_t w, int32_t h, int32_t bit_depth,
                             int32_t* out) {
  return guarded([&] {
    if (!path || !out) fail(SC_ERR_USAGE, "NULL argument");
    *out = yuv_frame_count(path, w, h, bit_depth);
  });
}

sc_status sc_yuv_load_luma(const char* path, int32_t w, int32_t h, int32_t poc,
                           int32_t bit_depth, uint16_t* out) {
  return guarded([&] {
    if (!path || !out) fail(SC_ERR_USAGE, "NULL argument");
    const int bps = yuv_bytes_per_sample(bit_depth);
    const size_t n = (size_t)w * h;
    if (bps == 2) {  // little-endian 16-bit containers (texture.cpp:64-72)
      std::vector<uint8_t> raw(n * 2);
      yuv_read_luma(path, w, h, bit_depth, poc, 1, raw.data());
      for (size_t i = 0; i < n; ++i) out[i] = (uint16_t)(raw[2 * i] | (raw[2 * i + 1] << 8));
    } else {
      std::vector<uint8_t> raw(n);
      yuv_read_luma(path, w, h, bit_depth, poc, 1, raw.data());
      for (size_t i = 0; i < n; ++i) out[i] = raw[i];
    }
  });
}

sc_status sc_yuv_read_luma(const char* path, int32_t w, int32_t h, int32_t bit_depth,
                           int32_t first, int32_t n, void* out) {
  return guarded([&] {
    if (!path || !out) fail(SC_ERR_USAGE, "NULL argument");
    yuv_read_luma(path, w, h, bit_depth, first, n, out);
  });
}

// Luma planes of a YUV file in the context's pinned staging buffer.
const void* yuv_stage(sc_ctx* ctx, const char* path, int w, int h, int bit_depth, int first,
                      int n) {
  const size_t plane = (size_t)w * h * yuv_bytes_per_sample(bit_depth);
  ctx->h_luma.ensure(plane * (size_t)std::max(n, 1));
  yuv_read_luma(path, w, h, bit_depth, first, n, ctx->h_luma.p);
  return ctx->h_luma.p;
}

sc_status sc_yuv_texture_moments(sc_ctx* ctx, const char* path, int32_t w, int32_t h,
                                 int32_t bit_depth, int32_t ctu, int32_t first, int32_t n,
                                 sc_ctu_record* out) {
  if (!ctx || !path || !out) return set_error(SC_ERR_USAGE, "NULL argument");
  const void* luma = nullptr;
  const sc_status st = guarded([&] { luma = yuv_stage(ctx, path, w, h, bit_depth, first, n); });
  if (st != SC_OK) return st;
  const int bps = bit_depth == 8 ? 1 : 2;
  return sc_texture_moments(ctx, luma, bps, w, h, (size_t)w * bps, (size_t)w * h * bps, ctu, n,
                            out);
}

sc_status sc_partition_yuv(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                           const char* path, int32_t bit_depth, int32_t first, int32_t n,
                           const double* est, sc_ctu_record* records_out, sc_search_result* out) {
  if (!ctx || !grid || !path) return set_error(SC_ERR_USAGE, "NULL argument");
  const void* luma = nullptr;
  const sc_status st = guarded([&] {
    luma = yuv_stage(ctx, path, grid->frame_width, grid->frame_height, bit_depth, first, n);
  });
  if (st != SC_OK) return st;
  const int bps = bit_depth == 8 ? 1 : 2;
  const int W = grid->frame_width, H = grid->frame_height;
  return sc_partition_frames(ctx, grid, cfg, luma, bps, (size_t)W * bps, (size_t)W * H * bps, est,
                             n, records_out, out);
}

sc_status sc_uniform_partition(const sc_grid* grid, int32_t n_slices, sc_partition* out) {
  return guarded([&] {
    if (!out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const UniformPartition u = uniform_or_fail(*grid, n_slices);
    std::memset(out, 0, sizeof(*out));
    if (n_slices > SC_MAX_SLICES) fail(SC_ERR_SIZE, "n_slices exceeds SC_MAX_SLICES");
    out->n_tile_cols = (int32_t)u.tile_cols.size();
    out->n_tile_rows = (int32_t)u.tile_rows.size();
    for (size_t i = 0; i < u.tile_cols.size(); ++i) out->tile_col_widths[i] = u.tile_cols[i];
    for (size_t i = 0; i < u.tile_rows.size(); ++i) out->tile_row_heights[i] = u.tile_rows[i];
    out->n_slices = n_slices;
    out->origin = SC_ORIGIN_UNIFORM;
    for (int i = 0; i < n_slices; ++i)
      out->slices[i] = sc_rect{u.rects[4 * i], u.rects[4 * i + 1], u.rects[4 * i + 2],
                               u.rects[4 * i + 3], i};
  });
}

sc_status sc_uniform_partition_n(const sc_grid* grid, int32_t n_slices, int32_t* tile_col_widths,
                                 int32_t* n_tile_cols, int32_t* tile_row_heights,
                                 int32_t* n_tile_rows, sc_rect* slices) {
  return guarded([&] {
    if (!tile_col_widths || !n_tile_cols || !tile_row_heights || !n_tile_rows || !slices)
      fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const UniformPartition u = uniform_or_fail(*grid, n_slices);
    *n_tile_cols = (int32_t)u.tile_cols.size();
    *n_tile_rows = (int32_t)u.tile_rows.size();
    for (size_t i = 0; i < u.tile_cols.size(); ++i) tile_col_widths[i] = u.tile_cols[i];
    for (size_t i = 0; i < u.tile_rows.size(); ++i) tile_row_heights[i] = u.tile_rows[i];
    for (int i = 0; i < n_slices; ++i)
      slices[i] = sc_rect{u.rects[4 * i], u.rects[4 * i + 1], u.rects[4 * i + 2],
                          u.rects[4 * i + 3], i};
  });
}

sc_status sc_partition_eval(sc_ctx* ctx, const sc_grid* grid, const sc_rect* slices,
                            int32_t n_slices, const double* est, const sc_ctu_record* records,
                            int32_t frames, sc_partition_stats* out, double* slice_times,
                            sc_ctu_record* slice_moments) {
  return guarded([&] {
    if (!ctx || !slices || !out) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    if (frames < 1) fail(SC_ERR_USAGE, "n_frames must be >= 1");
    if (n_slices < 1 || n_slices > SC_MAX_SLICES)
      fail(SC_ERR_SIZE, "slice count must be in [1, SC_MAX_SLICES]");
    std::vector<int> rects((size_t)n_slices * 4, 0);
    std::vector<char> seen((size_t)n_slices, 0);
    for (int i = 0; i < n_slices; ++i) {
      const sc_rect& r = slices[i];
      if (r.id < 0 || r.id >= n_slices || seen[(size_t)r.id])
        fail(SC_ERR_USAGE, "slice ids must be a permutation of 0..n_slices-1");
      if (r.w < 1 || r.h < 1 || r.x0 < 0 || r.y0 < 0 || r.x0 + r.w > grid->cols ||
          r.y0 + r.h > grid->rows)
        fail(SC_ERR_GEOMETRY, "slice outside the CTU grid");
      seen[(size_t)r.id] = 1;
      int* d = &rects[(size_t)r.id * 4];
      d[0] = r.x0, d[1] = r.y0, d[2] = r.w, d[3] = r.h;
    }
    if (records && !is_device_ptr(records))
      for (int f = 0; f < frames; ++f)
        validate_records(*grid, records + (size_t)f * grid->cols * grid->rows);
    SCB_CUDA(cudaSetDevice(ctx->device));
    const sc_partition_stats* h = eval_partition(ctx, *grid, rects, est, records, false, frames,
                                                main_stream(ctx), slice_times, slice_moments);
    for (int f = 0; f < frames; ++f) {
      out[f] = h[f];
      if (!est) out[f].max_us = out[f].total_us = 0.0, out[f].argmax = -1;
    }
  });
}

sc_status sc_shard_export(sc_ctx* ctx, int32_t step, int32_t frames, sc_shard_best* out) {
  return guarded([&] {
    if (!ctx || !out) fail(SC_ERR_USAGE, "NULL argument");
    if (step != 1 && step != 2) fail(SC_ERR_USAGE, "step must be 1 or 2");
    export_shards(ctx, step, frames, out);
  });
}

}  // extern "C"

namespace {
void export_shards(sc_ctx* ctx, int step, int frames, sc_shard_best* out) {
  {
    const auto& v = ctx->last_best[step - 1];
    if ((int)v.size() < frames) fail(SC_ERR_USAGE, "no step result for that many frames");
    for (int f = 0; f < frames; ++f) {
      sc_shard_best& s = out[f];
      std::memset(&s, 0, sizeof(s));
      const FrameBest& b = v[f];
      s.key_sse = b.sse;
      s.key_t = b.found ? b.t : ~0ull;
      s.item = b.found ? b.item : ~0ull;
      s.ord = b.found ? b.ord : ~0ull;
      s.count = b.count;
      s.count_hi = ctx->last_count_hi[step - 1];
      // leaves this shard actually scored (per frame; the walks count
      // candidate-frame scores for the whole warp)
      s.leaves = b.scored / (uint64_t)ctx->last_fpw;
      layout_from_snap(b, SC_MAX_SLICES, &s.layout);
    }
  }
}
}  // namespace

extern "C" {

sc_status sc_comm_unique_id(void* id_out) {
  return guarded([&] {
    if (!id_out) fail(SC_ERR_USAGE, "NULL argument");
    static_assert(sizeof(ncclUniqueId) == SC_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

sc_status sc_comm_detach(sc_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(SC_ERR_USAGE, "NULL argument");
    if (ctx->comm_kind == 1 && ctx->nccl_comm) nccl().commDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
    ctx->comm_kind = 0;
    ctx->comm_fn = nullptr;
    ctx->comm_user = nullptr;
    ctx->shard_rank = 0;
    ctx->shard_world = 1;
  });
}

sc_status sc_comm_init_nccl(sc_ctx* ctx, int32_t rank, int32_t world, const void* unique_id) {
  return guarded([&] {
    if (!ctx || !unique_id) fail(SC_ERR_USAGE, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) fail(SC_ERR_CONFIG, "bad shard rank/world");
    SCB_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    nccl_check(nccl().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
    if (ctx->comm_kind == 1 && ctx->nccl_comm) nccl().commDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = comm;
    ctx->comm_kind = 1;
    ctx->shard_rank = rank;
    ctx->shard_world = world;
  });
}

sc_status sc_comm_init_callback(sc_ctx* ctx, int32_t rank, int32_t world, sc_allgather_fn fn,
                                void* user) {
  return guarded([&] {
    if (!ctx || !fn) fail(SC_ERR_USAGE, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) fail(SC_ERR_CONFIG, "bad shard rank/world");
    if (ctx->comm_kind == 1 && ctx->nccl_comm) nccl().commDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
    ctx->comm_kind = 2;
    ctx->comm_fn = fn;
    ctx->comm_user = user;
    ctx->shard_rank = rank;
    ctx->shard_world = world;
  });
}

sc_status sc_shard_merge(int32_t step, int32_t world, int32_t frames,
                         const sc_shard_best* gathered, sc_search_result* inout) {
  return guarded([&] {
    if (!gathered || !inout) fail(SC_ERR_USAGE, "NULL argument");
    merge_shards(step, world, frames, gathered, inout);
  });
}

}  // extern "C"

namespace {
// The first-in-order winner of every frame over the ranks' records
// (rank-major), counts summed; throws NoCandidateError when no rank has one.
void merge_shards(int step, int world, int frames, const sc_shard_best* gathered,
                  sc_search_result* inout) {
  {
    for (int f = 0; f < frames; ++f) {
      int win = -1;
      unsigned __int128 total = 0;
      uint64_t leaves = 0;
      for (int r = 0; r < world; ++r) {
        const sc_shard_best& s = gathered[(size_t)r * frames + f];
        total += ((unsigned __int128)s.count_hi << 64) | s.count;
        leaves += s.leaves;
        if (s.item == ~0ull) continue;
        if (win < 0) { win = r; continue; }
        const sc_shard_best& b = gathered[(size_t)win * frames + f];
        bool less;
        if (step == 2 && s.key_sse != b.key_sse) less = s.key_sse < b.key_sse;
        else if (s.key_t != b.key_t) less = s.key_t < b.key_t;
        else if (s.item != b.item) less = s.item < b.item;
        else less = layout_less(s.layout, b.layout);
        if (less) win = r;
      }
      if (win < 0) fail(SC_ERR_NO_CANDIDATE, "no candidate on any shard");
      const sc_shard_best& b = gathered[(size_t)win * frames + f];
      sc_search_result& r = inout[f];
      const int n = r.argmin.n_slices ? r.argmin.n_slices : r.best.n_slices;
      sc_layout L = b.layout;
      L.n_slices = n;
      if (step == 1) {
        r.t_min_us = bits_to_double(b.key_t);
        r.argmin = L;
        r.candidates_step1 = (uint64_t)total;
        r.candidates_step1_hi = (uint64_t)(total >> 64);
        r.leaves_scored_step1 = leaves;
      } else {
        r.t_best_us = bits_to_double(b.key_t);
        r.sse_best = b.key_sse;
        r.best = L;
        r.candidates_step2 = (uint64_t)total;
        r.candidates_step2_hi = (uint64_t)(total >> 64);
        r.leaves_scored_step2 = leaves;
      }
      r.candidates_evaluated = r.candidates_step1 + r.candidates_step2;
    }
  }
}
}  // namespace

extern "C" {

sc_status sc_validate_partition(sc_ctx* ctx, const sc_grid* grid, int32_t n_tile_cols,
                                const int32_t* tile_col_widths, int32_t n_tile_rows,
                                const int32_t* tile_row_heights, const sc_rect* slices,
                                int32_t n_slices, int32_t* slice_map) {
  return guarded([&] {
    if (!ctx || (n_tile_cols > 0 && !tile_col_widths) || (n_tile_rows > 0 && !tile_row_heights) ||
        (n_slices > 0 && !slices))
      fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const sc_grid& g = *grid;
    // host part of validate_partition (grid.cpp:86-124): tiles, then each
    // slice's bounds and id, in list order
    if (n_tile_cols < 1 || n_tile_rows < 1)
      fail(SC_ERR_GEOMETRY, "tile grid must have at least one column and row");
    for (int i = 0; i < n_tile_cols; ++i)
      if (tile_col_widths[i] < 1) fail(SC_ERR_GEOMETRY, "tile column width must be >= 1");
    for (int i = 0; i < n_tile_rows; ++i)
      if (tile_row_heights[i] < 1) fail(SC_ERR_GEOMETRY, "tile row height must be >= 1");
    std::vector<int> bx(1, 0), by(1, 0);
    for (int i = 0; i < n_tile_cols; ++i) bx.push_back(bx.back() + tile_col_widths[i]);
    for (int i = 0; i < n_tile_rows; ++i) by.push_back(by.back() + tile_row_heights[i]);
    if (bx.back() != g.cols || by.back() != g.rows)
      fail(SC_ERR_GEOMETRY, "tile sums (" + std::to_string(bx.back()) + "x" +
                                std::to_string(by.back()) + ") do not match grid (" +
                                std::to_string(g.cols) + "x" + std::to_string(g.rows) + ")");
    if (n_slices < 1) fail(SC_ERR_COVERAGE, "partition has no slices");
    std::vector<char> seen((size_t)n_slices, 0);
    std::vector<int> rects((size_t)n_slices * 5);
    for (int i = 0; i < n_slices; ++i) {
      const sc_rect& r = slices[i];
      if (r.w < 1 || r.h < 1 || r.x0 < 0 || r.y0 < 0 || r.x0 + r.w > g.cols ||
          r.y0 + r.h > g.rows)
        fail(SC_ERR_GEOMETRY, "slice " + std::to_string(r.id) + " (" + std::to_string(r.x0) +
                                  "," + std::to_string(r.y0) + " " + std::to_string(r.w) + "x" +
                                  std::to_string(r.h) + ") outside the " + std::to_string(g.cols) +
                                  "x" + std::to_string(g.rows) + " grid");
      if (r.id < 0 || r.id >= n_slices || seen[(size_t)r.id])
        fail(SC_ERR_GEOMETRY, "slice ids must be a permutation of 0..n-1");
      seen[(size_t)r.id] = 1;
      int* d = &rects[(size_t)i * 5];
      d[0] = r.x0, d[1] = r.y0, d[2] = r.w, d[3] = r.h, d[4] = r.id;
    }
    // device part: exact disjoint cover, then structure (validate.cu)
    SCB_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = main_stream(ctx);
    const size_t cells = (size_t)g.cols * g.rows;
    const size_t nin = rects.size() + bx.size() + by.size();
    ctx->val_in.ensure(nin * sizeof(int) + cells * sizeof(int32_t) + sizeof(VCheck));
    int* d_rects = ctx->val_in.as<int>();
    int* d_bx = d_rects + rects.size();
    int* d_by = d_bx + bx.size();
    int32_t* d_map = d_by + by.size();
    VCheck* d_out = reinterpret_cast<VCheck*>(d_map + cells);
    ctx->owner.ensure(cells * sizeof(int));
    std::vector<int> in(rects);
    in.insert(in.end(), bx.begin(), bx.end());
    in.insert(in.end(), by.begin(), by.end());
    SCB_CUDA(cudaMemcpyAsync(d_rects, in.data(), nin * sizeof(int), cudaMemcpyHostToDevice, s));
    validate_device(n_slices, d_rects, (int)bx.size(), d_bx, (int)by.size(), d_by, g.cols, g.rows,
                    ctx->owner.as<int>(), d_map, d_out, s);
    VCheck v;
    SCB_CUDA(cudaMemcpyAsync(&v, d_out, sizeof(VCheck), cudaMemcpyDeviceToHost, s));
    if (slice_map)
      SCB_CUDA(cudaMemcpyAsync(slice_map, d_map, cells * sizeof(int32_t), cudaMemcpyDefault, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    const std::string cell = "(" + std::to_string(v.x) + "," + std::to_string(v.y) + ")";
    if (v.status == SC_ERR_OVERLAP)
      fail(SC_ERR_OVERLAP, "slices " + std::to_string(v.a) + " and " + std::to_string(v.b) +
                               " both cover cell " + cell);
    if (v.status == SC_ERR_COVERAGE)
      fail(SC_ERR_COVERAGE, "cell " + cell + " is not covered by any slice");
    if (v.status == SC_ERR_STRUCTURE)
      fail(SC_ERR_STRUCTURE, "slice " + std::to_string(v.a) +
                                 " is neither a rectangle of complete tiles nor a CTU-row run "
                                 "inside a single tile");
  });
}

sc_status sc_result_slice_maps(sc_ctx* ctx, int32_t step, int32_t n_frames, int32_t* out) {
  return guarded([&] {
    if (!ctx || !out) fail(SC_ERR_USAGE, "NULL argument");
    if (step != 1 && step != 2) fail(SC_ERR_USAGE, "step must be 1 or 2");
    const int have = ctx->maps_frames[step - 1];
    if (n_frames < 1 || n_frames > have)
      fail(SC_ERR_USAGE, "the last search returned no step-" + std::to_string(step) +
                             " partitions for that many frames");
    SCB_CUDA(cudaSetDevice(ctx->device));
    SCB_CUDA(cudaMemcpy(out, ctx->slice_maps.as<int32_t>() + (size_t)(step - 1) * have * ctx->maps_cells,
                        (size_t)n_frames * ctx->maps_cells * sizeof(int32_t), cudaMemcpyDefault));
  });
}

sc_status sc_enumerate_candidates(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                                  uint64_t first, uint64_t max_out, sc_layout* out,
                                  uint64_t* n_out, uint64_t* total) {
  return guarded([&] {
    if (!ctx || (max_out > 0 && !out)) fail(SC_ERR_USAGE, "NULL argument");
    check_grid(grid);
    const int maxc = check_cfg(*grid, cfg);
    const sc_grid& g = *grid;
    uint64_t n = 0, tot = 0;
    if (cfg->family == SC_FAMILY_UNIFORM_ONLY) {
      // for_each_candidate (search.cpp:308-312): the uniform partition if it
      // passes the area test; out[0].n_cols = 0 marks it (sc_uniform_partition)
      tot = uniform_area_ok(uniform_or_fail(g, cfg->n_slices), cfg->k_area) ? 1 : 0;
      if (tot && first == 0 && max_out > 0) {
        std::memset(out, 0, sizeof(sc_layout));
        out[0].n_slices = cfg->n_slices;
        n = 1;
      }
    } else {
      SCB_CUDA(cudaSetDevice(ctx->device));
      Plan* plan = get_plan(ctx, g, *cfg, maxc);
      upload_plan(ctx, plan);
      cudaStream_t s = main_stream(ctx);
      const uint32_t ni = (uint32_t)plan->items.size();
      if (!plan->have_enum) {
        const unsigned __int128 dp = plan_count(plan, g, *cfg);
        if (dp > ((unsigned __int128)1 << 36))
          fail(SC_ERR_SIZE, "candidate stream limited to 2^36 candidates (the family has more)");
        plan->d_enum_counts.ensure((size_t)ni * sizeof(uint64_t) + 8);
        plan->d_enum_offsets.ensure((size_t)ni * sizeof(uint64_t) + 8);
        enumerate_count_device(plan->d_items.as<WorkItem>(), ni, g.cols, g.rows, cfg->n_slices,
                               cfg->k_area, cfg->coverage, plan->d_enum_counts.as<uint64_t>(),
                               plan->d_enum_offsets.as<uint64_t>(), ctx->enum_temp, s);
        uint64_t last[2] = {0, 0};
        if (ni) {
          SCB_CUDA(cudaMemcpyAsync(&last[0], plan->d_enum_offsets.as<uint64_t>() + ni - 1, 8,
                                   cudaMemcpyDeviceToHost, s));
          SCB_CUDA(cudaMemcpyAsync(&last[1], plan->d_enum_counts.as<uint64_t>() + ni - 1, 8,
                                   cudaMemcpyDeviceToHost, s));
        }
        SCB_CUDA(cudaStreamSynchronize(s));
        plan->enum_total = last[0] + last[1];
        plan->have_enum = true;
        if ((unsigned __int128)plan->enum_total != dp)
          fail(SC_ERR_INTERNAL, "candidate stream count differs from the counting DP");
      }
      tot = plan->enum_total;
      n = first < tot ? std::min<uint64_t>(max_out, tot - first) : 0;
      if (n) {
        ctx->enum_out.ensure((size_t)n * kSnapBytes);
        enumerate_emit_device(plan->d_items.as<WorkItem>(), ni, g.cols, g.rows, cfg->n_slices,
                              cfg->k_area, cfg->coverage, plan->d_enum_counts.as<uint64_t>(),
                              plan->d_enum_offsets.as<uint64_t>(), first, n,
                              ctx->enum_out.as<uint8_t>(), s);
        std::vector<uint8_t> snaps((size_t)n * kSnapBytes);
        SCB_CUDA(cudaMemcpyAsync(snaps.data(), ctx->enum_out.p, snaps.size(),
                                 cudaMemcpyDeviceToHost, s));
        SCB_CUDA(cudaStreamSynchronize(s));
        FrameBest fb;
        for (uint64_t i = 0; i < n; ++i) {
          std::memcpy(fb.snap, snaps.data() + i * kSnapBytes, kSnapBytes);
          layout_from_snap(fb, cfg->n_slices, &out[i]);
        }
      }
    }
    if (n_out) *n_out = n;
    if (total) *total = tot;
  });
}

}  // extern "C"
