/*
 * slicecraft_b200.h — the C-ABI drop-in boundary of the B200-native TRS
 * partitioner core (arXiv 2012.14792, reference library `slicecraft`).
 *
 * Plain C: POD structs, caller-owned buffers, an opaque context, integer
 * status codes and a thread-local error string.  No torch or C++ types cross
 * this boundary.  The C++ drop-in layer (include/slicecraft/*.hpp, namespace
 * slicecraft) and the Python binding (paper_2012_14792_b200/) both sit on top
 * of these entry points.  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj).
 *
 * Pointers to frame data may be HOST or DEVICE pointers (detected with
 * cudaPointerGetAttributes); host inputs are staged through pinned buffers
 * owned by the context.  All calls are synchronous with respect to their
 * outputs.  A context is owned by one host thread at a time.
 */
#ifndef SLICECRAFT_B200_H
#define SLICECRAFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 2

/* Compile-time limits of the search kernels.  Larger requests fail with
 * SC_ERR_SIZE (the reference has no such limits). */
#define SC_MAX_SLICES 64
#define SC_MAX_COLS 16

/* One status per exception class of include/slicecraft/errors.hpp:10-85. */
typedef enum sc_status {
  SC_OK = 0,
  SC_ERR_GEOMETRY = 1,     /* GeometryError */
  SC_ERR_OVERLAP = 2,      /* OverlapError */
  SC_ERR_COVERAGE = 3,     /* CoverageError */
  SC_ERR_STRUCTURE = 4,    /* StructureError */
  SC_ERR_IO = 5,           /* IoError */
  SC_ERR_RANGE = 6,        /* RangeError */
  SC_ERR_FORMAT = 7,       /* FormatError */
  SC_ERR_CONFIG = 8,       /* ConfigError */
  SC_ERR_TRACE = 9,        /* TraceError */
  SC_ERR_NO_CANDIDATE = 10,/* NoCandidateError */
  SC_ERR_SIZE = 11,        /* SizeError */
  SC_ERR_USAGE = 12,       /* UsageError */
  SC_ERR_CUDA = 100,       /* CUDA runtime failure / no device */
  SC_ERR_INTERNAL = 101
} sc_status;

/* CtuGrid (grid.hpp:13-34). */
typedef struct sc_grid {
  int32_t frame_width;
  int32_t frame_height;
  int32_t ctu_size;
  int32_t cols;
  int32_t rows;
} sc_grid;

/* CtuRecord (texture.hpp:35-41). */
typedef struct sc_ctu_record {
  uint64_t count;
  uint64_t sum;
  uint64_t sumsq;
} sc_ctu_record;

/* CandidateFamily (search.hpp:17). */
enum { SC_FAMILY_COLUMN_SPLIT = 0, SC_FAMILY_UNIFORM_ONLY = 1 };
/* Candidate-space coverage: REFERENCE reproduces search.cpp:133-143 exactly
 * (tile widths sum to <= cols); COVERING keeps only sum == cols. */
enum { SC_COVERAGE_REFERENCE = 0, SC_COVERAGE_COVERING = 1 };
/* EXHAUSTIVE scores every candidate; PRUNED is an exact branch-and-bound
 * (identical results and counters, fewer leaves scored). */
enum { SC_MODE_EXHAUSTIVE = 0, SC_MODE_PRUNED = 1 };

/* SearchConfig (search.hpp:22-34) + B200 fields. */
typedef struct sc_search_cfg {
  int32_t n_slices;       /* >= 1 */
  double lambda;          /* >= 0, finite */
  double k_area;          /* > 1 */
  int32_t family;         /* SC_FAMILY_* */
  int32_t max_tile_cols;  /* 0 means n_slices */
  int32_t workers;        /* accepted for parity of SearchConfig::check; >= 1 */
  int32_t coverage;       /* SC_COVERAGE_* */
  int32_t mode;           /* SC_MODE_* */
} sc_search_cfg;

/* A ColumnSplit layout (search.cpp:41-45): tile columns, each cut into
 * full-width CTU-row runs.  run_heights is column-major. */
typedef struct sc_layout {
  int32_t n_cols;
  int32_t n_slices;
  int32_t col_widths[SC_MAX_COLS];
  int32_t runs_per_col[SC_MAX_COLS];
  int32_t run_heights[SC_MAX_SLICES];
} sc_layout;

/* RectSlice (grid.hpp:47-58): a slice in CTU units with its id. */
typedef struct sc_rect {
  int32_t x0, y0, w, h, id;
} sc_rect;

/* PartitionOrigin (grid.hpp:70): Proposed = a ColumnSplit layout (sc_layout),
 * Uniform = uniform_partition(grid, n) (sc_uniform_partition). */
enum { SC_ORIGIN_PROPOSED = 0, SC_ORIGIN_UNIFORM = 1 };

/* A general Partition (grid.hpp:60-77): tile grid + slices in id order. */
typedef struct sc_partition {
  int32_t n_tile_cols;
  int32_t n_tile_rows;
  int32_t tile_col_widths[SC_MAX_SLICES];
  int32_t tile_row_heights[SC_MAX_SLICES];
  int32_t n_slices;
  int32_t origin; /* SC_ORIGIN_* */
  sc_rect slices[SC_MAX_SLICES];
} sc_partition;

/* SliceTimeTable (cost.hpp:93-98) summary + partition_sse (texture.hpp:92),
 * per frame (sc_partition_eval). */
typedef struct sc_partition_stats {
  double max_us;    /* first-strict-> maximum of the slice times (cost.cpp:133-143) */
  double total_us;  /* slice times summed in id order */
  int64_t argmax;
  double sse;       /* slice SSEs summed in id order (texture.cpp:183-189) */
} sc_partition_stats;

/* SearchOutcome (search.hpp:36-49) + the step-1 argmin of min_time_search. */
typedef struct sc_search_result {
  double t_min_us;
  double t_best_us;
  double sse_best;
  uint64_t candidates_evaluated;
  uint64_t candidates_step1;
  uint64_t candidates_step2;
  double search_time_us;       /* device time of both steps (CUDA events) */
  double time_min_step_us;
  double clustering_step_us;
  uint64_t leaves_scored_step1; /* == candidates_step1 in EXHAUSTIVE mode */
  uint64_t leaves_scored_step2;
  sc_layout argmin;            /* step-1 first-in-order argmin */
  sc_layout best;              /* step-2 choice */
  /* bits 64..127 of the exact candidate counts (the low 64 bits are
   * candidates_step1/2, the reference's own uint64 counters): non-zero only
   * for spaces beyond 2^64 such as config 5 (~6.1e29). */
  uint64_t candidates_step1_hi;
  uint64_t candidates_step2_hi;
  /* SC_ORIGIN_UNIFORM for the UniformOnly family: argmin / best are then the
   * partition sc_uniform_partition(grid, n) returns (their sc_layout fields
   * are left empty: the uniform grid is not a ColumnSplit layout). */
  int32_t origin;
  int32_t pad;
} sc_search_result;

typedef struct sc_ctx sc_ctx;

/* ---- errors / version --------------------------------------------------- */
const char* sc_last_error(void);

/* Kernels the library has launched in this process so far (its own kernels
 * and the CUB kernels it instantiates; a CUDA-graph replay counts the kernels
 * captured in it).  For launch accounting in benchmarks (bench.py's
 * gpu_launches); no reference counterpart. */
uint64_t sc_kernel_launches(void);
int sc_abi_version(void);

/* ---- geometry (grid.cpp:9-32, CtuGrid::make) ---------------------------- */
sc_status sc_grid_make(int32_t frame_width, int32_t frame_height, int32_t ctu_size,
                       sc_grid* out);
/* temporal_layer_of_poc (cost.cpp:28-38, cost.hpp:39) */
sc_status sc_temporal_layer(int32_t poc, int32_t gop_size, int32_t* out);

/* SearchConfig::check (search.cpp:28-36): ConfigError for n_slices < 1,
 * k_area <= 1, lambda < 0 or not finite, workers < 1, max_tile_cols < 0. */
sc_status sc_search_cfg_check(const sc_search_cfg* cfg);

/* ---- context ------------------------------------------------------------ */
sc_status sc_ctx_create(int32_t device, sc_ctx** out);
sc_status sc_ctx_destroy(sc_ctx* ctx);
/* Bind the context to a rank of a candidate-space shard (multi-GPU):
 * rank r of world w scores the work items r, r+w, r+2w, ... ; results of
 * sc_search_* then hold this shard's best and must be merged with
 * sc_merge_results (an all-gather of sc_shard_best records). */
sc_status sc_ctx_set_shard(sc_ctx* ctx, int32_t rank, int32_t world);

/* Run all work of this context on the caller's CUDA stream (a cudaStream_t
 * passed as void*; NULL restores the context's own stream).  Calls stay
 * synchronous; events recorded on that stream bracket the device work. */
sc_status sc_ctx_set_stream(sc_ctx* ctx, void* cuda_stream);
/* Device time (CUDA events, microseconds) of the phases of the last
 * search call: [0] K1 texture, [1] K2/K3 tables, [2] step 1, [3] step 2,
 * [4] whole call (first to last event on the context's stream). */
sc_status sc_ctx_timings(sc_ctx* ctx, double out[5]);
/* The first n of: the five phases above, then [5] the time-table phase alone
 * (main stream: est -> K2/K3 -> ranks -> split table), [6] the moment tables
 * (side stream), [7] the device post-check and result copies. */
sc_status sc_ctx_timings_ex(sc_ctx* ctx, int32_t n, double* out);

/* ---- texture map (texture.cpp:145-169, ctu_stats) ------------------------ */
/* K1: per-CTU exact moments over n_frames frames.  luma: bytes_per_sample
 * 1 (uint8) or 2 (uint16 LE, values <= 65535), row pitch and frame stride in
 * bytes; host or device pointer.  out: n_frames * cols * rows records
 * (host or device pointer). */
sc_status sc_texture_moments(sc_ctx* ctx, const void* luma, int32_t bytes_per_sample,
                             int32_t width, int32_t height, size_t pitch_bytes,
                             size_t frame_stride_bytes, int32_t ctu_size,
                             int32_t n_frames, sc_ctu_record* out);
/* ---- raw YUV ingest (texture.cpp:9-81) ----------------------------------- */
/* yuv_frame_count: whole planar 4:2:0 frames in the file (bit_depth 8 or 10).
 * IoError (stat), FormatError (dimensions, bit depth, size not a multiple). */
sc_status sc_yuv_frame_count(const char* path, int32_t width, int32_t height,
                             int32_t bit_depth, int32_t* out);
/* load_yuv_frame: the luma plane of frame `poc`, widened to uint16 (out:
 * width * height).  RangeError for a poc outside the file. */
sc_status sc_yuv_load_luma(const char* path, int32_t width, int32_t height, int32_t poc,
                           int32_t bit_depth, uint16_t* out);
/* Raw luma planes of frames [first_poc, first_poc + n_frames), in the file's
 * own sample format (uint8, or uint16 LE for 10-bit), packed: n_frames *
 * width * height * bytes_per_sample bytes into a host buffer.  Chroma is
 * never read. */
sc_status sc_yuv_read_luma(const char* path, int32_t width, int32_t height, int32_t bit_depth,
                           int32_t first_poc, int32_t n_frames, void* out);
/* K1 straight from a YUV file: sc_yuv_read_luma into pinned staging, then
 * sc_texture_moments on the device (out: n_frames * cells records, host or
 * device). */
sc_status sc_yuv_texture_moments(sc_ctx* ctx, const char* path, int32_t width, int32_t height,
                                 int32_t bit_depth, int32_t ctu_size, int32_t first_poc,
                                 int32_t n_frames, sc_ctu_record* out);
/* sc_partition_frames on frames [first_poc, first_poc + n_frames) of a YUV
 * file (est: n_frames maps). */
sc_status sc_partition_yuv(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                           const char* path, int32_t bit_depth, int32_t first_poc,
                           int32_t n_frames, const double* est, sc_ctu_record* records_out,
                           sc_search_result* out);

/* TextureStats ctor validation (texture.cpp:90-111) of caller records. */
sc_status sc_texture_validate(const sc_grid* grid, const sc_ctu_record* records);

/* ---- grid tables (cost.cpp:97-115, texture.cpp:113-143) ----------------- */
/* K2+K3 on n_frames frames: est_times n_frames*cells doubles (host ptr),
 * records n_frames*cells (host ptr or NULL).  Outputs, host pointers, may be
 * NULL: rect_time / rect_sse n_frames * NXW * NYH doubles in rectangle order
 * xw(x0,w)*NYH + yh(y0,h), sat n_frames*(cols+1)*(rows+1). */
sc_status sc_grid_tables(sc_ctx* ctx, const sc_grid* grid, const double* est_times,
                         const sc_ctu_record* records, int32_t n_frames,
                         double* rect_time, double* rect_sse, double* sat);

/* ---- partitions (grid.cpp:186-262, cost.cpp:117-145, texture.cpp:171-189) */
/* uniform_partition (grid.cpp:186-262).  GeometryError if n_slices is not in
 * [1, cells]. */
sc_status sc_uniform_partition(const sc_grid* grid, int32_t n_slices, sc_partition* out);
/* uniform_partition for any n in [1, cells] into caller arrays of n_slices
 * entries each (tile widths, tile heights, slices in id order). */
sc_status sc_uniform_partition_n(const sc_grid* grid, int32_t n_slices, int32_t* tile_col_widths,
                                 int32_t* n_tile_cols, int32_t* tile_row_heights,
                                 int32_t* n_tile_rows, sc_rect* slices);
/* partition_time + partition_sse (+ slice_moments) of one partition on
 * n_frames frames, on the device.  slices: n_slices rects whose ids are a
 * permutation of 0..n_slices-1 (host pointer).  est_times / records: host or
 * device, either may be NULL (its outputs are then left untouched).  out:
 * n_frames summaries; slice_times (n_frames * n_slices doubles, by id) and
 * slice_moments (n_frames * n_slices records, by id) may be NULL. */
sc_status sc_partition_eval(sc_ctx* ctx, const sc_grid* grid, const sc_rect* slices,
                            int32_t n_slices, const double* est_times,
                            const sc_ctu_record* records, int32_t n_frames,
                            sc_partition_stats* out, double* slice_times,
                            sc_ctu_record* slice_moments);

/* ---- partition search (search.cpp:257-434) ------------------------------ */
/* min_time_search (search.cpp:328-332) for n_frames est maps. */
sc_status sc_min_time_search(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                             const double* est_times, int32_t n_frames,
                             sc_search_result* out);
/* constrained_clustering_search (search.cpp:334-405): t_min_us per frame. */
sc_status sc_constrained_clustering(sc_ctx* ctx, const sc_grid* grid,
                                    const sc_search_cfg* cfg, const double* est_times,
                                    const sc_ctu_record* records, const double* t_min_us,
                                    int32_t n_frames, sc_search_result* out);
/* two_step_partition (search.cpp:407-434) after the host-side estimate
 * (estimate_ctu_times, cost.cpp:66-95): est_times are the estimated maps. */
sc_status sc_two_step(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                      const double* est_times, const sc_ctu_record* records,
                      int32_t n_frames, sc_search_result* out);
/* The whole per-batch hot path in one call: K1 texture pass over the frames,
 * K2/K3 tables, step 1, step 2.  records_out may be NULL. */
sc_status sc_partition_frames(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                              const void* luma, int32_t bytes_per_sample,
                              size_t pitch_bytes, size_t frame_stride_bytes,
                              const double* est_times, int32_t n_frames,
                              sc_ctu_record* records_out, sc_search_result* out);
/* for_each_candidate / enumerate_candidates count (search.cpp:302-326). */
sc_status sc_count_candidates(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                              uint64_t* count);

/* ---- device post-check and candidate stream ---------------------------- */
/* validate_partition (grid.cpp:86-184): the tile and per-slice bound / id
 * checks on the host, then the exact-disjoint-cover and structure checks in
 * one device block, with the reference's error classes and first-failure
 * order (GeometryError, CoverageError, OverlapError, StructureError).
 * slice_map (cols*rows, host or device, may be NULL): the slice id of every
 * CTU (-1 where none) -- written on success and on Overlap/Coverage/Structure
 * failures. */
sc_status sc_validate_partition(sc_ctx* ctx, const sc_grid* grid, int32_t n_tile_cols,
                                const int32_t* tile_col_widths, int32_t n_tile_rows,
                                const int32_t* tile_row_heights, const sc_rect* slices,
                                int32_t n_slices, int32_t* slice_map);
/* The CTU -> slice-id maps (n_frames * cols * rows, -1 for cells outside the
 * layout's tile columns, as render_ascii's '?', grid.cpp:279-287) of the
 * step-1 argmin (step=1) or step-2 best (step=2) partitions the last search
 * call on this context returned.  Every returned partition passes the device
 * post-check (validate_partition over the columns its widths span) before
 * the call returns; SLICECRAFT_B200_POSTCHECK=0 skips it (no maps then). */
sc_status sc_result_slice_maps(sc_ctx* ctx, int32_t step, int32_t n_frames, int32_t* out);
/* for_each_candidate / enumerate_candidates (search.cpp:302-326) as a
 * device-materialised stream: the candidates with ordinals [first, first +
 * max_out) of the family's enumeration order, as layouts (out, host).
 * *n_out = candidates written, *total = family size.  The first call per
 * (grid, config) counts the family on the device (families above 2^36
 * candidates: SizeError).  UniformOnly: total is 0 or 1 and its candidate is
 * sc_uniform_partition(grid, n) (out[0].n_cols == 0). */
sc_status sc_enumerate_candidates(sc_ctx* ctx, const sc_grid* grid, const sc_search_cfg* cfg,
                                  uint64_t first, uint64_t max_out, sc_layout* out,
                                  uint64_t* n_out, uint64_t* total);

/* ---- host-side model pieces (no device needed) -------------------------- */
/* CostSource (cost.hpp:11-16). */
enum {
  SC_SOURCE_MEASURED = 0,
  SC_SOURCE_CO_TEMPORAL_LAYER = 1,
  SC_SOURCE_MOST_RECENT_ANY = 2,
  SC_SOURCE_UNIFORM = 3
};
/* CostHistory::append validation (cost.cpp:45-64) of a map about to join a
 * history whose maps carry history_pocs: GeometryError (grid, entry count),
 * FormatError (a time not finite or < 0), TraceError (duplicate poc). */
sc_status sc_cost_map_check(const sc_grid* history_grid, const sc_grid* map_grid,
                            const double* times, int64_t n_times, int32_t poc,
                            const int32_t* history_pocs, int32_t n_history);
/* estimate_ctu_times (cost.cpp:66-95) over a history of n_maps maps (encode
 * order; maps[i] points at cols*rows times, pocs / temporal_layers per map):
 * the most recent map of poc's temporal layer (gop_size, ConfigError), else
 * the most recent map, else all-ones.  out: cols*rows times; source
 * (SC_SOURCE_*), source_poc (-1 for Uniform) and the temporal layer of poc
 * (may be NULL). */
sc_status sc_estimate_ctu_times(const sc_grid* grid, int32_t gop_size, int32_t n_maps,
                                const double* const* maps, const int32_t* pocs,
                                const int32_t* temporal_layers, int32_t poc, double* out,
                                int32_t* source, int32_t* source_poc, int32_t* temporal_layer);
/* TextureStats ctor (texture.cpp:90-130): validates n_records records
 * (GeometryError on the count, FormatError on pixel counts / moments) and
 * builds the (cols+1)*(rows+1) u64 inclusion-exclusion tables (any output may
 * be NULL). */
sc_status sc_texture_tables(const sc_grid* grid, const sc_ctu_record* records, int64_t n_records,
                            uint64_t* pre_count, uint64_t* pre_sum, uint64_t* pre_sumsq);
/* SliceMoments::sse (texture.cpp:83-88). */
sc_status sc_moments_sse(const sc_ctu_record* moments, double* out);
/* PrefixSumTable (cost.cpp:97-112): the f64 summed-area table,
 * (cols+1)*(rows+1) doubles in the reference's operation order. */
sc_status sc_prefix_sum_table(const double* values, int64_t n_values, int32_t cols, int32_t rows,
                              double* table);
/* split_even (grid.cpp:52-60). */
sc_status sc_split_even(int32_t total, int32_t parts, int32_t* out);

/* ---- multi-GPU: the library owns the exchange between shards ---------- */
/* With a communicator attached (rank r of world w, on the context's device),
 * every search call shards the candidate space over the ranks (as
 * sc_ctx_set_shard) AND exchanges what the shards need, returning the merged,
 * global results on every rank: after step 1 the global t_min of each frame
 * (a u64 all-reduce-min of the time bits, on the device) sets step 2's
 * budget; in the pruned mode the frozen seed incumbents are all-reduced
 * (min) between phase A and phase B, so every shard prunes with the global
 * bound; at the end the per-frame shard bests are all-gathered and merged
 * (first in enumeration order, counts summed).  Every rank must make the
 * same calls in the same order.  Replaces the reference's per-flush
 * std::thread pool (search.cpp:198-249). */
#define SC_COMM_ID_BYTES 128
/* An all-gather between the ranks: send `bytes` bytes, receive world * bytes
 * in rank order into recv.  Returns 0 on success. */
typedef int (*sc_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);
/* NCCL unique id (ncclGetUniqueId; SC_COMM_ID_BYTES bytes) for rank 0 to
 * broadcast to the others by any means (the library loads libnccl.so.2 at
 * run time). */
sc_status sc_comm_unique_id(void* id_out);
/* NCCL transport (ncclCommInitRank on the context's device; over NVLink /
 * NVSwitch between the GPUs of one node). */
sc_status sc_comm_init_nccl(sc_ctx* ctx, int32_t rank, int32_t world, const void* unique_id);
/* Host transport: the library calls fn for every exchange (e.g. a gloo or MPI
 * all-gather); the device waits for it. */
sc_status sc_comm_init_callback(sc_ctx* ctx, int32_t rank, int32_t world, sc_allgather_fn fn,
                                void* user);
/* Detach (and destroy) the communicator; the context is a single shard again. */
sc_status sc_comm_detach(sc_ctx* ctx);

/* ---- multi-GPU shard merge (caller-owned exchange) ---------------------- */
/* Opaque per-frame shard best, exchanged by an all-gather (NCCL or gloo). */
typedef struct sc_shard_best {
  double key_sse;     /* step 2 key (inf in step 1) */
  uint64_t key_t;     /* f64 bits of t (non-negative => monotone) */
  uint64_t item;      /* global work-item index (lex order) */
  uint64_t ord;       /* candidate ordinal inside the item */
  uint64_t count;     /* this shard's candidate count (low 64 bits) */
  uint64_t leaves;    /* this shard's scored leaves */
  uint64_t count_hi;  /* high 64 bits of the count (pruned DP counts reach ~6e29) */
  sc_layout layout;
} sc_shard_best;
/* Export this context's last step-1 (step=1) or step-2 (step=2) shard bests. */
sc_status sc_shard_export(sc_ctx* ctx, int32_t step, int32_t n_frames, sc_shard_best* out);
/* Merge world*n_frames gathered records (rank-major) into per-frame results. */
sc_status sc_shard_merge(int32_t step, int32_t world, int32_t n_frames,
                         const sc_shard_best* gathered, sc_search_result* inout);

#ifdef __cplusplus
}
#endif

#endif /* SLICECRAFT_B200_H */
