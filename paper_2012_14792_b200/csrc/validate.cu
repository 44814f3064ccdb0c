// validate_partition (grid.cpp:86-184) as a device post-check, and the
// CTU -> slice-id maps of the partitions a search returns.
//
// The reference paints an owner map cell by cell and throws at the first
// conflict, in a fixed order: the first cell claimed twice (slices in list
// order, cells row-major inside a slice) -> OverlapError; else the first
// uncovered cell (row-major) -> CoverageError; else the first slice (list
// order) that is neither a union of complete tiles nor a row run inside one
// tile -> StructureError.  Here one block per partition computes, for every
// cell, the lowest list index covering it (atomicMin); a (slice, cell) pair
// whose cell has a lower owner is a conflict event, and the reference's first
// exception is the event minimal in (slice, y, x) -- found by one 64-bit
// atomicMin.  Coverage and structure reduce the same way, so the outcome
// (class and the cells/ids of its message) equals the reference's.
#include <climits>

#include "common.cuh"

namespace scb {

// One partition, one block.  rects: n x {x0, y0, w, h, id} in list order
// (bounds and ids already checked); bx / by: tile boundaries (nbx, nby
// entries, ascending from 0); cells with x >= span_cols are outside the
// partition's tile columns (a ColumnSplit layout whose widths sum to less
// than cols, search.cpp:133-143) and are neither required nor painted.
// owner: cols*rows ints of scratch; map (may be NULL): slice id per cell, -1
// where nothing covers it.
__device__ void check_partition(int n, const int* __restrict__ rects, int nbx,
                                const int* __restrict__ bx, int nby, const int* __restrict__ by,
                                int cols, int rows, int span_cols, int* owner, int32_t* map,
                                VCheck* out) {
  __shared__ unsigned long long s_ovl;
  __shared__ int s_cov, s_str;
  const int cells = cols * rows;
  if (threadIdx.x == 0) {
    s_ovl = ~0ull;
    s_cov = INT_MAX;
    s_str = INT_MAX;
  }
  for (int c = threadIdx.x; c < cells; c += blockDim.x) owner[c] = INT_MAX;
  __syncthreads();
  // lowest list index covering each cell
  for (int i = 0; i < n; ++i) {
    const int* r = rects + 5 * i;
    const int w = r[2], area = r[2] * r[3];
    for (int k = threadIdx.x; k < area; k += blockDim.x)
      atomicMin(&owner[(r[1] + k / w) * cols + r[0] + k % w], i);
  }
  __syncthreads();
  // first conflict event in (slice, y, x) order
  for (int i = 0; i < n; ++i) {
    const int* r = rects + 5 * i;
    const int w = r[2], area = r[2] * r[3];
    for (int k = threadIdx.x; k < area; k += blockDim.x) {
      const int x = r[0] + k % w, y = r[1] + k / w;
      if (owner[y * cols + x] < i)
        atomicMin(&s_ovl, ((unsigned long long)i << 40) | ((unsigned long long)y << 20) |
                              (unsigned long long)x);
    }
  }
  // first uncovered cell of the span, row-major
  for (int c = threadIdx.x; c < cells; c += blockDim.x)
    if (c % cols < span_cols && owner[c] == INT_MAX) atomicMin(&s_cov, c);
  // structural legality (grid.cpp:163-183): a union of complete tiles, or a
  // full-tile-width run of rows inside one tile
  auto on = [](const int* b, int nb, int v) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (b[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    return b[lo] == v;
  };
  auto interval = [](const int* b, int nb, int v) {  // i with b[i] <= v < b[i+1]
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (b[mid] <= v) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int* r = rects + 5 * i;
    const int x0 = r[0], y0 = r[1], x1 = r[0] + r[2], y1 = r[1] + r[3];
    if (on(bx, nbx, x0) && on(bx, nbx, x1) && on(by, nby, y0) && on(by, nby, y1)) continue;
    const int tc = interval(bx, nbx, x0), tr = interval(by, nby, y0);
    const bool run = tc + 1 < nbx && tr + 1 < nby && x0 == bx[tc] && x1 == bx[tc + 1] &&
                     y0 >= by[tr] && y1 <= by[tr + 1];
    if (!run) atomicMin(&s_str, i);
  }
  __syncthreads();
  if (map)
    for (int c = threadIdx.x; c < cells; c += blockDim.x)
      map[c] = owner[c] == INT_MAX ? -1 : rects[5 * owner[c] + 4];
  if (threadIdx.x == 0) {
    VCheck v{SC_OK, 0, 0, 0, 0};
    if (s_ovl != ~0ull) {
      const int i = (int)(s_ovl >> 40), y = (int)((s_ovl >> 20) & 0xfffff),
                x = (int)(s_ovl & 0xfffff);
      v = VCheck{SC_ERR_OVERLAP, rects[5 * owner[y * cols + x] + 4], rects[5 * i + 4], x, y};
    } else if (s_cov != INT_MAX) {
      v = VCheck{SC_ERR_COVERAGE, 0, 0, s_cov % cols, s_cov / cols};
    } else if (s_str != INT_MAX) {
      v = VCheck{SC_ERR_STRUCTURE, rects[5 * s_str + 4], 0, 0, 0};
    }
    *out = v;
  }
}

__global__ void k_validate(int n, const int* rects, int nbx, const int* bx, int nby, const int* by,
                           int cols, int rows, int* owner, int32_t* map, VCheck* out) {
  check_partition(n, rects, nbx, bx, nby, by, cols, rows, cols, owner, map, out);
}

// The partitions a search returns, straight from the device results: frame
// f's layout snapshot (W[16] R[16] H[64], FrameBest::snap) becomes the
// layout_to_partition slices (search.cpp:63-75; tiles = widths x {rows}) and
// goes through the same checks, restricted to the columns the widths span.
// blockIdx.y = step - 1 (both steps in one launch): the step's FrameBest,
// maps and verdicts sit `fb_stride` / `frames` entries apart.
// h_fb (optional): pinned host memory the block copies its FrameBest record
// into, so the call needs no device-to-host copy after this kernel (out0 may
// be pinned host memory as well).
__global__ void k_result_maps(const FrameBest* __restrict__ fb0, size_t fb_stride, int frames,
                              int first_step, int n, int cols, int rows, int* owner0,
                              int32_t* maps0, VCheck* out0, FrameBest* h_fb) {
  const int f = blockIdx.x, si = first_step - 1 + blockIdx.y;
  const FrameBest* fb = fb0 + (size_t)si * fb_stride;
  if (h_fb && threadIdx.x < sizeof(FrameBest) / 8) {
    static_assert(sizeof(FrameBest) % 8 == 0, "FrameBest is copied as 64-bit words");
    reinterpret_cast<uint64_t*>(h_fb + (size_t)si * fb_stride + f)[threadIdx.x] =
        reinterpret_cast<const uint64_t*>(fb + f)[threadIdx.x];
  }
  const size_t cells_ = (size_t)cols * rows;
  int* owner = owner0 + (size_t)blockIdx.y * frames * cells_;
  int32_t* maps = maps0 + (size_t)si * frames * cells_;
  VCheck* out = out0 + (size_t)si * frames;
  __shared__ int rects[5 * SC_MAX_SLICES];
  __shared__ int bx[SC_MAX_COLS + 1], by[2];
  __shared__ int s_c, s_span;
  const FrameBest& b = fb[f];
  if (threadIdx.x == 0) {
    int c = 0, x = 0, run = 0;
    bx[0] = 0;
    while (c < SC_MAX_COLS && b.snap[c] != 0) {
      const int w = b.snap[c], runs = b.snap[SC_MAX_COLS + c];
      int y = 0;
      for (int j = 0; j < runs && run < n; ++j, ++run) {
        const int h = b.snap[2 * SC_MAX_COLS + run];
        int* r = rects + 5 * run;
        r[0] = x, r[1] = y, r[2] = w, r[3] = h, r[4] = run;
        y += h;
      }
      x += w;
      bx[++c] = x;
    }
    by[0] = 0;
    by[1] = rows;
    s_c = c;
    s_span = x;
    // a snapshot that does not decode to n in-grid slices is malformed
    bool ok = b.found && run == n && x <= cols;
    for (int i = 0; i < run && ok; ++i)
      ok = rects[5 * i + 2] >= 1 && rects[5 * i + 3] >= 1 &&
           rects[5 * i + 1] + rects[5 * i + 3] <= rows;
    if (!ok) s_c = -1;
  }
  __syncthreads();
  const size_t cells = (size_t)cols * rows;
  if (s_c < 0) {  // not found (shard without a candidate) or malformed
    for (size_t c = threadIdx.x; c < cells; c += blockDim.x) maps[f * cells + c] = -1;
    if (threadIdx.x == 0)
      out[f] = VCheck{b.found ? SC_ERR_GEOMETRY : SC_OK, -1, 0, 0, 0};
    return;
  }
  check_partition(n, rects, s_c + 1, bx, 2, by, cols, rows, s_span, owner + f * cells,
                  maps + f * cells, out + f);
}

void validate_device(int n, const int* d_rects, int nbx, const int* d_bx, int nby, const int* d_by,
                     int cols, int rows, int* d_owner, int32_t* d_map, VCheck* d_out,
                     cudaStream_t st) {
  SCB_LAUNCH(k_validate<<<1, 256, 0, st>>>(n, d_rects, nbx, d_bx, nby, d_by, cols, rows, d_owner, d_map,
                                d_out));
  SCB_CUDA(cudaGetLastError());
}

void result_maps_device(const FrameBest* d_fb, size_t fb_stride, int frames, int first_step,
                        int steps, int n, int cols, int rows, int* d_owner, int32_t* d_maps,
                        VCheck* d_out, FrameBest* h_fb, cudaStream_t st) {
  SCB_LAUNCH(k_result_maps<<<dim3(frames, steps), 256, 0, st>>>(d_fb, fb_stride, frames, first_step, n, cols,
                                                     rows, d_owner, d_maps, d_out, h_fb));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
