// Time keys: per-frame exact ranks of the clamped rectangle times.
//
// The search only ever takes maxima of rectangle times and compares them (<,
// <=; search.cpp:77-83, 284, 380).  Replacing every time by its rank among the
// distinct times of its frame is injective and order-preserving, so all those
// operations give identical answers on ranks; the ranks fit 32 bits (a 8K
// frame has 1.09 M rectangles), halving the search tables.  A key maps back to
// its double through vals[f][key]; step 2's budget becomes the largest key
// whose time is <= t_min * (1 + lambda).
//
// Pipeline per call (after K3 wrote the frame-major clamped bits):
//   global stable radix sort of (bits, frame|rect), then a stable radix sort
//   by frame (one pass) -> (frame, bits) order; first-of-run flags ->
//   inclusive scan -> scatter keys into the search layout [group][rect][FPW]
//   and the distinct values into vals[f][key].  (Two global sorts instead of
//   a segmented sort, whose one-block-per-segment schedule crawls on the
//   1.09 M-rectangle frames of 8K.)
// The sort and scan are CUB (CUDA toolkit) device primitives: an O(R log R)
// preprocessing step per frame, not the search hot loop.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace scb {

// packed (frame, rect): rect < 2^22 (an 8K/CTU-64 grid has 4.3 M rectangles
// at most within the 7800-cell table limit), frame < 2^10
constexpr int kRectBits = 22;

__global__ void k_rank_prepare(uint32_t* __restrict__ packed, size_t nr, int frames) {
  const size_t total = nr * (size_t)frames;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    packed[i] = ((uint32_t)(i / nr) << kRectBits) | (uint32_t)(i % nr);
}

// after the first sort: frame of each element (second sort key) + position
__global__ void k_rank_split(const uint32_t* __restrict__ packed, uint32_t* __restrict__ fkey,
                             uint32_t* __restrict__ pos, size_t total) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    fkey[i] = packed[i] >> kRectBits;
    pos[i] = (uint32_t)i;
  }
}

// after the second sort: element i of the (frame, bits) order came from
// position pos[i] of the bits order
__global__ void k_rank_flags(const uint64_t* __restrict__ sorted_bits,
                             const uint32_t* __restrict__ pos, uint32_t* __restrict__ flags,
                             size_t nr, int frames) {
  const size_t total = nr * (size_t)frames;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    flags[i] = (i % nr == 0 || sorted_bits[pos[i]] != sorted_bits[pos[i - 1]]) ? 1u : 0u;
}

__global__ void k_rank_scatter(const uint64_t* __restrict__ sorted_bits,
                               const uint32_t* __restrict__ packed,
                               const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ flags,
                               const uint32_t* __restrict__ scan, size_t nr, int frames, int fpw,
                               uint32_t* __restrict__ keys, uint64_t* __restrict__ vals,
                               uint32_t* __restrict__ nvals) {
  const size_t total = nr * (size_t)frames;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t f = i / nr;
    const size_t start = f * nr;
    const uint32_t key = scan[i] - scan[start];
    const uint32_t p = pos[i];
    const uint32_t rect = packed[p] & ((1u << kRectBits) - 1u);
    const size_t g = f / fpw, slot = f % fpw;
    keys[(g * 2 * nr + rect) * fpw + slot] = key;  // [group][rt | rts][rect][fpw]
    if (flags[i]) vals[start + key] = sorted_bits[p];
    if (i == start + nr - 1) nvals[f] = key + 1;
  }
}

// bits_fm: [frames][nr] clamped time bits.  Outputs keys into the rt half of
// [groups][2][nr][fpw] (the rts half is the split table; slots of frames >=
// `frames` are left untouched), vals [frames][nr], nvals.
void rank_times_device(sc_ctx* ctx, const uint64_t* bits_fm, size_t nr, int frames, int fpw,
                       uint32_t* keys, uint64_t* vals, uint32_t* nvals, cudaStream_t st) {
  const size_t total = nr * (size_t)frames;
  if (nr >= (1u << kRectBits) || frames >= (1 << (32 - kRectBits)))
    fail(SC_ERR_SIZE, "too many rectangles or frames for the time-key pipeline");
  ctx->rk_idx.ensure(total * sizeof(uint32_t) * 6);
  ctx->rk_sorted.ensure(total * sizeof(uint64_t));
  ctx->rk_flags.ensure(total * sizeof(uint32_t) * 2);
  uint32_t* packed_in = ctx->rk_idx.as<uint32_t>();
  uint32_t* packed = packed_in + total;   // sorted by bits
  uint32_t* fkey_in = packed + total;
  uint32_t* fkey_out = fkey_in + total;
  uint32_t* pos_in = fkey_out + total;
  uint32_t* pos = pos_in + total;         // (frame, bits) order -> position
  uint64_t* sorted_bits = ctx->rk_sorted.as<uint64_t>();
  uint32_t* flags = ctx->rk_flags.as<uint32_t>();
  uint32_t* scan = flags + total;
  int fbits = 1;
  while ((1 << fbits) < frames) ++fbits;
  const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, (size_t)ctx->sm_count * 8);
  k_rank_prepare<<<blocks, 256, 0, st>>>(packed_in, nr, frames);
  SCB_CUDA(cudaGetLastError());
  size_t b1 = 0, b2 = 0, b3 = 0;
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, bits_fm, sorted_bits, packed_in, packed,
                                           (int)total, 0, 64, st));
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, fkey_in, fkey_out, pos_in, pos,
                                           (int)total, 0, fbits, st));
  SCB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b3, flags, scan, (int)total, st));
  ctx->rk_temp.ensure(std::max(b1, std::max(b2, b3)));
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(ctx->rk_temp.p, b1, bits_fm, sorted_bits, packed_in,
                                           packed, (int)total, 0, 64, st));
  k_rank_split<<<blocks, 256, 0, st>>>(packed, fkey_in, pos_in, total);
  SCB_CUDA(cudaGetLastError());
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(ctx->rk_temp.p, b2, fkey_in, fkey_out, pos_in, pos,
                                           (int)total, 0, fbits, st));
  k_rank_flags<<<blocks, 256, 0, st>>>(sorted_bits, pos, flags, nr, frames);
  SCB_CUDA(cudaGetLastError());
  SCB_CUDA(cub::DeviceScan::InclusiveSum(ctx->rk_temp.p, b3, flags, scan, (int)total, st));
  k_rank_scatter<<<blocks, 256, 0, st>>>(sorted_bits, packed, pos, flags, scan, nr, frames, fpw,
                                         keys, vals, nvals);
  SCB_CUDA(cudaGetLastError());
}

// Largest key whose time is <= b (as double), -1 when none: binary search
// over the frame's distinct values (ascending bit patterns of times >= +0.0).
__device__ __forceinline__ int64_t budget_key(const uint64_t* vals, uint32_t n, double b) {
  if (!(b >= 0.0)) return -1;  // negative or NaN budget: nothing feasible
  const uint64_t bits = (uint64_t)__double_as_longlong(b);
  uint32_t lo = 0, hi = n;  // first index with vals > bits
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (vals[mid] <= bits) lo = mid + 1;
    else hi = mid;
  }
  return (int64_t)lo - 1;
}

__global__ void k_budget_keys(const double* __restrict__ budgets, const uint64_t* __restrict__ vals,
                              const uint32_t* __restrict__ nvals, size_t nr, int frames,
                              int64_t* __restrict__ out) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < frames) out[f] = budget_key(vals + (size_t)f * nr, nvals[f], budgets[f]);
}

void budget_keys_device(const double* d_budgets, const uint64_t* vals, const uint32_t* nvals,
                        size_t nr, int frames, int64_t* out, cudaStream_t st) {
  k_budget_keys<<<(frames + 127) / 128, 128, 0, st>>>(d_budgets, vals, nvals, nr, frames, out);
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
