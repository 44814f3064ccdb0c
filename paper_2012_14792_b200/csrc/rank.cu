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

#include <cstdlib>

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
// The original two-sort pipeline (SLICECRAFT_B200_RANK=sort64).
void rank_times_sort64(sc_ctx* ctx, const uint64_t* bits_fm, size_t nr, int frames, int fpw,
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
  SCB_LAUNCH(k_rank_prepare<<<blocks, 256, 0, st>>>(packed_in, nr, frames));
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
  count_launches(10);  // CUB onesweep, 64-bit keys
  SCB_LAUNCH(k_rank_split<<<blocks, 256, 0, st>>>(packed, fkey_in, pos_in, total));
  SCB_CUDA(cudaGetLastError());
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(ctx->rk_temp.p, b2, fkey_in, fkey_out, pos_in, pos,
                                           (int)total, 0, fbits, st));
  count_launches(4);  // CUB onesweep (frame keys; at most two passes)
  SCB_LAUNCH(k_rank_flags<<<blocks, 256, 0, st>>>(sorted_bits, pos, flags, nr, frames));
  SCB_CUDA(cudaGetLastError());
  SCB_CUDA(cub::DeviceScan::InclusiveSum(ctx->rk_temp.p, b3, flags, scan, (int)total, st));
  count_launches(2);  // CUB scan: init + scan
  SCB_LAUNCH(k_rank_scatter<<<blocks, 256, 0, st>>>(sorted_bits, packed, pos, flags, scan, nr, frames, fpw,
                                         keys, vals, nvals));
  SCB_CUDA(cudaGetLastError());
}

// ---- the 32-bit pipeline ---------------------------------------------------------
// One 32-bit radix sort (4 passes) instead of a 64-bit one plus a frame sort:
// key32 = frame << qb | q, where q is an order-preserving quantisation of the
// time bits inside the frame's own range (0: +0.0, top: +inf, else
// 1 + (bits - lo) >> s, s chosen so the frame's finite range fits).  Equal q
// (a group) can still hold different times: groups are re-sorted by the full
// bits -- small ones by their first thread, large ones (rare: a frame whose
// times cluster far inside a huge range) by a counting rank in one block.
// Then the same first-of-run flags, scan and scatter as before.  Exact: the
// result (dense per-frame ranks, vals, nvals) equals the 64-bit sort's.
constexpr int kSmallGroup = 16;

__global__ void k_rank_range(const uint64_t* __restrict__ bits, size_t nr, uint64_t* lo,
                             uint64_t* hi) {
  const int f = blockIdx.y;
  const uint64_t* b = bits + (size_t)f * nr;
  uint64_t mn = ~0ull, mx = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nr;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t v = b[i];
    if (v != 0 && v < 0x7ff0000000000000ull) {  // positive finite (clamped: no negatives)
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, mn, o), c = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mn != ~0ull) atomicMin((unsigned long long*)&lo[f], (unsigned long long)mn);
    if (mx != 0) atomicMax((unsigned long long*)&hi[f], (unsigned long long)mx);
  }
}

__global__ void k_rank_key32(const uint64_t* __restrict__ bits, size_t nr, int frames, int fbits,
                             int kbits, const uint64_t* __restrict__ lo,
                             const uint64_t* __restrict__ hi, uint32_t* __restrict__ key,
                             uint32_t* __restrict__ val) {
  const int qb = kbits - fbits;
  const uint32_t qmax = qb >= 32 ? 0xffffffffu : (1u << qb) - 1u;
  const size_t total = nr * (size_t)frames;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / nr);
    const uint64_t v = bits[i];
    uint32_t q;
    if (v == 0) {
      q = 0;
    } else if (v >= 0x7ff0000000000000ull) {
      q = qmax;
    } else {
      const uint64_t l = lo[f], span = hi[f] - l;
      const int need = span ? 64 - __clzll((long long)span) : 0;  // bits of the span
      const int sh = need > qb - 2 ? need - (qb - 2) : 0;
      q = 1u + (uint32_t)((v - l) >> sh);
    }
    key[i] = (fbits ? ((uint32_t)f << qb) : 0u) | q;
    val[i] = (uint32_t)i;
  }
}

__device__ __forceinline__ bool bits_less(uint64_t a, uint32_t ia, uint64_t b, uint32_t ib) {
  return a < b || (a == b && ia < ib);
}

// Group starts: small groups sorted in place by (bits, index); large ones
// queued for k_rank_big.  The first-of-run flags come out of the same pass: a
// group's first element always starts a run (a smaller q is a smaller time),
// and inside a group the sorting thread compares neighbours; a group whose
// bits are all equal (tied times: a uniform estimate map ties every rectangle
// of the same area) needs no sorting at all.
__global__ void k_rank_groups(const uint32_t* __restrict__ key, uint32_t* __restrict__ idx,
                              const uint64_t* __restrict__ bits, size_t total,
                              uint32_t* big_count, uint2* big_list,
                              uint32_t* __restrict__ flags) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[i];
    if (i > 0 && key[i - 1] == k) continue;
    flags[i] = 1u;
    if (i + 1 >= total || key[i + 1] != k) continue;  // a group of one
    const uint64_t b0 = bits[idx[i]];
    bool alleq = true;
    size_t j = i + 1;
    while (j < total && key[j] == k) {
      alleq = alleq && bits[idx[j]] == b0;
      ++j;
    }
    if (alleq) {  // one run
      for (size_t a = i + 1; a < j; ++a) flags[a] = 0u;
      continue;
    }
    if (j - i > kSmallGroup) {  // k_rank_big sorts it and writes its flags
      const uint32_t slot = atomicAdd(big_count, 1u);
      big_list[slot] = make_uint2((uint32_t)i, (uint32_t)(j - i));
      continue;
    }
    uint32_t gi[kSmallGroup];
    uint64_t gb[kSmallGroup];
    const int n = (int)(j - i);
    for (int a = 0; a < n; ++a) {
      uint32_t e = idx[i + a];
      uint64_t be = bits[e];
      int b = a - 1;
      while (b >= 0 && bits_less(be, e, gb[b], gi[b])) {
        gb[b + 1] = gb[b];
        gi[b + 1] = gi[b];
        --b;
      }
      gb[b + 1] = be;
      gi[b + 1] = e;
    }
    for (int a = 0; a < n; ++a) {
      idx[i + a] = gi[a];
      if (a > 0) flags[i + a] = gb[a] != gb[a - 1] ? 1u : 0u;
    }
  }
}

// Large groups: the position of every element is the number of group
// elements before it in (bits, index) order.  One block per group at a time;
// then the group's first-of-run flags (its first element's is already set).
__global__ void k_rank_big(uint32_t* __restrict__ idx, const uint64_t* __restrict__ bits,
                           const uint32_t* big_count, const uint2* __restrict__ big_list,
                           uint32_t* __restrict__ tmp, uint32_t* __restrict__ flags) {
  for (uint32_t g = blockIdx.x; g < *big_count; g += gridDim.x) {
    const uint2 gr = big_list[g];
    for (uint32_t a = threadIdx.x; a < gr.y; a += blockDim.x) {
      const uint32_t e = idx[gr.x + a];
      const uint64_t be = bits[e];
      uint32_t r = 0;
      for (uint32_t c = 0; c < gr.y; ++c) {
        const uint32_t o = idx[gr.x + c];
        r += bits_less(bits[o], o, be, e) ? 1u : 0u;
      }
      tmp[gr.x + r] = e;
    }
    __syncthreads();
    for (uint32_t a = threadIdx.x; a < gr.y; a += blockDim.x) idx[gr.x + a] = tmp[gr.x + a];
    __syncthreads();
    for (uint32_t a = 1 + threadIdx.x; a < gr.y; a += blockDim.x)
      flags[gr.x + a] = bits[idx[gr.x + a]] != bits[idx[gr.x + a - 1]] ? 1u : 0u;
    __syncthreads();
  }
}

// nr: ranked rectangles per frame; nr_full / used: the grid's rectangle count
// and the ranked rectangles' indices (used == nullptr: all of them, in place)
__global__ void k_rank_scatter32(const uint32_t* __restrict__ idx, const uint64_t* __restrict__ bits,
                                 const uint32_t* __restrict__ flags,
                                 const uint32_t* __restrict__ scan, size_t nr, int frames, int fpw,
                                 size_t nr_full, const uint32_t* __restrict__ used,
                                 uint32_t* __restrict__ keys, uint64_t* __restrict__ vals,
                                 uint32_t* __restrict__ nvals) {
  const size_t total = nr * (size_t)frames;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t f = i / nr;
    const size_t start = f * nr;
    const uint32_t key = scan[i] - scan[start];
    const uint32_t e = idx[i];
    uint32_t rect = (uint32_t)(e - start);
    if (used) rect = used[rect];
    const size_t g = f / fpw, slot = f % fpw;
    keys[(g * 2 * nr_full + rect) * fpw + slot] = key;  // [group][rt | rts][rect][fpw]
    if (flags[i]) vals[f * nr_full + key] = bits[e];
    if (i == start + nr - 1) nvals[f] = key + 1;
  }
}

// bits_c[f][u] = bits[f][used[u]], and the frame's positive finite range
// (k_rank_range's job, in the same pass): blockIdx.y = frame
__global__ void k_rank_gather(const uint64_t* __restrict__ bits, size_t nr_full,
                              const uint32_t* __restrict__ used, size_t nu,
                              uint64_t* __restrict__ out, uint64_t* lo, uint64_t* hi) {
  const int f = blockIdx.y;
  const uint64_t* b = bits + (size_t)f * nr_full;
  uint64_t* o = out + (size_t)f * nu;
  uint64_t mn = ~0ull, mx = 0;
  for (size_t u = blockIdx.x * (size_t)blockDim.x + threadIdx.x; u < nu;
       u += (size_t)gridDim.x * blockDim.x) {
    const uint64_t v = b[used[u]];
    o[u] = v;
    if (v != 0 && v < 0x7ff0000000000000ull) {
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
  }
  for (int s = 16; s > 0; s >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, mn, s), c = __shfl_xor_sync(0xffffffffu, mx, s);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mn != ~0ull) atomicMin((unsigned long long*)&lo[f], (unsigned long long)mn);
    if (mx != 0) atomicMax((unsigned long long*)&hi[f], (unsigned long long)mx);
  }
}

bool rank64_requested() {
  const char* v = getenv("SLICECRAFT_B200_RANK");
  return v && std::string(v) == "sort64";
}

// used / nu: rank only these rectangles (the ones the plan's candidates use,
// trace.cu).  The caller keeps the other rectangles' keys "infinite" (all
// ones: a slice no candidate takes -- api.cu enqueue_time_tables); whatever
// they hold, no candidate reads them and a column bound (a minimum over
// splits) stays a valid lower bound.
void rank_times_device(sc_ctx* ctx, const uint64_t* bits_fm, size_t nr, int frames, int fpw,
                       uint32_t* keys, uint64_t* vals, uint32_t* nvals, const uint32_t* used,
                       size_t nu, size_t groups, cudaStream_t st) {
  if (rank64_requested()) {
    rank_times_sort64(ctx, bits_fm, nr, frames, fpw, keys, vals, nvals, st);
    return;
  }
  const size_t nr_full = nr;
  const uint64_t* bits_full = bits_fm;
  if (used) {
    ctx->rk_bits_c.ensure(nu * (size_t)frames * sizeof(uint64_t));
    bits_fm = ctx->rk_bits_c.as<uint64_t>();
    nr = nu;
  }
  const size_t total = nr * (size_t)frames;
  if (total >= (1ull << 32) || frames > (1 << 10))
    fail(SC_ERR_SIZE, "too many rectangles or frames for the time-key pipeline");
  int fbits = 0;
  while ((1 << fbits) < frames) ++fbits;
  // key width: 24 bits (3 radix passes) leave >= 2^14 buckets per frame even
  // at 1024 frames -- equal keys are re-sorted exactly by k_rank_groups --
  // and 32 bits (4 passes) only when the frame index needs more room
  const int kbits = fbits <= 10 ? 24 : 32;
  ctx->rk_idx.ensure(total * sizeof(uint32_t) * 6);
  ctx->rk_flags.ensure(total * sizeof(uint32_t) * 2);
  ctx->rk_sorted.ensure(((size_t)frames * 2 + 2) * sizeof(uint64_t) + (total / (kSmallGroup + 1) + 2) *
                        sizeof(uint2));
  uint32_t* key_in = ctx->rk_idx.as<uint32_t>();
  uint32_t* key_out = key_in + total;
  uint32_t* val_in = key_out + total;
  uint32_t* idx = val_in + total;
  uint32_t* tmp = idx + total;
  uint32_t* flags = ctx->rk_flags.as<uint32_t>();
  uint32_t* scan = flags + total;
  uint64_t* lo = ctx->rk_sorted.as<uint64_t>();
  uint64_t* hi = lo + frames;
  uint32_t* big_count = reinterpret_cast<uint32_t*>(hi + frames);
  uint2* big_list = reinterpret_cast<uint2*>(hi + frames + 2);
  const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, (size_t)ctx->sm_count * 8);
  SCB_CUDA(cudaMemsetAsync(lo, 0xff, (size_t)frames * sizeof(uint64_t), st));
  SCB_CUDA(cudaMemsetAsync(hi, 0, (size_t)frames * sizeof(uint64_t) + 16, st));  // + big_count
  const unsigned rb = (unsigned)std::max<size_t>(1, std::min<size_t>((nr + 255) / 256, 16));
  if (used)
    SCB_LAUNCH(k_rank_gather<<<dim3(rb, frames), 256, 0, st>>>(
        bits_full, nr_full, used, nu, ctx->rk_bits_c.as<uint64_t>(), lo, hi));
  else
    SCB_LAUNCH(k_rank_range<<<dim3(rb, frames), 256, 0, st>>>(bits_fm, nr, lo, hi));
  SCB_CUDA(cudaGetLastError());
  SCB_LAUNCH(k_rank_key32<<<blocks, 256, 0, st>>>(bits_fm, nr, frames, fbits, kbits, lo, hi, key_in, val_in));
  SCB_CUDA(cudaGetLastError());
  size_t b1 = 0, b3 = 0;
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, key_in, key_out, val_in, idx, (int)total,
                                           0, kbits, st));
  SCB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b3, flags, scan, (int)total, st));
  ctx->rk_temp.ensure(std::max(b1, b3));
  SCB_CUDA(cub::DeviceRadixSort::SortPairs(ctx->rk_temp.p, b1, key_in, key_out, val_in, idx,
                                           (int)total, 0, kbits, st));
  count_launches(2 + (kbits + 7) / 8);  // CUB onesweep: histogram, exclusive sum, one kernel per 8-bit pass
  SCB_LAUNCH(k_rank_groups<<<blocks, 256, 0, st>>>(key_out, idx, bits_fm, total, big_count, big_list,
                                                flags));
  SCB_CUDA(cudaGetLastError());
  SCB_LAUNCH(k_rank_big<<<ctx->sm_count, 256, 0, st>>>(idx, bits_fm, big_count, big_list, tmp, flags));
  SCB_CUDA(cudaGetLastError());
  SCB_CUDA(cub::DeviceScan::InclusiveSum(ctx->rk_temp.p, b3, flags, scan, (int)total, st));
  count_launches(2);  // CUB scan: init + scan
  SCB_LAUNCH(k_rank_scatter32<<<blocks, 256, 0, st>>>(idx, bits_fm, flags, scan, nr, frames, fpw, nr_full,
                                           used, keys, vals, nvals));
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
  SCB_LAUNCH(k_budget_keys<<<(frames + 127) / 128, 128, 0, st>>>(d_budgets, vals, nvals, nr, frames, out));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
