// The whole time-table phase of a small grid in one CTA per frame.
//
// For grids up to kSmallNR rectangles (cfg1 / cfg2: 15 x 9 CTUs = 5,400
// rectangles) the general pipeline -- K2 wavefront, K3, the rank pipeline
// (range, quantised keys, CUB radix sort, group fix-up, flags, scan, scatter)
// and the split table, ~20 launches -- is launch-latency bound: ~120 us per
// call for microseconds of work.  Here one CTA per frame does it all in
// shared memory, with the same arithmetic and the same results:
//   1. the f64 SAT by the anti-diagonal wavefront (cost.cpp:97-112 order);
//   2. every rectangle's time ((d - b) - c) + a, clamped to +0.0
//      (search.cpp:77-83), as u64 bits;
//   3. a bitonic sort of (bits, rect) in shared memory, first-of-run flags
//      and a block scan -> the exact per-frame ranks, vals[f][rank] and
//      nvals[f] (rank.cu);
//   4. the rt keys and the split table rts = max(run, forced rest) into the
//      search layout [group][rt | rts][rect][fpw].
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace scb {

constexpr int kSmallThreads = 512;
constexpr int kSmallItems = 16;
constexpr int kSmallNR = kSmallThreads * kSmallItems;  // 8,192 rectangles

__global__ void __launch_bounds__(kSmallThreads)
    k_small_tables(const double* __restrict__ est, int cols, int rows, int frames, int fpw,
                   const int16_t* __restrict__ dec, uint32_t* __restrict__ keys,
                   uint64_t* __restrict__ vals, uint32_t* __restrict__ nvals) {
  using Scan = cub::BlockScan<uint32_t, kSmallThreads>;
  extern __shared__ __align__(16) uint8_t sm_small[];
  __shared__ typename Scan::TempStorage scan_tmp;
  const int f = blockIdx.x;
  const int nyh = rows * (rows + 1) / 2, nxw = cols * (cols + 1) / 2;
  const int nr = nxw * nyh;
  int np = 1;  // sorted length: the next power of two
  while (np < nr) np <<= 1;
  const int stride = cols + 1, nsat = stride * (rows + 1);
  uint64_t* sk = reinterpret_cast<uint64_t*>(sm_small);  // [np] time bits, then sorted
  double* T = reinterpret_cast<double*>(sk + np);       // [nsat] SAT
  uint32_t* sv = reinterpret_cast<uint32_t*>(T + nsat);  // [np] rectangle of each key
  uint32_t* rank = sv + np;                              // [nr] rank of each rectangle
  const double* v = est + (size_t)f * cols * rows;
  // 1. f64 SAT, anti-diagonal wavefront: T = ((v + L) + U) - UL
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) T[i] = 0.0;
  __syncthreads();
  for (int s = 0; s <= cols + rows - 2; ++s) {
    for (int y = threadIdx.x; y < rows; y += blockDim.x) {
      const int x = s - y;
      if (x >= 0 && x < cols) {
        const int i = (y + 1) * stride + (x + 1);
        T[i] = __dsub_rn(__dadd_rn(__dadd_rn(v[y * cols + x], T[i - 1]), T[i - stride]),
                         T[i - stride - 1]);
      }
    }
    __syncthreads();
  }
  // 2. clamped time bits of every rectangle (padding sorts last)
  for (int rr = threadIdx.x; rr < np; rr += blockDim.x) {
    uint64_t b = ~0ull;
    if (rr < nr) {
      const int xw = rr / nyh, yh = rr % nyh;
      const int x0 = dec[xw], w = dec[nxw + xw], y0 = dec[2 * nxw + yh], h = dec[2 * nxw + nyh + yh];
      const int ia = y0 * stride + x0, ib = y0 * stride + x0 + w;
      const int ic = (y0 + h) * stride + x0, idd = (y0 + h) * stride + x0 + w;
      const double t = __dadd_rn(__dsub_rn(__dsub_rn(T[idd], T[ib]), T[ic]), T[ia]);
      b = t > 0.0 ? (uint64_t)__double_as_longlong(t) : 0ull;
    }
    sk[rr] = b;
    sv[rr] = (uint32_t)rr;
  }
  __syncthreads();
  // 3. bitonic sort of (bits, rect) in shared memory
  for (int size = 2; size <= np; size <<= 1) {
    for (int half = size >> 1; half > 0; half >>= 1) {
      for (int i = threadIdx.x; i < np / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (half - 1)), hi = lo + half;
        const bool up = (lo & size) == 0;
        const uint64_t a = sk[lo], b = sk[hi];
        const uint32_t va = sv[lo], vb = sv[hi];
        const bool gt = a > b || (a == b && va > vb);
        if (gt == up) {
          sk[lo] = b, sk[hi] = a;
          sv[lo] = vb, sv[hi] = va;
        }
      }
      __syncthreads();
    }
  }
  // first-of-run flags and their exclusive scan, kSmallItems positions per
  // thread (blocked) -> the rank of each distinct value
  const int p0 = threadIdx.x * kSmallItems;
  uint32_t cnt = 0;
  for (int j = 0; j < kSmallItems; ++j) {
    const int pos = p0 + j;
    cnt += (pos < nr && (pos == 0 || sk[pos] != sk[pos - 1])) ? 1u : 0u;
  }
  uint32_t run = 0;
  Scan(scan_tmp).ExclusiveSum(cnt, run);
  uint64_t* fv = vals + (size_t)f * nr;
  for (int j = 0; j < kSmallItems; ++j) {
    const int pos = p0 + j;
    if (pos >= nr) break;
    const bool first = pos == 0 || sk[pos] != sk[pos - 1];
    run += first ? 1u : 0u;
    const uint32_t key = run - 1;
    rank[sv[pos]] = key;
    if (first) fv[key] = sk[pos];
    if (pos == nr - 1) nvals[f] = key + 1;
  }
  __syncthreads();
  // 4. rt and the split table into [group][rt | rts][rect][fpw]
  const int g = f / fpw, slot = f % fpw;
  uint32_t* rt = keys + (size_t)g * 2 * nr * fpw;
  uint32_t* rts = rt + (size_t)nr * fpw;
  for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
    const uint32_t a = rank[rr];
    rt[(size_t)rr * fpw + slot] = a;
    const int xw = rr / nyh, yh = rr % nyh;
    const int y0 = dec[2 * nxw + yh], h = dec[2 * nxw + nyh + yh];
    uint32_t sp = 0;
    if (y0 + h < rows) {
      const uint32_t b = rank[xw * nyh + yh_index(rows, y0 + h, rows - y0 - h)];
      sp = a > b ? a : b;
    }
    rts[(size_t)rr * fpw + slot] = sp;
  }
}

size_t small_tables_smem(int cols, int rows) {
  const size_t nr = (size_t)cols * (cols + 1) / 2 * (rows * (rows + 1) / 2);
  size_t np = 1;
  while (np < nr) np <<= 1;
  return np * (sizeof(uint64_t) + sizeof(uint32_t)) +
         (size_t)(cols + 1) * (rows + 1) * sizeof(double) + nr * sizeof(uint32_t);
}

// true when the grid fits the one-CTA path (and it was launched)
bool small_tables_device(const double* d_est, int cols, int rows, int frames, int fpw,
                         const int16_t* d_dec, uint32_t* keys, uint64_t* vals, uint32_t* nvals,
                         cudaStream_t st) {
  const size_t nr = (size_t)cols * (cols + 1) / 2 * (rows * (rows + 1) / 2);
  if (nr > (size_t)kSmallNR) return false;
  const size_t smem = small_tables_smem(cols, rows);
  if (smem > (size_t)max_dynamic_smem((const void*)k_small_tables)) return false;
  once_per_device((const void*)k_small_tables, [] {
    SCB_CUDA(cudaFuncSetAttribute(k_small_tables, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dynamic_smem((const void*)k_small_tables)));
  });
  k_small_tables<<<frames, kSmallThreads, smem, st>>>(d_est, cols, rows, frames, fpw, d_dec, keys,
                                                      vals, nvals);
  SCB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace scb
