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
//   3. a 32-bit block radix sort of the range-quantised times (as rank.cu),
//      equal-key groups re-sorted by the full bits, first-of-run flags and a
//      block scan -> the exact per-frame ranks, vals[f][rank], nvals[f];
//   4. the rt keys and the split table rts = max(run, forced rest) into the
//      search layout [group][rt | rts][rect][fpw].
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace scb {

constexpr int kSmallThreads = 1024;
constexpr int kSmallItems = 8;
constexpr int kSmallNR = kSmallThreads * kSmallItems;  // 8,192 rectangles

using SmallSort = cub::BlockRadixSort<uint32_t, kSmallThreads, kSmallItems, uint32_t>;
using SmallScan = cub::BlockScan<uint32_t, kSmallThreads>;
union SmallTemp {
  typename SmallSort::TempStorage sort;
  typename SmallScan::TempStorage scan;
};

__global__ void __launch_bounds__(kSmallThreads)
    k_small_tables(const double* __restrict__ est, int cols, int rows, int frames, int fpw,
                   const int16_t* __restrict__ dec, uint32_t* __restrict__ keys,
                   uint64_t* __restrict__ vals, uint32_t* __restrict__ nvals) {
  extern __shared__ __align__(16) uint8_t sm_small[];
  SmallTemp& temp = *reinterpret_cast<SmallTemp*>(sm_small);
  __shared__ unsigned long long s_lo, s_hi;
  const int f = blockIdx.x;
  const int nyh = rows * (rows + 1) / 2, nxw = cols * (cols + 1) / 2;
  const int nr = nxw * nyh;
  const int stride = cols + 1, nsat = stride * (rows + 1);
  uint64_t* B = reinterpret_cast<uint64_t*>(sm_small + ((sizeof(SmallTemp) + 15) & ~size_t(15)));
  double* T = reinterpret_cast<double*>(B + nr);    // [nsat] SAT
  uint32_t* sidx = reinterpret_cast<uint32_t*>(T + nsat);  // [kSmallNR] sorted rectangles
  uint32_t* skey = sidx + kSmallNR;                  // [kSmallNR] sorted quantised keys
  uint32_t* rank = skey + kSmallNR;                  // [nr] rank of each rectangle
  const double* vg = est + (size_t)f * cols * rows;
  if (threadIdx.x == 0) s_lo = ~0ull, s_hi = 0;
  // 1. f64 SAT, anti-diagonal wavefront: T = ((v + L) + U) - UL; the frame's
  //    cells are staged in shared memory first (B is free until step 2), so
  //    the chain of dependent steps holds no global load
  double* v = reinterpret_cast<double*>(B);
  for (int i = threadIdx.x; i < cols * rows; i += blockDim.x) v[i] = vg[i];
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) T[i] = 0.0;
  __syncthreads();
  if (rows <= 32) {  // one warp owns the wavefront: a warp barrier per anti-diagonal
    if (threadIdx.x < 32) {
      const int y = threadIdx.x;
      for (int s = 0; s <= cols + rows - 2; ++s) {
        const int x = s - y;
        if (y < rows && x >= 0 && x < cols) {
          const int i = (y + 1) * stride + (x + 1);
          T[i] = __dsub_rn(__dadd_rn(__dadd_rn(v[y * cols + x], T[i - 1]), T[i - stride]),
                           T[i - stride - 1]);
        }
        __syncwarp();
      }
    }
    __syncthreads();
  } else {
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
  }
  // 2. clamped time bits of every rectangle and their positive finite range
  uint64_t mn = ~0ull, mx = 0;
  for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
    const int xw = rr / nyh, yh = rr % nyh;
    const int x0 = dec[xw], w = dec[nxw + xw], y0 = dec[2 * nxw + yh], h = dec[2 * nxw + nyh + yh];
    const int ia = y0 * stride + x0, ib = y0 * stride + x0 + w;
    const int ic = (y0 + h) * stride + x0, idd = (y0 + h) * stride + x0 + w;
    const double t = __dadd_rn(__dsub_rn(__dsub_rn(T[idd], T[ib]), T[ic]), T[ia]);
    const uint64_t b = t > 0.0 ? (uint64_t)__double_as_longlong(t) : 0ull;
    B[rr] = b;
    if (b != 0 && b < 0x7ff0000000000000ull) {
      mn = b < mn ? b : mn;
      mx = b > mx ? b : mx;
    }
  }
  atomicMin(&s_lo, (unsigned long long)mn);
  atomicMax(&s_hi, (unsigned long long)mx);
  __syncthreads();
  // 3. 32-bit order-preserving quantisation inside the frame's range (as
  //    rank.cu), a block radix sort, then equal-key groups re-sorted by the
  //    full bits -> the exact order of (bits, rectangle)
  const uint64_t lo = s_lo, span = s_hi > s_lo ? s_hi - s_lo : 0;
  const int need = span ? 64 - __clzll((long long)span) : 0;
  // 20-bit keys (5 radix passes instead of 8): <= 2^18 + 1 quantised values,
  // +inf and the padding above them; equal keys are re-sorted exactly below
  constexpr int kQBits = 20;
  const int sh = need > kQBits - 2 ? need - (kQBits - 2) : 0;
  uint32_t kk[kSmallItems], ki[kSmallItems];
  for (int j = 0; j < kSmallItems; ++j) {
    const int rr = threadIdx.x * kSmallItems + j;
    ki[j] = (uint32_t)rr;
    kk[j] = (1u << kQBits) - 1u;
    if (rr < nr) {
      const uint64_t b = B[rr];
      kk[j] = b == 0 ? 0u : (b >= 0x7ff0000000000000ull ? (1u << kQBits) - 2u
                                                        : 1u + (uint32_t)((b - lo) >> sh));
    }
  }
  SmallSort(temp.sort).SortBlockedToStriped(kk, ki, 0, kQBits);
  for (int j = 0; j < kSmallItems; ++j) {
    const int pos = j * kSmallThreads + threadIdx.x;  // striped
    skey[pos] = kk[j];
    sidx[pos] = ki[j];
  }
  __syncthreads();
  for (int pos = threadIdx.x; pos < nr; pos += blockDim.x) {
    if (pos > 0 && skey[pos - 1] == skey[pos]) continue;
    int e = pos + 1;
    while (e < nr && skey[e] == skey[pos]) ++e;
    for (int a = pos + 1; a < e; ++a) {  // insertion sort by (bits, rectangle)
      const uint32_t x = sidx[a];
      const uint64_t bx = B[x];
      int c = a - 1;
      while (c >= pos && (B[sidx[c]] > bx || (B[sidx[c]] == bx && sidx[c] > x))) {
        sidx[c + 1] = sidx[c];
        --c;
      }
      sidx[c + 1] = x;
    }
  }
  __syncthreads();
  // first-of-run flags and their exclusive scan, kSmallItems positions per
  // thread (blocked) -> the rank of each distinct value
  const int p0 = threadIdx.x * kSmallItems;
  uint32_t cnt = 0;
  for (int j = 0; j < kSmallItems; ++j) {
    const int pos = p0 + j;
    cnt += (pos < nr && (pos == 0 || B[sidx[pos]] != B[sidx[pos - 1]])) ? 1u : 0u;
  }
  uint32_t run = 0;
  SmallScan(temp.scan).ExclusiveSum(cnt, run);
  uint64_t* fv = vals + (size_t)f * nr;
  for (int j = 0; j < kSmallItems; ++j) {
    const int pos = p0 + j;
    if (pos >= nr) break;
    const uint64_t b = B[sidx[pos]];
    const bool first = pos == 0 || b != B[sidx[pos - 1]];
    run += first ? 1u : 0u;
    const uint32_t key = run - 1;
    rank[sidx[pos]] = key;
    if (first) fv[key] = b;
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
  return ((sizeof(SmallTemp) + 15) & ~size_t(15)) + nr * sizeof(uint64_t) +
         (size_t)(cols + 1) * (rows + 1) * sizeof(double) + 2 * (size_t)kSmallNR * sizeof(uint32_t) +
         nr * sizeof(uint32_t);
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
  SCB_LAUNCH(k_small_tables<<<frames, kSmallThreads, smem, st>>>(d_est, cols, rows, frames, fpw, d_dec, keys,
                                                      vals, nvals));
  SCB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace scb
