// K2 — summed-area tables; K3 — per-rectangle time and SSE tables.
//
// K2 (replaces PrefixSumTable ctor, cost.cpp:97-112, and the TextureStats
// SATs, texture.cpp:113-129): one CTA per frame.  The f64 table must follow the
// reference recurrence T = ((v + L) + U) - UL in row-major dependency order, so
// it is computed as an anti-diagonal wavefront (one thread per CTU row, one
// barrier per diagonal); a row-scan/column-scan would reassociate and differ.
// The three u64 tables are modular and order-free; they ride the same wavefront.
//
// K3 (replaces rect_sum, cost.hpp:75-81, and rect_moments + sse,
// texture.cpp:83-88/132-143): one thread per (frame, rectangle).  Times use
// the reference corner order ((d - b) - c) + a; SSE converts the exact
// 128-bit numerator count*sumsq - sum^2 to double with round-to-nearest-even
// (as GCC's __floattidf does) and divides by count.  The search-layout copies
// are frame-interleaved ([group][rect][FPW]) so that the lanes of a warp —
// one frame each — read one contiguous line per rectangle.
#include "common.cuh"

namespace scb {

__global__ void k_grid_sat(const double* __restrict__ est, const sc_ctu_record* __restrict__ rec,
                           int cols, int rows, double* __restrict__ sat_out,
                           uint64_t* __restrict__ usat_out) {
  extern __shared__ unsigned char smem[];
  const int stride = cols + 1;
  const int nsat = stride * (rows + 1);
  const int cells = cols * rows;
  double* T = reinterpret_cast<double*>(smem);
  uint64_t* U = reinterpret_cast<uint64_t*>(T + nsat);  // 3 tables
  // the frame's cells staged in shared memory first: the wavefront below is a
  // chain of dependent steps, and a global load inside every step would set
  // its pace
  double* V = reinterpret_cast<double*>(U + 3 * nsat);        // [cells] (est)
  uint64_t* R = reinterpret_cast<uint64_t*>(V + (est ? cells : 0));  // [3][cells] (records)
  const int f = blockIdx.x;
  const double* v = est ? est + (size_t)f * cells : nullptr;
  const sc_ctu_record* r = rec ? rec + (size_t)f * cells : nullptr;
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) {
    T[i] = 0.0;
    U[i] = 0;
    U[nsat + i] = 0;
    U[2 * nsat + i] = 0;
  }
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    if (v) V[i] = v[i];
    if (r) {
      const sc_ctu_record c = r[i];
      R[i] = c.count;
      R[cells + i] = c.sum;
      R[2 * cells + i] = c.sumsq;
    }
  }
  __syncthreads();
  auto cell = [&](int y, int x) {
    const int i = (y + 1) * stride + (x + 1), ci = y * cols + x;
    if (v)
      T[i] = __dsub_rn(__dadd_rn(__dadd_rn(V[ci], T[i - 1]), T[i - stride]), T[i - stride - 1]);
    if (r) {
      U[i] = R[ci] + U[i - 1] + U[i - stride] - U[i - stride - 1];
      U[nsat + i] =
          R[cells + ci] + U[nsat + i - 1] + U[nsat + i - stride] - U[nsat + i - stride - 1];
      U[2 * nsat + i] = R[2 * cells + ci] + U[2 * nsat + i - 1] + U[2 * nsat + i - stride] -
                        U[2 * nsat + i - stride - 1];
    }
  };
  if (rows <= 32) {  // one warp owns the wavefront: a warp barrier per anti-diagonal
    if (threadIdx.x < 32) {
      const int y = threadIdx.x;
      for (int s = 0; s <= cols + rows - 2; ++s) {
        const int x = s - y;
        if (y < rows && x >= 0 && x < cols) cell(y, x);
        __syncwarp();
      }
    }
    __syncthreads();
  } else {
    for (int s = 0; s <= cols + rows - 2; ++s) {
      for (int y = threadIdx.x; y < rows; y += blockDim.x) {
        const int x = s - y;
        if (x >= 0 && x < cols) cell(y, x);
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) {
    if (v) sat_out[(size_t)f * nsat + i] = T[i];
    if (r) {
      usat_out[((size_t)f * 3 + 0) * nsat + i] = U[i];
      usat_out[((size_t)f * 3 + 1) * nsat + i] = U[nsat + i];
      usat_out[((size_t)f * 3 + 2) * nsat + i] = U[2 * nsat + i];
    }
  }
}

// Unsigned 128-bit (hi, lo) -> double, round to nearest even.
__device__ __forceinline__ double u128_to_double_rn(uint64_t hi, uint64_t lo) {
  if (hi == 0) return __ull2double_rn(lo);
  const int s = __clzll((long long)hi);  // 0..63
  uint64_t top = s ? ((hi << s) | (lo >> (64 - s))) : hi;
  const uint64_t rest = lo << s;           // bits shifted out (s==0: all of lo)
  top |= (rest != 0) ? 1ull : 0ull;        // sticky below the rounding position
  return ldexp(__ull2double_rn(top), 64 - s);
}

// SliceMoments::sse (texture.cpp:83-88) with exact i128 arithmetic.
__device__ __forceinline__ double moments_sse(uint64_t c, uint64_t s, uint64_t q) {
  if (c == 0) return 0.0;
  uint64_t p1lo = c * q, p1hi = __umul64hi(c, q);
  uint64_t p2lo = s * s, p2hi = __umul64hi(s, s);
  uint64_t lo = p1lo - p2lo;
  uint64_t hi = p1hi - p2hi - (p1lo < p2lo ? 1ull : 0ull);
  double mag;
  if ((int64_t)hi < 0) {  // negative numerator (invalid records only)
    uint64_t nlo = ~lo + 1ull;
    uint64_t nhi = ~hi + (nlo == 0 ? 1ull : 0ull);
    mag = -u128_to_double_rn(nhi, nlo);
  } else {
    mag = u128_to_double_rn(hi, lo);
  }
  return __ddiv_rn(mag, (double)c);
}

struct RectDecode {
  const int16_t* xw_x0;
  const int16_t* xw_w;
  const int16_t* yh_y0;
  const int16_t* yh_h;
};

__global__ void k_rect_tables(const double* __restrict__ sat, const uint64_t* __restrict__ usat,
                              RectDecode dec, int cols, int rows, int frames, int fpw,
                              double* __restrict__ rect_t, double* __restrict__ rect_s,
                              uint64_t* __restrict__ rt_search, double* __restrict__ rs_search) {
  const int nyh = rows * (rows + 1) / 2;
  const int nr = cols * (cols + 1) / 2 * nyh;
  const int stride = cols + 1;
  const int nsat = stride * (rows + 1);
  const size_t total = (size_t)nr * frames;
  for (size_t id = blockIdx.x * (size_t)blockDim.x + threadIdx.x; id < total;
       id += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(id / nr);
    const int rr = (int)(id % nr);
    const int xw = rr / nyh, yh = rr % nyh;
    const int x0 = dec.xw_x0[xw], w = dec.xw_w[xw];
    const int y0 = dec.yh_y0[yh], h = dec.yh_h[yh];
    const int ia = y0 * stride + x0, ib = y0 * stride + x0 + w;
    const int ic = (y0 + h) * stride + x0, idd = (y0 + h) * stride + x0 + w;
    const int g = f / fpw, slot = f % fpw;
    const size_t so = ((size_t)g * nr + rr) * fpw + slot;
    if (sat) {
      const double* T = sat + (size_t)f * nsat;
      const double t = __dadd_rn(__dsub_rn(__dsub_rn(T[idd], T[ib]), T[ic]), T[ia]);
      if (rect_t) rect_t[(size_t)f * nr + rr] = t;
      // layout_time's running max starts at 0.0 and keeps it on ties/NaN
      // (search.cpp:77-83): clamp to +0.0 so u64 bit order == double order.
      // Frame-major bits, ranked into time keys by rank.cu.
      if (rt_search) rt_search[(size_t)f * nr + rr] =
          (t > 0.0) ? (uint64_t)__double_as_longlong(t) : 0ull;
    }
    if (usat) {
      const uint64_t* U = usat + (size_t)f * 3 * nsat;
      const uint64_t c = U[idd] - U[ib] - U[ic] + U[ia];
      const uint64_t s = U[nsat + idd] - U[nsat + ib] - U[nsat + ic] + U[nsat + ia];
      const uint64_t q = U[2 * nsat + idd] - U[2 * nsat + ib] - U[2 * nsat + ic] + U[2 * nsat + ia];
      const double e = moments_sse(c, s, q);
      if (rect_s) rect_s[(size_t)f * nr + rr] = e;
      if (rs_search) rs_search[so] = e;
    }
  }
}

// Split table (search_walk.cuh WalkEnv::rts): for every rectangle (x0,w,y0,h)
// with y0+h < rows, max(time(y0,h), time(y0+h, rows-y0-h)), i.e. a run and
// the forced remainder of its column, so the search scores a two-run split
// with one load.  Same [group][rect][FPW] layout as the time table.
// keys: [groups][2][nr][fpw] -- reads the rt half, writes the rts half
// list / nl: only these rectangles' entries (the split entries a plan's
// candidates read, trace.cu); nullptr: every rectangle
__global__ void k_split_table(uint32_t* __restrict__ keys, int cols, int rows,
                              size_t slots /* groups * fpw */, int fpw,
                              const uint32_t* __restrict__ list, size_t nl) {
  const int nyh = rows * (rows + 1) / 2;
  const size_t nr = (size_t)cols * (cols + 1) / 2 * nyh;
  const size_t per = list ? nl : nr;
  const size_t total = per * slots;
  for (size_t id = blockIdx.x * (size_t)blockDim.x + threadIdx.x; id < total;
       id += (size_t)gridDim.x * blockDim.x) {
    const size_t g = id / (per * fpw);
    const size_t rem = id % (per * fpw);
    const int slot = (int)(rem % fpw);
    const int rr = list ? (int)list[rem / fpw] : (int)(rem / fpw);
    const int xw = rr / nyh, yh = rr % nyh;
    // decode (y0, h) from yh: y0 is the largest y with yh(y, 1) <= yh
    int y0 = 0;
    while (y0 + 1 < rows && (y0 + 1) * rows - ((y0 + 1) * y0) / 2 <= yh) ++y0;
    const int h = yh - (y0 * rows - (y0 * (y0 - 1)) / 2) + 1;
    const uint32_t* rt = keys + g * 2 * nr * fpw;
    uint32_t v = 0;
    if (y0 + h < rows) {
      const uint32_t a = rt[(size_t)rr * fpw + slot];
      const int y1 = y0 + h, h1 = rows - y1;
      const int rr2 = xw * nyh + (y1 * rows - (y1 * (y1 - 1)) / 2 + h1 - 1);
      const uint32_t b = rt[(size_t)rr2 * fpw + slot];
      v = a > b ? a : b;
    }
    keys[g * 2 * nr * fpw + nr * fpw + (size_t)rr * fpw + slot] = v;
  }
}

void split_table_device(uint32_t* d_keys, int cols, int rows, int groups, int fpw, int sm_count,
                        const uint32_t* list, size_t nl, cudaStream_t st) {
  const size_t total =
      (list ? nl : (size_t)cols * (cols + 1) / 2 * (rows * (rows + 1) / 2)) * groups * fpw;
  size_t blocks = (total + 255) / 256;
  const size_t cap = (size_t)sm_count * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  SCB_LAUNCH(k_split_table<<<(unsigned)blocks, 256, 0, st>>>(d_keys, cols, rows, (size_t)groups * fpw, fpw,
                                                  list, nl));
  SCB_CUDA(cudaGetLastError());
}

// partition_time (cost.cpp:117-145) + slice_moments / partition_sse
// (texture.cpp:171-189) of one partition on every frame: one CTA per frame,
// one thread per slice for the rectangle sums, then thread 0 folds in id
// order exactly like the reference (max from slice 0 with strict >, totals
// summed in id order).  rects: {x0, y0, w, h} indexed by slice id.
__global__ void k_partition_eval(const double* __restrict__ sat, const uint64_t* __restrict__ usat,
                                 const int4* __restrict__ rects, int n, int cols, int rows,
                                 sc_partition_stats* __restrict__ out,
                                 double* __restrict__ slice_times,
                                 sc_ctu_record* __restrict__ slice_mom) {
  __shared__ double st[SC_MAX_SLICES], ss[SC_MAX_SLICES];
  const int f = blockIdx.x;
  const int stride = cols + 1;
  const int nsat = stride * (rows + 1);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int4 r = rects[j];
    const int ia = r.y * stride + r.x, ib = r.y * stride + r.x + r.z;
    const int ic = (r.y + r.w) * stride + r.x, idd = (r.y + r.w) * stride + r.x + r.z;
    if (sat) {
      const double* T = sat + (size_t)f * nsat;
      st[j] = __dadd_rn(__dsub_rn(__dsub_rn(T[idd], T[ib]), T[ic]), T[ia]);
      if (slice_times) slice_times[(size_t)f * n + j] = st[j];
    }
    if (usat) {
      const uint64_t* U = usat + (size_t)f * 3 * nsat;
      const uint64_t c = U[idd] - U[ib] - U[ic] + U[ia];
      const uint64_t sm = U[nsat + idd] - U[nsat + ib] - U[nsat + ic] + U[nsat + ia];
      const uint64_t q = U[2 * nsat + idd] - U[2 * nsat + ib] - U[2 * nsat + ic] + U[2 * nsat + ia];
      ss[j] = moments_sse(c, sm, q);
      if (slice_mom) slice_mom[(size_t)f * n + j] = sc_ctu_record{c, sm, q};
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sc_partition_stats& o = out[f];
    if (sat) {
      o.max_us = st[0];
      o.argmax = 0;
      o.total_us = 0.0;
      for (int j = 0; j < n; ++j) {
        o.total_us = __dadd_rn(o.total_us, st[j]);
        if (st[j] > o.max_us) {
          o.max_us = st[j];
          o.argmax = j;
        }
      }
    }
    if (usat) {
      double tot = 0.0;
      for (int j = 0; j < n; ++j) tot = __dadd_rn(tot, ss[j]);
      o.sse = tot;
    }
  }
}

void partition_eval_device(const double* d_sat, const uint64_t* d_usat, const int* d_rects, int n,
                           int cols, int rows, int frames, sc_partition_stats* d_out,
                           double* d_slice_times, sc_ctu_record* d_slice_mom, cudaStream_t st) {
  SCB_LAUNCH(k_partition_eval<<<frames, 64, 0, st>>>(d_sat, d_usat, reinterpret_cast<const int4*>(d_rects),
                                          n, cols, rows, d_out, d_slice_times, d_slice_mom));
  SCB_CUDA(cudaGetLastError());
}

void grid_sat_device(const double* d_est, const sc_ctu_record* d_rec, int cols, int rows,
                     int frames, double* d_sat, uint64_t* d_usat, cudaStream_t st) {
  const int nsat = (cols + 1) * (rows + 1);
  const size_t smem = (size_t)nsat * (8 + 24) +
                      (size_t)cols * rows * ((d_est ? 8 : 0) + (d_rec ? 24 : 0));
  if (smem > 227 * 1024) fail(SC_ERR_SIZE, "CTU grid too large for the shared-memory SAT");
  once_per_device((const void*)k_grid_sat, [] {
    SCB_CUDA(cudaFuncSetAttribute(k_grid_sat, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
  });
  int threads = rows < 128 ? 128 : (rows > 1024 ? 1024 : ((rows + 31) / 32) * 32);
  SCB_LAUNCH(k_grid_sat<<<frames, threads, smem, st>>>(d_est, d_rec, cols, rows, d_sat, d_usat));
  SCB_CUDA(cudaGetLastError());
}

void rect_tables_device(const double* d_sat, const uint64_t* d_usat, const int16_t* d_dec,
                        int cols, int rows, int frames, int fpw, double* d_rect_t,
                        double* d_rect_s, uint64_t* d_rt, double* d_rs, int sm_count,
                        cudaStream_t st) {
  const int nxw = cols * (cols + 1) / 2, nyh = rows * (rows + 1) / 2;
  RectDecode dec{d_dec, d_dec + nxw, d_dec + 2 * nxw, d_dec + 2 * nxw + nyh};
  const size_t total = (size_t)nxw * nyh * frames;
  size_t blocks = (total + 255) / 256;
  const size_t cap = (size_t)sm_count * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  SCB_LAUNCH(k_rect_tables<<<(unsigned)blocks, 256, 0, st>>>(d_sat, d_usat, dec, cols, rows, frames, fpw,
                                                  d_rect_t, d_rect_s, d_rt, d_rs));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
