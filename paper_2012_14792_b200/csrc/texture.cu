// K1 — per-CTU texture moments (replaces ctu_stats, texture.cpp:145-169).
//
// One CTA per (frame, CTU).  The CTA streams the CTU tile row by row with
// 128-bit read-only loads (ld.global.nc.L1::no_allocate), all PASSES loads of a
// thread issued before any is consumed, so every SM keeps ~32 KB per CTA in
// flight.  Per-thread partials are exact (u32 sum, u64 sum of squares via
// IMAD.WIDE), then a warp-shuffle and a shared-memory reduction produce the
// u64 {count, sum, sumsq} record.  count is the geometric pixel count of the
// (possibly partial, border) CTU — identical to the reference's per-pixel
// count (grid.cpp:26-32).  The kernel is HBM-bound: algorithmic bytes per
// frame = W*H*bytes_per_sample read + cells*24 written.
#include "common.cuh"

namespace scb {

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int BPS>
__device__ __forceinline__ void acc_word(uint32_t x, uint32_t& s, uint64_t& q) {
  if (BPS == 2) {
    uint32_t lo = x & 0xFFFFu, hi = x >> 16;
    s += lo + hi;
    q += (uint64_t)lo * lo;
    q += (uint64_t)hi * hi;
  } else {
    s = __dp4a(x, 0x01010101u, s);
    q += (uint64_t)__dp4a(x, x, 0u);
  }
}

template <int BPS>
__device__ __forceinline__ uint32_t ld_sample(const uint8_t* row, int x) {
  return BPS == 2 ? (uint32_t)reinterpret_cast<const uint16_t*>(row)[x] : (uint32_t)row[x];
}

template <int NT>
__device__ __forceinline__ void block_reduce_store(uint32_t s, uint64_t q, uint64_t count,
                                                   sc_ctu_record* out) {
  constexpr int NW = NT / 32;
  __shared__ uint64_t sh_s[NW], sh_q[NW];
  uint64_t s64 = s;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s64 += __shfl_xor_sync(0xffffffffu, s64, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sh_s[wid] = s64;
    sh_q[wid] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t ts = 0, tq = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      ts += sh_s[i];
      tq += sh_q[i];
    }
    out->count = count;
    out->sum = ts;
    out->sumsq = tq;
  }
}

// Vector path: base, pitch and frame stride 16-byte aligned.
template <int CTU, int BPS>
__global__ void __launch_bounds__((CTU * CTU * BPS / 16) < 256 ? (CTU * CTU * BPS / 16) : 256)
    k_texture_vec(const uint8_t* __restrict__ base, size_t pitch, size_t fstride, int W,
                  int H, int cols, int cells, sc_ctu_record* __restrict__ out) {
  constexpr int CPR = CTU * BPS / 16;  // 16-byte chunks per CTU row
  constexpr int EPC = 16 / BPS;        // samples per chunk
  constexpr int NT = (CTU * CPR) < 256 ? (CTU * CPR) : 256;
  constexpr int RPP = NT / CPR;        // rows per pass
  constexpr int PASSES = CTU / RPP;

  const int cell = blockIdx.x % cells;
  const int frame = blockIdx.x / cells;
  const int cx = cell % cols, cy = cell / cols;
  const int x0 = cx * CTU, y0 = cy * CTU;
  const int cw = min(CTU, W - x0), ch = min(CTU, H - y0);
  const int cc = threadIdx.x % CPR, r0 = threadIdx.x / CPR;
  const uint8_t* tile = base + (size_t)frame * fstride + (size_t)y0 * pitch + (size_t)x0 * BPS +
                        (size_t)cc * 16;
  uint32_t s = 0;
  uint64_t q = 0;
  if (cw == CTU && ch == CTU) {
    uint4 v[PASSES];
#pragma unroll
    for (int p = 0; p < PASSES; ++p) v[p] = ld_stream(tile + (size_t)(r0 + p * RPP) * pitch);
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      acc_word<BPS>(v[p].x, s, q);
      acc_word<BPS>(v[p].y, s, q);
      acc_word<BPS>(v[p].z, s, q);
      acc_word<BPS>(v[p].w, s, q);
    }
  } else {
    const int e0 = cc * EPC;
    const bool full_chunk = e0 + EPC <= cw;
    const bool part_chunk = !full_chunk && e0 < cw;
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      const int r = r0 + p * RPP;
      if (r < ch) {
        const uint8_t* rp = tile + (size_t)r * pitch;
        if (full_chunk) {
          uint4 v = ld_stream(rp);
          acc_word<BPS>(v.x, s, q);
          acc_word<BPS>(v.y, s, q);
          acc_word<BPS>(v.z, s, q);
          acc_word<BPS>(v.w, s, q);
        } else if (part_chunk) {
          for (int e = 0; e < cw - e0; ++e) {
            uint32_t x = ld_sample<BPS>(rp, e);
            s += x;
            q += (uint64_t)x * x;
          }
        }
      }
    }
  }
  block_reduce_store<NT>(s, q, (uint64_t)cw * (uint64_t)ch, out + blockIdx.x);
}

// Scalar path for unaligned pitches (any W, H, CTU).
template <int BPS>
__global__ void __launch_bounds__(256)
    k_texture_scalar(const uint8_t* __restrict__ base, size_t pitch, size_t fstride, int W,
                     int H, int ctu, int cols, int cells, sc_ctu_record* __restrict__ out) {
  const int cell = blockIdx.x % cells;
  const int frame = blockIdx.x / cells;
  const int cx = cell % cols, cy = cell / cols;
  const int x0 = cx * ctu, y0 = cy * ctu;
  const int cw = min(ctu, W - x0), ch = min(ctu, H - y0);
  uint32_t s = 0;
  uint64_t q = 0;
  const uint8_t* fb = base + (size_t)frame * fstride;
  for (int i = threadIdx.x; i < cw * ch; i += 256) {
    const int yy = i / cw, xx = i % cw;
    uint32_t x = ld_sample<BPS>(fb + (size_t)(y0 + yy) * pitch, x0 + xx);
    s += x;
    q += (uint64_t)x * x;
  }
  block_reduce_store<256>(s, q, (uint64_t)cw * (uint64_t)ch, out + blockIdx.x);
}

template <int CTU, int BPS>
static void launch_vec(const uint8_t* base, size_t pitch, size_t fstride, int W, int H,
                       int cols, int cells, int frames, sc_ctu_record* out, cudaStream_t st) {
  constexpr int CPR = CTU * BPS / 16;
  constexpr int NT = (CTU * CPR) < 256 ? (CTU * CPR) : 256;
  k_texture_vec<CTU, BPS><<<cells * frames, NT, 0, st>>>(base, pitch, fstride, W, H, cols,
                                                           cells, out);
}

// Launch K1 on device-resident frames.
void texture_moments_device(const void* d_luma, int bps, int W, int H, size_t pitch,
                            size_t fstride, int ctu, int frames, int cols, int rows,
                            sc_ctu_record* d_out, cudaStream_t st) {
  const uint8_t* base = static_cast<const uint8_t*>(d_luma);
  const int cells = cols * rows;
  const bool aligned = ((uintptr_t)base % 16 == 0) && (pitch % 16 == 0) && (fstride % 16 == 0);
  if (aligned) {
    if (bps == 2) {
      if (ctu == 128) launch_vec<128, 2>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
      else if (ctu == 64) launch_vec<64, 2>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
      else launch_vec<32, 2>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
    } else {
      if (ctu == 128) launch_vec<128, 1>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
      else if (ctu == 64) launch_vec<64, 1>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
      else launch_vec<32, 1>(base, pitch, fstride, W, H, cols, cells, frames, d_out, st);
    }
  } else {
    if (bps == 2)
      k_texture_scalar<2><<<cells * frames, 256, 0, st>>>(base, pitch, fstride, W, H, ctu, cols,
                                                          cells, d_out);
    else
      k_texture_scalar<1><<<cells * frames, 256, 0, st>>>(base, pitch, fstride, W, H, ctu, cols,
                                                          cells, d_out);
  }
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
