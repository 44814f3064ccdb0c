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
#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime: no libcuda link)

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

// ---- TMA path ---------------------------------------------------------------------
// The same pass with the CTU tiles staged in shared memory by the tensor
// memory accelerator: a persistent grid (one CTA per SM), a ring of STAGES
// tile buffers, one elected thread issuing cp.async.bulk.tensor (3-D map:
// x, y, frame; box = one CTU) that completes on the stage's mbarrier; the 256
// threads then read the tile with conflict-free 128-bit shared loads.  The
// tensor map zero-fills outside the frame, so partial border CTUs need no
// special path (zeros add nothing; count is geometric).  Bytes in flight per
// SM: (STAGES - 1) tiles (96 KB at CTU 128 / 10 bit).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (spin > (1u << 24)) __trap();  // a lost transaction must not hang the device
  }
}

template <int CTU, int BPS, int STAGES>
__global__ void __launch_bounds__(256)
    k_texture_tma(const __grid_constant__ CUtensorMap tmap, int W, int H, int cols, int cells,
                  int tiles, sc_ctu_record* __restrict__ out) {
  constexpr int TILE = CTU * CTU * BPS;  // bytes
  constexpr int NT = 256;
  constexpr int PER = TILE / 16 / NT;    // 128-bit chunks per thread
  static_assert(TILE % (16 * NT) == 0, "tile must split over the block");
  extern __shared__ __align__(128) uint8_t tex_sm[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int mine = tiles > (int)blockIdx.x ? (tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto issue = [&](int i) {  // tile i of this CTA into stage i % STAGES (one thread)
    const int t = (int)blockIdx.x + i * (int)gridDim.x;
    const int cell = t % cells, frame = t / cells;
    const int x0 = (cell % cols) * CTU, y0 = (cell / cols) * CTU;
    const uint32_t bar = smem_u32(&full[i % STAGES]);
    const uint32_t dst = smem_u32(tex_sm + (size_t)(i % STAGES) * TILE);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(frame), "r"(bar)
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < STAGES - 1 && i < mine; ++i) issue(i);
  for (int i = 0; i < mine; ++i) {
    if (threadIdx.x == 0 && i + STAGES - 1 < mine) {
      // the stage was read (generic proxy) in iteration i - 1; order those
      // reads before the async-proxy write that refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + STAGES - 1);
    }
    mbar_wait(smem_u32(&full[i % STAGES]), (uint32_t)((i / STAGES) & 1));
    const uint4* tile = reinterpret_cast<const uint4*>(tex_sm + (size_t)(i % STAGES) * TILE);
    uint32_t s = 0;
    uint64_t q = 0;
    uint4 v[PER];
#pragma unroll
    for (int p = 0; p < PER; ++p) v[p] = tile[threadIdx.x + p * NT];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      acc_word<BPS>(v[p].x, s, q);
      acc_word<BPS>(v[p].y, s, q);
      acc_word<BPS>(v[p].z, s, q);
      acc_word<BPS>(v[p].w, s, q);
    }
    const int t = (int)blockIdx.x + i * (int)gridDim.x;
    const int cell = t % cells;
    const int x0 = (cell % cols) * CTU, y0 = (cell / cols) * CTU;
    const int cw = min(CTU, W - x0), ch = min(CTU, H - y0);
    block_reduce_store<NT>(s, q, (uint64_t)cw * (uint64_t)ch, out + t);
    __syncthreads();  // the stage and the reduction scratch are free again
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// SLICECRAFT_B200_K1: "tma" / "ldg" force a path; default: see texture_moments_device
static int k1_choice() {
  const char* v = getenv("SLICECRAFT_B200_K1");
  if (v && v[0] == 't') return 1;
  if (v && v[0] == 'l') return 0;
  return -1;
}

template <int CTU, int BPS, int STAGES>
static bool launch_tma_s(const uint8_t* base, size_t pitch, size_t fstride, int W, int H, int cols,
                         int cells, int frames, int sm_count, int ctas, sc_ctu_record* out,
                         cudaStream_t st) {
  constexpr int TILE = CTU * CTU * BPS;
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)fstride};  // bytes, dims 1..2
  const cuuint32_t box[3] = {(cuuint32_t)CTU, (cuuint32_t)CTU, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, BPS == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
          const_cast<uint8_t*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  auto kern = k_texture_tma<CTU, BPS, STAGES>;
  const size_t smem = (size_t)STAGES * TILE;
  once_per_device((const void*)kern, [&] {
    SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  const int tiles = cells * frames;
  const int blocks = std::min(tiles, sm_count * ctas);
  SCB_LAUNCH(kern<<<blocks, 256, smem, st>>>(tm, W, H, cols, cells, tiles, out));
  return true;
}

// CTAs per SM x ring stages: 2 x 3 by default (192 KB of tiles per SM at CTU
// 128 / 10 bit: one CTA reduces while the other's tiles land);
// SLICECRAFT_B200_K1_CTAS = 1 (4 stages) / 2 (3) / 3 (2) for A/B runs
template <int CTU, int BPS>
static bool launch_tma(const uint8_t* base, size_t pitch, size_t fstride, int W, int H, int cols,
                       int cells, int frames, int sm_count, sc_ctu_record* out, cudaStream_t st) {
  int ctas = 2;
  if (const char* v = getenv("SLICECRAFT_B200_K1_CTAS")) ctas = std::max(1, std::min(3, atoi(v)));
  if (ctas == 1)
    return launch_tma_s<CTU, BPS, 4>(base, pitch, fstride, W, H, cols, cells, frames, sm_count, 1,
                                     out, st);
  if (ctas == 2)
    return launch_tma_s<CTU, BPS, 3>(base, pitch, fstride, W, H, cols, cells, frames, sm_count, 2,
                                     out, st);
  return launch_tma_s<CTU, BPS, 2>(base, pitch, fstride, W, H, cols, cells, frames, sm_count, 3,
                                   out, st);
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

constexpr bool kK1DefaultTma = false;  // the direct-load kernel stays the default (measured)

template <int CTU, int BPS>
static void launch_vec(const uint8_t* base, size_t pitch, size_t fstride, int W, int H,
                       int cols, int cells, int frames, sc_ctu_record* out, cudaStream_t st) {
  constexpr int CPR = CTU * BPS / 16;
  constexpr int NT = (CTU * CPR) < 256 ? (CTU * CPR) : 256;
  SCB_LAUNCH(k_texture_vec<CTU, BPS><<<cells * frames, NT, 0, st>>>(base, pitch, fstride, W, H, cols,
                                                           cells, out));
}

// Launch K1 on device-resident frames.
void texture_moments_device(const void* d_luma, int bps, int W, int H, size_t pitch,
                            size_t fstride, int ctu, int frames, int cols, int rows,
                            sc_ctu_record* d_out, cudaStream_t st) {
  const uint8_t* base = static_cast<const uint8_t*>(d_luma);
  const int cells = cols * rows;
  const bool aligned = ((uintptr_t)base % 16 == 0) && (pitch % 16 == 0) && (fstride % 16 == 0);
  // TMA staging (CTU 128; tensor-map strides are multiples of 16 bytes) where
  // it is chosen: SLICECRAFT_B200_K1=tma, or by default for batches with at
  // least a few tiles per SM.  Measured against the direct-load kernel in
  // profiles/ (DESIGN.md 3.1).
  if (aligned && ctu == 128 && k1_choice() != 0 && pitch < (1ull << 40) &&
      (k1_choice() == 1 || kK1DefaultTma)) {
    int dev = 0, sms = 0;
    SCB_CUDA(cudaGetDevice(&dev));
    SCB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool ok = bps == 2 ? launch_tma<128, 2>(base, pitch, fstride, W, H, cols, cells, frames,
                                                  sms, d_out, st)
                             : launch_tma<128, 1>(base, pitch, fstride, W, H, cols, cells, frames,
                                                  sms, d_out, st);
    if (ok) {
      SCB_CUDA(cudaGetLastError());
      return;
    }
  }
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
      SCB_LAUNCH(k_texture_scalar<2><<<cells * frames, 256, 0, st>>>(base, pitch, fstride, W, H, ctu, cols,
                                                          cells, d_out));
    else
      SCB_LAUNCH(k_texture_scalar<1><<<cells * frames, 256, 0, st>>>(base, pitch, fstride, W, H, ctu, cols,
                                                          cells, d_out));
  }
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
