// for_each_candidate / enumerate_candidates (search.cpp:302-326) as a
// device-materialised candidate stream.
//
// The search walks (search_walk.cuh) never materialise a candidate; this is
// the API for callers that want the candidates themselves, meant for small
// spaces or for paging through a window of a large one.  One thread per work
// item (a lex-ordered width prefix, plan.h) runs the reference's generator
// below its prefix -- remaining widths, runs per column, run heights with the
// area test k*(double)amin > (double)amax (search.cpp:120-190) -- twice: a
// count pass (per-item counts, scanned into offsets once per plan) and an
// emit pass that writes the candidates whose global ordinal falls in the
// requested window as 96-byte snapshots (W[16] R[16] H[64]).
#include <cub/cub.cuh>

#include "common.cuh"

namespace scb {

template <bool EMIT>
__global__ void k_enumerate(const WorkItem* __restrict__ items, uint32_t n_items, int cols,
                            int rows, int n, double k, int covering,
                            uint64_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                            uint64_t first, uint64_t limit, uint8_t* __restrict__ out) {
  const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  uint64_t ord = 0;
  if (EMIT) {
    ord = offsets[it];
    if (ord >= first + limit || ord + counts[it] <= first) return;  // outside the window
  }
  const WorkItem wi = items[it];
  const int c = wi.c, d = wi.d;
  int W[SC_MAX_COLS], R[SC_MAX_COLS], CL[SC_MAX_COLS + 1], SL[SC_MAX_COLS + 1];
  // per run (column-major): width, first-run flag, height, area bounds before it
  int RW[SC_MAX_SLICES], H[SC_MAX_SLICES], RLeft[SC_MAX_SLICES], RL[SC_MAX_SLICES];
  int AMIN[SC_MAX_SLICES], AMAX[SC_MAX_SLICES];
  bool LAST[SC_MAX_SLICES];
  uint64_t local = 0;
  CL[0] = cols;
  for (int i = 0; i < d; ++i) {
    W[i] = wi.w[i];
    CL[i + 1] = CL[i] - W[i];
  }
  // ---- widths below the prefix (rec_widths, search.cpp:133-143)
  int pos = d;
  const bool fixed = d == c;
  if (!fixed) W[pos] = 0;
  while (true) {
    if (!fixed) {
      bool got = false;
      while (true) {
        const int maxw = CL[pos] - (c - pos - 1);
        int wv;
        if (covering && pos == c - 1) wv = W[pos] == 0 ? maxw : maxw + 1;  // sum == cols
        else wv = W[pos] + 1;
        if (wv > maxw) {
          if (pos == d) break;
          --pos;
          continue;
        }
        W[pos] = wv;
        CL[pos + 1] = CL[pos] - wv;
        if (pos == c - 1) {
          got = true;
          break;
        }
        W[++pos] = 0;
      }
      if (!got) break;
    }
    // ---- runs per column (rec_runs, search.cpp:145-161)
    int rp = 0;
    SL[0] = n;
    R[0] = max(1, n - (c - 1) * rows) - 1;
    while (rp >= 0) {
      const int after = c - rp - 1;
      const int hi = min(rows, SL[rp] - after);
      if (++R[rp] > hi) {
        --rp;
        continue;
      }
      SL[rp + 1] = SL[rp] - R[rp];
      if (rp < c - 1) {
        ++rp;
        R[rp] = max(1, SL[rp] - (c - rp - 1) * rows) - 1;
        continue;
      }
      if (SL[c] != 0) continue;
      // ---- run heights (rec_heights, search.cpp:163-190)
      int t = 0;
      for (int i = 0; i < c; ++i)
        for (int j = 0; j < R[i]; ++j, ++t) {
          RW[t] = W[i];
          RLeft[t] = R[i] - j;  // runs left in the column, this one included
          LAST[t] = j == R[i] - 1;
        }
      t = 0;
      RL[0] = rows;
      AMIN[0] = 0x7fffffff;
      AMAX[0] = 0;
      H[0] = (LAST[0] ? RL[0] : 1) - 1;
      while (t >= 0) {
        const int hi_h = RL[t] - (RLeft[t] - 1);
        const int h = ++H[t];
        if (h > hi_h) {
          --t;
          continue;
        }
        const int area = RW[t] * h;
        const int na = min(AMIN[t], area), nx = max(AMAX[t], area);
        if (!(k * (double)na > (double)nx)) continue;
        if (t == n - 1) {
          if (EMIT) {
            const uint64_t o = ord + local;
            if (o >= first && o < first + limit) {
              uint8_t* s = out + (o - first) * kSnapBytes;
              for (int i = 0; i < SC_MAX_COLS; ++i) {
                s[i] = (uint8_t)(i < c ? W[i] : 0);
                s[SC_MAX_COLS + i] = (uint8_t)(i < c ? R[i] : 0);
              }
              for (int i = 0; i < SC_MAX_SLICES; ++i)
                s[2 * SC_MAX_COLS + i] = (uint8_t)(i < n ? H[i] : 0);
            }
          }
          ++local;
          continue;
        }
        AMIN[t + 1] = na;
        AMAX[t + 1] = nx;
        RL[t + 1] = LAST[t] ? rows : RL[t] - h;
        ++t;
        H[t] = (LAST[t] ? RL[t] : 1) - 1;
      }
    }
    if (fixed) break;
  }
  if (!EMIT) counts[it] = local;
}

// Per-item counts and their exclusive scan (offsets), total into *total_host.
void enumerate_count_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                            double k, int covering, uint64_t* d_counts, uint64_t* d_offsets,
                            DevBuf& temp, cudaStream_t st) {
  if (!n_items) return;
  SCB_LAUNCH(k_enumerate<false><<<(n_items + 127) / 128, 128, 0, st>>>(
      d_items, n_items, cols, rows, n, k, covering, d_counts, nullptr, 0, 0, nullptr));
  SCB_CUDA(cudaGetLastError());
  size_t tb = 0;
  SCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_counts, d_offsets, (int)n_items, st));
  temp.ensure(tb + 16);
  SCB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, d_counts, d_offsets, (int)n_items, st));
  count_launches(2);  // CUB scan: init + scan
}

void enumerate_emit_device(const WorkItem* d_items, uint32_t n_items, int cols, int rows, int n,
                           double k, int covering, const uint64_t* d_counts,
                           const uint64_t* d_offsets, uint64_t first, uint64_t limit,
                           uint8_t* d_out, cudaStream_t st) {
  if (!n_items || !limit) return;
  SCB_LAUNCH(k_enumerate<true><<<(n_items + 127) / 128, 128, 0, st>>>(
      d_items, n_items, cols, rows, n, k, covering, const_cast<uint64_t*>(d_counts), d_offsets,
      first, limit, d_out));
  SCB_CUDA(cudaGetLastError());
}

}  // namespace scb
