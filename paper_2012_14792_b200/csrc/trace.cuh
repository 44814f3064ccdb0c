// The candidate family compiled into a time-evaluation program ("trace").
//
// The ColumnSplit enumeration (search.cpp:110-196) does not depend on the
// frame: for a given grid and configuration it always yields the same
// candidates in the same order.  Step 1 of the exhaustive search only needs,
// per candidate, the maximum of its slices' time keys.  So instead of
// re-running the DFS (widths, runs, heights, area windows) for every call --
// which is what the warp-uniform walk in search_walk.cuh does, and where most
// of its instructions go -- the DFS runs ONCE per plan and writes its
// pre-order as a stream of 32-bit ops; the per-call kernel (trace.cu) is an
// interpreter that keeps one running maximum per DFS depth:
//
//   SKEL  ld        new skeleton (widths + runs): P[0] = 0, its leaf depth ld
//   FIX   idx, tag  P[0] = max(P[0], rt[idx])          a one-run column (tag:
//                   the multi-run columns left of it, its place in the slice
//                   order for the step-2 SSE fold)
//   PUSH  d, kidx   P[d+1] = max(P[d], keys[kidx])     a run of a multi-run
//                   column; keys = rt | rts (the time keys, then the split
//                   table: run + forced rest of its column), kidx = idx for
//                   rt and NR + idx for the column's second-to-last run
//                   (PUSHL: the same op at depth ld - 1, right above a LEAF)
//   LEAF  idx, cnt  candidates time max(P[ld], rts[idx + i]), i < cnt (<= 31): the
//                   last decision run takes cnt consecutive heights (its
//                   forced rest and any later one-run columns are in the key);
//                   longer runs of heights are several LEAF ops
//   LEAF  -, 0      the skeleton's single candidate (no decision run): P[ld]
//
// Only ops that lead to a candidate are emitted (a PUSH is written lazily,
// right before the first LEAF below it), so the trace holds every candidate
// exactly once, in the reference's enumeration order: candidate ordinals are
// the running sum of the LEAF counts.  The trace is independent of k, of the
// coverage flag and of the frame: those only decide which ops exist.
//
// Written as __host__ __device__ code: the generator runs on the device (two
// passes over the plan's work items, trace.cu) and, for the CPU test suite,
// on the host (tests/emu), together with a scalar reference interpreter.
#pragma once

#include <math.h>
#include <stdint.h>

#include "plan.h"
#include "slicecraft_b200.h"

#ifdef __CUDACC__
#define SCB_TR_HD __host__ __device__ __forceinline__
#else
#define SCB_TR_HD inline
#endif

namespace scb {

constexpr uint32_t kOpPush = 0u, kOpPushL = 1u, kOpLeaf = 2u, kOpSkel = 3u;  // bits 31..30
constexpr int kTrIdxBits = 22;                                 // rectangle index
constexpr uint32_t kTrIdxMask = (1u << kTrIdxBits) - 1u;
constexpr uint32_t kTrKeyMask = (1u << (kTrIdxBits + 1)) - 1u;  // rt | rts key index
constexpr int kTrLeafMax = 31;                                  // heights per LEAF op

// Encoding.  Every op that reads a key holds its key index (rt | rts) in bits
// 27..5, i.e. already multiplied by 32 -- the element offset of the key's line
// in the [rect][32 frames] table -- so the interpreter's address is one AND
// and one multiply-add.  The small field (a PUSH's depth, a FIX's tag, a
// LEAF's count) is in bits 4..0 (+ bit 28 for depths / tags above 31).
//   PUSH  (code 0)  depth d; PUSHL (code 1) the same with d == ld - 1: the
//                   push right above a LEAF, which the step-1 interpreter
//                   fuses with that LEAF (the next op) and keeps in a register
//   LEAF  (code 2)  key index NR + idx (the split table), count 0..31
//   SKEL  (code 3, bit 29 clear)  leaf depth in bits 5..0
//   FIX   (code 3, bit 29 set)    rectangle idx, tag
SCB_TR_HD uint32_t tr_small(int v) { return ((uint32_t)v & 31u) | (((uint32_t)v & 32u) << 23); }
SCB_TR_HD uint32_t op_push(int d, uint32_t kidx, bool to_leaf) {
  return ((to_leaf ? kOpPushL : kOpPush) << 30) | (kidx << 5) | tr_small(d);
}
SCB_TR_HD uint32_t op_leaf(uint32_t kidx, int cnt) {
  return (kOpLeaf << 30) | (kidx << 5) | (uint32_t)cnt;
}
SCB_TR_HD uint32_t op_skel(int ld) { return (kOpSkel << 30) | (uint32_t)ld; }
// FIX: tag = the number of multi-run columns left of the column (its place in
// the slice order, for the step-2 SSE fold)
SCB_TR_HD uint32_t op_fix(uint32_t idx, int tag) {
  return (kOpSkel << 30) | (1u << 29) | (idx << 5) | tr_small(tag);
}
// decoders
SCB_TR_HD uint32_t tr_code(uint32_t op) { return op >> 30; }
SCB_TR_HD bool tr_is_push(uint32_t op) { return (op >> 31) == 0u; }  // PUSH or PUSHL
SCB_TR_HD bool tr_is_fix(uint32_t op) { return (op >> 29) == 7u; }
SCB_TR_HD uint32_t tr_kidx(uint32_t op) { return (op >> 5) & kTrKeyMask; }
SCB_TR_HD uint32_t tr_koff32(uint32_t op) { return op & (kTrKeyMask << 5); }  // kidx * 32
SCB_TR_HD int tr_small_of(uint32_t op) { return (int)((op & 31u) | ((op >> 23) & 32u)); }
SCB_TR_HD int tr_leaf_cnt(uint32_t op) { return (int)(op & 31u); }
SCB_TR_HD int tr_skel_ld(uint32_t op) { return (int)(op & 63u); }

SCB_TR_HD int tr_xw(int cols, int x0, int w) { return x0 * cols - (x0 * (x0 - 1)) / 2 + (w - 1); }
SCB_TR_HD int tr_yh(int rows, int y0, int h) { return y0 * rows - (y0 * (y0 - 1)) / 2 + (h - 1); }
// inverse of tr_xw / tr_yh: the origin a (largest with tr(n, a, 1) <= v) and
// the extent v - tr(n, a, 1) + 1; closed form plus an exact fix-up
SCB_TR_HD void tr_unrank(int n, int v, int& a, int& ext) {
  const float b = (float)(2 * n + 1);
  float disc = b * b - 8.0f * (float)v;
  disc = disc > 0.0f ? disc : 0.0f;
  int g = (int)((b - sqrtf(disc)) * 0.5f);
  g = g < 0 ? 0 : (g > n - 1 ? n - 1 : g);
  while (g + 1 < n && tr_xw(n, g + 1, 1) <= v) ++g;
  while (g > 0 && tr_xw(n, g, 1) > v) --g;
  a = g;
  ext = v - tr_xw(n, g, 1) + 1;
}

// Counting sink (pass 1) and writing sink (pass 2) of the generator.
struct TraceCount {
  uint64_t ops = 0, cands = 0, skels = 0;
  SCB_TR_HD void skel(int) { ++ops; ++skels; }
  SCB_TR_HD void fix(uint32_t, int) { ++ops; }
  SCB_TR_HD void push(int, uint32_t, bool) { ++ops; }
  SCB_TR_HD void leaf(uint32_t, int cnt) { ++ops; cands += cnt ? (uint64_t)cnt : 1u; }
};
struct TraceWrite {
  uint32_t* ops;          // this item's ops
  uint64_t pos = 0;       // ops written
  uint64_t cand;          // global ordinal of the next candidate
  uint32_t* skel_pos;     // this item's skeleton starts: global op index
  uint64_t* skel_ord;     // and the ordinal of their first candidate
  uint64_t op_base;       // global index of ops[0]
  uint64_t nsk = 0;
  SCB_TR_HD void skel(int ld) {
    skel_pos[nsk] = (uint32_t)(op_base + pos);
    skel_ord[nsk] = cand;
    ++nsk;
    ops[pos++] = op_skel(ld);
  }
  SCB_TR_HD void fix(uint32_t idx, int tag) { ops[pos++] = op_fix(idx, tag); }
  SCB_TR_HD void push(int d, uint32_t kidx, bool to_leaf) { ops[pos++] = op_push(d, kidx, to_leaf); }
  SCB_TR_HD void leaf(uint32_t kidx, int cnt) {
    ops[pos++] = op_leaf(kidx, cnt);
    cand += cnt ? (uint64_t)cnt : 1u;
  }
};

// The enumeration below the width prefix of one work item (plan.h), in the
// reference's order: remaining widths (search.cpp:133-143; covering: the last
// width closes the grid), runs per column (145-161), run heights with the
// area test k * (double)amin > (double)amax (163-190).  The area test prunes
// partial candidates exactly as the reference does (adding areas only
// tightens it), so the emitted candidates are the reference's.
template <class Sink>
SCB_TR_HD void trace_item(const WorkItem& wi, int cols, int rows, int n, double k, int covering,
                          Sink& out) {
  const int c = wi.c, d = wi.d;
  const int nyh = rows * (rows + 1) / 2;
  const uint32_t nr = (uint32_t)(cols * (cols + 1) / 2 * nyh);
  int W[SC_MAX_COLS], R[SC_MAX_COLS], CL[SC_MAX_COLS + 1], SL[SC_MAX_COLS + 1];
  // decision runs (every run of a multi-run column but its last), in order
  int Dx0[SC_MAX_SLICES], Dw[SC_MAX_SLICES], Dleft[SC_MAX_SLICES];  // runs left incl. this
  int H[SC_MAX_SLICES], Y0[SC_MAX_SLICES], AMIN[SC_MAX_SLICES + 1], AMAX[SC_MAX_SLICES + 1];
  uint32_t FIXI[SC_MAX_COLS];
  int FIXT[SC_MAX_COLS];  // multi-run columns left of each one-run column
  CL[0] = cols;
  for (int i = 0; i < d; ++i) {
    W[i] = wi.w[i];
    CL[i + 1] = CL[i] - W[i];
  }
  int pos = d;
  const bool fixed = d == c;
  if (!fixed) W[pos] = 0;
  while (true) {
    if (!fixed) {
      bool got = false;
      while (true) {
        const int maxw = CL[pos] - (c - pos - 1);
        const int wv = (covering && pos == c - 1) ? (W[pos] == 0 ? maxw : maxw + 1) : W[pos] + 1;
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
    // ---- runs per column (rec_runs)
    int rp = 0;
    SL[0] = n;
    R[0] = (n - (c - 1) * rows > 1 ? n - (c - 1) * rows : 1) - 1;
    while (rp >= 0) {
      const int hi_r = rows < SL[rp] - (c - rp - 1) ? rows : SL[rp] - (c - rp - 1);
      if (++R[rp] > hi_r) {
        --rp;
        continue;
      }
      SL[rp + 1] = SL[rp] - R[rp];
      if (rp < c - 1) {
        ++rp;
        const int lo_r = SL[rp] - (c - rp - 1) * rows;
        R[rp] = (lo_r > 1 ? lo_r : 1) - 1;
        continue;
      }
      if (SL[c] != 0) continue;
      // ---- one skeleton: fixed one-run columns, then the decision runs
      int amin = 0x7fffffff, amax = 0, nl = 0, nfix = 0, x0 = 0, nmulti = 0;
      bool ok = true;
      for (int i = 0; i < c; ++i) {
        if (R[i] == 1) {
          const int a = W[i] * rows;
          amin = a < amin ? a : amin;
          amax = a > amax ? a : amax;
          ok = ok && (k * (double)amin > (double)amax);
          FIXT[nfix] = nmulti;
          FIXI[nfix++] = (uint32_t)(tr_xw(cols, x0, W[i]) * nyh + tr_yh(rows, 0, rows));
        } else {
          for (int j = 0; j < R[i] - 1; ++j, ++nl) {
            Dx0[nl] = x0;
            Dw[nl] = W[i];
            Dleft[nl] = R[i] - j;
          }
          ++nmulti;
        }
        x0 += W[i];
      }
      if (!ok) continue;
      bool skel_out = false;
      int emitted = 0;  // PUSH depths already written for the current path
      if (nl == 0) {    // the skeleton is one candidate
        out.skel(0);
        for (int i = 0; i < nfix; ++i) out.fix(FIXI[i], FIXT[i]);
        out.leaf(0, 0);
        continue;
      }
      // heights DFS over the decision runs; depth nl-1 is the leaf
      int t = 0;
      AMIN[0] = amin;
      AMAX[0] = amax;
      Y0[0] = 0;
      H[0] = 0;
      while (t >= 0) {
        const int w = Dw[t], left = Dleft[t], y0 = Y0[t];
        const int rl = rows - y0;
        const int hmax = rl - (left - 1);  // leave one row per later run of the column
        if (t < nl - 1) {
          int h = ++H[t];
          if (h > hmax) {
            --t;
            if (t >= 0 && emitted > t) emitted = t;
            continue;
          }
          int na = AMIN[t] < w * h ? AMIN[t] : w * h, nx = AMAX[t] > w * h ? AMAX[t] : w * h;
          if (left == 2) {  // the forced rest of the column
            const int a2 = w * (rl - h);
            na = a2 < na ? a2 : na;
            nx = a2 > nx ? a2 : nx;
          }
          if (emitted > t) emitted = t;
          if (!(k * (double)na > (double)nx)) continue;
          AMIN[t + 1] = na;
          AMAX[t + 1] = nx;
          Y0[t + 1] = left == 2 ? 0 : y0 + h;
          H[t + 1] = 0;
          ++t;
          continue;
        }
        // leaf: the column's second-to-last run takes every admissible height;
        // maximal runs of consecutive heights become one LEAF op each
        const uint32_t base = (uint32_t)(tr_xw(cols, Dx0[t], w) * nyh + tr_yh(rows, y0, 1));
        int h = 1;
        while (h <= rl - 1) {
          int h0 = -1;
          for (; h <= rl - 1; ++h) {
            const int a1 = w * h, a2 = w * (rl - h);
            const int na = AMIN[t] < (a1 < a2 ? a1 : a2) ? AMIN[t] : (a1 < a2 ? a1 : a2);
            const int nx = AMAX[t] > (a1 > a2 ? a1 : a2) ? AMAX[t] : (a1 > a2 ? a1 : a2);
            const bool adm = k * (double)na > (double)nx;
            if (adm && h0 < 0) h0 = h;
            if (!adm && h0 >= 0) break;
          }
          if (h0 < 0) break;
          if (!skel_out) {
            out.skel(nl - 1);
            for (int i = 0; i < nfix; ++i) out.fix(FIXI[i], FIXT[i]);
            skel_out = true;
            emitted = 0;
          }
          for (int dd = emitted; dd < nl - 1; ++dd)
            out.push(dd,
                     (Dleft[dd] == 2 ? nr : 0u) + (uint32_t)(tr_xw(cols, Dx0[dd], Dw[dd]) * nyh +
                                                             tr_yh(rows, Y0[dd], H[dd])),
                     dd == nl - 2);
          emitted = nl - 1;
          // h - h0 <= rows - 2 <= 253 heights, kTrLeafMax per LEAF op
          uint32_t lk = nr + base + (uint32_t)(h0 - 1);
          int left_h = h - h0;
          for (; left_h > kTrLeafMax; left_h -= kTrLeafMax, lk += kTrLeafMax)
            out.leaf(lk, kTrLeafMax);
          out.leaf(lk, left_h);
        }
        --t;
      }
    }
    if (fixed) break;
  }
}

// The layout of one candidate from its skeleton's one-run columns (fixes,
// rectangle indices), its decision path (path[0..ld-1]: the rectangle index
// of each PUSH) and its leaf run (leaf: rectangle index, or ~0u for a
// skeleton without decision runs).  Writes the 96-byte snapshot W[16] R[16]
// H[64] of search.cu (columns by x, runs column-major).
SCB_TR_HD void trace_snapshot(const uint32_t* fixes, int nfix, const uint32_t* path, int ld,
                              uint32_t leaf, int cols, int rows, uint8_t* snap) {
  const int nyh = rows * (rows + 1) / 2;
  auto decode = [&](uint32_t idx, int& x0, int& w, int& y0, int& h) {
    const int xw = (int)(idx / (uint32_t)nyh), yh = (int)(idx % (uint32_t)nyh);
    tr_unrank(cols, xw, x0, w);
    tr_unrank(rows, yh, y0, h);
  };
  int cx0[SC_MAX_COLS], cw[SC_MAX_COLS], cr[SC_MAX_COLS], cs[SC_MAX_COLS], nc = 0;
  uint8_t hh[SC_MAX_SLICES];  // heights in path order, then re-ordered by column
  int hcol[SC_MAX_SLICES], nh = 0;
  for (int i = 0; i < nfix; ++i) {
    int x0, w, y0, h;
    decode(fixes[i], x0, w, y0, h);
    cx0[nc] = x0, cw[nc] = w, cr[nc] = 1;
    hcol[nh] = nc, hh[nh++] = (uint8_t)rows;
    ++nc;
  }
  if (leaf != ~0u) {
    for (int dd = 0; dd <= ld; ++dd) {
      int x0, w, y0, h;
      decode(dd == ld ? leaf : path[dd], x0, w, y0, h);
      int col = -1;
      for (int i = 0; i < nc; ++i)
        if (cx0[i] == x0) col = i;
      if (col < 0) {
        col = nc++;
        cx0[col] = x0, cw[col] = w, cr[col] = 0;
      }
      ++cr[col];
      hcol[nh] = col, hh[nh++] = (uint8_t)h;
      // the column's second-to-last run (the leaf, or a PUSH whose next
      // decision run is in another column): its forced rest follows
      bool closes = dd == ld;
      if (!closes) {
        int nx0, nw, ny0, nhh;
        decode(dd + 1 == ld ? leaf : path[dd + 1], nx0, nw, ny0, nhh);
        closes = nx0 != x0;
      }
      if (closes) {
        ++cr[col];
        hcol[nh] = col, hh[nh++] = (uint8_t)(rows - y0 - h);
      }
    }
  }
  // columns by x; a column's runs keep their path order (top to bottom)
  for (int i = 0; i < nc; ++i) cs[i] = i;
  for (int i = 0; i < nc; ++i)
    for (int j = i + 1; j < nc; ++j)
      if (cx0[cs[j]] < cx0[cs[i]]) {
        const int t = cs[i];
        cs[i] = cs[j];
        cs[j] = t;
      }
  int run = 0;
  for (int i = 0; i < SC_MAX_COLS; ++i) {
    snap[i] = (uint8_t)(i < nc ? cw[cs[i]] : 0);
    snap[SC_MAX_COLS + i] = (uint8_t)(i < nc ? cr[cs[i]] : 0);
    if (i < nc)
      for (int q = 0; q < nh; ++q)
        if (hcol[q] == cs[i]) snap[2 * SC_MAX_COLS + run++] = hh[q];
  }
  for (; run < SC_MAX_SLICES; ++run) snap[2 * SC_MAX_COLS + run] = 0;
}

// Sequential replay of one skeleton's ops (host emulator; the device uses a
// warp-parallel replay in trace.cu): the candidate at position `which`.
SCB_TR_HD bool trace_layout(const uint32_t* ops, uint64_t nops, uint64_t which, int cols, int rows,
                            int n, uint8_t* snap) {
  const int nyh = rows * (rows + 1) / 2;
  const uint32_t nr = (uint32_t)(cols * (cols + 1) / 2 * nyh);
  uint32_t path[SC_MAX_SLICES];
  uint32_t fixes[SC_MAX_COLS];
  int nfix = 0, ld = 0;
  uint64_t seen = 0;
  (void)n;
  for (uint64_t p = 0; p < nops; ++p) {
    const uint32_t op = ops[p];
    if (tr_code(op) == kOpSkel) {
      if (tr_is_fix(op)) fixes[nfix++] = tr_kidx(op);
      else if (p == 0) ld = tr_skel_ld(op);
      else return false;  // next skeleton: `which` was not in this one
      continue;
    }
    if (tr_is_push(op)) {
      const uint32_t kidx = tr_kidx(op);
      path[tr_small_of(op)] = kidx >= nr ? kidx - nr : kidx;
      continue;
    }
    const int cnt = tr_leaf_cnt(op);
    const uint64_t m = cnt ? (uint64_t)cnt : 1u;
    if (which >= seen + m) {
      seen += m;
      continue;
    }
    trace_snapshot(fixes, nfix, path, ld, cnt ? tr_kidx(op) - nr + (uint32_t)(which - seen) : ~0u,
                   cols, rows, snap);
    return true;
  }
  return false;
}

}  // namespace scb
