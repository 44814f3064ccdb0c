"""Python mirror of the reference partitioner API (proj/include/slicecraft).

Same names, argument meaning and error behaviour as the reference C++ API, so
the parity tests read like the reference's own (absent) tests:

  texture map         ctu_stats                       texture.hpp:83
  CTU-complexity      temporal_layer_of_poc,          cost.hpp:39
                      CostHistory.append,              cost.hpp:43-58
                      estimate_ctu_times              cost.hpp:64
  partition search    min_time_search,                search.hpp:66-67
                      constrained_clustering_search,  search.hpp:72-75
                      two_step_partition              search.hpp:80-82

Every compute call goes through the C-ABI (include/slicecraft_b200.h) into the
sm_100a kernels; the host-side pieces here are the O(cells) cost-history
bookkeeping the reference also keeps on the host (cost.cpp:56-95).
Errors surface as SlicecraftError whose ``kind`` names the reference class.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._abi import (ALLGATHER_FN, SC_COMM_ID_BYTES, SC_ORIGIN_UNIFORM, CtuRecord, Grid, Layout,
                   PartitionC, PartitionStats, Rect, SearchCfg, SearchResult, ShardBest,
                   SlicecraftError, check, lib)

COLUMN_SPLIT, UNIFORM_ONLY = 0, 1
COVERAGE_REFERENCE, COVERAGE_COVERING = 0, 1
MODE_EXHAUSTIVE, MODE_PRUNED = 0, 1

RECORD_DTYPE = np.dtype([("count", "<u8"), ("sum", "<u8"), ("sumsq", "<u8")])


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


@dataclass(frozen=True)
class CtuGrid:
    """CtuGrid (grid.hpp:13-34); build with CtuGrid.make."""
    frame_width: int
    frame_height: int
    ctu_size: int
    cols: int
    rows: int

    @staticmethod
    def make(frame_width: int, frame_height: int, ctu_size: int = 128) -> "CtuGrid":
        g = Grid()
        check(lib().sc_grid_make(frame_width, frame_height, ctu_size, C.byref(g)))
        return CtuGrid(g.frame_width, g.frame_height, g.ctu_size, g.cols, g.rows)

    def cell_count(self) -> int:
        return self.cols * self.rows

    def c(self) -> Grid:
        return Grid(self.frame_width, self.frame_height, self.ctu_size, self.cols, self.rows)

    @property
    def n_rects(self) -> int:
        return self.cols * (self.cols + 1) // 2 * (self.rows * (self.rows + 1) // 2)


@dataclass
class SearchConfig:
    """SearchConfig (search.hpp:22-34) + coverage / mode (B200 additions)."""
    n_slices: int = 4
    lambda_: float = 0.0
    k_area: float = 3.0
    family: int = COLUMN_SPLIT
    max_tile_cols: int = 0
    workers: int = 1
    coverage: int = COVERAGE_REFERENCE
    mode: int = MODE_EXHAUSTIVE

    def c(self) -> SearchCfg:
        return SearchCfg(self.n_slices, self.lambda_, self.k_area, self.family,
                         self.max_tile_cols, self.workers, self.coverage, self.mode)


def temporal_layer_of_poc(poc: int, gop_size: int) -> int:
    out = C.c_int32()
    check(lib().sc_temporal_layer(poc, gop_size, C.byref(out)))
    return out.value


# CostSource (cost.hpp:11-16)
MEASURED, CO_TEMPORAL_LAYER, MOST_RECENT_ANY, UNIFORM = 0, 1, 2, 3


@dataclass
class CostMap:
    """CostMap (cost.hpp:21-34): per-CTU times in microseconds, row-major."""
    grid: CtuGrid
    times_us: np.ndarray
    poc: int = 0
    temporal_layer: int = 0
    qp: int = 0
    source: int = MEASURED
    source_poc: int = -1


class CostHistory:
    """CostHistory (cost.hpp:43-58; append validation cost.cpp:56-75)."""

    def __init__(self, grid: CtuGrid, gop_size: int = 16):
        temporal_layer_of_poc(0, gop_size)  # validates the GOP eagerly
        self.grid = grid
        self.gop_size = gop_size
        self.maps: List[CostMap] = []

    def append(self, m: CostMap) -> None:
        """CostHistory::append: validated by sc_cost_map_check (cost.cpp:45-64)."""
        t = np.ascontiguousarray(m.times_us, dtype=np.float64).reshape(-1)
        pocs = np.array([x.poc for x in self.maps], dtype=np.int32)
        check(lib().sc_cost_map_check(C.byref(self.grid.c()), C.byref(m.grid.c()), _ptr(t),
                                      t.size, m.poc, _ptr(pocs), len(pocs)))
        m.times_us = t
        self.maps.append(m)


def estimate_ctu_times(history: CostHistory, poc: int) -> CostMap:
    """estimate_ctu_times (cost.cpp:66-95) via sc_estimate_ctu_times: co-TL,
    else most recent, else ones."""
    n = len(history.maps)
    arrs = [np.ascontiguousarray(m.times_us, dtype=np.float64) for m in history.maps]
    ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
    pocs = np.array([m.poc for m in history.maps], dtype=np.int32)
    tls = np.array([m.temporal_layer for m in history.maps], dtype=np.int32)
    out = np.empty(history.grid.cell_count())
    src, src_poc, tl = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().sc_estimate_ctu_times(C.byref(history.grid.c()), history.gop_size, n,
                                      C.cast(ptrs, C.c_void_p), _ptr(pocs), _ptr(tls), poc,
                                      _ptr(out), C.byref(src), C.byref(src_poc), C.byref(tl)))
    qp = next((m.qp for m in history.maps if m.poc == src_poc.value), 0) if n else 0
    return CostMap(history.grid, out, poc, tl.value, qp, src.value, src_poc.value)


class PrefixSumTable:
    """PrefixSumTable (cost.hpp:67-89) built by sc_prefix_sum_table."""

    def __init__(self, values, cols: int, rows: int):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        self.cols, self.rows = cols, rows
        self.table = np.empty((rows + 1) * (cols + 1))
        check(lib().sc_prefix_sum_table(_ptr(v), v.size, cols, rows, _ptr(self.table)))

    def rect_sum(self, x0: int, y0: int, w: int, h: int) -> float:
        s, t = self.cols + 1, self.table
        return ((t[(y0 + h) * s + x0 + w] - t[y0 * s + x0 + w]) - t[(y0 + h) * s + x0]) + \
            t[y0 * s + x0]


def split_even(total: int, parts: int) -> List[int]:
    """split_even (grid.cpp:52-60)."""
    out = (C.c_int32 * max(parts, 1))()
    check(lib().sc_split_even(total, parts, out))
    return list(out[:parts])


def moments_sse(count: int, sum_: int, sumsq: int) -> float:
    """SliceMoments::sse (texture.cpp:83-88)."""
    out = C.c_double()
    check(lib().sc_moments_sse(C.byref(CtuRecord(count, sum_, sumsq)), C.byref(out)))
    return out.value


def texture_tables(grid: CtuGrid, records: np.ndarray):
    """TextureStats ctor (texture.cpp:90-130): validation + the three u64 SATs."""
    rec = np.ascontiguousarray(records)
    n = (grid.cols + 1) * (grid.rows + 1)
    tabs = [np.empty(n, np.uint64) for _ in range(3)]
    check(lib().sc_texture_tables(C.byref(grid.c()), _ptr(rec), rec.shape[0] if rec.ndim else 0,
                                  *[_ptr(t) for t in tabs]))
    return tabs


@dataclass
class TextureStats:
    """TextureStats (texture.hpp:54-79): per-CTU records of one frame."""
    grid: CtuGrid
    records: np.ndarray  # RECORD_DTYPE, cols*rows
    poc: int = 0


@dataclass
class Slice:
    x0: int
    y0: int
    w: int
    h: int
    id: int


@dataclass
class Partition:
    """Partition (grid.hpp:62-71) as produced by layout_to_partition (search.cpp:63-75)."""
    grid: CtuGrid
    col_widths: List[int]
    row_heights: List[int]
    slices: List[Slice] = field(default_factory=list)
    origin: str = "proposed"  # PartitionOrigin (grid.hpp:70)

    @staticmethod
    def from_layout(grid: CtuGrid, L: Layout) -> "Partition":
        p = Partition(grid, [L.col_widths[i] for i in range(L.n_cols)], [grid.rows])
        x, run, sid = 0, 0, 0
        for col in range(L.n_cols):
            w = L.col_widths[col]
            y = 0
            for _ in range(L.runs_per_col[col]):
                h = L.run_heights[run]
                p.slices.append(Slice(x, y, w, h, sid))
                sid += 1
                run += 1
                y += h
            x += w
        return p

    @staticmethod
    def uniform(grid: CtuGrid, n_slices: int) -> "Partition":
        """uniform_partition (grid.cpp:186-262) via sc_uniform_partition."""
        out = PartitionC()
        check(lib().sc_uniform_partition(C.byref(grid.c()), n_slices, C.byref(out)))
        p = Partition(grid, [out.tile_col_widths[i] for i in range(out.n_tile_cols)],
                      [out.tile_row_heights[i] for i in range(out.n_tile_rows)])
        p.slices = [Slice(r.x0, r.y0, r.w, r.h, r.id) for r in out.slices[:out.n_slices]]
        p.origin = "uniform"
        return p

    @staticmethod
    def from_result(grid: CtuGrid, r: SearchResult, L: Layout) -> "Partition":
        if r.origin == SC_ORIGIN_UNIFORM:
            return Partition.uniform(grid, L.n_slices)
        return Partition.from_layout(grid, L)

    def rects(self):
        return [(s.x0, s.y0, s.w, s.h, s.id) for s in self.slices]


@dataclass
class SearchOutcome:
    """SearchOutcome (search.hpp:36-49) + the step-1 argmin."""
    best: Optional[Partition]
    argmin: Optional[Partition]
    t_min_us: float
    t_best_us: float
    sse_best: float
    candidates_evaluated: int
    candidates_step1: int
    candidates_step2: int
    search_time_us: float
    time_min_step_us: float
    clustering_step_us: float
    leaves_scored_step1: int = 0
    leaves_scored_step2: int = 0
    est_source: int = UNIFORM
    est_source_poc: int = -1


def _outcome(grid: CtuGrid, r: SearchResult, step1: bool, step2: bool) -> SearchOutcome:
    return SearchOutcome(
        best=Partition.from_result(grid, r, r.best) if step2 else None,
        argmin=Partition.from_result(grid, r, r.argmin) if step1 else None,
        t_min_us=r.t_min_us, t_best_us=r.t_best_us, sse_best=r.sse_best,
        candidates_evaluated=r.candidates_evaluated, candidates_step1=r.candidates_step1,
        candidates_step2=r.candidates_step2, search_time_us=r.search_time_us,
        time_min_step_us=r.time_min_step_us, clustering_step_us=r.clustering_step_us,
        leaves_scored_step1=r.leaves_scored_step1, leaves_scored_step2=r.leaves_scored_step2)


class Partitioner:
    """One device context (sc_ctx) with the partitioner entry points."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().sc_ctx_create(device, C.byref(self._h)))

    def close(self) -> None:
        if self._h:
            lib().sc_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_shard(self, rank: int, world: int) -> None:
        check(lib().sc_ctx_set_shard(self._h, rank, world))

    def comm_init_nccl(self, rank: int, world: int, unique_id: bytes) -> None:
        """Shard over `world` GPUs with the library's own NCCL exchange
        (sc_comm_init_nccl): every search call returns the merged results."""
        buf = (C.c_uint8 * SC_COMM_ID_BYTES).from_buffer_copy(unique_id)
        check(lib().sc_comm_init_nccl(self._h, rank, world, C.cast(buf, C.c_void_p)))

    def comm_init_callback(self, rank: int, world: int, allgather) -> None:
        """Shard with a host transport: allgather(send: bytes) -> bytes
        (world * len(send), rank order), e.g. torch.distributed gloo."""
        def fn(_user, send, nbytes, recv):
            try:
                got = allgather(C.string_at(send, nbytes))
                C.memmove(recv, got, len(got))
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failure
                return 1
        self._comm_fn = ALLGATHER_FN(fn)  # keep the trampoline alive
        check(lib().sc_comm_init_callback(self._h, rank, world, self._comm_fn, None))

    def comm_detach(self) -> None:
        check(lib().sc_comm_detach(self._h))


    # ---- texture map --------------------------------------------------------
    def timings(self) -> dict:
        """Device time (us, CUDA events) of the phases of the last search call."""
        t = (C.c_double * 5)()
        check(lib().sc_ctx_timings(self._h, t))
        return dict(zip(("texture", "tables", "step1", "step2", "total"), list(t)))

    def ctu_stats_batch(self, frames: np.ndarray, ctu_size: int = 128) -> np.ndarray:
        """K1 over a [F, H, W] uint8/uint16 array (host numpy or any array
        exposing ``data_ptr``/``ctypes``); returns [F, rows*cols] records."""
        if frames.ndim == 2:
            frames = frames[None]
        F, H, W = frames.shape
        bps = frames.dtype.itemsize
        if frames.dtype not in (np.uint8, np.uint16):
            raise SlicecraftError(7, "luma must be uint8 or uint16")
        frames = np.ascontiguousarray(frames)
        g = CtuGrid.make(W, H, ctu_size)
        out = np.zeros((F, g.cell_count()), dtype=RECORD_DTYPE)
        check(lib().sc_texture_moments(self._h, _ptr(frames), bps, W, H, W * bps, W * H * bps,
                                       ctu_size, F, _ptr(out)))
        return out

    def ctu_stats(self, luma: np.ndarray, grid: CtuGrid, poc: int = 0) -> TextureStats:
        """ctu_stats (texture.cpp:145-169)."""
        if luma.shape != (grid.frame_height, grid.frame_width):
            raise SlicecraftError(1, "plane dimensions do not match the grid")
        return TextureStats(grid, self.ctu_stats_batch(luma, grid.ctu_size)[0], poc)

    def grid_tables(self, grid: CtuGrid, est: np.ndarray, records: Optional[np.ndarray] = None):
        """K2/K3: per-rectangle times (and SSEs) for F frames, rectangle order
        xw(x0,w)*NYH + yh(y0,h).  Returns (rect_time, rect_sse, sat)."""
        est = np.ascontiguousarray(est, dtype=np.float64).reshape(-1, grid.cell_count())
        F = est.shape[0]
        nr = grid.n_rects
        rt = np.zeros((F, nr))
        rs = np.zeros((F, nr)) if records is not None else None
        sat = np.zeros((F, (grid.cols + 1) * (grid.rows + 1)))
        rec = None if records is None else np.ascontiguousarray(records).reshape(F, -1)
        check(lib().sc_grid_tables(self._h, C.byref(grid.c()), _ptr(est), _ptr(rec), F, _ptr(rt),
                                   _ptr(rs), _ptr(sat)))
        return rt, rs, sat

    # ---- partition search ---------------------------------------------------
    def min_time_search_batch(self, grid: CtuGrid, est: np.ndarray, cfg: SearchConfig):
        est = np.ascontiguousarray(est, dtype=np.float64).reshape(-1, grid.cell_count())
        F = est.shape[0]
        res = (SearchResult * F)()
        check(lib().sc_min_time_search(self._h, C.byref(grid.c()), C.byref(cfg.c()), _ptr(est),
                                       F, C.cast(res, C.c_void_p)))
        return [_outcome(grid, r, True, False) for r in res]

    def min_time_search(self, est: CostMap, cfg: SearchConfig):
        """min_time_search (search.cpp:328-332) -> (t_min, argmin Partition)."""
        o = self.min_time_search_batch(est.grid, est.times_us, cfg)[0]
        return o.t_min_us, o.argmin

    def constrained_clustering_batch(self, grid: CtuGrid, est: np.ndarray, records: np.ndarray,
                                     t_min: Sequence[float], cfg: SearchConfig):
        est = np.ascontiguousarray(est, dtype=np.float64).reshape(-1, grid.cell_count())
        F = est.shape[0]
        rec = np.ascontiguousarray(records).reshape(F, -1)
        tm = np.ascontiguousarray(np.asarray(t_min, dtype=np.float64).reshape(F))
        res = (SearchResult * F)()
        check(lib().sc_constrained_clustering(self._h, C.byref(grid.c()), C.byref(cfg.c()),
                                              _ptr(est), _ptr(rec), _ptr(tm), F,
                                              C.cast(res, C.c_void_p)))
        return [_outcome(grid, r, False, True) for r in res]

    def constrained_clustering_search(self, est: CostMap, stats: TextureStats, t_min_us: float,
                                      cfg: SearchConfig) -> SearchOutcome:
        """constrained_clustering_search (search.cpp:334-405)."""
        if stats.grid != est.grid:
            raise SlicecraftError(1, "texture stats grid does not match the cost map grid")
        return self.constrained_clustering_batch(est.grid, est.times_us, stats.records,
                                                 [t_min_us], cfg)[0]

    def two_step_batch(self, grid: CtuGrid, est: np.ndarray, records: np.ndarray,
                       cfg: SearchConfig):
        est = np.ascontiguousarray(est, dtype=np.float64).reshape(-1, grid.cell_count())
        F = est.shape[0]
        rec = np.ascontiguousarray(records).reshape(F, -1)
        res = (SearchResult * F)()
        check(lib().sc_two_step(self._h, C.byref(grid.c()), C.byref(cfg.c()), _ptr(est),
                                _ptr(rec), F, C.cast(res, C.c_void_p)))
        return [_outcome(grid, r, True, True) for r in res]

    def two_step_partition(self, history: CostHistory, stats: TextureStats, poc: int,
                           cfg: SearchConfig) -> SearchOutcome:
        """two_step_partition (search.cpp:407-434)."""
        if stats.grid != history.grid:
            raise SlicecraftError(1, "texture stats grid does not match the history grid")
        est = estimate_ctu_times(history, poc)
        o = self.two_step_batch(history.grid, est.times_us, stats.records, cfg)[0]
        o.est_source, o.est_source_poc = est.source, est.source_poc
        return o

    def partition_frames(self, grid: CtuGrid, luma: np.ndarray, est: np.ndarray,
                         cfg: SearchConfig, records_out: Optional[np.ndarray] = None):
        """Whole hot path for a batch: K1 -> K2/K3 -> step 1 -> step 2."""
        F = est.shape[0]
        bps = luma.dtype.itemsize
        est = np.ascontiguousarray(est, dtype=np.float64)
        res = (SearchResult * F)()
        W, H = grid.frame_width, grid.frame_height
        check(lib().sc_partition_frames(self._h, C.byref(grid.c()), C.byref(cfg.c()),
                                        _ptr(luma), bps, W * bps, W * H * bps, _ptr(est), F,
                                        _ptr(records_out), C.cast(res, C.c_void_p)))
        return res

    def partition_eval(self, p: "Partition", est: Optional[np.ndarray] = None,
                       records: Optional[np.ndarray] = None, slice_values: bool = False):
        """partition_time (cost.cpp:117-145) and partition_sse / slice_moments
        (texture.cpp:171-189) of one partition on a batch of frames, on the
        device.  Returns a list of dicts (max_us, total_us, argmax, sse) and,
        with slice_values, the per-slice times [F][n] and moments [F][n]."""
        g = p.grid
        n = len(p.slices)
        rects = (Rect * n)(*[Rect(s.x0, s.y0, s.w, s.h, s.id) for s in p.slices])
        e = None if est is None else np.ascontiguousarray(est, dtype=np.float64).reshape(
            -1, g.cell_count())
        r = None if records is None else np.ascontiguousarray(records).reshape(-1, g.cell_count())
        F = (e if e is not None else r).shape[0]
        out = (PartitionStats * F)()
        st = np.zeros((F, n)) if slice_values and e is not None else None
        sm = np.zeros((F, n), RECORD_DTYPE) if slice_values and r is not None else None
        check(lib().sc_partition_eval(self._h, C.byref(g.c()), C.cast(rects, C.c_void_p), n,
                                      _ptr(e), _ptr(r), F, C.cast(out, C.c_void_p), _ptr(st),
                                      _ptr(sm)))
        res = [dict(max_us=o.max_us, total_us=o.total_us, argmax=o.argmax, sse=o.sse)
               for o in out]
        return (res, st, sm) if slice_values else res

    def ctu_stats_yuv(self, path: str, grid: CtuGrid, bit_depth: int, first_poc: int = 0,
                      n_frames: int = 1) -> np.ndarray:
        """K1 straight from a planar 4:2:0 file: luma planes only, no widening."""
        out = np.zeros((n_frames, grid.cell_count()), RECORD_DTYPE)
        check(lib().sc_yuv_texture_moments(self._h, path.encode(), grid.frame_width,
                                           grid.frame_height, bit_depth, grid.ctu_size, first_poc,
                                           n_frames, _ptr(out)))
        return out

    def partition_yuv(self, grid: CtuGrid, path: str, bit_depth: int, first_poc: int,
                      est: np.ndarray, cfg: SearchConfig, records_out: Optional[np.ndarray] = None):
        """partition_frames over frames [first_poc, first_poc + len(est)) of a YUV file."""
        est = np.ascontiguousarray(est, dtype=np.float64).reshape(-1, grid.cell_count())
        F = est.shape[0]
        res = (SearchResult * F)()
        check(lib().sc_partition_yuv(self._h, C.byref(grid.c()), C.byref(cfg.c()), path.encode(),
                                     bit_depth, first_poc, F, _ptr(est), _ptr(records_out),
                                     C.cast(res, C.c_void_p)))
        return res

    def validate_partition(self, grid: CtuGrid, col_widths: Sequence[int],
                           row_heights: Sequence[int], slices: Sequence[Slice]) -> np.ndarray:
        """validate_partition (grid.cpp:86-184) on the device; returns the
        CTU -> slice-id map (rows x cols)."""
        cw = np.ascontiguousarray(col_widths, dtype=np.int32)
        rh = np.ascontiguousarray(row_heights, dtype=np.int32)
        n = len(slices)
        rects = (Rect * max(n, 1))(*[Rect(q.x0, q.y0, q.w, q.h, q.id) for q in slices])
        out = np.empty((grid.rows, grid.cols), np.int32)
        check(lib().sc_validate_partition(self._h, C.byref(grid.c()), len(cw), _ptr(cw), len(rh),
                                          _ptr(rh), C.cast(rects, C.c_void_p), n, _ptr(out)))
        return out

    def result_slice_maps(self, grid: CtuGrid, step: int, frames: int) -> np.ndarray:
        """CTU -> slice-id maps [F, rows, cols] of the last search's argmin
        (step 1) / best (step 2) partitions (-1 outside the layout's columns)."""
        out = np.empty((frames, grid.rows, grid.cols), np.int32)
        check(lib().sc_result_slice_maps(self._h, step, frames, _ptr(out)))
        return out

    def enumerate_layouts(self, grid: CtuGrid, cfg: SearchConfig, first: int = 0,
                          max_out: int = 1 << 16):
        """A window of the family's candidate stream (search.cpp:302-326) as
        layouts: (layouts, total)."""
        buf = (Layout * max(max_out, 1))()
        n, tot = C.c_uint64(), C.c_uint64()
        check(lib().sc_enumerate_candidates(self._h, C.byref(grid.c()), C.byref(cfg.c()), first,
                                            max_out, C.cast(buf, C.c_void_p), C.byref(n),
                                            C.byref(tot)))
        return list(buf[:n.value]), tot.value

    def for_each_candidate(self, grid: CtuGrid, cfg: SearchConfig, sink, page: int = 1 << 16):
        """for_each_candidate (search.cpp:302-320): every admissible candidate
        in enumeration order, as a Partition, through `sink`."""
        first = 0
        while True:
            lays, tot = self.enumerate_layouts(grid, cfg, first, page)
            for L in lays:
                sink(Partition.uniform(grid, cfg.n_slices) if L.n_cols == 0
                     else Partition.from_layout(grid, L))
            first += len(lays)
            if first >= tot or not lays:
                return

    def enumerate_candidates(self, grid: CtuGrid, cfg: SearchConfig) -> List["Partition"]:
        """enumerate_candidates (search.cpp:322-326)."""
        out: List[Partition] = []
        self.for_each_candidate(grid, cfg, out.append)
        return out

    def count_candidates(self, grid: CtuGrid, cfg: SearchConfig) -> int:
        n = C.c_uint64()
        check(lib().sc_count_candidates(self._h, C.byref(grid.c()), C.byref(cfg.c()), C.byref(n)))
        return n.value

    def shard_export(self, step: int, frames: int):
        out = (ShardBest * frames)()
        check(lib().sc_shard_export(self._h, step, frames, C.cast(out, C.c_void_p)))
        return out


def shard_merge(step: int, world: int, frames: int, gathered: bytes, results) -> None:
    """sc_shard_merge over rank-major gathered ShardBest records."""
    buf = (ShardBest * (world * frames)).from_buffer_copy(gathered)
    check(lib().sc_shard_merge(step, world, frames, C.cast(buf, C.c_void_p),
                               C.cast(results, C.c_void_p)))


def yuv_frame_count(path: str, width: int, height: int, bit_depth: int) -> int:
    """yuv_frame_count (texture.cpp:25-40)."""
    n = C.c_int32()
    check(lib().sc_yuv_frame_count(path.encode(), width, height, bit_depth, C.byref(n)))
    return n.value


def load_yuv_frame(path: str, width: int, height: int, poc: int, bit_depth: int) -> np.ndarray:
    """load_yuv_frame (texture.cpp:42-81): the luma plane widened to uint16."""
    out = np.empty((height, width), np.uint16)
    check(lib().sc_yuv_load_luma(path.encode(), width, height, poc, bit_depth, _ptr(out)))
    return out


def read_yuv_luma(path: str, width: int, height: int, bit_depth: int, first_poc: int,
                  n_frames: int) -> np.ndarray:
    """Raw luma planes (uint8, or uint16 for 10-bit) of consecutive frames."""
    out = np.empty((n_frames, height, width), np.uint8 if bit_depth == 8 else np.uint16)
    check(lib().sc_yuv_read_luma(path.encode(), width, height, bit_depth, first_poc, n_frames,
                                 _ptr(out)))
    return out


def texture_validate(grid: CtuGrid, records: np.ndarray) -> None:
    rec = np.ascontiguousarray(records)
    check(lib().sc_texture_validate(C.byref(grid.c()), _ptr(rec)))


def comm_unique_id() -> bytes:
    """An NCCL unique id for sc_comm_init_nccl (rank 0 makes it, all ranks use it)."""
    buf = (C.c_uint8 * SC_COMM_ID_BYTES)()
    check(lib().sc_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)
