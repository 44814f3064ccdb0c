"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the CPU oracle.

* ``Oracle``  — liboracle.so, the plain-C restatement (sc_oracle.c).  Travels
  to the GPU box; the GPU parity tests check the CUDA path against it.
* ``Ref``     — _ref/libslicecraft_ref.so, the UNMODIFIED reference compiled
  in place + ref_shim.cpp.  Built only where /root/reference exists; used to
  pin the oracle and to generate tests/golden fixtures.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libslicecraft_ref.so")

ORC_MAX_COLS = 64
ORC_MAX_SLICES = 128


class OrcLayout(C.Structure):
    _fields_ = [("n_cols", C.c_int32), ("col_widths", C.c_int32 * ORC_MAX_COLS),
                ("runs_per_col", C.c_int32 * ORC_MAX_COLS),
                ("run_heights", C.c_int32 * ORC_MAX_SLICES)]

    def slices(self, rows):
        out, x, run, sid = [], 0, 0, 0
        for c in range(self.n_cols):
            y = 0
            for _ in range(self.runs_per_col[c]):
                h = self.run_heights[run]
                out.append((x, y, self.col_widths[c], h, sid))
                sid += 1
                run += 1
                y += h
            x += self.col_widths[c]
        return out


class OrcResult(C.Structure):
    _fields_ = [("t_min_us", C.c_double), ("candidates_step1", C.c_uint64),
                ("argmin1", OrcLayout), ("t_best_us", C.c_double), ("sse_best", C.c_double),
                ("candidates_step2", C.c_uint64), ("best", OrcLayout)]


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        self.L = C.CDLL(path)

    def ctu_stats(self, plane: np.ndarray, ctu: int = 128) -> np.ndarray:
        H, W = plane.shape
        plane = np.ascontiguousarray(plane)
        bps = plane.dtype.itemsize
        cols, rows = -(-W // ctu), -(-H // ctu)
        out = np.zeros(cols * rows * 3, dtype=np.uint64)
        st = self.L.orc_ctu_stats(_p(plane), bps, W, H, C.c_size_t(W * bps), ctu, _p(out))
        if st:
            raise RuntimeError(f"oracle status {st}")
        return out.reshape(-1, 3)

    def rect_times(self, times: np.ndarray, cols: int, rows: int) -> np.ndarray:
        t = np.ascontiguousarray(times, dtype=np.float64)
        out = np.zeros(cols * (cols + 1) // 2 * (rows * (rows + 1) // 2))
        self.L.orc_rect_times(_p(t), cols, rows, _p(out))
        return out

    def rect_sse(self, fw, fh, ctu, records) -> np.ndarray:
        cols, rows = -(-fw // ctu), -(-fh // ctu)
        rec = np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        out = np.zeros(cols * (cols + 1) // 2 * (rows * (rows + 1) // 2))
        st = self.L.orc_rect_sse(fw, fh, ctu, _p(rec), _p(out))
        if st:
            raise RuntimeError(f"oracle status {st}")
        return out

    def search(self, fw, fh, ctu, est, records, n, lam=0.0, k=3.0, max_cols=0, coverage=0,
               step=3, t_min=0.0):
        r = OrcResult()
        e = np.ascontiguousarray(est, dtype=np.float64)
        rec = None if records is None else np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        self.L.orc_search.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                      C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                      C.c_double, C.c_void_p]
        st = self.L.orc_search(fw, fh, ctu, _p(e), _p(rec), n, lam, k, max_cols, coverage, step,
                               t_min, C.byref(r))
        return st, r

    def search_pruned(self, fw, fh, ctu, est, records, n, lam=0.0, k=3.0, max_cols=0,
                      coverage=0, step=3, t_min=0.0):
        """Independent branch-and-bound restatement (counts not enumerated)."""
        r = OrcResult()
        e = np.ascontiguousarray(est, dtype=np.float64)
        rec = None if records is None else np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        self.L.orc_search_pruned.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                             C.c_int, C.c_double, C.c_void_p]
        st = self.L.orc_search_pruned(fw, fh, ctu, _p(e), _p(rec), n, lam, k, max_cols, coverage,
                                      step, t_min, C.byref(r))
        return st, r

    def count(self, cols, rows, n, k=3.0, max_cols=0, coverage=0) -> int:
        out = C.c_uint64()
        self.L.orc_count.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                     C.c_void_p]
        self.L.orc_count(cols, rows, n, k, max_cols, coverage, C.byref(out))
        return out.value


class RefLayout(C.Structure):
    _fields_ = [("n_cols", C.c_int32), ("n_slices", C.c_int32),
                ("col_widths", C.c_int32 * 64), ("row_heights", C.c_int32 * 64),
                ("n_tile_rows", C.c_int32), ("slices", (C.c_int32 * 5) * 128)]

    def rects(self):
        return [tuple(self.slices[i][j] for j in range(5)) for i in range(self.n_slices)]

    def widths(self):
        return [self.col_widths[i] for i in range(self.n_cols)]


class RefOutcome(C.Structure):
    _fields_ = [("t_min_us", C.c_double), ("t_best_us", C.c_double), ("sse_best", C.c_double),
                ("candidates_evaluated", C.c_uint64), ("candidates_step1", C.c_uint64),
                ("candidates_step2", C.c_uint64), ("search_time_us", C.c_double),
                ("time_min_step_us", C.c_double), ("clustering_step_us", C.c_double),
                ("est_source", C.c_int32), ("est_source_poc", C.c_int32), ("best", RefLayout)]


class Ref:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle ref` where "
                               "/root/reference exists")
        self.L = C.CDLL(path)
        self.L.ref_last_error.restype = C.c_char_p
        D, I, P = C.c_double, C.c_int, C.c_void_p
        self.L.ref_min_time_search.argtypes = [I, I, I, P, I, D, D, I, I, I, P, P]
        self.L.ref_constrained_clustering.argtypes = [I, I, I, P, P, D, I, D, D, I, I, I, P]
        self.L.ref_two_step.argtypes = [I, I, I, I, I, P, P, P, P, I, I, D, D, I, I, I, P]
        self.L.ref_enumerate.argtypes = [I, I, I, I, D, I, I, P, P, C.c_uint64]
        self.L.ref_estimate.argtypes = [I, I, I, I, I, P, P, P, I, P, P, P]
        self.L.ref_partition_eval.argtypes = [I, I, I, I, P, I, P, I, P, P, P, I, P, P, P, P]
        self.L.ref_uniform_partition.argtypes = [I, I, I, I, P]

    def err(self):
        return self.L.ref_last_error().decode()

    def ctu_stats(self, plane16: np.ndarray, bit_depth: int, ctu: int = 128):
        H, W = plane16.shape
        p = np.ascontiguousarray(plane16, dtype=np.uint16)
        cols, rows = -(-W // ctu), -(-H // ctu)
        out = np.zeros(cols * rows * 3, dtype=np.uint64)
        st = self.L.ref_ctu_stats(_p(p), W, H, bit_depth, ctu, 0, _p(out))
        return st, out.reshape(-1, 3)

    def rect_times(self, times, cols, rows):
        t = np.ascontiguousarray(times, dtype=np.float64)
        out = np.zeros(cols * (cols + 1) // 2 * (rows * (rows + 1) // 2))
        st = self.L.ref_rect_times(_p(t), cols, rows, _p(out))
        return st, out

    def rect_sse(self, fw, fh, ctu, records):
        cols, rows = -(-fw // ctu), -(-fh // ctu)
        rec = np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        out = np.zeros(cols * (cols + 1) // 2 * (rows * (rows + 1) // 2))
        st = self.L.ref_rect_sse(fw, fh, ctu, _p(rec), _p(out), None)
        return st, out

    def enumerate(self, fw, fh, ctu, n, k=3.0, family=0, max_cols=0, max_out=0):
        cnt = C.c_uint64()
        buf = (RefLayout * max_out)() if max_out else None
        st = self.L.ref_enumerate(fw, fh, ctu, n, k, family, max_cols, C.byref(cnt),
                                  C.cast(buf, C.c_void_p) if buf is not None else None, max_out)
        return st, cnt.value, (list(buf)[:min(max_out, cnt.value)] if buf is not None else [])

    def min_time_search(self, fw, fh, ctu, est, n, lam=0.0, k=3.0, family=0, max_cols=0,
                        workers=1):
        t = C.c_double()
        lay = RefLayout()
        e = np.ascontiguousarray(est, dtype=np.float64)
        st = self.L.ref_min_time_search(fw, fh, ctu, _p(e), n, lam, k, family, max_cols, workers,
                                        C.byref(t), C.byref(lay))
        return st, t.value, lay

    def constrained(self, fw, fh, ctu, est, records, t_min, n, lam=0.0, k=3.0, family=0,
                    max_cols=0, workers=1):
        o = RefOutcome()
        e = np.ascontiguousarray(est, dtype=np.float64)
        rec = np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        st = self.L.ref_constrained_clustering(fw, fh, ctu, _p(e), _p(rec), t_min, n, lam, k,
                                               family, max_cols, workers, C.byref(o))
        return st, o

    def two_step(self, fw, fh, ctu, gop, maps, pocs, tls, records, poc, n, lam=0.0, k=3.0,
                 family=0, max_cols=0, workers=1):
        o = RefOutcome()
        m = np.ascontiguousarray(maps, dtype=np.float64)
        pc = np.ascontiguousarray(pocs, dtype=np.int32)
        tl = np.ascontiguousarray(tls, dtype=np.int32)
        rec = np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        st = self.L.ref_two_step(fw, fh, ctu, gop, len(pocs), _p(m), _p(pc), _p(tl), _p(rec), poc,
                                 n, lam, k, family, max_cols, workers, C.byref(o))
        return st, o

    def temporal_layer(self, poc, gop):
        tl = C.c_int()
        st = self.L.ref_temporal_layer(poc, gop, C.byref(tl))
        return st, tl.value

    def estimate(self, fw, fh, ctu, gop, maps, pocs, tls, poc):
        cols, rows = -(-fw // ctu), -(-fh // ctu)
        m = np.ascontiguousarray(maps, dtype=np.float64)
        pc = np.ascontiguousarray(pocs, dtype=np.int32)
        tl = np.ascontiguousarray(tls, dtype=np.int32)
        est = np.zeros(cols * rows)
        src, srcp = C.c_int(), C.c_int()
        st = self.L.ref_estimate(fw, fh, ctu, gop, len(pocs), _p(m), _p(pc), _p(tl), poc,
                                 _p(est), C.byref(src), C.byref(srcp))
        return st, est, src.value, srcp.value

    def yuv_frame_count(self, path, w, h, bit_depth):
        n = C.c_int()
        st = self.L.ref_yuv_frame_count(path.encode(), w, h, bit_depth, C.byref(n))
        return st, n.value

    def load_yuv_frame(self, path, w, h, poc, bit_depth):
        out = np.zeros((h, w), np.uint16)
        st = self.L.ref_load_yuv_frame(path.encode(), w, h, poc, bit_depth, _p(out))
        return st, out

    def uniform_partition(self, fw, fh, ctu, n):
        """uniform_partition (grid.cpp:186-262) -> (status, RefLayout)."""
        lay = RefLayout()
        st = self.L.ref_uniform_partition(fw, fh, ctu, n, C.byref(lay))
        return st, lay

    def partition_eval(self, fw, fh, ctu, col_widths, row_heights, slices, times=None,
                       records=None, validate=False):
        cw = np.ascontiguousarray(col_widths, dtype=np.int32)
        rh = np.ascontiguousarray(row_heights, dtype=np.int32)
        sl = np.ascontiguousarray(np.asarray(slices, dtype=np.int32).reshape(-1))
        t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
        rec = None if records is None else np.ascontiguousarray(records, dtype=np.uint64).reshape(-1)
        mx, tot, sse = C.c_double(), C.c_double(), C.c_double()
        am = C.c_int64()
        st = self.L.ref_partition_eval(fw, fh, ctu, len(cw), _p(cw), len(rh), _p(rh),
                                       len(slices), _p(sl), _p(t), _p(rec), int(validate),
                                       C.byref(mx), C.byref(tot), C.byref(am), C.byref(sse))
        return st, mx.value, tot.value, am.value, sse.value
