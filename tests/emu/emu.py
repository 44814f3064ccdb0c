"""TEST-ONLY ctypes wrapper of the host emulator of the search kernels."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libsearch_emu.so")


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class Emu:
    def __init__(self):
        if not os.path.exists(SO):
            raise RuntimeError(f"{SO} missing: make -C tests/emu")
        self.L = C.CDLL(SO)
        I, D, P = C.c_int, C.c_double, C.c_void_p
        self.SEED_CB = C.CFUNCTYPE(None, C.POINTER(C.c_uint64), C.c_int)
        self.L.emu_search.argtypes = [I, I, I, D, I, I, I, I, I, P, P, P, I, C.c_size_t, I, I, P, P, P, P,
                                      P, P, P, I, I, I, self.SEED_CB]

    def trace_search(self, cols, rows, n, k, max_cols, coverage, rect_time, item_target=16):
        """Exhaustive step 1 through the host build of the candidate trace
        (csrc/trace.cuh): (t_min, count, ordinal, snapshot, found, n_ops)."""
        rt = np.ascontiguousarray(rect_time, dtype=np.float64)
        F = rt.shape[0]
        t = np.zeros(F)
        cnt = np.zeros(F, dtype=np.uint64)
        ordn = np.zeros(F, dtype=np.uint64)
        snap = np.zeros((F, 96), dtype=np.uint8)
        found = np.zeros(F, dtype=np.int32)
        nops = C.c_uint64()
        I, D, P = C.c_int, C.c_double, C.c_void_p
        self.L.emu_trace_search.argtypes = [I, I, I, D, I, I, I, P, C.c_size_t, P, P, P, P, P, P]
        st = self.L.emu_trace_search(cols, rows, n, k, max_cols, coverage, F, _p(rt), item_target,
                                     _p(t), _p(cnt), _p(ordn), _p(snap), _p(found),
                                     C.byref(nops))
        assert st == 0, st
        return t, cnt, ordn, snap, found, nops.value

    def trace_step2(self, cols, rows, n, k, max_cols, coverage, rect_time, rect_sse, budget,
                    item_target=16):
        """Step 2 through the host build of the trace: (t, sse, ordinal,
        snapshot, found)."""
        rt = np.ascontiguousarray(rect_time, dtype=np.float64)
        rs = np.ascontiguousarray(rect_sse, dtype=np.float64)
        b = np.ascontiguousarray(budget, dtype=np.float64)
        F = rt.shape[0]
        t, sse = np.zeros(F), np.zeros(F)
        ordn = np.zeros(F, dtype=np.uint64)
        snap = np.zeros((F, 96), dtype=np.uint8)
        found = np.zeros(F, dtype=np.int32)
        I, D, P = C.c_int, C.c_double, C.c_void_p
        self.L.emu_trace_step2.argtypes = [I, I, I, D, I, I, I, P, P, P, C.c_size_t, P, P, P, P, P]
        st = self.L.emu_trace_step2(cols, rows, n, k, max_cols, coverage, F, _p(rt), _p(rs), _p(b),
                                    item_target, _p(t), _p(sse), _p(ordn), _p(snap), _p(found))
        assert st == 0, st
        return t, sse, ordn, snap, found

    def search(self, cols, rows, n, k, max_cols, coverage, step, rect_time, rect_sse=None,
               budget=None, warps=3, item_target=16, offset=0, stride=1, full=False, prune=0,
               order=0, split=1, split_depth=1, seed_allreduce=None):
        """seed_allreduce(list[int]) -> list[int]: the shards' all-reduce-min
        of the frozen seed incumbents (pruned step 1), or None."""
        rt = np.ascontiguousarray(rect_time, dtype=np.float64)
        F = rt.shape[0]
        rs = None if rect_sse is None else np.ascontiguousarray(rect_sse, dtype=np.float64)
        b = None if budget is None else np.ascontiguousarray(budget, dtype=np.float64)
        t = np.zeros(F)
        sse = np.zeros(F)
        cnt = np.zeros(F, dtype=np.uint64)
        snap = np.zeros((F, 96), dtype=np.uint8)
        found = np.zeros(F, dtype=np.int32)
        item = np.zeros(F, dtype=np.uint64)
        ordn = np.zeros(F, dtype=np.uint64)
        st = self.L.emu_search(cols, rows, n, k, max_cols, coverage, step, prune, F, _p(rt), _p(rs),
                               _p(b),
                               warps, item_target, offset, stride, _p(t), _p(sse), _p(cnt),
                               _p(snap), _p(found), _p(item), _p(ordn), order, split,
                               split_depth, self._seed_cb(seed_allreduce))
        assert st == 0
        if full:
            return t, sse, cnt, snap, found, item, ordn
        return t, sse, cnt, snap, found

    def _seed_cb(self, fn):
        if fn is None:
            return self.SEED_CB()

        def cb(ptr, n):
            vals = fn([ptr[i] for i in range(n)])
            for i in range(n):
                ptr[i] = vals[i]
        self._cb_keep = self.SEED_CB(cb)
        return self._cb_keep

    @staticmethod
    def slices(snap_row, n, rows):
        W = [int(x) for x in snap_row[:16]]
        R = [int(x) for x in snap_row[16:32]]
        H = [int(x) for x in snap_row[32:32 + n]]
        out, x, run, sid = [], 0, 0, 0
        c = 0
        while c < 16 and W[c]:
            c += 1
        for i in range(c):
            y = 0
            for _ in range(R[i]):
                out.append((x, y, W[i], H[run], sid))
                y += H[run]
                run += 1
                sid += 1
            x += W[i]
        return out
