"""Phase timings (sc_ctx_timings_ex, CUDA events) of the cfg3 call in three
shapes: the whole batch path with device luma (K1 on the side stream), two_step
with device records (no K1), and min_time_search alone (no side stream) -- to
see what the time-table phase costs by itself and what K1 adds to it."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_14792_b200 import Partitioner, lib  # noqa: E402
from paper_2012_14792_b200 import workloads as wl  # noqa: E402
from paper_2012_14792_b200._abi import SearchResult, check  # noqa: E402
import bench  # noqa: E402

w = wl.WORKLOADS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
F, g, bps = w.frames, w.grid(), w.bps
luma_h, est_h = bench.make_inputs(w, 0, F)
luma_d, est_d = luma_h.cuda(), est_h.cuda()
part = Partitioner(0)
rec_d = torch.empty(F * g.cell_count() * 24, dtype=torch.uint8, device="cuda")
res = (SearchResult * F)()
tim = (C.c_double * 8)()
gc, cc = g.c(), w.cfg().c()
names = ["texture", "tables", "step1", "step2", "call", "time_tables_main", "moment_side", "post"]


def run(kind):
    if kind == "partition_frames":
        check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc),
                                        C.c_void_p(luma_d.data_ptr()), bps, w.width * bps,
                                        w.width * w.height * bps, C.c_void_p(est_d.data_ptr()), F,
                                        C.c_void_p(rec_d.data_ptr()), C.cast(res, C.c_void_p)))
    elif kind == "two_step":
        check(lib().sc_two_step(part._h, C.byref(gc), C.byref(cc), C.c_void_p(est_d.data_ptr()),
                                C.c_void_p(rec_d.data_ptr()), F, C.cast(res, C.c_void_p)))
    else:
        check(lib().sc_min_time_search(part._h, C.byref(gc), C.byref(cc),
                                       C.c_void_p(est_d.data_ptr()), F, C.cast(res, C.c_void_p)))
    check(lib().sc_ctx_timings_ex(part._h, 8, tim))
    return np.array([tim[i] for i in range(8)])


out = {}
for kind in ["partition_frames", "two_step", "min_time"]:
    for _ in range(3):
        run(kind)
    acc = np.mean([run(kind) for _ in range(10)], axis=0)
    out[kind] = {n: round(float(v), 1) for n, v in zip(names, acc)}
print(json.dumps(out, indent=1))
