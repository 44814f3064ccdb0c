"""Single-frame device latency of sc_two_step (the paper's per-frame call,
PAPER.md:169) on the cfg1 and cfg3 grids, exhaustive and pruned: warm calls,
CUDA-event phases (sc_ctx_timings_ex) and the whole call's device time."""
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

names = ["texture", "tables", "step1", "step2", "call", "time_tables_main", "moment_side", "post"]
out = {}
part = Partitioner(0)
for ci in (1, 3):
    w = wl.WORKLOADS[ci]
    g, bps = w.grid(), w.bps
    luma_h, est_h = bench.make_inputs(w, 0, 1)
    luma_d, est_d = luma_h.cuda(), est_h.cuda()
    rec_d = torch.empty(g.cell_count() * 24, dtype=torch.uint8, device="cuda")
    res = (SearchResult * 1)()
    tim = (C.c_double * 8)()
    for mode in (0, 1):
        cc, gc = w.cfg(mode=mode).c(), g.c()

        def call():
            check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc),
                                            C.c_void_p(luma_d.data_ptr()), bps, w.width * bps,
                                            w.width * w.height * bps, C.c_void_p(est_d.data_ptr()),
                                            1, C.c_void_p(rec_d.data_ptr()),
                                            C.cast(res, C.c_void_p)))
            check(lib().sc_ctx_timings_ex(part._h, 8, tim))
            return np.array([tim[i] for i in range(8)])
        for _ in range(5):
            call()
        acc = np.median(np.stack([call() for _ in range(20)]), axis=0)
        out[f"cfg{ci}_F1_{'pruned' if mode else 'exhaustive'}"] = {
            n: round(float(v), 1) for n, v in zip(names, acc)}
print(json.dumps(out, indent=1))
