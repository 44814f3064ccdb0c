"""cfg1 single-frame calls only (for an ncu capture of the small-grid kernels)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_14792_b200 import Partitioner, lib  # noqa: E402
from paper_2012_14792_b200 import workloads as wl  # noqa: E402
from paper_2012_14792_b200._abi import SearchResult, check  # noqa: E402
import bench  # noqa: E402

w = wl.WORKLOADS[1]
g, bps = w.grid(), w.bps
luma_h, est_h = bench.make_inputs(w, 0, 1)
luma_d, est_d = luma_h.cuda(), est_h.cuda()
part = Partitioner(0)
res = (SearchResult * 1)()
cc, gc = w.cfg().c(), g.c()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    check(lib().sc_partition_frames(part._h, C.byref(gc), C.byref(cc), C.c_void_p(luma_d.data_ptr()),
                                    bps, w.width * bps, w.width * w.height * bps,
                                    C.c_void_p(est_d.data_ptr()), 1, None, C.cast(res, C.c_void_p)))
torch.cuda.synchronize()
print("ok")
