"""CPU tests of the boundary and the host logic: the C-ABI library loads and
exports every symbol include/slicecraft_b200.h declares, host-side entry
points behave like the reference (errors, temporal layers, estimator
fallbacks, record validation), and the synthetic generator is deterministic.
No compute entry point is called here (no GPU)."""
import ctypes as C
import hashlib
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "slicecraft_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2012_14792_b200 import lib
    from paper_2012_14792_b200._abi import SIGNATURES
    L = lib()
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(n for n, _, _ in SIGNATURES) == syms  # the ctypes mirror is complete
    assert L.sc_abi_version() == 2


def test_struct_layouts_match_header():
    """ctypes mirror sizes == the C compiler's sizes of the header structs."""
    import subprocess
    import tempfile
    from paper_2012_14792_b200 import _abi
    src = """#include <stdio.h>
#include "slicecraft_b200.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sc_grid),
 sizeof(sc_ctu_record), sizeof(sc_search_cfg), sizeof(sc_layout), sizeof(sc_search_result),
 sizeof(sc_shard_best), sizeof(sc_status), sizeof(sc_rect), sizeof(sc_partition),
 sizeof(sc_partition_stats));return 0;}"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        sizes = list(map(int, subprocess.run([exe], capture_output=True, text=True,
                                             check=True).stdout.split()))
    mine = [C.sizeof(_abi.Grid), C.sizeof(_abi.CtuRecord), C.sizeof(_abi.SearchCfg),
            C.sizeof(_abi.Layout), C.sizeof(_abi.SearchResult), C.sizeof(_abi.ShardBest), 4,
            C.sizeof(_abi.Rect), C.sizeof(_abi.PartitionC), C.sizeof(_abi.PartitionStats)]
    assert sizes == mine


def test_uniform_partition_matches_reference_golden():
    """sc_uniform_partition (host code) == the reference's uniform_partition
    (grid.cpp:186-262) on factorizable, prime-fallback and too-many-slice
    cases (tests/golden/uniform.json)."""
    import json
    from paper_2012_14792_b200 import CtuGrid, SlicecraftError
    from paper_2012_14792_b200.partitioner import Partition
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "uniform.json")))["partitions"]
    for c in gold:
        g = CtuGrid.make(c["cols"] * 32, c["rows"] * 32, 32)
        if c["status"] != 0:
            with pytest.raises(SlicecraftError) as e:
                Partition.uniform(g, c["n"])
            assert e.value.status == c["status"], c
            continue
        if c["n"] > 64:
            continue  # beyond SC_MAX_SLICES
        p = Partition.uniform(g, c["n"])
        assert p.col_widths == c["tile_cols"], c
        assert p.row_heights == c["tile_rows"], c
        assert p.rects() == [tuple(x) for x in c["slices"]], c


def test_grid_make_matches_reference_rules():
    from paper_2012_14792_b200 import CtuGrid, SlicecraftError
    g = CtuGrid.make(1920, 1080)
    assert (g.cols, g.rows) == (15, 9)
    g = CtuGrid.make(3840, 2160)
    assert (g.cols, g.rows) == (30, 17)
    g = CtuGrid.make(7680, 4320)
    assert (g.cols, g.rows) == (60, 34)
    with pytest.raises(SlicecraftError) as e:
        CtuGrid.make(100, 100, 48)
    assert e.value.kind == "GeometryError"
    with pytest.raises(SlicecraftError) as e:
        CtuGrid.make(0, 100)
    assert e.value.kind == "GeometryError"


def test_temporal_layers_and_estimator_vs_golden():
    from paper_2012_14792_b200 import (CostHistory, CostMap, CtuGrid, SlicecraftError,
                                       estimate_ctu_times, temporal_layer_of_poc)
    from paper_2012_14792_b200.partitioner import (CO_TEMPORAL_LAYER, MOST_RECENT_ANY,
                                                   UNIFORM)
    k = json.load(open(os.path.join(GOLDEN, "spec_kats.json")))
    for poc, gop, tl in k["temporal_layers"]:
        assert temporal_layer_of_poc(poc, gop) == tl
    with pytest.raises(SlicecraftError) as e:
        temporal_layer_of_poc(3, 12)
    assert e.value.kind == "ConfigError"
    g = CtuGrid.make(128, 128, 32)
    est = k["estimate"]
    # history {0 (TL0)=1.0, 16 (TL0)=2.0, 8 (TL1)=3.0}
    h = CostHistory(g, 16)
    for v, poc, tl in [(1.0, 0, 0), (2.0, 16, 0), (3.0, 8, 1)]:
        h.append(CostMap(g, np.full(16, v), poc, tl))
    e24 = estimate_ctu_times(h, 24)
    assert e24.times_us[0] == est["24:0,16,8"]["est0"] and e24.source == CO_TEMPORAL_LAYER
    assert e24.source_poc == est["24:0,16,8"]["source_poc"] == 8
    e6 = estimate_ctu_times(h, 6)
    assert e6.source == MOST_RECENT_ANY == est["6:0,16,8"]["source"]
    assert e6.source_poc == 8
    e5 = estimate_ctu_times(CostHistory(g, 16), 5)
    assert e5.source == UNIFORM and np.all(e5.times_us == 1.0)
    with pytest.raises(SlicecraftError) as e:
        h.append(CostMap(g, np.ones(16), 8, 1))
    assert e.value.kind == "TraceError"
    with pytest.raises(SlicecraftError) as e:
        h.append(CostMap(g, -np.ones(16), 9, 4))
    assert e.value.kind == "FormatError"


def test_texture_validate_matches_reference_rules():
    from paper_2012_14792_b200 import RECORD_DTYPE, CtuGrid, SlicecraftError, texture_validate
    g = CtuGrid.make(200, 100, 64)  # partial border cells: widths 64,64,64,8; heights 64,36
    rec = np.zeros(g.cell_count(), RECORD_DTYPE)
    for y in range(g.rows):
        for x in range(g.cols):
            cnt = min(64, 200 - 64 * x) * min(64, 100 - 64 * y)
            rec[y * g.cols + x] = (cnt, 5 * cnt, 25 * cnt)
    texture_validate(g, rec)
    bad = rec.copy()
    bad[3]["count"] += 1
    with pytest.raises(SlicecraftError) as e:
        texture_validate(g, bad)
    assert e.value.kind == "FormatError"
    bad = rec.copy()
    bad[0]["sumsq"] = 0  # count*sumsq < sum^2
    with pytest.raises(SlicecraftError) as e:
        texture_validate(g, bad)
    assert e.value.kind == "FormatError"


def test_no_gpu_fails_loudly():
    """Without a device the product path refuses (no CPU fallback)."""
    import torch
    from paper_2012_14792_b200 import Partitioner, SlicecraftError
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(SlicecraftError) as e:
        Partitioner(0)
    assert e.value.kind == "CudaError"


def test_synthetic_generator_is_deterministic():
    from paper_2012_14792_b200 import workloads as wl
    a = wl.synth_luma(wl.WORKLOADS[1])
    b = wl.synth_luma(wl.WORKLOADS[1])
    assert np.array_equal(a, b) and a.dtype == np.uint8 and a.shape == (1, 1080, 1920)
    # golden hash of cfg1 records (golden file was made from these very bytes)
    from oracle.oracle import Oracle
    rec = Oracle().ctu_stats(a[0], 128)
    gold = json.load(open(os.path.join(GOLDEN, "configs.json")))["1"]["frames"][0]
    assert hashlib.sha256(np.ascontiguousarray(rec).tobytes()).hexdigest()[:16] == \
        gold["records_hash"]
    t = wl.synth_times(wl.WORKLOADS[3], 5, 510)
    assert np.all(t > 0) and np.array_equal(t, t.astype(np.float32).astype(np.float64))
    tr = wl.cost_trace(wl.WORKLOADS[2], frames=6)
    assert tr.est_source_poc == [0, 1, 1, 3, 3, 2]  # POC 6 is TL 3 like POC 2


def test_shard_merge_picks_first_in_order():
    """sc_shard_merge: per frame, min (key, item, position in the item = the
    layout's lex order); counts summed."""
    from paper_2012_14792_b200._abi import SearchResult, ShardBest, check, lib
    world, F = 3, 2
    recs = (ShardBest * (world * F))()
    vals = {  # (rank, frame): (t bits proxy, item, ord)
        (0, 0): (5, 10, 3), (1, 0): (5, 4, 9), (2, 0): (7, 1, 0),
        (0, 1): (9, 2, 2), (1, 1): (8, 30, 1), (2, 1): (8, 30, 0)}
    for (r, f), (t, it, o) in vals.items():
        s = recs[r * F + f]
        s.key_t, s.item, s.ord, s.count, s.key_sse = t, it, o, 100 + r, 0.0
        s.layout.n_cols = 1
        s.layout.col_widths[0] = r + 1
    res = (SearchResult * F)()
    for f in range(F):
        res[f].argmin.n_slices = 1
    check(lib().sc_shard_merge(1, world, F, C.cast(recs, C.c_void_p), C.cast(res, C.c_void_p)))
    assert res[0].argmin.col_widths[0] == 2  # rank 1: t=5, item 4 < 10
    assert res[1].argmin.col_widths[0] == 2  # t=8, item 30 tie: layout [2] < [3]
    assert res[0].candidates_step1 == 303


def test_shard_merge_wide_counts():
    """Pruned-mode DP counts exceed 64 bits (cfg5: ~6.1e29 per frame and step):
    sc_shard_best carries count_hi and the merge sums 128-bit counts."""
    from paper_2012_14792_b200._abi import SearchResult, ShardBest, check, lib
    world, F = 2, 1
    recs = (ShardBest * (world * F))()
    total = 610308283606383278175018310268  # cfg5's count
    for r in range(world):
        s = recs[r]
        s.key_t, s.item, s.ord, s.key_sse = 5 + r, 1, 0, 0.0
        s.layout.n_cols = 1
        s.layout.col_widths[0] = 1
    recs[0].count, recs[0].count_hi = total & ((1 << 64) - 1), total >> 64  # rank 0 carries it
    res = (SearchResult * F)()
    res[0].argmin.n_slices = 1
    check(lib().sc_shard_merge(1, world, F, C.cast(recs, C.c_void_p), C.cast(res, C.c_void_p)))
    assert res[0].candidates_step1 | (res[0].candidates_step1_hi << 64) == total


def test_synthetic_inputs_reproduce_the_golden_hashes():
    """synth/libscsynth.so regenerates the very estimate maps the reference
    fixtures were made from (configs.json cfg1-3, ladder.json cfg4 / cfg5)."""
    from paper_2012_14792_b200 import workloads as wl

    def h(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    cfgs = json.load(open(os.path.join(GOLDEN, "configs.json")))
    for ci in ("1", "2", "3"):
        fr = cfgs[ci]["frames"][0]
        tr = wl.cost_trace(wl.WORKLOADS[int(ci)], frames=fr["poc"])
        assert h(tr.est[fr["poc"] - 1]) == fr["est_hash"], ci
    lad = json.load(open(os.path.join(GOLDEN, "ladder.json")))["grids"]
    for ci in ("4", "5"):
        tr = wl.cost_trace(wl.WORKLOADS[int(ci)], frames=1)
        assert h(tr.est[0]) == lad[ci]["est_hash"], ci
