"""GPU tests of the round-2 C-ABI additions, through the C-ABI:

* validate_partition as a device post-check (grid.cpp:86-184) against the
  reference's own status + message on 400 valid / mutated partitions
  (tests/golden/validate.json), and the CTU -> slice-id map it writes;
* the device-materialised candidate stream (for_each_candidate /
  enumerate_candidates, search.cpp:302-326) against the reference's ordered
  lists (tests/golden/enumerate.json), including windows (paging);
* the per-frame CTU -> slice-id maps of the partitions a search returns
  (sc_result_slice_maps) against maps painted from the returned layouts;
* the reference's +inf rule for step 1 (search.cpp:277-292);
* the cfg4 / cfg5 grids (30x17, 60x34) against the unmodified reference on
  the ladder of spaces it can enumerate (tests/golden/ladder.json, SURVEY.md
  §8c): exhaustive and pruned modes, and the oracle's independent
  branch-and-bound restatement, bit-exact.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _paint(cols, rows, rects):
    m = np.full((rows, cols), -1, np.int32)
    for x0, y0, w, h, sid in rects:
        m[y0:y0 + h, x0:x0 + w] = sid
    return m


def test_validate_partition_vs_reference(part):
    from paper_2012_14792_b200 import CtuGrid, SlicecraftError
    from paper_2012_14792_b200.partitioner import Slice
    cases = json.load(open(os.path.join(GOLDEN, "validate.json")))
    seen = set()
    for i, c in enumerate(cases):
        g = CtuGrid.make(c["cols"] * 32, c["rows"] * 32, 32)
        sl = [Slice(*q) for q in c["slices"]]
        if c["status"]:
            with pytest.raises(SlicecraftError) as e:
                part.validate_partition(g, c["tile_cols"], c["tile_rows"], sl)
            assert e.value.status == c["status"], (i, c["kind"])
            assert str(e.value).split(": ", 1)[1] == c["message"], (i, c["kind"])
        else:
            m = part.validate_partition(g, c["tile_cols"], c["tile_rows"], sl)
            assert np.array_equal(m, _paint(g.cols, g.rows, c["slices"])), i
        seen.add(c["status"])
    assert seen == {0, 1, 2, 3, 4}  # every class of validate_partition exercised


def test_validate_partition_large_grid(part):
    """A full 8K grid (60x34) of single-CTU slices (2040 slices, beyond the
    search's SC_MAX_SLICES): valid, then one overlap."""
    from paper_2012_14792_b200 import CtuGrid, SlicecraftError
    from paper_2012_14792_b200.partitioner import Slice
    g = CtuGrid.make(7680, 4320, 128)
    sl = [Slice(x, y, 1, 1, y * g.cols + x) for y in range(g.rows) for x in range(g.cols)]
    m = part.validate_partition(g, [1] * g.cols, [1] * g.rows, sl)
    assert np.array_equal(m.reshape(-1), np.arange(g.cell_count()))
    sl[100] = Slice(sl[99].x0, sl[99].y0, 1, 1, 100)
    with pytest.raises(SlicecraftError) as e:
        part.validate_partition(g, [1] * g.cols, [1] * g.rows, sl)
    assert e.value.kind == "OverlapError"
    assert "slices 99 and 100 both cover cell (39,1)" in str(e.value)


def test_enumerate_candidates_vs_reference(part):
    from paper_2012_14792_b200 import CtuGrid, SearchConfig, SlicecraftError
    cases = json.load(open(os.path.join(GOLDEN, "enumerate.json")))
    for i, c in enumerate(cases):
        g = CtuGrid.make(c["w"], c["h"], c["ctu"])
        cfg = SearchConfig(n_slices=c["n"], k_area=c["k"], family=c["family"],
                           max_tile_cols=c["max_tile_cols"])
        if c["status"]:
            with pytest.raises(SlicecraftError) as e:
                part.enumerate_candidates(g, cfg)
            assert e.value.status == c["status"], i
            continue
        if c["count"] > 200000:
            continue
        got = [[list(s) for s in p.rects()] for p in part.enumerate_candidates(g, cfg)]
        assert len(got) == c["count"], i
        if c["count"]:
            assert hashlib.sha256(json.dumps(got).encode()).hexdigest() == c["sha256"], i
        if "list" in c:
            assert got == c["list"], i
        elif c["count"]:
            assert got[:40] == c["head"] and got[-40:] == c["tail"], i


def test_enumerate_windows_page_in_order(part):
    """Windows [first, first + k) of the stream concatenate to the whole
    stream; the total equals the counting DP (sc_count_candidates)."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    g = CtuGrid.make(1920, 1080, 128)
    for cfg in [SearchConfig(n_slices=8, max_tile_cols=4), SearchConfig(n_slices=5, coverage=1),
                SearchConfig(n_slices=4, k_area=1.3)]:
        whole, tot = part.enumerate_layouts(g, cfg, 0, 1 << 20)
        assert tot == len(whole) == part.count_candidates(g, cfg)
        # order: column count ascending, then (widths, runs, heights) lexicographic
        key = [(L.n_cols, list(L.col_widths[:L.n_cols]), list(L.runs_per_col[:L.n_cols]),
                list(L.run_heights[:cfg.n_slices])) for L in whole]
        assert key == sorted(key)
        pages, first = [], 0
        while first < tot:
            lay, t2 = part.enumerate_layouts(g, cfg, first, 777)
            assert t2 == tot and lay
            pages += lay
            first += len(lay)
        assert [bytes(a) for a in pages] == [bytes(b) for b in whole]
        lay, _ = part.enumerate_layouts(g, cfg, tot, 10)
        assert lay == []


def test_result_slice_maps(part, oracle):
    """The CTU -> slice-id maps of the returned partitions (device post-check
    output) equal the maps painted from the returned layouts; cells right of
    a reference-family layout's columns are -1."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    from paper_2012_14792_b200.partitioner import Partition
    rng = np.random.default_rng(5)
    g = CtuGrid.make(1920, 1080, 128)
    F = 6
    est = rng.lognormal(0, 0.7, (F, g.cell_count()))
    luma = rng.integers(0, 1024, (F, 1080, 1920)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 128)
    for cov in (0, 1):
        res = part.two_step_batch(g, est, rec, SearchConfig(n_slices=6, lambda_=0.2, coverage=cov))
        m1 = part.result_slice_maps(g, 1, F)
        m2 = part.result_slice_maps(g, 2, F)
        for f in range(F):
            assert np.array_equal(m1[f], _paint(g.cols, g.rows, res[f].argmin.rects()))
            assert np.array_equal(m2[f], _paint(g.cols, g.rows, res[f].best.rects()))
            if cov:
                assert (m2[f] >= 0).all()


def test_step1_infinite_times(part, oracle):
    """run_step1 keeps `t < best_t` from best_t = +inf (search.cpp:277-292): a
    family whose every layout_time is +inf has no argmin (NoCandidateError;
    the reference raises it on these grids, checked when the fixtures were
    made).  Elsewhere inf times turn summed-area-table entries into NaN
    (inf - inf), which layout_time's max from 0.0 skips: the results must
    still be the oracle's, bit for bit."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig, SlicecraftError
    for mode in (0, 1):
        for W, n, est in [(128, 1, [np.inf]), (256, 1, [np.inf, 1.0]), (256, 2, [np.inf, 1.0])]:
            g = CtuGrid.make(W, 128, 128)
            with pytest.raises(SlicecraftError) as e:
                part.min_time_search_batch(g, np.array(est), SearchConfig(n_slices=n, mode=mode))
            assert e.value.kind == "NoCandidateError"
        g = CtuGrid.make(640, 384, 128)
        cfg = SearchConfig(n_slices=3, mode=mode)
        for est in [np.full(g.cell_count(), np.inf), np.where(np.arange(15) % 5 == 0, np.inf, 1.0),
                    np.where(np.arange(15) == 7, np.inf, 2.0)]:
            o = part.min_time_search_batch(g, est, cfg)[0]
            st, exp = oracle.search(640, 384, 128, est, None, 3, 0.0, 3.0, 0, 0, 1)
            assert st == 0 and o.t_min_us == exp.t_min_us
            assert o.argmin.rects() == exp.argmin1.slices(g.rows)


# ---- cfg4 / cfg5 grids against the reference ------------------------------------
def _ladder_inputs(gr):
    from paper_2012_14792_b200 import RECORD_DTYPE, CtuGrid
    g = CtuGrid.make(gr["width"], gr["height"], gr["ctu"])
    est = np.array(gr["est"], dtype=np.float64)
    r3 = np.array(gr["records"], dtype=np.uint64)
    rec = np.zeros(g.cell_count(), RECORD_DTYPE)
    rec["count"], rec["sum"], rec["sumsq"] = r3[:, 0], r3[:, 1], r3[:, 2]
    assert hashlib.sha256(np.ascontiguousarray(est).tobytes()).hexdigest()[:16] == gr["est_hash"]
    return g, est, rec, r3


LADDER = json.load(open(os.path.join(GOLDEN, "ladder.json")))


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("ci", range(len(LADDER["cases"])))
def test_ladder_vs_reference(part, oracle, ci, mode):
    """two_step_partition on the real cfg4 (30x17) / cfg5 (60x34) grids at every
    space the reference enumerates here (up to 3.1e8 candidates per step):
    exhaustive and pruned GPU walks == the unmodified reference, bit-exact,
    including the counters; and the oracle's branch-and-bound restatement
    (the cfg4 / cfg5 checker) == the reference too."""
    from paper_2012_14792_b200 import SearchConfig
    from paper_2012_14792_b200.partitioner import Partition
    c = LADDER["cases"][ci]
    g, est, rec, r3 = _ladder_inputs(LADDER["grids"][str(c["cfg"])])
    cfg = SearchConfig(n_slices=c["n"], lambda_=c["lambda"], k_area=c["k"],
                       max_tile_cols=c["max_tile_cols"], mode=mode)
    o = part.two_step_batch(g, est[None], rec[None], cfg)[0]
    assert o.t_min_us == c["t_min"] and o.t_best_us == c["t_best"] and o.sse_best == c["sse_best"]
    assert o.best.rects() == [tuple(x) for x in c["best"]]
    assert o.candidates_step1 == c["candidates_step1"]
    assert o.candidates_step2 == c["candidates_step2"]
    if mode == 1:
        st, e = oracle.search_pruned(g.frame_width, g.frame_height, g.ctu_size, est, r3, c["n"],
                                     c["lambda"], c["k"], c["max_tile_cols"], 0, 3)
        assert st == 0
        assert e.t_min_us == c["t_min"] and e.t_best_us == c["t_best"]
        assert e.sse_best == c["sse_best"]
        assert e.best.slices(g.rows) == [tuple(x) for x in c["best"]]
    assert Partition  # noqa
