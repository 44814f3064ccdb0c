"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle and the
golden fixtures generated from the unmodified reference.

Bar: bit-exact for every integer / index artefact (CTU records, chosen
layouts, candidate counts) and for every double the reference computes with
the same operation order (times, SSEs, t_min, t_best, sse_best) — the
north_star's 1e-6 relative tolerance is therefore met with margin 0.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(2012_14792)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


# ---- K1 texture ---------------------------------------------------------------
@pytest.mark.parametrize("shape", [(64, 64, 32), (100, 70, 32), (1920, 1080, 128),
                                   (333, 129, 64), (3840, 2160, 128), (1000, 1000, 64),
                                   (127, 33, 32), (1, 1, 32), (129, 257, 128)])
@pytest.mark.parametrize("depth", [8, 10, 16])
def test_texture_matches_oracle(part, oracle, shape, depth):
    W, H, ctu = shape
    hi = (1 << depth)
    dt = np.uint8 if depth == 8 else np.uint16
    frames = RNG.integers(0, hi, size=(3, H, W)).astype(dt)
    frames[1] = hi - 1  # saturated plane: largest sums
    got = part.ctu_stats_batch(frames, ctu)
    for f in range(3):
        exp = oracle.ctu_stats(frames[f], ctu)
        g = np.stack([got[f]["count"], got[f]["sum"], got[f]["sumsq"]], axis=1)
        assert np.array_equal(g, exp), (shape, depth, f)


@pytest.mark.parametrize("shape", [(1920, 1080, 128), (3840, 2160, 128), (129, 257, 128),
                                   (7680, 4320, 128), (144, 128, 128)])
@pytest.mark.parametrize("depth", [8, 10])
@pytest.mark.parametrize("ctas", ["1", "2", "3"])
def test_texture_tma_path_matches_oracle(part, oracle, shape, depth, ctas, monkeypatch):
    """K1 through the TMA-staged kernel (SLICECRAFT_B200_K1=tma; the ring of 4 / 3 / 2
    stages with 1 / 2 / 3 CTAs per SM): tensor-map zero fill handles the partial border
    CTUs.  Same records as the oracle's ctu_stats (texture.cpp:145-169)."""
    monkeypatch.setenv("SLICECRAFT_B200_K1", "tma")
    monkeypatch.setenv("SLICECRAFT_B200_K1_CTAS", ctas)
    W, H, ctu = shape
    hi = (1 << depth)
    dt = np.uint8 if depth == 8 else np.uint16
    nf = 2 if W < 7680 else 1
    frames = RNG.integers(0, hi, size=(nf, H, W)).astype(dt)
    frames[nf - 1] = hi - 1
    got = part.ctu_stats_batch(frames, ctu)
    for f in range(nf):
        exp = oracle.ctu_stats(frames[f], ctu)
        g = np.stack([got[f]["count"], got[f]["sum"], got[f]["sumsq"]], axis=1)
        assert np.array_equal(g, exp), (shape, depth, f)


def test_texture_spec_kats(part):
    k = json.load(open(os.path.join(GOLDEN, "spec_kats.json")))
    c = k["constant_100"]
    got = part.ctu_stats_batch(np.full((c["h"], c["w"]), 100, np.uint8), c["ctu"])[0]
    assert [list(r) for r in got.tolist()] == c["records"]
    wp = k["white_pixel"]
    p = np.zeros((wp["h"], wp["w"]), np.uint8)
    p[wp["pixel"][1], wp["pixel"][0]] = 255
    got = part.ctu_stats_batch(p, wp["ctu"])[0]
    assert [list(r) for r in got.tolist()] == wp["records"]


# ---- K2/K3 tables ---------------------------------------------------------------
@pytest.mark.parametrize("grid", [(15, 9), (30, 17), (7, 5), (1, 1), (60, 34)])
def test_rect_tables_bit_exact(part, oracle, grid):
    from paper_2012_14792_b200 import CtuGrid
    cols, rows = grid
    g = CtuGrid.make(cols * 128 - 50, rows * 128 - 3, 128)
    F = 3
    est = RNG.lognormal(0, 0.8, size=(F, cols * rows))
    est[1] = np.round(est[1] * 4) / 4
    luma = RNG.integers(0, 1024, size=(F, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 128)
    rt, rs, sat = part.grid_tables(g, est, rec)
    for f in range(F):
        exp_t = oracle.rect_times(est[f], cols, rows)
        assert np.array_equal(_bits(rt[f]), _bits(exp_t))
        r3 = np.stack([rec[f]["count"], rec[f]["sum"], rec[f]["sumsq"]], axis=1)
        exp_s = oracle.rect_sse(g.frame_width, g.frame_height, 128, r3)
        assert np.array_equal(_bits(rs[f]), _bits(exp_s))


# ---- K4/K5 search -----------------------------------------------------------------
# search modes under test: exhaustive (step 2 bounded by its budget), the
# same with an unbounded step-2 walk, the exact pruned mode, and the pruned
# mode with every work item shared by several warps (forced on small grids,
# where the default keeps one warp per item)
# exhaustive step 1 runs the candidate-trace interpreter (trace.cu) by
# default; "exhaustive-dfs" forces the warp-uniform DFS walk instead
MODES = ["exhaustive", "exhaustive-full", "exhaustive-dfs", "pruned", "pruned-split"]


def _mode(monkeypatch, m):
    if m == "exhaustive-full":
        monkeypatch.setenv("SLICECRAFT_B200_STEP2_BOUND", "0")
    if m == "exhaustive-dfs":
        monkeypatch.setenv("SLICECRAFT_B200_TRACE", "0")
    if m == "pruned-split":
        monkeypatch.setenv("SLICECRAFT_B200_SPLIT", "5")
        monkeypatch.setenv("SLICECRAFT_B200_SPLIT2", "3")
        monkeypatch.setenv("SLICECRAFT_B200_SPLIT_DEPTH", "3")
    return 1 if m.startswith("pruned") else 0


def _rec3(rec):
    return np.stack([rec["count"], rec["sum"], rec["sumsq"]], axis=1)


@pytest.mark.parametrize("m", MODES)
def test_search_small_golden(part, monkeypatch, m):
    """200 reference-generated instances: step 1 and step 2, bit-exact, in the
    exhaustive and the exact pruned mode."""
    from paper_2012_14792_b200 import RECORD_DTYPE, CtuGrid, SearchConfig, SlicecraftError
    mode = _mode(monkeypatch, m)
    cases = json.load(open(os.path.join(GOLDEN, "search_small.json")))
    for i, c in enumerate(cases):
        g = CtuGrid.make(c["w"], c["h"], c["ctu"])
        cfg = SearchConfig(n_slices=c["n"], lambda_=c["lambda"], k_area=c["k"],
                           max_tile_cols=c["max_tile_cols"], mode=mode)
        rec = np.zeros(g.cell_count(), RECORD_DTYPE)
        r3 = np.array(c["records"], dtype=np.uint64)
        rec["count"], rec["sum"], rec["sumsq"] = r3[:, 0], r3[:, 1], r3[:, 2]
        est = np.array(c["est"])
        if c["status1"] != 0:
            with pytest.raises(SlicecraftError) as e:
                part.two_step_batch(g, est, rec, cfg)
            assert e.value.status == c["status1"], i
            continue
        o = part.two_step_batch(g, est, rec, cfg)[0]
        assert o.t_min_us == c["t_min"], i
        assert o.argmin.rects() == [tuple(x) for x in c["argmin"]], i
        assert o.candidates_step1 == c["candidates"], i
        assert o.t_best_us == c["t_best"], i
        assert o.sse_best == c["sse_best"], i
        assert o.best.rects() == [tuple(x) for x in c["best"]], i
        assert o.candidates_step2 == c["candidates_step2"], i


@pytest.mark.parametrize("m", MODES)
@pytest.mark.parametrize("coverage", [0, 1])
@pytest.mark.parametrize("seed", range(6))
def test_search_random_vs_oracle(part, oracle, monkeypatch, coverage, seed, m):
    from paper_2012_14792_b200 import CtuGrid, SearchConfig, SlicecraftError
    mode = _mode(monkeypatch, m)
    rng = np.random.default_rng(seed + 100 * coverage)
    for trial in range(12):
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        g = CtuGrid.make(cols * 64, rows * 64 - int(rng.integers(0, 60)), 64)
        n = int(rng.integers(1, min(9, g.cell_count()) + 1))
        mc = int(rng.integers(0, 5))
        lam = float(rng.choice([0.0, 0.1, 0.3, 1.0]))
        k = float(rng.choice([3.0, 2.5, 2.0, 1.2]))  # 1.2: single areas can fail (patho)
        F = int(rng.integers(1, 5))
        est = rng.lognormal(0, 0.6, size=(F, g.cell_count()))
        if trial % 3 == 0:
            est = np.round(est)
        luma = rng.integers(0, 1024, size=(F, g.frame_height, g.frame_width)).astype(np.uint16)
        rec = part.ctu_stats_batch(luma, 64)
        cfg = SearchConfig(n_slices=n, lambda_=lam, k_area=k, max_tile_cols=mc, coverage=coverage,
                           mode=mode)
        exp = [oracle.search(g.frame_width, g.frame_height, 64, est[f], _rec3(rec[f]), n, lam, k,
                             mc, coverage, 3) for f in range(F)]
        if any(st != 0 for st, _ in exp):
            with pytest.raises(SlicecraftError):
                part.two_step_batch(g, est, rec, cfg)
            continue
        got = part.two_step_batch(g, est, rec, cfg)
        for f in range(F):
            _, e = exp[f]
            o = got[f]
            ctx = (seed, trial, f, cols, rows, n, mc, lam, k)
            assert o.t_min_us == e.t_min_us, ctx
            assert o.argmin.rects() == e.argmin1.slices(rows), ctx
            assert o.candidates_step1 == e.candidates_step1, ctx
            assert o.t_best_us == e.t_best_us, ctx
            assert o.sse_best == e.sse_best, ctx
            assert o.best.rects() == e.best.slices(rows), ctx
            assert o.candidates_step2 == e.candidates_step2, ctx


def test_constrained_with_given_tmin(part, oracle):
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    g = CtuGrid.make(8 * 64, 6 * 64, 64)
    est = RNG.lognormal(0, 0.7, size=(2, g.cell_count()))
    luma = RNG.integers(0, 1024, size=(2, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 64)
    cfg = SearchConfig(n_slices=5, lambda_=0.3)
    tm = [float(est[0].sum() / 3), float(est[1].max() * 2)]
    got = part.constrained_clustering_batch(g, est, rec, tm, cfg)
    for f in range(2):
        st, e = oracle.search(g.frame_width, g.frame_height, 64, est[f], _rec3(rec[f]), 5, 0.3, 3.0,
                              0, 0, 2, tm[f])
        assert st == 0
        assert got[f].t_best_us == e.t_best_us and got[f].sse_best == e.sse_best
        assert got[f].best.rects() == e.best.slices(g.rows)
        assert got[f].candidates_step2 == e.candidates_step2


def test_min_time_search_api(part, oracle):
    from paper_2012_14792_b200 import CostMap, CtuGrid, SearchConfig
    g = CtuGrid.make(1920, 1080)
    est = RNG.lognormal(0, 0.5, g.cell_count())
    t, p = part.min_time_search(CostMap(g, est), SearchConfig(n_slices=4, max_tile_cols=2))
    st, e = oracle.search(1920, 1080, 128, est, None, 4, 0.0, 3.0, 2, 0, 1)
    assert t == e.t_min_us and p.rects() == e.argmin1.slices(g.rows)


# ---- BASELINE configs on their synthetic inputs ------------------------------------
def _config_inputs(ci, frames):
    from paper_2012_14792_b200 import workloads as wl
    w = wl.WORKLOADS[ci]
    frames = w.frames if frames is None else frames
    return w, wl.cost_trace(w, frames=frames), wl.synth_luma(w, frames=frames)


@pytest.mark.parametrize("m", MODES)
@pytest.mark.parametrize("ci", [1, 2, 3])
def test_baseline_configs_vs_reference_golden(part, monkeypatch, ci, m):
    """cfg1 (all), cfg2 (POC 1..4), cfg3 (POC 1) against the reference itself."""
    import hashlib
    mode = _mode(monkeypatch, m)
    from paper_2012_14792_b200 import workloads as wl
    gold = json.load(open(os.path.join(GOLDEN, "configs.json")))[str(ci)]
    F = max(fr["poc"] for fr in gold["frames"])
    w, tr, luma = _config_inputs(ci, F)
    g = w.grid()
    rec = np.zeros((F, g.cell_count()), dtype=__import__(
        "paper_2012_14792_b200").RECORD_DTYPE)
    res = part.partition_frames(g, luma, tr.est, w.cfg(mode=mode), records_out=rec)
    for fr in gold["frames"]:
        p = fr["poc"]
        r3 = np.ascontiguousarray(_rec3(rec[p - 1]), dtype=np.uint64)
        assert hashlib.sha256(r3.tobytes()).hexdigest()[:16] == fr["records_hash"]
        assert hashlib.sha256(np.ascontiguousarray(tr.est[p - 1]).tobytes()).hexdigest()[:16] == \
            fr["est_hash"]
        r = res[p - 1]
        from paper_2012_14792_b200.partitioner import Partition
        assert r.t_min_us == fr["t_min"]
        assert r.t_best_us == fr["t_best"]
        assert r.sse_best == fr["sse_best"]
        assert Partition.from_layout(g, r.best).rects() == [tuple(x) for x in fr["best"]]
        assert r.candidates_step1 == fr["candidates_step1"]
        assert r.candidates_step2 == fr["candidates_step2"]
        assert tr.est_source[p - 1] == fr["est_source"]
        assert tr.est_source_poc[p - 1] == fr["est_source_poc"]
    assert wl  # noqa


@pytest.mark.parametrize("m", ["exhaustive", "pruned"])
@pytest.mark.parametrize("ci", [1, 2, 3])
def test_baseline_configs_lambda_vs_reference_golden(part, monkeypatch, ci, m):
    """lambda in {0.1, 0.3} on cfg1 (POC 1), cfg2 (POC 1..2) and
    cfg3 (POC 1) against the reference's own two_step_partition outputs."""
    import hashlib
    mode = _mode(monkeypatch, m)
    from paper_2012_14792_b200 import RECORD_DTYPE
    from paper_2012_14792_b200.partitioner import Partition
    gold = json.load(open(os.path.join(GOLDEN, "configs_lambda.json")))[str(ci)]
    F = max(fr["poc"] for fr in gold["frames"])
    w, tr, luma = _config_inputs(ci, F)
    g = w.grid()
    for lam in sorted({fr["lambda"] for fr in gold["frames"]}):
        rec = np.zeros((F, g.cell_count()), dtype=RECORD_DTYPE)
        res = part.partition_frames(g, luma, tr.est, w.cfg(mode=mode, lambda_=lam),
                                    records_out=rec)
        for fr in gold["frames"]:
            if fr["lambda"] != lam:
                continue
            p = fr["poc"]
            r3 = np.ascontiguousarray(_rec3(rec[p - 1]), dtype=np.uint64)
            assert hashlib.sha256(r3.tobytes()).hexdigest()[:16] == fr["records_hash"]
            r = res[p - 1]
            ctx = (ci, p, lam, m)
            assert r.t_min_us == fr["t_min"], ctx
            assert r.t_best_us == fr["t_best"], ctx
            assert r.sse_best == fr["sse_best"], ctx
            assert Partition.from_layout(g, r.best).rects() == [tuple(x) for x in fr["best"]], ctx
            assert r.candidates_step1 == fr["candidates_step1"], ctx
            assert r.candidates_step2 == fr["candidates_step2"], ctx


@pytest.mark.parametrize("m", ["exhaustive", "pruned"])
@pytest.mark.parametrize("ci,frames", [(1, 1), (2, 2), (3, 1)])
def test_baseline_configs_covering_vs_oracle(part, oracle, monkeypatch, ci, frames, m):
    """The covering family (sum of widths = cols) on the
    cfg1-3 inputs, lambda 0 and 0.3, against the C oracle (pinned to the
    reference's primitives in test_oracle_pin)."""
    mode = _mode(monkeypatch, m)
    from paper_2012_14792_b200 import RECORD_DTYPE
    from paper_2012_14792_b200.partitioner import Partition
    w, tr, luma = _config_inputs(ci, frames)
    g = w.grid()
    for lam in (0.0, 0.3):
        rec = np.zeros((frames, g.cell_count()), dtype=RECORD_DTYPE)
        res = part.partition_frames(g, luma, tr.est, w.cfg(mode=mode, lambda_=lam, coverage=1),
                                    records_out=rec)
        for f in range(frames):
            st, e = oracle.search(w.width, w.height, w.ctu, tr.est[f], _rec3(rec[f]), w.n_slices,
                                  lam, 3.0, w.max_tile_cols, 1, 3)
            assert st == 0
            r = res[f]
            ctx = (ci, f, lam, m)
            assert r.t_min_us == e.t_min_us, ctx
            assert r.t_best_us == e.t_best_us and r.sse_best == e.sse_best, ctx
            assert Partition.from_layout(g, r.best).rects() == e.best.slices(g.rows), ctx
            assert r.candidates_step1 == e.candidates_step1, ctx
            assert r.candidates_step2 == e.candidates_step2, ctx
            assert sum(Partition.from_layout(g, r.best).col_widths) == g.cols, ctx


def test_cfg2_all_frames_vs_oracle(part, oracle):
    """All 64 frames of config 2 (two GPU frame groups) against the C oracle."""
    w, tr, luma = _config_inputs(2, 64)
    g = w.grid()
    from paper_2012_14792_b200 import RECORD_DTYPE
    rec = np.zeros((64, g.cell_count()), dtype=RECORD_DTYPE)
    res = part.partition_frames(g, luma, tr.est, w.cfg(), records_out=rec)
    from paper_2012_14792_b200.partitioner import Partition
    for f in range(0, 64, 3):
        st, e = oracle.search(w.width, w.height, 128, tr.est[f], _rec3(rec[f]), 8, 0.0, 3.0, 4, 0, 3)
        assert st == 0
        r = res[f]
        assert r.t_min_us == e.t_min_us and r.t_best_us == e.t_best_us and r.sse_best == e.sse_best
        assert Partition.from_layout(g, r.best).rects() == e.best.slices(g.rows)
        assert r.candidates_step1 == e.candidates_step1 == 171788


@pytest.mark.parametrize("m", MODES)
@pytest.mark.parametrize("world", [2, 3])
def test_candidate_space_shards(part, oracle, monkeypatch, m, world):
    """Candidate-space sharding through the product library: shard r walks
    work items r, r+world, ... (sc_ctx_set_shard), exports its per-frame best
    (sc_shard_export), and sc_shard_merge combines the rank-major records --
    step 1, then step 2 under the merged t_min.  The shards run one after the
    other on this GPU (no rank waits on another); the merge equals the oracle."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    from paper_2012_14792_b200._abi import SearchResult
    from paper_2012_14792_b200.partitioner import Partition, shard_merge
    mode = _mode(monkeypatch, m)
    rng = np.random.default_rng(11 + world)
    g = CtuGrid.make(7 * 64, 6 * 64, 64)
    F, n, lam = 3, 6, 0.25
    est = rng.lognormal(0, 0.5, size=(F, g.cell_count()))
    luma = rng.integers(0, 1024, size=(F, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 64)
    cfg = SearchConfig(n_slices=n, lambda_=lam, k_area=3.0, max_tile_cols=4, mode=mode)
    merged = {}
    try:
        for step in (1, 2):
            blobs = b""
            for r in range(world):
                part.set_shard(r, world)
                if step == 1:
                    part.min_time_search_batch(g, est, cfg)
                else:
                    tmin = np.array([merged[1][f].t_min_us for f in range(F)])
                    part.constrained_clustering_batch(g, est, rec, tmin, cfg)
                blobs += bytes(part.shard_export(step, F))
            res = (SearchResult * F)()
            for f in range(F):
                res[f].argmin.n_slices = n
                res[f].best.n_slices = n
            shard_merge(step, world, F, blobs, res)
            merged[step] = res
    finally:
        part.set_shard(0, 1)
    for f in range(F):
        st, e = oracle.search(g.frame_width, g.frame_height, 64, est[f], _rec3(rec[f]), n, lam, 3.0,
                              4, 0, 3)
        assert st == 0
        r1, r2 = merged[1][f], merged[2][f]
        assert r1.t_min_us == e.t_min_us and r1.candidates_step1 == e.candidates_step1, (m, f)
        assert Partition.from_layout(g, r1.argmin).rects() == e.argmin1.slices(g.rows), (m, f)
        assert r2.t_best_us == e.t_best_us and r2.sse_best == e.sse_best, (m, f)
        assert r2.candidates_step2 == e.candidates_step2, (m, f)
        assert Partition.from_layout(g, r2.best).rects() == e.best.slices(g.rows), (m, f)


def test_cost_ordered_schedule_keeps_first_in_order(part, oracle):
    """The first exhaustive call measures each work item's walk cost, later
    calls take the items by decreasing cost; with heavily tied times the
    argmin is still the reference's first-in-order one on every call."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    from paper_2012_14792_b200.partitioner import Partition
    rng = np.random.default_rng(99)
    g = CtuGrid.make(9 * 64, 7 * 64, 64)
    F = 6
    est = np.round(rng.lognormal(0, 0.3, size=(F, g.cell_count())) * 2) / 2
    cfg = SearchConfig(n_slices=6, lambda_=0.0, k_area=3.0, max_tile_cols=4)
    exp = [oracle.search(g.frame_width, g.frame_height, 64, est[f], None, 6, 0.0, 3.0, 4, 0, 1)
           for f in range(F)]
    for call in range(3):
        out = part.min_time_search_batch(g, est, cfg)
        for f in range(F):
            st, e = exp[f]
            assert st == 0
            assert out[f].t_min_us == e.t_min_us, (call, f)
            assert out[f].argmin.rects() == e.argmin1.slices(g.rows), (call, f)
            assert out[f].candidates_step1 == e.candidates_step1


@pytest.mark.parametrize("chunks", ["1", "64", "100000"])
@pytest.mark.parametrize("coverage", [0, 1])
def test_trace_chunk_cuts_inside_skeletons(oracle, chunks, coverage, monkeypatch):
    """The trace is cut into chunks at SKEL ops and at depth-0 pushes (a chunk
    that starts inside a skeleton replays its SKEL + FIX prologue).  Whatever
    the chunk size (SLICECRAFT_B200_TRACE_CHUNKS, read when the plan's trace
    is built: one chunk per SM ... 16-op chunks), both trace walks return the
    oracle's results: t_min, argmin, (sse, t, first-in-order) winner, counts."""
    from paper_2012_14792_b200 import CtuGrid, Partitioner, SearchConfig
    monkeypatch.setenv("SLICECRAFT_B200_TRACE_CHUNKS", chunks)
    monkeypatch.setenv("SLICECRAFT_B200_TRACE2", "1")
    rng = np.random.default_rng(4178)
    g = CtuGrid.make(14 * 64, 10 * 64, 64)
    F = 5
    # coarse values: many tied times and SSEs, so order decides
    est = np.round(rng.lognormal(0, 0.4, size=(F, g.cell_count())) * 4) / 4
    rec = np.zeros((F, g.cell_count(), 3), np.uint64)
    rec[..., 0] = 64 * 64
    mean = rng.integers(0, 64, size=(F, g.cell_count())).astype(np.uint64) * 16
    rec[..., 1] = mean * 4096
    rec[..., 2] = mean * mean * 4096 + rng.integers(0, 8, size=mean.shape).astype(np.uint64) * 4096
    cfg = SearchConfig(n_slices=7, lambda_=0.25, k_area=3.0, max_tile_cols=0,
                       coverage=coverage)
    exp = [oracle.search(g.frame_width, g.frame_height, 64, est[f], rec[f], 7, 0.25, 3.0, 0,
                         coverage, 3) for f in range(F)]
    p = Partitioner(0)
    try:
        for call in range(2):
            res = p.two_step_batch(g, est, rec, cfg)
            for f in range(F):
                st, e = exp[f]
                assert st == 0
                r = res[f]
                assert r.t_min_us == e.t_min_us and r.t_best_us == e.t_best_us, (call, f)
                assert r.sse_best == e.sse_best, (call, f)
                assert r.candidates_step1 == e.candidates_step1
                assert r.candidates_step2 == e.candidates_step2
                assert r.best.rects() == e.best.slices(g.rows), (call, f)
                assert r.argmin.rects() == e.argmin1.slices(g.rows), (call, f)
    finally:
        p.close()


def test_cfg3_counts_all_frames(part):
    """Size-independent checks on the full cfg3 batch: counts, budget, feasibility."""
    w, tr, luma = _config_inputs(3, 32)
    g = w.grid()
    res = part.partition_frames(g, luma, tr.est, w.cfg())
    for r in res:
        assert r.candidates_step1 == r.candidates_step2 == 66007331
        assert r.t_best_us <= r.t_min_us * (1.0 + 0.0)  # lambda = 0: t_best == t_min
        assert r.t_best_us == r.t_min_us


# ---- configs 4 and 5 (exact pruned mode) ---------------------------------------------
# Survey-verified exact candidate counts (reference enumeration ladder + the
# counting DP): the reference's own counters.
CFG_COUNTS = {4: 5362975262506, 5: 610308283606383278175018310268}


def _check_result_properties(oracle, w, g, est, rec, r, lam=0.0):
    """Size-independent checks of one frame's result: the returned layouts are
    admissible, their times / SSE recomputed by the CPU oracle from its own
    rectangle tables equal t_min / t_best / sse_best, t_best is within budget."""
    from paper_2012_14792_b200.partitioner import Partition
    nyh = g.rows * (g.rows + 1) // 2
    rt = oracle.rect_times(est, g.cols, g.rows)
    rs = oracle.rect_sse(w.width, w.height, w.ctu, _rec3(rec))

    def rid(s):
        return (s[0] * g.cols - s[0] * (s[0] - 1) // 2 + s[2] - 1) * nyh + \
            (s[1] * g.rows - s[1] * (s[1] - 1) // 2 + s[3] - 1)
    for L, tref in ((r.argmin, r.t_min_us), (r.best, r.t_best_us)):
        rects = Partition.from_layout(g, L).rects()
        assert len(rects) == w.n_slices
        areas = [s[2] * s[3] for s in rects]
        assert 3.0 * min(areas) > max(areas)
        t = 0.0
        for s in rects:
            t = max(t, rt[rid(s)])
        assert t == tref
    sse = 0.0
    for s in Partition.from_layout(g, r.best).rects():
        sse += rs[rid(s)]
    assert sse == r.sse_best
    assert r.t_best_us <= r.t_min_us * (1.0 + lam)


@pytest.mark.parametrize("ci", [4, 5])
def test_cfg4_cfg5_pruned(part, oracle, ci):
    """Every frame of configs 4 and 5: the GPU's exact pruned search against the
    oracle's independent branch-and-bound restatement (bit-exact), the exact
    counts, and size-independent properties of the returned partitions."""
    from paper_2012_14792_b200 import RECORD_DTYPE
    from paper_2012_14792_b200.partitioner import Partition
    w, tr, luma = _config_inputs(ci, None)
    g = w.grid()
    F = w.frames
    rec = np.zeros((F, g.cell_count()), dtype=RECORD_DTYPE)
    res = part.partition_frames(g, luma, tr.est, w.cfg(mode=1), records_out=rec)
    for f in range(F):
        r = res[f]
        cnt = r.candidates_step1 | (r.candidates_step1_hi << 64)
        assert cnt == CFG_COUNTS[ci] == (r.candidates_step2 | (r.candidates_step2_hi << 64))
        _check_result_properties(oracle, w, g, tr.est[f], rec[f], r)
        st, e = oracle.search_pruned(w.width, w.height, w.ctu, tr.est[f], _rec3(rec[f]),
                                     w.n_slices, 0.0, 3.0, w.max_tile_cols, 0, 3)
        assert st == 0
        assert r.t_min_us == e.t_min_us and r.t_best_us == e.t_best_us
        assert r.sse_best == e.sse_best
        assert Partition.from_layout(g, r.argmin).rects() == e.argmin1.slices(g.rows)
        assert Partition.from_layout(g, r.best).rects() == e.best.slices(g.rows)


@pytest.mark.parametrize("ci", [2, 3])
def test_exhaustive_and_pruned_agree_all_frames(part, ci):
    """Both search modes give identical results on every frame of cfg2/cfg3."""
    w, tr, luma = _config_inputs(ci, None)
    g = w.grid()
    a = part.partition_frames(g, luma, tr.est, w.cfg(mode=0))
    b = part.partition_frames(g, luma, tr.est, w.cfg(mode=1))
    from paper_2012_14792_b200.partitioner import Partition
    for x, y in zip(a, b):
        assert x.t_min_us == y.t_min_us and x.t_best_us == y.t_best_us and x.sse_best == y.sse_best
        assert x.candidates_step1 == y.candidates_step1 and x.candidates_step2 == y.candidates_step2
        assert Partition.from_layout(g, x.argmin).rects() == Partition.from_layout(g, y.argmin).rects()
        assert Partition.from_layout(g, x.best).rects() == Partition.from_layout(g, y.best).rects()


# ---- error behaviour -----------------------------------------------------------------
def test_errors(part):
    from paper_2012_14792_b200 import CtuGrid, SearchConfig, SlicecraftError
    g = CtuGrid.make(256, 128, 128)  # 2x1 cells
    est = np.ones((1, 2))
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g, est, SearchConfig(n_slices=3))
    assert e.value.kind == "GeometryError"
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g, est, SearchConfig(n_slices=1, k_area=1.0))
    assert e.value.kind == "ConfigError"
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g, est, SearchConfig(n_slices=1, lambda_=float("nan")))
    assert e.value.kind == "ConfigError"
    # k so tight that no candidate is admissible -> NoCandidateError
    g4 = CtuGrid.make(4 * 128, 128, 128)
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g4, np.ones((1, 4)), SearchConfig(n_slices=3, k_area=1.0001,
                                                                    max_tile_cols=1))
    assert e.value.kind == "NoCandidateError"
    from paper_2012_14792_b200 import RECORD_DTYPE
    bad = np.zeros((1, 2), RECORD_DTYPE)
    with pytest.raises(SlicecraftError) as e:
        part.two_step_batch(g, est, bad, SearchConfig(n_slices=1))
    assert e.value.kind == "FormatError"


@pytest.mark.parametrize("m", MODES)
def test_edge_shapes_vs_oracle(part, oracle, monkeypatch, m):
    """Edge shapes: one cell; one column of 64 rows cut into the maximum 64
    slices (63-level heights DFS); a single-row grid; partial border CTUs; a
    ragged frame batch (35 frames = one full 32-frame group + 3 in the next)."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    from paper_2012_14792_b200.partitioner import Partition
    mode = _mode(monkeypatch, m)
    rng = np.random.default_rng(77)
    cases = [((64, 64, 64), 1, 0, 1), ((64, 64 * 64, 64), 64, 0, 1),
             ((64, 18 * 64, 64), 12, 1, 2), ((12 * 64, 64, 64), 5, 0, 3),
             ((5 * 64 - 17, 4 * 64 - 33, 64), 6, 0, 2), ((6 * 64, 5 * 64, 64), 5, 4, 35)]
    for (W, H, ctu), n, mc, F in cases:
        g = CtuGrid.make(W, H, ctu)
        est = rng.lognormal(0, 0.5, size=(F, g.cell_count()))
        luma = rng.integers(0, 1024, size=(F, H, W)).astype(np.uint16)
        rec = part.ctu_stats_batch(luma, ctu)
        cfg = SearchConfig(n_slices=n, lambda_=0.2, k_area=3.0, max_tile_cols=mc, mode=mode)
        got = part.two_step_batch(g, est, rec, cfg)
        for f in range(F):
            st, e = oracle.search(W, H, ctu, est[f], _rec3(rec[f]), n, 0.2, 3.0, mc, 0, 3)
            ctx = (W, H, n, mc, F, f, m)
            assert st == 0, ctx
            o = got[f]
            assert o.t_min_us == e.t_min_us and o.candidates_step1 == e.candidates_step1, ctx
            assert o.argmin.rects() == e.argmin1.slices(g.rows), ctx
            assert o.t_best_us == e.t_best_us and o.sse_best == e.sse_best, ctx
            assert o.best.rects() == e.best.slices(g.rows), ctx
            assert o.candidates_step2 == e.candidates_step2, ctx


def test_graph_replay_sees_new_inputs(part, oracle):
    """The time-table phase is captured into a CUDA graph on the second call of
    a shape and replayed afterwards: every call must still read its own
    estimate maps (new data in the same buffers) and match the oracle."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    g = CtuGrid.make(9 * 64, 7 * 64, 64)
    rng = np.random.default_rng(5)
    cfg = SearchConfig(n_slices=6, lambda_=0.1, max_tile_cols=3)
    luma = rng.integers(0, 1024, size=(3, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 64)
    for call in range(4):
        est = rng.lognormal(0, 0.6, size=(3, g.cell_count()))
        got = part.two_step_batch(g, est, rec, cfg)
        for f in range(3):
            st, e = oracle.search(g.frame_width, g.frame_height, 64, est[f], _rec3(rec[f]), 6,
                                  0.1, 3.0, 3, 0, 3)
            assert st == 0
            assert got[f].t_min_us == e.t_min_us and got[f].sse_best == e.sse_best, (call, f)
            assert got[f].best.rects() == e.best.slices(g.rows), (call, f)


def test_size_limits(part):
    """Requests beyond the compiled limits fail with SizeError,
    the reference's own checks keep their classes."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig, SlicecraftError
    g = CtuGrid.make(64, 65 * 64, 64)  # 1 x 65 cells
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g, np.ones((1, 65)), SearchConfig(n_slices=65))
    assert e.value.kind == "SizeError"
    g = CtuGrid.make(256 * 64, 64, 64)  # 256 columns
    with pytest.raises(SlicecraftError) as e:
        part.min_time_search_batch(g, np.ones((1, 256)), SearchConfig(n_slices=2))
    assert e.value.kind == "SizeError"


# ---- UniformOnly family and partition evaluation -----------
def _uniform_gold():
    return json.load(open(os.path.join(GOLDEN, "uniform.json")))


def test_uniform_only_family_vs_reference_golden(part):
    """min_time_search / constrained_clustering_search / two_step with the
    UniformOnly family (search.cpp:265-275, 349-364) against the reference:
    values, counts, the uniform Partition, and the NoCandidateError cases
    (area constraint; time budget)."""
    from paper_2012_14792_b200 import RECORD_DTYPE, CtuGrid, SearchConfig, SlicecraftError
    for i, c in enumerate(_uniform_gold()["searches"]):
        g = CtuGrid.make(c["w"], c["h"], c["ctu"])
        cfg = SearchConfig(n_slices=c["n"], lambda_=c["lambda"], k_area=c["k"], family=1)
        est = np.array(c["est"])[None]
        rec = np.zeros((1, g.cell_count()), RECORD_DTYPE)
        r3 = np.array(c["records"], dtype=np.uint64)
        rec["count"], rec["sum"], rec["sumsq"] = r3[:, 0], r3[:, 1], r3[:, 2]
        if c["status1"] != 0:
            with pytest.raises(SlicecraftError) as e:
                part.min_time_search_batch(g, est, cfg)
            assert e.value.status == c["status1"], i
            assert part.count_candidates(g, cfg) == 0
            continue
        assert part.count_candidates(g, cfg) == 1
        o1 = part.min_time_search_batch(g, est, cfg)[0]
        assert o1.t_min_us == c["t_min"], i
        assert o1.argmin.rects() == [tuple(x) for x in c["argmin"]], i
        assert o1.argmin.origin == "uniform"
        o2 = part.constrained_clustering_batch(g, est, rec, [c["t_min"]], cfg)[0]
        assert c["status2"] == 0
        assert o2.t_best_us == c["t_best"] and o2.sse_best == c["sse_best"], i
        assert o2.best.rects() == [tuple(x) for x in c["best"]], i
        assert o2.candidates_step2 == c["candidates_step2"] == 1
        assert o2.candidates_evaluated == c["candidates_evaluated"]
        o3 = part.two_step_batch(g, est, rec, cfg)[0]
        assert (o3.t_min_us, o3.t_best_us, o3.sse_best) == (c["t_min"], c["t_best"], c["sse_best"])
        assert (o3.candidates_step1, o3.candidates_step2, o3.candidates_evaluated) == (1, 1, 2)
        over = SearchConfig(n_slices=c["n"], lambda_=0.0, k_area=c["k"], family=1)
        with pytest.raises(SlicecraftError) as e:
            part.constrained_clustering_batch(g, est, rec, [c["t_min"] * 0.5], over)
        assert e.value.status == c["status_over"] == 10


def test_partition_eval_vs_reference_golden(part):
    """sc_partition_eval == partition_time (cost.cpp:117-145: max from slice 0
    with strict >, total in id order, raw sums incl. negative times) and
    partition_sse (texture.cpp:183-189) of the reference, bit for bit; the
    per-slice values equal the oracle's rectangle tables."""
    from paper_2012_14792_b200 import RECORD_DTYPE, CtuGrid
    from paper_2012_14792_b200.partitioner import Partition, Slice
    for i, c in enumerate(_uniform_gold()["evals"]):
        g = CtuGrid.make(c["w"], c["h"], c["ctu"])
        p = Partition(g, [], [g.rows], [Slice(*s) for s in c["slices"]])
        rec = np.zeros((1, g.cell_count()), RECORD_DTYPE)
        r3 = np.array(c["records"], dtype=np.uint64)
        rec["count"], rec["sum"], rec["sumsq"] = r3[:, 0], r3[:, 1], r3[:, 2]
        est = np.array(c["est"])[None]
        res, st, sm = part.partition_eval(p, est, rec, slice_values=True)
        assert c["status"] == 0
        r = res[0]
        assert (r["max_us"], r["total_us"], r["argmax"], r["sse"]) == \
            (c["max_us"], c["total_us"], c["argmax"], c["sse"]), i
        for s in c["slices"]:  # slice moments by id
            x0, y0, w, h, sid = s
            cells = [(y, x) for y in range(y0, y0 + h) for x in range(x0, x0 + w)]
            tot = r3[[y * g.cols + x for y, x in cells]].sum(axis=0)
            assert tuple(int(v) for v in sm[0][sid]) == tuple(int(v) for v in tot), (i, sid)
    # batch of frames, est only / records only
    g = CtuGrid.make(8 * 32, 5 * 32, 32)
    p = Partition.uniform(g, 6)
    rng = np.random.default_rng(5)
    est = rng.lognormal(0, 0.5, size=(7, g.cell_count()))
    res = part.partition_eval(p, est=est)
    assert len(res) == 7 and all(r["argmax"] >= 0 for r in res)
