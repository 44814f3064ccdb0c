"""CPU check of the search-kernel LOGIC: the very walk code the GPU runs
(csrc/search_walk.cuh), compiled for the host by the test-only emulator in
tests/emu and executed lane by lane, against the C oracle on seeded random
instances -- both steps, both coverage modes, every frames-per-warp width
(hence every leaf-loop split J = 32 / FPW), several work-item granularities.
The GPU parity tests (test_gpu_parity.py) then check the compiled kernels."""
import numpy as np
import pytest


def _case(rng, max_cells=9):
    cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    n = int(rng.integers(1, min(max_cells, cols * rows) + 1))
    return cols, rows, n


@pytest.mark.parametrize("prune", [0, 1])
@pytest.mark.parametrize("seed", range(4))
def test_step1_vs_oracle(emu, oracle, seed, prune):
    from emu.emu import Emu
    rng = np.random.default_rng(seed)
    for trial in range(60):
        cols, rows, n = _case(rng, 10)
        mc = int(rng.integers(0, 5))
        k = float(rng.choice([3.0, 2.5, 2.0, 1.5]))
        cov = int(rng.integers(0, 2))
        F = int(rng.choice([1, 2, 3, 4, 8, 32]))
        est = rng.lognormal(0, 0.6, size=(F, cols * rows))
        if trial % 3 == 0:
            est = np.round(est)
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        tgt = int(rng.choice([1, 16, 100000]))
        t, _, cnt, snap, found = emu.search(cols, rows, n, k, mc, cov, 1, rt, item_target=tgt,
                                            warps=int(rng.integers(1, 5)), prune=prune)
        for f in range(F):
            st, r = oracle.search(cols * 64, rows * 64, 64, est[f], None, n, 0.0, k, mc, cov, 1)
            if st:
                assert not found[f]
                continue
            ctx = (seed, trial, f, cols, rows, n, mc, k, cov, F)
            assert t[f] == r.t_min_us, ctx
            assert cnt[f] == r.candidates_step1, ctx
            assert Emu.slices(snap[f], n, rows) == r.argmin1.slices(rows), ctx


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("seed", range(3))
def test_step1_any_item_order(emu, oracle, seed, order):
    """Exhaustive step 1 with the work items taken out of enumeration order
    (reversed / permuted, as the cost-ordered schedule does): the lanes' tie
    rule still returns the reference's first-in-order argmin.  Times are
    rounded hard so that many candidates tie."""
    from emu.emu import Emu
    rng = np.random.default_rng(500 + seed)
    for trial in range(40):
        cols, rows, n = _case(rng, 9)
        mc = int(rng.integers(0, 5))
        cov = int(rng.integers(0, 2))
        F = int(rng.choice([1, 2, 4, 8, 32]))
        est = np.round(rng.lognormal(0, 0.4, size=(F, cols * rows)) * 2) / 2
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        t, _, cnt, snap, found = emu.search(cols, rows, n, 3.0, mc, cov, 1, rt,
                                            item_target=int(rng.choice([1, 16, 64])),
                                            warps=int(rng.integers(1, 5)), order=order)
        for f in range(F):
            st, r = oracle.search(cols * 64, rows * 64, 64, est[f], None, n, 0.0, 3.0, mc, cov, 1)
            if st:
                continue
            ctx = (seed, trial, f, cols, rows, n, mc, cov, F)
            assert t[f] == r.t_min_us and cnt[f] == r.candidates_step1, ctx
            assert Emu.slices(snap[f], n, rows) == r.argmin1.slices(rows), ctx


@pytest.mark.parametrize("split,depth", [(3, 0), (8, 1), (5, 2)])
def test_pruned_split_items_vs_oracle(emu, oracle, split, depth):
    """Pruned mode with `split` warps per work item: the heights subtrees below
    level `depth` (or whole small skeletons) are dealt out by a hash of their
    identity; both steps still equal the oracle."""
    from emu.emu import Emu
    rng = np.random.default_rng(700 + split)
    for trial in range(40):
        cols, rows, n = _case(rng, 10)
        mc = int(rng.integers(0, 5))
        cov = int(rng.integers(0, 2))
        lam = float(rng.choice([0.0, 0.2]))
        F = int(rng.choice([1, 2, 4, 8]))
        W, H = cols * 64, rows * 64
        est = rng.lognormal(0, 0.6, size=(F, cols * rows))
        if trial % 3 == 0:
            est = np.round(est)
        luma = rng.integers(0, 1024, size=(F, H, W)).astype(np.uint16)
        recs = [oracle.ctu_stats(luma[f], 64) for f in range(F)]
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        rs = np.stack([oracle.rect_sse(W, H, 64, recs[f]) for f in range(F)])
        res = [oracle.search(W, H, 64, est[f], recs[f], n, lam, 3.0, mc, cov, 3) for f in range(F)]
        kw = dict(item_target=int(rng.choice([1, 16])), warps=int(rng.integers(1, 5)), prune=1,
                  split=split, split_depth=depth)
        t, _, _, snap, found = emu.search(cols, rows, n, 3.0, mc, cov, 1, rt, **kw)
        for f in range(F):
            st, r = res[f]
            ctx = (split, depth, trial, f, cols, rows, n, mc, cov, F)
            if st:
                assert not found[f], ctx
                continue
            assert t[f] == r.t_min_us, ctx
            assert Emu.slices(snap[f], n, rows) == r.argmin1.slices(rows), ctx
        if any(st for st, _ in res):
            continue
        budget = np.array([r.t_min_us * (1.0 + lam) for _, r in res])
        t2, sse, _, snap2, _ = emu.search(cols, rows, n, 3.0, mc, cov, 2, rt, rs, budget, **kw)
        for f in range(F):
            r = res[f][1]
            ctx = (split, depth, trial, f, cols, rows, n, mc, cov, lam, F)
            assert t2[f] == r.t_best_us and sse[f] == r.sse_best, ctx
            assert Emu.slices(snap2[f], n, rows) == r.best.slices(rows), ctx


@pytest.mark.parametrize("prune", [0, 1])
@pytest.mark.parametrize("seed", range(3))
def test_step2_vs_oracle(emu, oracle, seed, prune):
    from emu.emu import Emu
    rng = np.random.default_rng(100 + seed)
    for trial in range(40):
        cols, rows, n = _case(rng, 9)
        mc = int(rng.integers(0, 5))
        k = float(rng.choice([3.0, 2.5, 2.0]))
        cov = int(rng.integers(0, 2))
        lam = float(rng.choice([0.0, 0.1, 0.3, 1.0]))
        F = int(rng.choice([1, 2, 3, 4, 8]))
        W, H = cols * 64, rows * 64 - int(rng.integers(0, 60))
        est = rng.lognormal(0, 0.6, size=(F, cols * rows))
        if trial % 3 == 0:
            est = np.round(est)
        luma = rng.integers(0, 1024, size=(F, H, W)).astype(np.uint16)
        if trial % 4 == 0:
            luma[:] = 7  # flat frames: SSE ties at 0
        recs = [oracle.ctu_stats(luma[f], 64) for f in range(F)]
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        rs = np.stack([oracle.rect_sse(W, H, 64, recs[f]) for f in range(F)])
        res = [oracle.search(W, H, 64, est[f], recs[f], n, lam, k, mc, cov, 3) for f in range(F)]
        if any(st != 0 for st, _ in res):
            continue
        budget = np.array([r.t_min_us * (1.0 + lam) for _, r in res])
        t, sse, cnt, snap, found = emu.search(cols, rows, n, k, mc, cov, 2, rt, rs, budget,
                                              prune=prune)
        for f in range(F):
            r = res[f][1]
            ctx = (seed, trial, f, cols, rows, n, mc, k, cov, lam, F)
            assert t[f] == r.t_best_us and sse[f] == r.sse_best, ctx
            assert cnt[f] == r.candidates_step2, ctx
            assert Emu.slices(snap[f], n, rows) == r.best.slices(rows), ctx


def test_dp_counts_match_enumeration(emu, oracle):
    """The exact counting DP (pruned mode's counters) == the oracle's
    enumerated counts on 40 random grids up to 7x7."""
    rng = np.random.default_rng(9)
    for _ in range(40):
        cols, rows = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        n = int(rng.integers(1, min(9, cols * rows) + 1))
        mc = int(rng.integers(0, 5))
        k = float(rng.choice([3.0, 2.5, 2.0, 1.5]))
        cov = int(rng.integers(0, 2))
        rt = np.ones((1, cols * (cols + 1) // 2 * (rows * (rows + 1) // 2)))
        _, _, cnt, _, _ = emu.search(cols, rows, n, k, mc, cov, 1, rt, prune=1)
        assert cnt[0] == oracle.count(cols, rows, n, k, mc, cov)


def test_baseline_grid_counts(emu, oracle):
    """cfg1 / cfg2 grids: counts of both families equal the oracle's."""
    for (cols, rows, n, mc) in [(15, 9, 4, 2), (15, 9, 8, 4)]:
        est = np.ones((1, cols * rows))
        rt = np.stack([oracle.rect_times(est[0], cols, rows)])
        for cov in (0, 1):
            _, _, cnt, _, _ = emu.search(cols, rows, n, 3.0, mc, cov, 1, rt, item_target=512)
            assert cnt[0] == oracle.count(cols, rows, n, 3.0, mc, cov)


def test_dp_counts_match_reference_ladder(emu):
    """The counting DP == the counts the UNMODIFIED reference enumerated on the
    real cfg4 (30x17) and cfg5 (60x34) grids (tests/golden/ladder.json,
    SURVEY.md §8c: 480 ... 314,959,056 candidates) and on the SPEC / survey
    instances of spec_kats.json."""
    import json
    import os
    from conftest import GOLDEN
    lad = json.load(open(os.path.join(GOLDEN, "ladder.json")))
    for c in lad["cases"]:
        cols, rows = (30, 17) if c["cfg"] == 4 else (60, 34)
        rt = np.ones((1, cols * (cols + 1) // 2 * (rows * (rows + 1) // 2)))
        _, _, cnt, _, _ = emu.search(cols, rows, c["n"], c["k"], c["max_tile_cols"], 0, 1, rt,
                                     prune=1)
        assert cnt[0] == c["candidates_step1"] == c["candidates_step2"], c
    kats = json.load(open(os.path.join(GOLDEN, "spec_kats.json")))["enumeration_counts"]
    for key, want in kats.items():
        dims, ctu, n, mc = key.split("/")
        fw, fh = map(int, dims.split("x"))
        ctu, n, mc = int(ctu), int(n[1:]), int(mc[1:])
        cols, rows = -(-fw // ctu), -(-fh // ctu)
        rt = np.ones((1, cols * (cols + 1) // 2 * (rows * (rows + 1) // 2)))
        _, _, cnt, _, _ = emu.search(cols, rows, n, 3.0, mc, 0, 1, rt, prune=1)
        assert cnt[0] == want, key


@pytest.mark.parametrize("seed", range(4))
def test_trace_step1_matches_oracle(emu, oracle, seed):
    """The candidate trace (csrc/trace.cuh, the exhaustive step-1 program):
    host build of the generator + a scalar interpreter == the oracle's
    exhaustive step 1 (t_min bit-exact, first-in-order argmin, count), on
    random grids, both families, k down to the pathological 1.05, with items
    split at several prefix depths."""
    rng = np.random.default_rng(700 + seed)
    for case in range(30):
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        n = int(rng.integers(1, min(9, cols * rows) + 1))
        mc = int(rng.integers(0, 5))
        k = float(rng.choice([3.0, 2.5, 1.5, 1.05]))
        cov = int(rng.integers(0, 2))
        F = 3
        est = rng.lognormal(0, 0.7, (F, cols * rows))
        est[1] = np.round(est[1])      # ties
        est[2, :cols * rows // 3] *= -1  # non-positive slices (clamped by the max from 0.0)
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        t, cnt, ordn, snap, found, nops = emu.trace_search(cols, rows, n, k, mc, cov, rt,
                                                           item_target=int(rng.integers(1, 64)))
        for f in range(F):
            st, e = oracle.search(cols * 32, rows * 32, 32, est[f], None, n, 0.0, k, mc, cov, 1)
            ctx = (cols, rows, n, mc, k, cov, f)
            if st != 0:
                assert not found[f] and cnt[f] == 0, ctx
                continue
            assert found[f] and cnt[f] == e.candidates_step1, ctx
            assert t[f] == e.t_min_us, ctx
            assert emu.slices(snap[f], n, rows) == e.argmin1.slices(rows), ctx


def test_trace_cfg_grids_counts_and_size(emu, oracle):
    """cfg1 / cfg2 / cfg3 grids: trace candidate counts (= the reference's);
    the trace stays within two ops per candidate."""
    for cols, rows, n, mc, want in [(15, 9, 4, 2, 1232), (15, 9, 8, 4, 171788),
                                    (30, 17, 8, 0, 66007331)]:
        est = np.ones((1, cols * rows))
        rt = np.stack([oracle.rect_times(est[0], cols, rows)])
        _, cnt, _, _, found, nops = emu.trace_search(cols, rows, n, 3.0, mc, 0, rt,
                                                     item_target=4096)
        assert cnt[0] == want
        assert nops < 2 * want


@pytest.mark.parametrize("seed", range(4))
def test_trace_step2_matches_oracle(emu, oracle, seed):
    """Step 2 through the candidate trace (host build): the SSE of every
    feasible candidate folded in slice order from the FIX tags and the
    decision path == the oracle's constrained clustering (t_best, sse_best
    bit-exact, the chosen layout), both families, several lambdas."""
    rng = np.random.default_rng(900 + seed)
    for case in range(25):
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        n = int(rng.integers(1, min(9, cols * rows) + 1))
        mc = int(rng.integers(0, 5))
        k = float(rng.choice([3.0, 2.0, 1.5]))
        cov = int(rng.integers(0, 2))
        lam = float(rng.choice([0.0, 0.1, 0.3, 1.0, 5.0]))
        F = 2
        W, H = cols * 32, rows * 32
        est = rng.lognormal(0, 0.7, (F, cols * rows))
        est[1] = np.round(est[1])
        rec = [oracle.ctu_stats(rng.integers(0, 1024, (H, W)).astype(np.uint16), 32)
               for _ in range(F)]
        rt = np.stack([oracle.rect_times(est[f], cols, rows) for f in range(F)])
        rs = np.stack([oracle.rect_sse(W, H, 32, rec[f]) for f in range(F)])
        exp = [oracle.search(W, H, 32, est[f], rec[f], n, lam, k, mc, cov, 3) for f in range(F)]
        budget = np.array([e.t_min_us * (1.0 + lam) if st == 0 else -1.0 for st, e in exp])
        t, sse, ordn, snap, found = emu.trace_step2(cols, rows, n, k, mc, cov, rt, rs, budget,
                                                    item_target=int(rng.integers(1, 64)))
        for f in range(F):
            st, e = exp[f]
            ctx = (cols, rows, n, mc, k, cov, lam, f)
            if st != 0:
                assert not found[f], ctx
                continue
            assert found[f], ctx
            assert t[f] == e.t_best_us and sse[f] == e.sse_best, ctx
            assert emu.slices(snap[f], n, rows) == e.best.slices(rows), ctx


def test_trace_encoding_and_rect_decode(emu):
    """The trace op encoding round-trips every field (csrc/trace.cuh), and the
    closed-form rectangle decode used by the finalize kernels (tr_unrank)
    inverts tr_xw / tr_yh for every (origin, extent) of every axis length."""
    assert emu.L.emu_trace_encoding_check() == 0
    for n in list(range(1, 70)) + [127, 128, 200, 255]:
        assert emu.L.emu_unrank_check(n) == 0, n
