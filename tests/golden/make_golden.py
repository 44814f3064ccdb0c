"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel to the GPU box; the reference does not.

Contents
  spec_kats.json   known-answer tests taken from the reference's SPEC examples
                   that the compiled reference passes: texture
                   (SPEC.md:134-135, 145), cost
                   plus the enumeration counts of SURVEY.md §8c.
  search_small.json  200 seeded random small instances (grids <= 6x6, n <= 6,
                   lambda in {0, .1, .3, 1}, k in {3, 2.5, 1.5}): the reference's
                   min_time_search + constrained_clustering_search outputs.
  uniform.json     UniformOnly family: uniform_partition
                   shapes, min_time_search / constrained_clustering_search
                   outputs, and partition_time / partition_sse of random
                   column partitions (ids permuted, some negative times).
  configs.json     BASELINE configs on their real synthetic inputs: cfg1 (all),
                   cfg2 (POC 1..4), cfg3 (POC 1): two_step_partition outputs,
                   with a hash of the estimate maps / records that were used.
  configs_lambda.json  the same inputs with lambda in {0.1, 0.3} (SURVEY.md
                   §8d): cfg1 (POC 1), cfg2 (POC 1..2), cfg3 (POC 1).
  validate.json    validate_partition (grid.cpp:86-184) on valid partitions and
                   on mutations hitting every error class: status + message.
  enumerate.json   for_each_candidate (search.cpp:302-320): the ordered candidate
                   lists of small spaces (full lists, or count + sha256 of the
                   list + its first / last 40 for larger ones).
  ladder.json      the reference-checkable ladder on the REAL cfg4 / cfg5 grids
                   (SURVEY.md §8c): cfg4's POC-1 inputs (30x17) at n=16 cap 1/2
                   and n=8 cap 4; cfg5's POC-1 inputs (60x34) at n=4, n=6,
                   n=8 cap 2 and n=32 cap 1 (several lambdas): the reference's
                   two_step_partition outputs (search.cpp:407-434) with the
                   estimate maps and records that were used.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_2012_14792_b200 import workloads as wl  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def h(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def spec_kats(r: Ref) -> dict:
    k = {}
    # SPEC.md:134 constant plane value 100, 2x2 CTUs of 64^2
    st, rec = r.ctu_stats(np.full((128, 128), 100, np.uint16), 8, 64)
    k["constant_100"] = {"w": 128, "h": 128, "ctu": 64, "value": 100, "records": rec.tolist()}
    # SPEC.md:135 one white pixel (255) else 0
    p = np.zeros((128, 128), np.uint16)
    p[70, 9] = 255
    st, rec = r.ctu_stats(p, 8, 64)
    k["white_pixel"] = {"w": 128, "h": 128, "ctu": 64, "pixel": [9, 70], "records": rec.tolist()}
    # SPEC.md:145 two-tone frame: left half 0, right half 200, 8x8 grid (ctu 32)
    p = np.zeros((256, 256), np.uint16)
    p[:, 128:] = 200
    st, rec = r.ctu_stats(p, 8, 32)
    vert = r.partition_eval(256, 256, 32, [4, 4], [8], [(0, 0, 4, 8, 0), (4, 0, 4, 8, 1)],
                            records=rec, validate=True)
    horz = r.partition_eval(256, 256, 32, [8], [8], [(0, 0, 8, 4, 0), (0, 4, 8, 4, 1)],
                            records=rec, validate=True)
    k["two_tone"] = {"records": rec.tolist(), "sse_vertical": vert[4], "sse_horizontal": horz[4]}
    # SPEC.md:192-194 temporal layers at gop 16
    k["temporal_layers"] = [[poc, 16, r.temporal_layer(poc, 16)[1]] for poc in range(0, 33)]
    # SPEC.md:210 [[1,2],[3,4]], two row slices -> {3,7}, T = 7
    st, mx, tot, am, _ = r.partition_eval(64, 64, 32, [2], [1, 1], [(0, 0, 2, 1, 0), (0, 1, 2, 1, 1)],
                                          times=np.array([1.0, 2.0, 3.0, 4.0]), validate=True)
    k["row_slices_2x2"] = {"times": [1, 2, 3, 4], "max_us": mx, "total_us": tot, "argmax": am}
    # SPEC.md:201-203 estimator fallbacks
    g = (128, 128, 32)
    maps = np.stack([np.full(16, v) for v in (1.0, 2.0, 3.0)])
    est = {}
    for poc, pocs, tls in [(24, [0, 16, 8], [0, 0, 1]), (5, [], []), (6, [0, 16, 8], [0, 0, 1])]:
        mm = maps[: len(pocs)] if pocs else np.zeros((0, 16))
        st, e, src, srcp = r.estimate(*g, 16, mm, pocs, tls, poc)
        est[str(poc) + ":" + ",".join(map(str, pocs))] = {"est0": e[0], "source": src,
                                                          "source_poc": srcp}
    k["estimate"] = est
    # enumeration counts, compat = reference family
    cnt = {}
    for (fw, fh, ctu, n, mc) in [(64, 64, 32, 2, 0), (128, 32, 32, 2, 0), (1920, 1080, 128, 1, 0),
                                 (1920, 1080, 128, 2, 0), (1920, 1080, 128, 4, 0),
                                 (128, 128, 32, 4, 0), (192, 192, 32, 4, 0),
                                 (1920, 1080, 128, 4, 2), (1920, 1080, 128, 8, 4)]:
        st, c, _ = r.enumerate(fw, fh, ctu, n, 3.0, 0, mc)
        cnt[f"{fw}x{fh}/{ctu}/n{n}/c{mc}"] = c
    k["enumeration_counts"] = cnt
    return k


def search_small(r: Ref, n_cases: int = 200) -> list:
    rng = np.random.default_rng(20121479)
    cases = []
    while len(cases) < n_cases:
        ctu = 32
        cols, rows = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        W = max(1, cols * ctu - int(rng.integers(0, ctu)))
        H = max(1, rows * ctu - int(rng.integers(0, ctu)))
        cols, rows = -(-W // ctu), -(-H // ctu)
        n = int(rng.integers(1, min(6, cols * rows) + 1))
        mc = int(rng.integers(0, 4))
        lam = float(rng.choice([0.0, 0.1, 0.3, 1.0]))
        k = float(rng.choice([3.0, 2.5, 1.5]))
        est = rng.lognormal(0, 0.7, cols * rows)
        if len(cases) % 7 == 0:
            est = np.round(est * 2) / 2  # force ties
        plane = rng.integers(0, 1024, size=(H, W)).astype(np.uint16)
        if len(cases) % 5 == 0:
            plane[:] = int(rng.integers(0, 1024))
        _, rec = r.ctu_stats(plane, 10, ctu)
        st1, t1, lay1 = r.min_time_search(W, H, ctu, est, n, lam, k, 0, mc)
        case = {"w": W, "h": H, "ctu": ctu, "n": n, "max_tile_cols": mc, "lambda": lam, "k": k,
                "est": est.tolist(), "records": rec.tolist(), "status1": st1}
        if st1 == 0:
            st2, o = r.constrained(W, H, ctu, est, rec, t1, n, lam, k, 0, mc)
            _, cnt, _ = r.enumerate(W, H, ctu, n, k, 0, mc)
            case.update({"t_min": t1, "argmin": lay1.rects(), "argmin_widths": lay1.widths(),
                         "status2": st2, "t_best": o.t_best_us, "sse_best": o.sse_best,
                         "best": o.best.rects(), "best_widths": o.best.widths(),
                         "candidates": cnt, "candidates_step2": o.candidates_step2})
        cases.append(case)
    return cases


def configs(r: Ref, lambdas=(0.0,), plan=None) -> dict:
    out = {}
    plan = plan or {1: [1], 2: [1, 2, 3, 4], 3: [1]}
    for ci, pocs in plan.items():
        w = wl.WORKLOADS[ci]
        F = max(pocs)
        tr = wl.cost_trace(w, frames=F)
        luma = wl.synth_luma(w, frames=F)
        maps = np.stack([m.times_us for m in tr.history_maps])
        hpocs = [m.poc for m in tr.history_maps]
        htls = [m.temporal_layer for m in tr.history_maps]
        res = []
        for p in pocs:
            st, rec = r.ctu_stats(luma[p - 1].astype(np.uint16), w.bit_depth, w.ctu)
            for lam in lambdas:
                t0 = time.time()
                # history visible to frame p: POCs 0..p-1
                st, o = r.two_step(w.width, w.height, w.ctu, 16, maps[:p], hpocs[:p], htls[:p],
                                   rec, p, w.n_slices, lam, 3.0, 0, w.max_tile_cols)
                assert st == 0, r.err()
                fr = {"poc": p, "records_hash": h(rec), "est_hash": h(tr.est[p - 1]),
                      "records": rec.tolist() if ci == 1 else None,
                      "t_min": o.t_min_us, "t_best": o.t_best_us, "sse_best": o.sse_best,
                      "best": o.best.rects(), "best_widths": o.best.widths(),
                      "candidates_step1": o.candidates_step1,
                      "candidates_step2": o.candidates_step2,
                      "est_source": o.est_source, "est_source_poc": o.est_source_poc,
                      "ref_seconds": time.time() - t0}
                if lam != 0.0 or len(lambdas) > 1:
                    fr["lambda"] = lam
                res.append(fr)
                print(f"cfg{ci} poc {p} lambda {lam}: {time.time() - t0:.1f}s", flush=True)
        out[str(ci)] = {"name": w.name, "frames": res}
    return out


LADDER = [  # (cfg, n, max_tile_cols, lambda); candidate counts from SURVEY.md §8c
    (4, 16, 1, 0.0), (4, 16, 2, 0.0), (4, 8, 4, 0.0), (4, 8, 4, 0.3),
    (4, 16, 2, 1.0), (5, 32, 1, 0.0), (5, 32, 1, 0.3), (5, 4, 0, 0.0), (5, 4, 0, 0.1),
    (5, 4, 0, 2.0), (5, 6, 0, 0.0), (5, 6, 0, 0.3), (5, 8, 2, 0.0), (5, 8, 2, 0.5),
]


def ladder(r: Ref) -> dict:
    """two_step_partition of the unmodified reference on the cfg4 / cfg5 grids
    (30x17, 60x34) at the candidate spaces it can enumerate (<= 3.2e8)."""
    from concurrent.futures import ThreadPoolExecutor

    inputs = {}
    for ci in (4, 5):
        w = wl.WORKLOADS[ci]
        tr = wl.cost_trace(w, frames=1)
        luma = wl.synth_luma(w, frames=1)
        st, rec = r.ctu_stats(luma[0].astype(np.uint16), w.bit_depth, w.ctu)
        assert st == 0
        maps = np.stack([m.times_us for m in tr.history_maps[:1]])
        inputs[ci] = {"w": w, "rec": rec, "maps": maps, "est": tr.est[0],
                      "hpocs": [tr.history_maps[0].poc], "htls": [tr.history_maps[0].temporal_layer]}

    def run(case):
        ci, n, mc, lam = case
        I = inputs[ci]
        w = I["w"]
        t0 = time.time()
        st, o = r.two_step(w.width, w.height, w.ctu, 16, I["maps"], I["hpocs"], I["htls"], I["rec"],
                           1, n, lam, 3.0, 0, mc)
        assert st == 0, r.err()
        dt = time.time() - t0
        print(f"ladder cfg{ci} n={n} cap={mc} lambda={lam}: {o.candidates_step1} cand, {dt:.1f}s",
              flush=True)
        return {"cfg": ci, "n": n, "max_tile_cols": mc, "lambda": lam, "k": 3.0,
                "t_min": o.t_min_us, "t_best": o.t_best_us, "sse_best": o.sse_best,
                "best": o.best.rects(), "best_widths": o.best.widths(),
                "candidates_step1": o.candidates_step1, "candidates_step2": o.candidates_step2,
                "est_source": o.est_source, "est_source_poc": o.est_source_poc,
                "ref_seconds": dt}

    with ThreadPoolExecutor(max_workers=min(len(LADDER), os.cpu_count() or 1)) as ex:
        cases = list(ex.map(run, LADDER))
    grids = {}
    for ci, I in inputs.items():
        w = I["w"]
        grids[str(ci)] = {"name": w.name, "width": w.width, "height": w.height, "ctu": w.ctu,
                          "poc": 1, "est": I["est"].tolist(), "records": I["rec"].tolist(),
                          "est_hash": h(I["est"]), "records_hash": h(I["rec"])}
    return {"grids": grids, "cases": cases}


def validate(r: Ref) -> list:
    """validate_partition on valid partitions and on mutations of them."""
    rng = np.random.default_rng(86184)
    cases = []

    def rec(cols, rows, cw, rh, sl, kind):
        st, *_ = r.partition_eval(cols * 32, rows * 32, 32, cw, rh, sl, validate=True)
        cases.append({"cols": cols, "rows": rows, "tile_cols": list(map(int, cw)),
                      "tile_rows": list(map(int, rh)),
                      "slices": [list(map(int, q)) for q in sl], "kind": kind, "status": st,
                      "message": r.err() if st else ""})

    while len(cases) < 400:
        cols, rows = int(rng.integers(1, 10)), int(rng.integers(1, 10))
        # random tile grid, then slices: some tiles whole, some cut into row runs
        def comp(total):
            out, left = [], total
            while left:
                v = int(rng.integers(1, left + 1))
                out.append(v)
                left -= v
            return out
        cw, rh = comp(cols), comp(rows)
        sl, x = [], 0
        for w in cw:
            y = 0
            for h in rh:
                if rng.random() < 0.5:
                    sl.append([x, y, w, h])
                else:
                    yy = y
                    for hh in comp(h):
                        sl.append([x, yy, w, hh])
                        yy += hh
                y += h
            x += w
        perm = rng.permutation(len(sl))
        sl = [q + [int(perm[i])] for i, q in enumerate(sl)]
        order = rng.permutation(len(sl))
        sl = [sl[i] for i in order]
        rec(cols, rows, cw, rh, sl, "valid")
        m = int(rng.integers(0, 9))
        sl2 = [list(q) for q in sl]
        if m == 0 and len(sl2) > 1:  # drop a slice -> coverage (ids break too)
            del sl2[int(rng.integers(0, len(sl2)))]
            for i, q in enumerate(sorted(sl2, key=lambda q: q[4])):
                q[4] = i
            rec(cols, rows, cw, rh, sl2, "drop")
        elif m == 1:  # grow a slice -> overlap / bounds
            q = sl2[int(rng.integers(0, len(sl2)))]
            q[2 + int(rng.integers(0, 2))] += 1
            rec(cols, rows, cw, rh, sl2, "grow")
        elif m == 2:  # duplicate id
            if len(sl2) > 1:
                sl2[0][4] = sl2[1][4]
            rec(cols, rows, cw, rh, sl2, "dup_id")
        elif m == 3:  # tile grid that cuts slices -> structure
            if cols > 1:
                cw2 = [1] * cols
                rec(cols, rows, cw2, rh, sl2, "fine_tiles")
        elif m == 4:  # bad tiles
            rec(cols, rows, cw + [1], rh, sl2, "tile_sum")
            rec(cols, rows, [0] + cw, rh, sl2, "tile_zero")
            rec(cols, rows, [], rh, sl2, "tile_empty")
        elif m == 5:  # overlapping duplicate appended with a fresh id
            q = list(sl2[int(rng.integers(0, len(sl2)))])
            q[4] = len(sl2)
            sl2.insert(int(rng.integers(0, len(sl2) + 1)), q)
            rec(cols, rows, cw, rh, sl2, "overlap")
        elif m == 6:  # shift a slice by one cell
            q = sl2[int(rng.integers(0, len(sl2)))]
            q[int(rng.integers(0, 2))] += 1 if rng.random() < 0.7 else -1
            rec(cols, rows, cw, rh, sl2, "shift")
        elif m == 7:
            rec(cols, rows, cw, rh, [], "empty")
        else:  # merge two vertically adjacent runs across a tile row -> structure or ok
            rec(cols, rows, [cols], [rows], sl2, "one_tile")
    return cases


def enumerate_lists(r: Ref) -> list:
    """Ordered candidate streams of the reference's for_each_candidate."""
    rng = np.random.default_rng(302326)
    out = []
    inst = [(64, 64, 32, 2, 3.0, 0, 0), (128, 32, 32, 2, 3.0, 0, 0), (192, 192, 32, 4, 3.0, 0, 0),
            (1920, 1080, 128, 4, 3.0, 0, 2), (1920, 1080, 128, 1, 3.0, 0, 0),
            (1920, 1080, 128, 2, 3.0, 0, 0), (1920, 1080, 128, 4, 3.0, 0, 0),
            (1920, 1080, 128, 8, 3.0, 0, 4), (256, 256, 32, 5, 1.2, 0, 0),
            (256, 160, 32, 6, 2.0, 0, 3), (1920, 1080, 128, 6, 3.0, 1, 0)]
    while len(inst) < 40:
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        n = int(rng.integers(1, min(7, cols * rows) + 1))
        inst.append((cols * 32 - int(rng.integers(0, 32)), rows * 32 - int(rng.integers(0, 32)),
                     32, n, float(rng.choice([3.0, 2.0, 1.5, 1.1])), 0, int(rng.integers(0, 4))))
    for fw, fh, ctu, n, k, fam, mc in inst:
        st, cnt, _ = r.enumerate(fw, fh, ctu, n, k, fam, mc)
        case = {"w": fw, "h": fh, "ctu": ctu, "n": n, "k": k, "family": fam,
                "max_tile_cols": mc, "status": st, "count": cnt}
        if st == 0 and cnt:
            _, _, lays = r.enumerate(fw, fh, ctu, n, k, fam, mc, max_out=cnt)
            rects = [[list(q) for q in L.rects()] for L in lays]
            case["sha256"] = hashlib.sha256(json.dumps(rects).encode()).hexdigest()
            if cnt <= 3000:
                case["list"] = rects
            else:
                case["head"], case["tail"] = rects[:40], rects[-40:]
        out.append(case)
    return out


def uniform(r: Ref) -> dict:
    """UniformOnly family: uniform_partition shapes, the family's search
    outputs, and partition_time / partition_sse of arbitrary partitions."""
    rng = np.random.default_rng(1479)
    parts = []
    for cols, rows in [(15, 9), (30, 17), (60, 34), (7, 5), (1, 1), (3, 11), (13, 2)]:
        for n in [1, 2, 3, 4, 5, 6, 7, 8, 12, 13, 16, 17, 31, 32, 37, 64, 65]:
            st, lay = r.uniform_partition(cols * 32, rows * 32, 32, n)
            parts.append({"cols": cols, "rows": rows, "n": n, "status": st,
                          "tile_cols": lay.widths() if st == 0 else [],
                          "tile_rows": [lay.row_heights[i] for i in range(lay.n_tile_rows)]
                          if st == 0 else [],
                          "slices": lay.rects() if st == 0 else []})
    searches = []
    while len(searches) < 60:
        ctu = 32
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        W, H = cols * ctu - int(rng.integers(0, ctu)), rows * ctu - int(rng.integers(0, ctu))
        n = int(rng.integers(1, min(12, cols * rows) + 1))
        lam = float(rng.choice([0.0, 0.1, 1.0]))
        k = float(rng.choice([3.0, 2.0, 1.2]))
        est = rng.lognormal(0, 0.7, cols * rows)
        plane = rng.integers(0, 1024, size=(H, W)).astype(np.uint16)
        _, rec = r.ctu_stats(plane, 10, ctu)
        st1, t1, lay1 = r.min_time_search(W, H, ctu, est, n, lam, k, 1, 0)
        case = {"w": W, "h": H, "ctu": ctu, "n": n, "lambda": lam, "k": k, "est": est.tolist(),
                "records": rec.tolist(), "status1": st1}
        if st1 == 0:
            case.update({"t_min": t1, "argmin": lay1.rects()})
            # the reference's step 2 with its own t_min, and with a t_min that
            # puts the uniform candidate over budget
            st2, o = r.constrained(W, H, ctu, est, rec, t1, n, lam, k, 1, 0)
            st3, _ = r.constrained(W, H, ctu, est, rec, t1 * 0.5, n, 0.0, k, 1, 0)
            case.update({"status2": st2, "t_best": o.t_best_us, "sse_best": o.sse_best,
                         "best": o.best.rects(), "candidates_step2": o.candidates_step2,
                         "candidates_evaluated": o.candidates_evaluated, "status_over": st3})
        searches.append(case)
    evals = []
    for i in range(40):
        cols, rows = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        ctu = 32
        W, H = cols * ctu, rows * ctu
        # a random column layout: widths, then each column cut into runs
        widths, x = [], 0
        while x < cols:
            w = int(rng.integers(1, cols - x + 1))
            widths.append(w)
            x += w
        slices, x = [], 0
        for w in widths:
            y = 0
            while y < rows:
                h = int(rng.integers(1, rows - y + 1))
                slices.append([x, y, w, h])
                y += h
            x += w
        perm = rng.permutation(len(slices))
        slices = [s + [int(perm[j])] for j, s in enumerate(slices)]
        est = rng.lognormal(0, 0.7, cols * rows) * (1 if i % 4 else -1)  # negative times too
        plane = rng.integers(0, 1024, size=(H, W)).astype(np.uint16)
        _, rec = r.ctu_stats(plane, 10, ctu)
        res = r.partition_eval(W, H, ctu, widths, [rows], slices, times=est, records=rec)
        evals.append({"w": W, "h": H, "ctu": ctu, "slices": slices, "est": est.tolist(),
                      "records": rec.tolist(), "status": res[0], "max_us": res[1],
                      "total_us": res[2], "argmax": res[3], "sse": res[4]})
    return {"partitions": parts, "searches": searches, "evals": evals}


def main():
    r = Ref()
    which = sys.argv[1:] or ["kats", "small", "uniform", "configs"]
    if "kats" in which:
        with open(os.path.join(OUT, "spec_kats.json"), "w") as f:
            json.dump(spec_kats(r), f, indent=1)
    if "small" in which:
        with open(os.path.join(OUT, "search_small.json"), "w") as f:
            json.dump(search_small(r), f)
    if "uniform" in which:
        with open(os.path.join(OUT, "uniform.json"), "w") as f:
            json.dump(uniform(r), f)
    if "configs" in which:
        with open(os.path.join(OUT, "configs.json"), "w") as f:
            json.dump(configs(r), f, indent=1)
    if "validate" in which:
        with open(os.path.join(OUT, "validate.json"), "w") as f:
            json.dump(validate(r), f)
    if "enumerate" in which:
        with open(os.path.join(OUT, "enumerate.json"), "w") as f:
            json.dump(enumerate_lists(r), f)
    if "ladder" in which:
        with open(os.path.join(OUT, "ladder.json"), "w") as f:
            json.dump(ladder(r), f)
    if "lambda" in which:
        with open(os.path.join(OUT, "configs_lambda.json"), "w") as f:
            json.dump(configs(r, lambdas=(0.1, 0.3), plan={1: [1], 2: [1, 2], 3: [1]}), f,
                      indent=1)


if __name__ == "__main__":
    main()
