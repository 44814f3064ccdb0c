"""CPU tests of the host-side model pieces behind the C-ABI (no device
needed): estimate_ctu_times and CostHistory::append validation (cost.cpp:45-95),
the TextureStats tables and SliceMoments::sse (texture.cpp:83-143),
PrefixSumTable (cost.cpp:97-112) and split_even (grid.cpp:52-60), checked
against the SPEC known answers the reference passes (tests/golden/spec_kats.json)
and against exact restatements written here."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

RNG = np.random.default_rng(97112)


def test_estimate_matches_spec_kats():
    """sc_estimate_ctu_times through the C-ABI == the reference's estimator
    (SPEC.md:201-203 fallbacks, generated from oracle/_ref)."""
    from paper_2012_14792_b200 import CostHistory, CostMap, CtuGrid, estimate_ctu_times
    k = json.load(open(os.path.join(GOLDEN, "spec_kats.json")))["estimate"]
    g = CtuGrid.make(128, 128, 32)
    for key, exp in k.items():
        poc, pocs = key.split(":")
        pocs = [int(p) for p in pocs.split(",")] if pocs else []
        tls = {0: 0, 16: 0, 8: 1}
        h = CostHistory(g, 16)
        for i, p in enumerate(pocs):
            h.append(CostMap(g, np.full(16, float(i + 1)), p, tls[p]))
        e = estimate_ctu_times(h, int(poc))
        assert e.times_us[0] == exp["est0"], key
        assert e.source == exp["source"] and e.source_poc == exp["source_poc"], key
        assert np.all(e.times_us == e.times_us[0])


def test_estimate_raw_abi_sources_and_layers():
    """The raw entry point: co-temporal-layer pick, most-recent fallback,
    all-ones fallback, temporal layer output, gop error."""
    from paper_2012_14792_b200 import CtuGrid, lib
    from paper_2012_14792_b200._abi import SlicecraftError, check
    g = CtuGrid.make(96, 64, 32)
    cells = g.cell_count()
    maps = [RNG.random(cells) for _ in range(4)]
    pocs = np.array([0, 16, 8, 4], np.int32)
    tls = np.array([0, 0, 1, 2], np.int32)
    ptrs = (C.c_void_p * 4)(*[m.ctypes.data for m in maps])
    out = np.empty(cells)
    src, sp, tl = C.c_int32(), C.c_int32(), C.c_int32()

    def est(poc, n=4, gop=16):
        check(lib().sc_estimate_ctu_times(C.byref(g.c()), gop, n, C.cast(ptrs, C.c_void_p),
                                          C.c_void_p(pocs.ctypes.data),
                                          C.c_void_p(tls.ctypes.data), poc,
                                          C.c_void_p(out.ctypes.data), C.byref(src),
                                          C.byref(sp), C.byref(tl)))
        return src.value, sp.value, tl.value

    assert est(32) == (1, 16, 0) and np.array_equal(out, maps[1])   # TL 0: POC 16
    assert est(24) == (1, 8, 1) and np.array_equal(out, maps[2])    # TL 1: POC 8
    assert est(12) == (1, 4, 2) and np.array_equal(out, maps[3])    # TL 2: POC 4
    assert est(3) == (2, 4, 4) and np.array_equal(out, maps[3])     # TL 4: most recent
    assert est(3, n=0) == (3, -1, 4) and np.all(out == 1.0)         # empty: all ones
    with pytest.raises(SlicecraftError) as e:
        est(3, gop=12)
    assert e.value.kind == "ConfigError"


def test_cost_history_append_errors():
    """CostHistory::append (cost.cpp:45-64): grid, size, values, duplicate poc."""
    from paper_2012_14792_b200 import CostHistory, CostMap, CtuGrid, SlicecraftError
    g = CtuGrid.make(96, 64, 32)
    h = CostHistory(g, 16)
    h.append(CostMap(g, np.ones(6), 0, 0))
    cases = [(CostMap(CtuGrid.make(64, 64, 32), np.ones(4), 1, 4), "GeometryError"),
             (CostMap(g, np.ones(5), 1, 4), "GeometryError"),
             (CostMap(g, np.array([1, 2, 3, -1e-300, 5, 6.0]), 1, 4), "FormatError"),
             (CostMap(g, np.array([1, 2, np.inf, 4, 5, 6.0]), 1, 4), "FormatError"),
             (CostMap(g, np.array([1, 2, np.nan, 4, 5, 6.0]), 1, 4), "FormatError"),
             (CostMap(g, np.ones(6), 0, 0), "TraceError")]
    for m, kind in cases:
        with pytest.raises(SlicecraftError) as e:
            h.append(m)
        assert e.value.kind == kind
    h.append(CostMap(g, np.zeros(6), 1, 4))  # zeros are legal
    assert len(h.maps) == 2
    with pytest.raises(SlicecraftError) as e:
        CostHistory(g, 6)
    assert e.value.kind == "ConfigError"


def _records(g, depth=10):
    from paper_2012_14792_b200 import RECORD_DTYPE
    rec = np.zeros(g.cell_count(), RECORD_DTYPE)
    for y in range(g.rows):
        for x in range(g.cols):
            w = min(g.ctu_size, g.frame_width - x * g.ctu_size)
            h = min(g.ctu_size, g.frame_height - y * g.ctu_size)
            px = RNG.integers(0, 1 << depth, size=w * h).astype(np.uint64)
            i = y * g.cols + x
            rec[i] = (w * h, int(px.sum()), int((px * px).sum()))
    return rec


def test_texture_tables_exact_and_validation():
    """TextureStats ctor: u64 SATs (modular, texture.cpp:113-129) and its
    validation classes (texture.cpp:90-111)."""
    from paper_2012_14792_b200 import CtuGrid, SlicecraftError, texture_tables
    for W, H, ctu in [(200, 100, 32), (1920, 1080, 128), (33, 1, 32)]:
        g = CtuGrid.make(W, H, ctu)
        rec = _records(g)
        tabs = texture_tables(g, rec)
        for tab, field in zip(tabs, ("count", "sum", "sumsq")):
            v = rec[field].reshape(g.rows, g.cols).astype(object)
            exp = np.zeros((g.rows + 1, g.cols + 1), dtype=object)
            exp[1:, 1:] = v.cumsum(0).cumsum(1)
            assert [int(t) for t in tab] == [int(e) % (1 << 64) for e in exp.reshape(-1)]
    g = CtuGrid.make(200, 100, 32)
    rec = _records(g)
    with pytest.raises(SlicecraftError) as e:
        texture_tables(g, rec[:-1])
    assert e.value.kind == "GeometryError"
    bad = rec.copy()
    bad[3]["count"] += 1
    with pytest.raises(SlicecraftError) as e:
        texture_tables(g, bad)
    assert e.value.kind == "FormatError" and "(3,0)" in str(e.value)
    bad = rec.copy()
    bad[7]["sumsq"] = 0
    with pytest.raises(SlicecraftError) as e:
        texture_tables(g, bad)
    assert e.value.kind == "FormatError" and "sum^2" in str(e.value)


def test_moments_sse_exact():
    """SliceMoments::sse: exact 128-bit numerator, round-to-nearest-even to
    double, one division (texture.cpp:83-88); Python ints + float() are the
    same IEEE operations."""
    from paper_2012_14792_b200 import moments_sse
    cases = [(0, 0, 0), (1, 5, 25), (4, 6, 10), ((1 << 64) - 1, (1 << 64) - 1, (1 << 64) - 1),
             (16384, 16384 * 1023, 16384 * 1023 * 1023), (3, 1, 1 << 63)]
    for _ in range(2000):
        n = int(RNG.integers(1, 1 << 40))
        s = int(RNG.integers(0, 1 << 62))
        cases.append((n, s, int(RNG.integers(0, 1 << 63)) * 2 + 1))
    for n, s, q in cases:
        exp = 0.0 if n == 0 else float(n * q - s * s) / float(n)
        assert moments_sse(n, s, q) == exp, (n, s, q)


def test_prefix_sum_table_order():
    """PrefixSumTable: ((v + left) + up) - up_left, row-major (cost.cpp:97-112),
    bit-exact against the same recurrence in Python floats; rect_sum as
    cost.hpp:75-81."""
    from paper_2012_14792_b200 import PrefixSumTable, SlicecraftError
    for cols, rows in [(15, 9), (1, 1), (7, 3), (60, 34)]:
        v = RNG.lognormal(0, 1.0, cols * rows) * RNG.choice([1, -1, 1e-300, 1e300], cols * rows)
        t = PrefixSumTable(v, cols, rows)
        s = cols + 1
        exp = [0.0] * (s * (rows + 1))
        for y in range(rows):
            for x in range(cols):
                i = (y + 1) * s + x + 1
                exp[i] = v[y * cols + x] + exp[i - 1] + exp[i - s] - exp[i - s - 1]
        assert np.array_equal(t.table.view(np.uint64), np.array(exp).view(np.uint64))
        assert t.rect_sum(0, 0, cols, rows) == ((exp[-1] - exp[cols]) - exp[rows * s]) + exp[0]
    with pytest.raises(SlicecraftError) as e:
        PrefixSumTable(np.ones(5), 2, 3)
    assert e.value.kind == "GeometryError"


def test_split_even():
    from paper_2012_14792_b200 import split_even
    for total in range(1, 40):
        for parts in range(1, total + 1):
            got = split_even(total, parts)
            assert sum(got) == total and len(got) == parts
            assert got == sorted(got, reverse=True) and max(got) - min(got) <= 1
