"""Simulator: the spec's worked examples and properties."""
import numpy as np
import pytest


def test_amdahl_bound_examples():
    from paper_2012_14792_b200.simulate import amdahl_bound
    assert round(amdahl_bound(0.04, 4), 3) == 3.571   # SPEC.md:354, paper §3.2
    assert amdahl_bound(0.04, 8) == pytest.approx(6.25)
    assert round(amdahl_bound(0.04, 12), 3) == 8.333
    assert amdahl_bound(0.0, 7) == pytest.approx(7.0) and amdahl_bound(1.0, 7) == 1.0


def test_encode_order_ra_gop16():
    from paper_2012_14792_b200.simulate import encode_order
    assert encode_order(17, 16) == [0, 16, 8, 4, 2, 1, 3, 6, 5, 7, 12, 10, 9, 11, 14, 13, 15]
    o = encode_order(40, 16)
    assert sorted(o) == list(range(40)) and o[:2] == [0, 16] and o[17] == 32


def _setup(part, F, cols, rows, seed, const=False):
    from paper_2012_14792_b200 import CtuGrid
    g = CtuGrid.make(cols * 64, rows * 64, 64)
    rng = np.random.default_rng(seed)
    luma = rng.integers(0, 1024, size=(F, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 64)
    if const:
        maps = np.full((F, g.cell_count()), 2.5)
    else:
        maps = rng.lognormal(0, 0.6, size=(F, g.cell_count()))
    return g, rec, maps


@pytest.mark.gpu
def test_simulate_frame_examples(part):
    from paper_2012_14792_b200 import CostMap, CtuGrid
    from paper_2012_14792_b200.partitioner import Partition
    from paper_2012_14792_b200.simulate import simulate_frame
    g = CtuGrid.make(8 * 64, 4 * 64, 64)
    p = Partition.uniform(g, 4)
    m = CostMap(g, np.full(g.cell_count(), 100.0 / g.cell_count()))
    assert simulate_frame(part, m, p, 0.04) == pytest.approx(28.0)
    rng = np.random.default_rng(1)
    m2 = CostMap(g, rng.lognormal(0, 0.5, g.cell_count()))
    st = part.partition_eval(p, est=m2.times_us[None])[0]
    assert simulate_frame(part, m2, p, 0.0) == st["max_us"]
    assert simulate_frame(part, m2, p, 1.0) == pytest.approx(float(np.sum(m2.times_us)))


@pytest.mark.gpu
def test_balanced_trace_reaches_amdahl(part):
    """Equal CTU times, exact divisibility, search time excluded: sigma ==
    amdahl_bound(s, n) within 1e-9."""
    from paper_2012_14792_b200.simulate import SimConfig, amdahl_bound, simulate_sequence
    g, rec, maps = _setup(part, 5, 8, 4, 2, const=True)
    cfg = SimConfig(n_threads=4, qps=(22, 37), seq_frac=0.04, search_time="zero")
    rep = simulate_sequence(part, g, {22: maps, 37: maps}, rec, cfg)
    assert rep["proposed"].sigma == pytest.approx(amdahl_bound(0.04, 4), rel=1e-9)
    assert rep["uniform"].sigma == pytest.approx(amdahl_bound(0.04, 4), rel=1e-9)


@pytest.mark.gpu
def test_causality_and_proposed_beats_uniform(part):
    """17-frame GOP-16 trace: every frame's estimate comes from the most recent
    same-TL frame in encode order, else the most recent;
    with estimates equal to the truth (identical maps), lambda = 0 and no
    search time, the proposed sigma is >= uniform's."""
    from paper_2012_14792_b200 import temporal_layer_of_poc
    from paper_2012_14792_b200.simulate import SimConfig, encode_order, simulate_sequence
    g, rec, maps = _setup(part, 17, 9, 6, 3)
    cfg = SimConfig(n_threads=6, qps=(27,), seq_frac=0.04, search_time="zero")
    rep = simulate_sequence(part, g, {27: maps}, rec, cfg)["proposed"]
    order = encode_order(17, 16)
    seen = []
    for poc in order:
        row = next(r for r in rep.rows if r.poc == poc)
        tl = temporal_layer_of_poc(poc, 16)
        same = [q for q in seen if temporal_layer_of_poc(q, 16) == tl]
        exp = same[-1] if same else (seen[-1] if seen else -1)
        assert row.est_source_poc == exp, poc
        seen.append(poc)
    same_map = np.repeat(maps[:1], 17, axis=0)
    both = simulate_sequence(part, g, {27: same_map}, rec,
                             SimConfig(n_threads=6, qps=(27,), search_time="zero"))
    assert both["proposed"].sigma >= both["uniform"].sigma - 1e-12
    assert both["proposed"].sigma <= both["proposed"].sigma_max * (1 + 1e-6)


@pytest.mark.gpu
def test_report_and_table(part):
    from paper_2012_14792_b200.simulate import SimConfig, compare_baseline, simulate_sequence
    g, rec, maps = _setup(part, 9, 7, 5, 4)
    trace = {qp: maps * (1 + 0.1 * i) for i, qp in enumerate((22, 27, 32, 37))}
    rep = simulate_sequence(part, g, trace, rec, SimConfig(n_threads=4, lambda_=0.1))
    p, u = rep["proposed"], rep["uniform"]
    assert len(p.rows) == 36 and set(p.per_qp) == {22, 27, 32, 37}
    assert p.theta > 0 and u.theta == 0
    assert all(r.t_true <= r.frame_total + 1e-9 for r in p.rows)
    assert "sigma" in compare_baseline(p, u)
    assert '"method": "proposed"' in p.to_json()
