"""Encoding-parallelism simulator (module `simulate`).

The reference ships this module as a specification only (no code in
proj/src); SURVEY.md §8f ranks it fourth among the rows beside the hot path.
It replays a cost trace in random-access encode order, partitions every frame
with the two-step search (fed only by the maps of frames already encoded:
causality), and simulates N-thread encoding of each frame:

    simulate_frame = s * frame_total + (1 - s) * max_j T(slice_j)       (Eq. 1, §3.2)
    sigma_qp       = T_O / T_R,  T_O = sum frame_total,
                     T_R = sum (simulate_frame + search_time)           (Eq. 5)
    sigma          = mean over the QPs,  sigma_max = amdahl_bound(s, N)  (Eq. 6)
    theta          = 100 * sum search_time / sum T_R                   (§3.1)

B200 shape: the estimates of a whole QP pass are known once the trace is
loaded (each frame only reads maps of earlier-encoded frames), so all frames
of a pass are partitioned in ONE batched device call (sc_two_step), and the
true-map slice times of all chosen partitions come from device partition
evaluations (sc_partition_eval).  search_time is the device time of the
batched search divided evenly over its frames (or 0 for property tests).
"""
from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from .partitioner import (COLUMN_SPLIT, COVERAGE_COVERING, CostHistory, CostMap, CtuGrid,
                          Partition, Partitioner, SearchConfig, estimate_ctu_times,
                          temporal_layer_of_poc)


@dataclass
class SimConfig:
    """SimConfig."""
    n_threads: int = 4                     # N = slices per frame
    qps: Sequence[int] = (22, 27, 32, 37)
    seq_frac: float = 0.04                 # s, the sequential part of a frame
    lambda_: float = 0.0
    gop_size: int = 16
    baseline: Optional[str] = "uniform"    # "uniform" or None
    k_area: float = 3.0
    max_tile_cols: int = 0
    mode: int = 0                          # SC_MODE_EXHAUSTIVE / SC_MODE_PRUNED
    # The reference family (widths summing to <= cols, search.cpp:133-143) can
    # leave CTUs outside every slice, which an encoder cannot do; simulations
    # use the covering family unless told otherwise.
    coverage: int = COVERAGE_COVERING
    search_time: str = "measured"          # "measured" or "zero" (property tests)

    def check(self) -> None:
        if not (0.0 <= self.seq_frac < 1.0):
            raise ValueError("sequential fraction must be in [0, 1)")
        if not self.qps:
            raise ValueError("qps must be non-empty")
        if self.n_threads < 1:
            raise ValueError("n_threads must be >= 1")


def amdahl_bound(s: float, n: int) -> float:
    """amdahl_bound (Eq. 6): 1 / (s + (1 - s) / n)."""
    return 1.0 / (s + (1.0 - s) / n)


def encode_order(n_frames: int, gop_size: int) -> List[int]:
    """Random-access hierarchical-B encode order of POCs 0..n_frames-1
    (SPEC.md:368): POC 0, then per GOP its last frame and a binary split of
    the rest (16, 8, 4, 2, 1, 3, 6, 5, 7, 12, 10, 9, 11, 14, 13, 15)."""
    def split(lo: int, hi: int, out: List[int]) -> None:
        if hi - lo < 2:
            return
        mid = (lo + hi) // 2
        out.append(mid)
        split(lo, mid, out)
        split(mid, hi, out)

    order = [0] if n_frames > 0 else []
    start = 0
    while start + 1 < n_frames:
        end = min(start + gop_size, n_frames - 1)
        order.append(end)
        mids: List[int] = []
        split(start, end, mids)
        order.extend(mids)
        start = end
    return order


@dataclass
class FrameRow:
    poc: int
    qp: int
    tl: int
    t_true: float       # simulate_frame on the true map
    t_est: float        # the search's estimated slowest slice (t_best_us)
    sse: float
    search_time: float
    frame_total: float
    est_source_poc: int


@dataclass
class SimReport:
    """SimReport for one method."""
    method: str
    rows: List[FrameRow] = field(default_factory=list)
    per_qp: Dict[int, Dict[str, float]] = field(default_factory=dict)
    sigma: float = 0.0
    sigma_max: float = 0.0
    theta: float = 0.0
    total_sse: float = 0.0

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=1)


def simulate_frame(part: Partitioner, costs: CostMap, p: Partition, s: float) -> float:
    """simulate_frame: s * frame_total + (1 - s) * the slowest
    slice of `p` on the true map (slice times from the device)."""
    if costs.grid != p.grid:
        from ._abi import SlicecraftError
        raise SlicecraftError(1, "cost map grid does not match the partition grid")
    st = part.partition_eval(p, est=np.asarray(costs.times_us, dtype=np.float64)[None])[0]
    total = float(np.sum(costs.times_us))
    return s * total + (1.0 - s) * st["max_us"]


def _frame_times(part: Partitioner, grid: CtuGrid, parts: List[Partition],
                 true_maps: np.ndarray, s: float) -> List[float]:
    out = []
    for p, t in zip(parts, true_maps):
        st = part.partition_eval(p, est=t[None])[0]
        out.append(s * float(np.sum(t)) + (1.0 - s) * st["max_us"])
    return out


def simulate_sequence(part: Partitioner, grid: CtuGrid, trace: Dict[int, np.ndarray],
                      records: np.ndarray, cfg: SimConfig) -> Dict[str, SimReport]:
    """simulate_sequence + compare_baseline's inputs.

    trace: qp -> true per-CTU time maps [F][cells] in POC order; records:
    texture records [F][cells] (RECORD_DTYPE) of the same frames.  Returns
    {"proposed": report, "uniform": report} (uniform only if cfg.baseline)."""
    cfg.check()
    F = records.shape[0]
    for qp in cfg.qps:
        if qp not in trace:
            from ._abi import SlicecraftError
            raise SlicecraftError(9, f"missing cost maps for qp {qp}")
        if trace[qp].shape != (F, grid.cell_count()):
            from ._abi import SlicecraftError
            raise SlicecraftError(9, f"qp {qp}: expected {F} maps of {grid.cell_count()} CTUs")
    order = encode_order(F, cfg.gop_size)
    scfg = SearchConfig(n_slices=cfg.n_threads, lambda_=cfg.lambda_, k_area=cfg.k_area,
                        family=COLUMN_SPLIT, max_tile_cols=cfg.max_tile_cols,
                        coverage=cfg.coverage, mode=cfg.mode)
    methods = ["proposed"] + (["uniform"] if cfg.baseline == "uniform" else [])
    reports = {m: SimReport(m, sigma_max=amdahl_bound(cfg.seq_frac, cfg.n_threads))
               for m in methods}
    uni = Partition.uniform(grid, cfg.n_threads) if "uniform" in methods else None
    for qp in cfg.qps:
        maps = np.ascontiguousarray(trace[qp], dtype=np.float64)
        # causal estimates in encode order (cost.cpp:66-95), then one batched search
        hist = CostHistory(grid, cfg.gop_size)
        est, src = np.zeros_like(maps), {}
        for poc in order:
            e = estimate_ctu_times(hist, poc)
            est[poc] = e.times_us
            src[poc] = e.source_poc
            hist.append(CostMap(grid, maps[poc], poc, temporal_layer_of_poc(poc, cfg.gop_size),
                                qp))
        outs = part.two_step_batch(grid, est, records, scfg)
        per_frame_search = part.timings()["total"] / F if cfg.search_time == "measured" else 0.0
        for m in methods:
            parts = [o.best for o in outs] if m == "proposed" else [uni] * F
            t_true = _frame_times(part, grid, parts, maps, cfg.seq_frac)
            rep = reports[m]
            T_O = T_R = S = 0.0
            for poc in order:
                stime = per_frame_search if m == "proposed" else 0.0
                total = float(np.sum(maps[poc]))
                if m == "proposed":
                    sse, t_est = outs[poc].sse_best, outs[poc].t_best_us
                else:
                    ev = part.partition_eval(uni, est=est[poc][None], records=records[poc][None])[0]
                    sse, t_est = ev["sse"], ev["max_us"]
                rep.rows.append(FrameRow(poc, qp, temporal_layer_of_poc(poc, cfg.gop_size),
                                         t_true[poc], t_est, sse, stime, total, src[poc]))
                T_O += total
                T_R += t_true[poc] + stime
                S += stime
                rep.total_sse += sse
            rep.per_qp[qp] = {"T_O": T_O, "T_R": T_R, "sigma": T_O / T_R, "search": S}
    for rep in reports.values():
        rep.sigma = float(np.mean([v["sigma"] for v in rep.per_qp.values()]))
        T_R = sum(v["T_R"] for v in rep.per_qp.values())
        rep.theta = 100.0 * sum(v["search"] for v in rep.per_qp.values()) / T_R
    return reports


def compare_baseline(proposed: SimReport, uniform: SimReport) -> str:
    """compare_baseline: a Table-1-shaped text table (BDR is
    replaced by the SSE proxy and labelled as such)."""
    lines = ["| metric | Unif. | Proposed |", "|---|---|---|",
             f"| SSE proxy | {uniform.total_sse:.6g} | {proposed.total_sse:.6g} |",
             f"| sigma | {uniform.sigma:.4f} | {proposed.sigma:.4f} |",
             f"| theta (%) | {uniform.theta:.4f} | {proposed.theta:.4f} |",
             f"| sigma_max | {uniform.sigma_max:.4f} | {proposed.sigma_max:.4f} |"]
    return "\n".join(lines)
