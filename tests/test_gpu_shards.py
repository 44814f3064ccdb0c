"""The library-owned exchange between candidate-space shards
(sc_comm_init_callback; sc_comm_init_nccl uses the same hooks with NCCL
collectives): `world` contexts, one per host thread, each a shard; the
library all-reduces step 1's t_min (step 2's budget) and, in the pruned mode,
the frozen seed incumbents, and all-gathers + merges the shard bests -- every
rank must return the single-context result, bit for bit.

The shards run on the one GPU of the test box from different host threads:
their kernels never wait on one another (the exchange is a host callback
between launches), so this checks the sharding and the exchange logic, not
multi-GPU performance."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class ThreadAllGather:
    """all-gather between `world` host threads (rank order)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def make(self, rank):
        def gather(data: bytes) -> bytes:
            self.slots[rank] = data
            self.bar.wait()
            out = b"".join(self.slots)
            self.bar.wait()
            return out
        return gather


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_library_exchange_matches_single_context(part, mode, world):
    from paper_2012_14792_b200 import CtuGrid, Partitioner, SearchConfig
    rng = np.random.default_rng(100 + world + 10 * mode)
    g = CtuGrid.make(9 * 64, 6 * 64, 64)
    F = 3
    est = rng.lognormal(0, 0.6, size=(F, g.cell_count()))
    luma = rng.integers(0, 1024, size=(F, g.frame_height, g.frame_width)).astype(np.uint16)
    rec = part.ctu_stats_batch(luma, 64)
    cases = [SearchConfig(n_slices=6, lambda_=0.25, max_tile_cols=4, mode=mode),
             SearchConfig(n_slices=5, lambda_=0.3, coverage=1, mode=mode)]
    for cfg in cases:
        ref = part.two_step_batch(g, est, rec, cfg)
        ag = ThreadAllGather(world)
        got, errs = [None] * world, []

        def run(r):
            try:
                p = Partitioner(0)
                p.comm_init_callback(r, world, ag.make(r))
                got[r] = p.two_step_batch(g, est, rec, cfg)
                p.comm_detach()
                p.close()
            except Exception as e:  # noqa: BLE001
                errs.append(e)
                ag.bar.abort()
        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for r in range(world):
            for f in range(F):
                a, b = got[r][f], ref[f]
                ctx = (world, mode, cfg.coverage, r, f)
                assert a.t_min_us == b.t_min_us and a.t_best_us == b.t_best_us, ctx
                assert a.sse_best == b.sse_best, ctx
                assert a.argmin.rects() == b.argmin.rects(), ctx
                assert a.best.rects() == b.best.rects(), ctx
                assert a.candidates_step1 == b.candidates_step1, ctx
                assert a.candidates_step2 == b.candidates_step2, ctx
