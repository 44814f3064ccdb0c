"""Raw planar 4:2:0 YUV ingest (texture.cpp:9-81): frame counting, luma
loading and its errors against the unmodified reference (oracle/_ref), and
(GPU) K1 / the whole hot path straight from a file."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write_yuv(path, w, h, frames, bit_depth, seed):
    rng = np.random.default_rng(seed)
    dt = np.uint8 if bit_depth == 8 else np.dtype("<u2")
    top = 255 if bit_depth == 8 else 1023
    cw, ch = (w + 1) // 2, (h + 1) // 2
    planes = []
    with open(path, "wb") as f:
        for _ in range(frames):
            y = rng.integers(0, top + 1, size=(h, w)).astype(dt)
            f.write(y.tobytes())
            f.write(rng.integers(0, top + 1, size=2 * cw * ch).astype(dt).tobytes())
            planes.append(y)
    return np.stack(planes)


def _ref():
    from oracle.oracle import Ref
    try:
        return Ref()
    except RuntimeError:
        pytest.skip("oracle/_ref not built (needs /root/reference)")


@pytest.mark.parametrize("bit_depth", [8, 10])
@pytest.mark.parametrize("dims", [(35, 21), (64, 64), (130, 7)])
def test_yuv_count_and_load_match_reference(tmp_path, bit_depth, dims):
    from paper_2012_14792_b200 import load_yuv_frame, read_yuv_luma, yuv_frame_count
    r = _ref()
    w, h = dims
    p = str(tmp_path / "clip.yuv")
    planes = _write_yuv(p, w, h, 3, bit_depth, w * h + bit_depth)
    st, n = r.yuv_frame_count(p, w, h, bit_depth)
    assert st == 0 and n == 3 == yuv_frame_count(p, w, h, bit_depth)
    for poc in range(3):
        st, ref_plane = r.load_yuv_frame(p, w, h, poc, bit_depth)
        got = load_yuv_frame(p, w, h, poc, bit_depth)
        assert st == 0 and np.array_equal(got, ref_plane)
        assert np.array_equal(got, planes[poc].astype(np.uint16))
    raw = read_yuv_luma(p, w, h, bit_depth, 1, 2)
    assert raw.dtype == (np.uint8 if bit_depth == 8 else np.uint16)
    assert np.array_equal(raw, planes[1:3])


def test_yuv_errors_match_reference(tmp_path):
    from paper_2012_14792_b200 import SlicecraftError, load_yuv_frame, yuv_frame_count
    r = _ref()
    p = str(tmp_path / "clip.yuv")
    _write_yuv(p, 16, 8, 2, 8, 1)

    def status(fn):
        try:
            fn()
            return 0
        except SlicecraftError as e:
            return e.status

    cases = [
        (lambda: yuv_frame_count(p, 16, 8, 9), r.yuv_frame_count(p, 16, 8, 9)[0]),  # bit depth
        (lambda: yuv_frame_count(p, 0, 8, 8), r.yuv_frame_count(p, 0, 8, 8)[0]),  # dims
        (lambda: yuv_frame_count(p, 15, 8, 8), r.yuv_frame_count(p, 15, 8, 8)[0]),  # size
        (lambda: yuv_frame_count(p + ".missing", 16, 8, 8),
         r.yuv_frame_count(p + ".missing", 16, 8, 8)[0]),  # stat
        (lambda: load_yuv_frame(p, 16, 8, 2, 8), r.load_yuv_frame(p, 16, 8, 2, 8)[0]),  # range
        (lambda: load_yuv_frame(p, 16, 8, -1, 8), r.load_yuv_frame(p, 16, 8, -1, 8)[0]),
    ]
    for fn, ref_status in cases:
        assert ref_status != 0
        assert status(fn) == ref_status


@pytest.mark.gpu
@pytest.mark.parametrize("bit_depth", [8, 10])
def test_yuv_texture_and_partition_on_device(tmp_path, part, oracle, bit_depth):
    """K1 straight from the file == the oracle on the loaded planes, and the
    hot path from the file == the hot path from the same planes in memory."""
    from paper_2012_14792_b200 import CtuGrid, SearchConfig
    w, h, F = 700, 390, 3
    p = str(tmp_path / "clip.yuv")
    planes = _write_yuv(p, w, h, F + 1, bit_depth, 7 + bit_depth)
    g = CtuGrid.make(w, h, 64)
    rec = part.ctu_stats_yuv(p, g, bit_depth, 1, F)
    for f in range(F):
        exp = oracle.ctu_stats(planes[1 + f].astype(np.uint16), 64)
        got = np.stack([rec[f]["count"], rec[f]["sum"], rec[f]["sumsq"]], axis=1)
        assert np.array_equal(got, exp)
    est = np.random.default_rng(3).lognormal(0, 0.5, size=(F, g.cell_count()))
    cfg = SearchConfig(n_slices=5, lambda_=0.2, max_tile_cols=3)
    a = part.partition_yuv(g, p, bit_depth, 1, est, cfg)
    b = part.partition_frames(g, np.ascontiguousarray(planes[1:]), est, cfg)
    for x, y in zip(a, b):
        assert (x.t_min_us, x.t_best_us, x.sse_best) == (y.t_min_us, y.t_best_us, y.sse_best)
        assert x.candidates_step1 == y.candidates_step1
