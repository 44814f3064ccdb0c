"""ctypes mirror of include/slicecraft_b200.h (the C-ABI drop-in boundary).

The product library is ``libslicecraft_b200.so`` built in-tree by ``make``
(or ``__graft_entry__.build()``).  Loading fails loudly when it is missing:
there is no CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLICECRAFT_B200_LIB", os.path.join(HERE, "libslicecraft_b200.so"))

SC_MAX_SLICES = 64
SC_MAX_COLS = 16

# sc_status, one per exception class of slicecraft/errors.hpp:10-85
SC_OK = 0
STATUS_NAMES = {
    1: "GeometryError", 2: "OverlapError", 3: "CoverageError", 4: "StructureError",
    5: "IoError", 6: "RangeError", 7: "FormatError", 8: "ConfigError", 9: "TraceError",
    10: "NoCandidateError", 11: "SizeError", 12: "UsageError", 100: "CudaError",
    101: "InternalError",
}


class Grid(C.Structure):
    _fields_ = [("frame_width", C.c_int32), ("frame_height", C.c_int32),
                ("ctu_size", C.c_int32), ("cols", C.c_int32), ("rows", C.c_int32)]


class CtuRecord(C.Structure):
    _fields_ = [("count", C.c_uint64), ("sum", C.c_uint64), ("sumsq", C.c_uint64)]


class SearchCfg(C.Structure):
    _fields_ = [("n_slices", C.c_int32), ("lambda_", C.c_double), ("k_area", C.c_double),
                ("family", C.c_int32), ("max_tile_cols", C.c_int32), ("workers", C.c_int32),
                ("coverage", C.c_int32), ("mode", C.c_int32)]


class Layout(C.Structure):
    _fields_ = [("n_cols", C.c_int32), ("n_slices", C.c_int32),
                ("col_widths", C.c_int32 * SC_MAX_COLS),
                ("runs_per_col", C.c_int32 * SC_MAX_COLS),
                ("run_heights", C.c_int32 * SC_MAX_SLICES)]


class SearchResult(C.Structure):
    _fields_ = [("t_min_us", C.c_double), ("t_best_us", C.c_double), ("sse_best", C.c_double),
                ("candidates_evaluated", C.c_uint64), ("candidates_step1", C.c_uint64),
                ("candidates_step2", C.c_uint64), ("search_time_us", C.c_double),
                ("time_min_step_us", C.c_double), ("clustering_step_us", C.c_double),
                ("leaves_scored_step1", C.c_uint64), ("leaves_scored_step2", C.c_uint64),
                ("argmin", Layout), ("best", Layout),
                ("candidates_step1_hi", C.c_uint64), ("candidates_step2_hi", C.c_uint64),
                ("origin", C.c_int32), ("pad", C.c_int32)]


SC_ORIGIN_PROPOSED, SC_ORIGIN_UNIFORM = 0, 1
SC_COMM_ID_BYTES = 128
# int (*)(void* user, const void* send, size_t bytes, void* recv)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Rect(C.Structure):
    _fields_ = [("x0", C.c_int32), ("y0", C.c_int32), ("w", C.c_int32), ("h", C.c_int32),
                ("id", C.c_int32)]


class PartitionC(C.Structure):
    _fields_ = [("n_tile_cols", C.c_int32), ("n_tile_rows", C.c_int32),
                ("tile_col_widths", C.c_int32 * SC_MAX_SLICES),
                ("tile_row_heights", C.c_int32 * SC_MAX_SLICES),
                ("n_slices", C.c_int32), ("origin", C.c_int32),
                ("slices", Rect * SC_MAX_SLICES)]


class PartitionStats(C.Structure):
    _fields_ = [("max_us", C.c_double), ("total_us", C.c_double), ("argmax", C.c_int64),
                ("sse", C.c_double)]


class ShardBest(C.Structure):
    _fields_ = [("key_sse", C.c_double), ("key_t", C.c_uint64), ("item", C.c_uint64),
                ("ord", C.c_uint64), ("count", C.c_uint64), ("leaves", C.c_uint64),
                ("count_hi", C.c_uint64), ("layout", Layout)]


# (name, restype, argtypes) for every symbol declared in the header.
_P = C.c_void_p
SIGNATURES = [
    ("sc_last_error", C.c_char_p, []),
    ("sc_kernel_launches", C.c_uint64, []),
    ("sc_abi_version", C.c_int, []),
    ("sc_grid_make", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(Grid)]),
    ("sc_temporal_layer", C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
    ("sc_search_cfg_check", C.c_int, [C.POINTER(SearchCfg)]),
    ("sc_ctx_create", C.c_int, [C.c_int32, C.POINTER(_P)]),
    ("sc_ctx_destroy", C.c_int, [_P]),
    ("sc_ctx_set_shard", C.c_int, [_P, C.c_int32, C.c_int32]),
    ("sc_ctx_set_stream", C.c_int, [_P, _P]),
    ("sc_ctx_timings", C.c_int, [_P, _P]),
    ("sc_ctx_timings_ex", C.c_int, [_P, C.c_int32, _P]),
    ("sc_uniform_partition", C.c_int, [C.POINTER(Grid), C.c_int32, C.POINTER(PartitionC)]),
    ("sc_uniform_partition_n", C.c_int, [C.POINTER(Grid), C.c_int32, _P, C.POINTER(C.c_int32),
                                         _P, C.POINTER(C.c_int32), _P]),
    ("sc_yuv_frame_count", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(C.c_int32)]),
    ("sc_yuv_load_luma", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    ("sc_yuv_read_luma", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_int32, _P]),
    ("sc_yuv_texture_moments", C.c_int, [_P, C.c_char_p, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_int32, _P]),
    ("sc_partition_yuv", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), C.c_char_p,
                                   C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    ("sc_partition_eval", C.c_int, [_P, C.POINTER(Grid), _P, C.c_int32, _P, _P, C.c_int32, _P,
                                    _P, _P]),
    ("sc_texture_moments", C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_size_t,
                                     C.c_size_t, C.c_int32, C.c_int32, _P]),
    ("sc_texture_validate", C.c_int, [C.POINTER(Grid), _P]),
    ("sc_grid_tables", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int32, _P, _P, _P]),
    ("sc_min_time_search", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), _P,
                                     C.c_int32, _P]),
    ("sc_constrained_clustering", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), _P,
                                            _P, _P, C.c_int32, _P]),
    ("sc_two_step", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), _P, _P, C.c_int32,
                              _P]),
    ("sc_partition_frames", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), _P,
                                      C.c_int32, C.c_size_t, C.c_size_t, _P, C.c_int32, _P,
                                      _P]),
    ("sc_count_candidates", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg),
                                      C.POINTER(C.c_uint64)]),
    ("sc_validate_partition", C.c_int, [_P, C.POINTER(Grid), C.c_int32, _P, C.c_int32, _P, _P,
                                        C.c_int32, _P]),
    ("sc_result_slice_maps", C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    ("sc_enumerate_candidates", C.c_int, [_P, C.POINTER(Grid), C.POINTER(SearchCfg), C.c_uint64,
                                          C.c_uint64, _P, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)]),
    ("sc_cost_map_check", C.c_int, [C.POINTER(Grid), C.POINTER(Grid), _P, C.c_int64, C.c_int32,
                                    _P, C.c_int32]),
    ("sc_estimate_ctu_times", C.c_int, [C.POINTER(Grid), C.c_int32, C.c_int32, _P, _P, _P,
                                        C.c_int32, _P, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("sc_texture_tables", C.c_int, [C.POINTER(Grid), _P, C.c_int64, _P, _P, _P]),
    ("sc_moments_sse", C.c_int, [C.POINTER(CtuRecord), C.POINTER(C.c_double)]),
    ("sc_prefix_sum_table", C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, _P]),
    ("sc_split_even", C.c_int, [C.c_int32, C.c_int32, _P]),
    ("sc_comm_unique_id", C.c_int, [_P]),
    ("sc_comm_init_nccl", C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    ("sc_comm_init_callback", C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    ("sc_comm_detach", C.c_int, [_P]),
    ("sc_shard_export", C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    ("sc_shard_merge", C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P, _P]),
]

_lib = None


def lib() -> C.CDLL:
    """Load the product library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                "the B200 path has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class SlicecraftError(RuntimeError):
    """Raised for a non-OK sc_status; ``kind`` is the reference exception name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {message}")


def check(status: int) -> None:
    if status != SC_OK:
        msg = lib().sc_last_error()
        raise SlicecraftError(status, msg.decode() if msg else "")
