"""B200-native core of the dynamic TRS partitioner (arXiv 2012.14792).

A drop-in for the reference `slicecraft` partitioner API: texture map,
CTU-complexity model and ColumnSplit two-step search, computed by sm_100a
kernels behind the C-ABI in include/slicecraft_b200.h.
"""
from ._abi import LIB_PATH, SlicecraftError, lib
from .partitioner import (COLUMN_SPLIT, COVERAGE_COVERING, COVERAGE_REFERENCE, MODE_EXHAUSTIVE,
                          MODE_PRUNED, RECORD_DTYPE, UNIFORM_ONLY, CostHistory, CostMap, CtuGrid,
                          Partition, Partitioner, PrefixSumTable, SearchConfig, SearchOutcome,
                          TextureStats, estimate_ctu_times, load_yuv_frame, moments_sse,
                          read_yuv_luma, shard_merge, split_even, temporal_layer_of_poc,
                          texture_tables, texture_validate, yuv_frame_count)

__all__ = [
    "LIB_PATH", "SlicecraftError", "lib", "COLUMN_SPLIT", "UNIFORM_ONLY", "COVERAGE_REFERENCE",
    "COVERAGE_COVERING", "MODE_EXHAUSTIVE", "MODE_PRUNED", "RECORD_DTYPE", "CostHistory",
    "CostMap", "CtuGrid", "Partition", "Partitioner", "SearchConfig", "SearchOutcome",
    "TextureStats", "estimate_ctu_times", "shard_merge", "temporal_layer_of_poc",
    "texture_validate", "yuv_frame_count", "load_yuv_frame", "read_yuv_luma", "PrefixSumTable",
    "split_even", "moments_sse", "texture_tables",
]
