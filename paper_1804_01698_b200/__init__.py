"""B200-native hash SpGEMM (Gustavson row-wise, hash accumulator, two phases)
after Nagasaka, Matsuoka, Azad, Buluc, arXiv:1804.01698.

The compute lives in libspgemm.so (hand-written sm_100a CUDA kernels behind
the C ABI of include/spgemm.h).  This package is a thin binding: it never
computes on the CPU and never imports the oracle.
"""
from .api import (Context, DeviceCSR, default_context, mask_sum, plan_export,  # noqa: F401
                  row_blocks_by_bytes, rows_to_parts, spg_numeric, spg_symbolic, spgemm,
                  triangle_count, triangle_count_rows, validate, masked_sum,
                  triangle_count_fused, degree_relabel, triangle_count_graph,
                  probe_stats, masked_sum_int, spgemm_onephase, rows_to_parts_bytes)
from . import _lib  # noqa: F401

__all__ = ["Context", "DeviceCSR", "default_context", "spgemm", "spg_symbolic", "spg_numeric",
           "plan_export", "rows_to_parts", "mask_sum", "validate", "triangle_count",
           "row_blocks_by_bytes", "triangle_count_rows", "masked_sum", "triangle_count_fused",
           "degree_relabel", "triangle_count_graph", "probe_stats", "masked_sum_int", "spgemm_onephase",
           "rows_to_parts_bytes"]
