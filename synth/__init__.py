"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the ArborKV method (no scoring,
allocation, selection, compaction or attention).  It only draws trees,
node features, K/V/Q tensors and DPTS transition schedules with the
shapes and structure of the paper's workloads (§5.1
"Tree-search configurations"; SURVEY.md §8(d) recipe), so that
both sides of every parity test see byte-identical inputs.
"""
from .trees import (SynthTree, full_tree, search_tree, leaves_of, highest_v_leaf,
                    dpts_initial_leaves, dpts_schedule, tot_expansion)
from .tensors import bf16_round_np, make_kv, make_queries, heavy_positions, hindsight_labels

__all__ = [
    "SynthTree", "full_tree", "search_tree", "leaves_of", "highest_v_leaf",
    "dpts_initial_leaves", "dpts_schedule", "tot_expansion",
    "bf16_round_np", "make_kv", "make_queries", "heavy_positions",
]
