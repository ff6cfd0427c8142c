"""B200-native ArborKV per-step KV-eviction path (arXiv 2605.22106).

The product is ``libarbor.so`` (C ABI, include/arbor.h) built from ``csrc/`` for sm_100a;
``arbor.py`` is its thin ctypes binding and ``workload.py`` drives the synthetic
ToT/DPTS workloads through it.  There is no CPU fallback.
"""
from .arbor import (ArborError, ArborKV, ArborParams, TreeArgs, load_library, make_params,
                    params_from_dict, min_feasible_budget, nccl_unique_id, validate_tree,
                    LIB_PATH, STAGES)

__all__ = ["ArborError", "ArborKV", "ArborParams", "TreeArgs", "load_library", "make_params",
           "params_from_dict", "min_feasible_budget", "nccl_unique_id", "validate_tree",
           "LIB_PATH", "STAGES"]
