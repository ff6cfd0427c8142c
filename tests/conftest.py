import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_sessionfinish(session, exitstatus):
    """GPU sessions: write the observed error of every tolerance check (gpu_helpers.TOL_LOG)."""
    try:
        import gpu_helpers
    except Exception:
        return
    if not gpu_helpers.TOL_LOG:
        return
    import json
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    worst = {}
    for e in gpu_helpers.TOL_LOG:
        w = worst.get(e["what"])
        if w is None or e["max_err_over_bound"] > w["max_err_over_bound"]:
            worst[e["what"]] = dict(e, checks=0)
        worst[e["what"]]["checks"] = worst[e["what"]].get("checks", 0) + 1
    with open(os.path.join(out, "tolerance_report.json"), "w") as f:
        json.dump(dict(checks=len(gpu_helpers.TOL_LOG), worst_per_check=worst), f, indent=1)
