"""f3 measurement: arbor_boundary_uncertainty (Eq. 1) on Llama-3-sized logits.
One row per active leaf at a block boundary: batch ∈ {1, 16, 64} × vocab 128,256, f32 and
bf16.  HBM-bound: algorithmic bytes = batch · vocab · element size (one read); CUDA-event
time of the launch (mean of 50 after 10 warm-up) with the logits flushed from L2 between
launches (a 256 MB write).  Usage: python profiles/f3_uncertainty_bench.py [--out f.json]"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_22106_b200 import workload
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ctx = workload.make_context(workload.PRESETS["c1"], workload.build_tree(workload.PRESETS["c1"], 0))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    rows = []
    for dtype in (torch.float32, torch.bfloat16):
        for B in (1, 16, 64):
            V = 128256
            z = torch.randn((B, V), device="cuda").to(dtype)
            u = torch.empty(B, device="cuda")
            for _ in range(10):
                ctx.arbor_boundary_uncertainty(z, u)
            ms = []
            for _ in range(50):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                ctx.arbor_boundary_uncertainty(z, u)
                e1.record(s)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = sum(ms) / len(ms)
            byts = B * V * z.element_size()
            rows.append({"dtype": str(dtype).split(".")[-1], "batch": B, "vocab": V, "us": t * 1e3,
                         "bytes": byts, "GBps": byts / (t / 1e3) / 1e9,
                         "frac_measured_hbm": byts / (t / 1e3) / 1e9 / peak})
            print(json.dumps(rows[-1]), flush=True)
    if a.out:
        json.dump({"kernel": "uncertainty_kernel (f3, Eq. 1)", "peak_GBps": peak, "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
