"""Stress: many arbor_decode_step calls on a preset (default c3: 16 leaves, NQ = 48 tiles)
with a device sync every 50 steps; prints progress.  A pipeline deadlock hangs the stream:
faulthandler prints the Python stack after 90 s and exits.  A debug build with
ARBOR_NVCC_FLAGS=-DARBOR_MBAR_WATCHDOG turns it into a CUDA error (bounded mbarrier waits
that __trap(), tile.cuh).

    python profiles/stress_decode.py [c3] [steps]
"""
from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(90, exit=True)   # a hang prints the Python stack
    import torch
    from paper_2605_22106_b200 import workload

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    print(f"{cfg}: setup", flush=True)
    sc = workload.setup(cfg, 0)
    torch.cuda.synchronize()
    print(f"{cfg}: setup done", flush=True)
    ctx, tree = sc.ctx, sc.tree
    nA = len(tree.active)
    qs = [sc.queries(i, nA) for i in range(4)]
    out = torch.empty_like(qs[0])
    lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device=qs[0].device)
    t0 = time.time()
    for i in range(steps):
        ctx.arbor_decode_step(tree, qs[i % 4], out, lse)
        if i % 50 == 49 or i < 3:
            torch.cuda.synchronize()
            print(f"{cfg}: {i + 1} steps ok ({time.time() - t0:.1f} s)", flush=True)
    torch.cuda.synchronize()
    print(f"{cfg}: done {steps} steps", flush=True)


if __name__ == "__main__":
    main()
