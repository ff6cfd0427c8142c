import json, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import synth
from gpu_helpers import Pair
d = json.load(open("scratch/alloc_fail.json"))
N = len(d["n"]); n = np.array(d["n"], np.int32)
tree = synth.SynthTree(np.array(d["parent"], np.int32), np.concatenate([[0], np.cumsum(n[:-1])]).astype(np.int64), n,
                       np.zeros(N, np.uint8), np.full(N, .5, np.float32), np.full(N, .5, np.float32), d["active"])
preset = dict(tree=None, L=1, H=1, Hq=1, d=64, dtype="f32", P=4, rho=0.5, params={}, active=None)
pr = Pair(preset, seed=0, tree=tree, params_over=d["params"])
s = np.array(d["s"], np.float32)
k = torch.full((N,), -1, dtype=torch.int32, device="cuda")
pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(s, device="cuda"), d["B"], k)
torch.cuda.synchronize()
print("got ", k.cpu().tolist())
print("want", d["want"])
try:
    pr.ctx.arbor_sync(); print("sync ok")
except Exception as e:
    print("sync err", e)
