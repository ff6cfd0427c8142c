"""Moved rows per (node, row) of one C2 eviction from full retention under the two slot
layouts (Q23*): the round-1 prefix [0, k_app) and the end window [n − k_app, n).
The oracle's own state on the C2 tree and K/V (first 2 layers, one leaf-cycling warm-up
pass), its allocation and retained sets.  A design-time measurement, not a test:

    python tests/window_estimate.py
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2605_22106_b200 import workload
from oracle.state import ArborOracle, default_params
from oracle import geometry, msve, tae
from oracle.select import retained_set
p = dict(workload.PRESETS['c2']); L1 = 2
tree = workload.build_tree(p, 0)
K, V, E = synth.make_kv(p['L'], p['H'], tree.total_tokens, p['d'], p['dtype'], 0, tree.span_start, tree.span_len, device='cpu')
K = K[:L1].float(); V = V[:L1].float()
params = default_params(**p['params'])
o = ArborOracle(K.double().numpy(), V.double().numpy(), p['Hq'], p['P'], 4096, params, num_layers_global=L1, num_q_heads_global=p['Hq'])
for i in range(tree.num_nodes):
    o.open_node(i, int(tree.span_start[i])); o.append(i, int(tree.span_len[i])); o.close_node(i)
order = [leaf for leaf in workload.leaf_cycle_order(tree, 0) for _ in range(1)]
for j, leaf in enumerate(order):
    tree.active = [leaf]
    q = synth.make_queries(1, p['L'], p['Hq'], p['d'], p['dtype'], workload.query_seed(0, j), E, device='cpu').float()[:, :L1]
    o.score_accumulate(tree, q.double().numpy())
leaf = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[0]
tree.active = [leaf]
N = tree.num_nodes
mass = o.masses()
s = [float(np.float32(msve.msve_score(params['theta'], float(tree.v[i]), float(tree.u[i]), msve.attention_feature(mass[i], o.Mclose[i], o.Nq[i], L1, p['Hq'])))) for i in range(N)]
parent = [int(x) for x in tree.parent]
B = int(math.floor(p['rho'] * tree.total_tokens))
st, k, _ = tae.allocate(0, s, geometry.depths(parent), geometry.delta(parent, tree.active), [i in geometry.path_star(parent, tree.active) for i in range(N)], [False]*N, [int(x) for x in tree.span_len], params, B)
tot_f = tot_e = 0; cnt = 0
A = o.A  # inspect layout
for i in range(N):
    n = int(tree.span_len[i]); ki = int(k[i])
    if ki >= n: continue
    for l in range(L1):
        for h in range(p['H']):
            a = A[l][h][int(tree.span_start[i]): int(tree.span_start[i]) + n] if not hasattr(A, 'shape') else A[l, h, int(tree.span_start[i]): int(tree.span_start[i]) + n]
            kept = retained_set(list(range(n)), n, ki, params['l_tail'], np.asarray(a, dtype=np.float32), params['select_mode'], params['n_sinks'], is_root=(parent[i] < 0))
            kept = set(int(x) for x in kept)
            tot_f += sum(1 for s_ in kept if s_ >= ki); tot_e += sum(1 for s_ in kept if s_ < n - ki); cnt += 1
print('items', cnt, 'front moves/item', tot_f / cnt, 'end moves/item', tot_e / cnt)
print('k hist', np.unique([int(x) for x in k], return_counts=True))
