#!/usr/bin/env python3
"""Short run of every kernel family for ncu: K1/K3 (C4 re-plan), K2 batch,
K4 branch-and-bound (k=8), K5 simulations, K6 snapshots."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_2505_15536_b200 import instances, replan
from paper_2505_15536_b200.engine import Engine
from paper_2505_15536_b200.enumeration import composition_table, decode_indices
from paper_2505_15536_b200.layout import PackedInstance
from test_bnb import _many_group_instance

eng = Engine(0)
m, t, g = instances.load("c4")
p = PackedInstance(m, t, g, 1.25)
for _ in range(3):
    b, info = eng.replan(p)
total = eng.space_size()
idx = np.random.default_rng(1).integers(0, total, 200_000)
o, c, bm = decode_indices(80, 4, idx, composition_table(80, 4))
cost, st = eng.eval_batch(o, c, bm)
feas = np.nonzero(np.isfinite(cost))[0][:20000]
eng.sim_candidates(o[feas], c[feas], bm[feas], 1, 0.0)
mk, tk, gk = _many_group_instance(8, 80, 8)
eng.load(PackedInstance(mk, tk, gk, 1.25))
print("k8 bnb", eng.argmin_bnb().cost)
spec = instances.config("c2")
m2, t2, g2 = instances.build(spec)
p2 = PackedInstance(m2, t2, g2, 1.25)
bws = replan.bandwidth_matrices(p2, [instances.snapshot_multipliers(spec, j) for j in range(1000)])
eng.load(p2)
bests, sts = eng.replan_snapshots(bws)
print("ok", b.cost, int((sts == 0).sum()))
