"""Median wall time of the bench's e2e step (replan.replan_snapshots of S C4
snapshots from pinned host matrices) for the engine build in GP_ENGINE_LIB."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import SearchConfig, instances, replan  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import packed_instance  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
spec = instances.config("c4")
model, topo, groups = instances.build(spec)
packed = packed_instance(model, topo, groups, 1.25)
eng = Engine(0).load(packed)
bws = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec, j) for j in range(S)])
bws_p = torch.from_numpy(bws).pin_memory().numpy()
cfg = SearchConfig(seed=0)
lat = []
for i in range(reps + 5):
    t0 = time.perf_counter()
    res = replan.replan_snapshots(model, topo, groups, cfg, bws_p, engine=eng)
    if i >= 5:
        lat.append(time.perf_counter() - t0)
tot = eng.space_size() * S
print(f"{os.environ.get('GP_ENGINE_LIB', 'default')}: e2e p50 {statistics.median(lat) * 1e3:.3f} ms "
      f"min {min(lat) * 1e3:.3f} mean {statistics.mean(lat) * 1e3:.3f} -> {tot / statistics.median(lat):.3e} cand/s")
