"""Latency / throughput of K7 grouping on C4 p_t snapshots (bench helper)."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import grouping as GR, instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402

eng = Engine(0)
_, t4, _ = instances.load("c4")
ids4, pt4, bw4, pc4 = GR.topology_arrays(t4)
for n in (1, 1000):
    pts = np.repeat(pt4[None], n, axis=0)
    GR.group_hierarchies(pts, bw4, pc4, engine=eng)
    lat = []
    for _ in range(10):
        t0 = time.perf_counter()
        GR.group_hierarchies(pts, bw4, pc4, engine=eng)
        lat.append(time.perf_counter() - t0)
    print(f"K7 C4 x{n}: {statistics.median(lat) * 1e3:.3f} ms per call")
