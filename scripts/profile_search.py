"""Host-side profile of the drop-in search_plan at C4 (cProfile over 20 calls)."""
import cProfile
import logging
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import SearchConfig, instances, search_plan  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402

logging.disable(logging.WARNING)
model, topo, groups = instances.load("c4")
eng = Engine(0)
cfg = SearchConfig(seed=0)
for _ in range(3):
    search_plan(model, topo, groups, cfg, engine=eng)
lat = []
for _ in range(20):
    t0 = time.perf_counter()
    search_plan(model, topo, groups, cfg, engine=eng)
    lat.append(time.perf_counter() - t0)
print(f"search_plan C4 p50 {statistics.median(lat) * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    search_plan(model, topo, groups, cfg, engine=eng)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
