"""Host-side profile of the drop-in exhaustive_plan(model, topology, groups,
config) at C4 (cProfile over 200 calls after warm-up) and its p50 latency."""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import SearchConfig, exhaustive_plan, instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402

model, topo, groups = instances.load("c4")
eng = Engine(0)
cfg = SearchConfig(seed=0)
for _ in range(10):
    exhaustive_plan(model, topo, groups, cfg, engine=eng)
lat = []
for _ in range(200):
    t0 = time.perf_counter()
    exhaustive_plan(model, topo, groups, cfg, engine=eng)
    lat.append(time.perf_counter() - t0)
print(f"exhaustive_plan C4 p50 {statistics.median(lat) * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    exhaustive_plan(model, topo, groups, cfg, engine=eng)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
