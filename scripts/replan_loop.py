"""20 exact C4 re-plans through gp_replan (the e2e path), for launch lists."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

packs = [PackedInstance(*instances.load("c4", snapshot=j), 1.25) for j in range(4)]
eng = Engine(0)
for i in range(20):
    t0 = time.perf_counter()
    best, info = eng.replan(packs[i % 4])
    if i >= 16:
        print(f"replan {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms cost {best.cost}")
