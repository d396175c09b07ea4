"""Latency of the e2e re-plan path (gp_replan) on C4 snapshots: host wall
clock of the C-ABI call and device time of its CUDA graph (events around the
graph launch), p10/p50/p90 over many calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402


def pct(v):
    v = sorted(v)
    q = lambda p: v[int(p * (len(v) - 1))]
    return f"p10 {q(0.1):.4f} p50 {q(0.5):.4f} p90 {q(0.9):.4f} min {v[0]:.4f}"


packs = [PackedInstance(*instances.load("c4", snapshot=j), 1.25) for j in range(4)]
eng = Engine(0)
for timed in (False, True):
    eng.replan_timing(timed)
    host, dev, ph = [], [], []
    for i in range(400):
        t0 = time.perf_counter()
        best, info = eng.replan(packs[i % 4])
        el = time.perf_counter() - t0
        if i >= 50:
            host.append(el * 1e3)
            if timed:
                dev.append(eng.replan_timing(True))
                ph.append(eng.replan_host_us())
    print(f"gp_replan C4 host ms ({'with' if timed else 'without'} graph events): {pct(host)}")
    if timed:
        print(f"gp_replan C4 graph device ms: {pct(dev)}")
        import numpy as np
        med = np.median(np.array(ph), axis=0)
        print("host phases p50 us: arena fill %.1f, graph launch %.1f, wait %.1f, decode %.1f"
              % tuple(med))
