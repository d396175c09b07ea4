#!/usr/bin/env python3
"""Time K4 branch-and-bound vs the K3 exhaustive sweep (device time, CUDA events)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2505_15536_b200 import instances as I
from paper_2505_15536_b200.engine import Engine
from paper_2505_15536_b200.layout import PackedInstance
from test_bnb import _many_group_instance

eng = Engine(0)


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    return (time.perf_counter() - t0) / reps * 1e3, r


for name in ("c2", "c4"):
    m, tp, g = I.load(name)
    eng.load(PackedInstance(m, tp, g, 1.25))
    total = eng.space_size()
    ms_ex, ex = t(lambda: eng.argmin_range(0, total))
    ms_bb, bb = t(lambda: eng.argmin_bnb())
    print(f"{name}: space {total:.3e}  sweep {ms_ex:.3f} ms  bnb {ms_bb:.3f} ms  same={ex.index == bb.index}")
for k, n, seed in [(6, 40, 5), (6, 80, 6), (8, 48, 7), (8, 80, 8), (10, 80, 9)]:
    m, tp, g = _many_group_instance(k, n, seed)
    eng.load(PackedInstance(m, tp, g, 1.25))
    total = eng.space_size()
    ms_bb, bb = t(lambda: eng.argmin_bnb(), reps=2)
    line = f"k={k} n={n}: space {total:.3e}  bnb {ms_bb:.3f} ms cost {bb.cost:.6g}"
    if total < 2e10:
        ms_ex, ex = t(lambda: eng.argmin_range(0, total), reps=1)
        line += f"  sweep {ms_ex:.3f} ms same={ex.index == bb.index}"
    print(line, flush=True)
