#!/usr/bin/env python3
"""Short K3 run for ncu: load an App. D config, 5 exhaustive re-plans."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances
from paper_2505_15536_b200.engine import Engine
from paper_2505_15536_b200.layout import PackedInstance

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
m, t, g = instances.load(name)
eng = Engine(0).load(PackedInstance(m, t, g, 1.25))
total = eng.space_size()
for _ in range(5):
    best = eng.argmin_range(0, total)
print(name, total, best.cost, best.index)
