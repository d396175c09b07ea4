import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2505_15536_b200 import grouping as GR, instances
from paper_2505_15536_b200.engine import Engine
eng = Engine(0)
_, t4, _ = instances.load("c4")
ids4, pt4, bw4, pc4 = GR.topology_arrays(t4)
GR.group_hierarchies(pt4[None], bw4, pc4, engine=eng)
