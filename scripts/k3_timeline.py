"""Per-CTA timeline of one C4 k3_sweep launch (needs a -DK3_PROFILE build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

m, t, g = instances.load("c4")
eng = Engine(0).load(PackedInstance(m, t, g, 1.25))
total = eng.space_size()
for _ in range(3):
    eng.argmin_range(0, total)
