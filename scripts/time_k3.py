"""Median device time of the C4 exhaustive K3 launch (L2 flushed between
launches) for one or more engine builds: GP_ENGINE_LIB=<so> per process.
Usage: python scripts/time_k3.py [reps]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
m, t, g = instances.load("c4")
eng = Engine(0).load(PackedInstance(m, t, g, 1.25))
if os.environ.get("K3_MODE"):
    eng.set_k3_mode(int(os.environ["K3_MODE"]))
total = eng.space_size()
stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", 0))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
ms = []
for i in range(reps + 5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        flush.zero_()
        a.record(stream)
    eng.argmin_range_async(0, total)
    with torch.cuda.stream(stream):
        b.record(stream)
    torch.cuda.synchronize()
    if i >= 5:
        ms.append(a.elapsed_time(b))
try:
    best = eng.argmin_fetch()
    res = f"cost {best.cost} index {best.index}"
except Exception as e:  # diagnostic builds (e.g. -DK3_NOLOOP) find no winner
    res = f"no result ({type(e).__name__})"
print(f"{os.environ.get('GP_ENGINE_LIB', 'default')} mode {os.environ.get('K3_MODE', 'auto')}: median {statistics.median(ms) * 1e3:.1f} us "
      f"min {min(ms) * 1e3:.1f} us  {res}")
