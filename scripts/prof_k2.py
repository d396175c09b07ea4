"""One large K2 explicit batch (2x10^7 random C4 candidates) for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.enumeration import composition_table, decode_indices  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

m, t, g = instances.load("c4")
eng = Engine(0).load(PackedInstance(m, t, g, 1.25))
total = eng.space_size()
N = 20_000_000
idx = np.random.default_rng(4).integers(0, total, size=N)
order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
dev = torch.device("cuda", 0)
d_o = torch.from_numpy(np.ascontiguousarray(order)).to(dev)
d_c = torch.from_numpy(np.ascontiguousarray(counts)).to(dev)
d_b = torch.from_numpy(np.ascontiguousarray(bm)).to(dev)
d_cost = torch.empty(N, dtype=torch.float64, device=dev)
d_st = torch.empty(N, dtype=torch.uint8, device=dev)
for _ in range(3):
    eng.eval_batch_device(4, N, d_o.data_ptr(), d_c.data_ptr(), d_b.data_ptr(), d_cost.data_ptr(),
                          d_st.data_ptr())
torch.cuda.synchronize()
# timing (CUDA events on the engine stream, 20 launches)
stream = torch.cuda.ExternalStream(eng.stream, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    a.record(stream)
for _ in range(20):
    eng.eval_batch_device(4, N, d_o.data_ptr(), d_c.data_ptr(), d_b.data_ptr(), d_cost.data_ptr(),
                          d_st.data_ptr())
with torch.cuda.stream(stream):
    b.record(stream)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
print(f"K2 2e7: {ms * 1e3:.1f} us per launch, {N / (ms * 1e-3):.3g} candidates/s")
