"""Device time of one K2 explicit batch of 2x10^7 random C4 candidates (as in
bench.py) for the engine build in GP_ENGINE_LIB (default: in-tree)."""
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
N = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
idx = np.random.default_rng(4).integers(0, total, size=N)
order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
dev = torch.device("cuda", 0)
d_o, d_c, d_b = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (order, counts, bm))
d_cost = torch.empty(N, dtype=torch.float64, device=dev)
d_st = torch.empty(N, dtype=torch.uint8, device=dev)
stream = torch.cuda.ExternalStream(eng.stream, device=dev)
run = lambda: eng.eval_batch_device(4, N, d_o.data_ptr(), d_c.data_ptr(), d_b.data_ptr(),
                                    d_cost.data_ptr(), d_st.data_ptr())
run()
torch.cuda.synchronize()
ref = d_cost.cpu().numpy().view(np.uint64).copy()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with torch.cuda.stream(stream):
    ev[0].record(stream)
for _ in range(20):
    run()
with torch.cuda.stream(stream):
    ev[1].record(stream)
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 20
digest = int(np.bitwise_xor.reduce(ref))
print(f"{os.environ.get('GP_ENGINE_LIB', 'default')}: K2 {ms * 1e3:.1f} us per {N:.0e} -> "
      f"{N / (ms * 1e-3):.3e} cand/s; cost digest {digest:#x}, feasible {np.isfinite(d_cost.cpu().numpy()).mean():.3f}")
