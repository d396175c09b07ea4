"""Device time of the bench step (K6 patch + sweep over S C4 bandwidth
snapshots, L2 flushed between steps) and a digest of the winners, for the
engine build in GP_ENGINE_LIB (default: in-tree).  Usage:
python scripts/time_k6.py [snapshots] [reps]"""
import hashlib
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances, replan  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import packed_instance  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
spec = instances.config("c4")
m, t, g = instances.build(spec)
packed = packed_instance(m, t, g, 1.25)
eng = Engine(0).load(packed)
total = eng.space_size()
dev = torch.device("cuda", 0)
bws = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec, j) for j in range(S)])
d_bw = torch.from_numpy(np.ascontiguousarray(bws)).to(dev)
d_keys = torch.zeros((S, 2), dtype=torch.int64, device=dev)
d_flags = torch.zeros(S, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.ExternalStream(eng.stream, device=dev)
ms = []
for i in range(reps + 3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        flush.zero_()
        a.record(stream)
    eng.replan_snapshots_async(d_bw.data_ptr(), S, d_keys.data_ptr(), d_flags.data_ptr())
    with torch.cuda.stream(stream):
        b.record(stream)
    torch.cuda.synchronize()
    if i >= 3:
        ms.append(a.elapsed_time(b))
keys = d_keys.cpu().numpy()
dig = hashlib.sha1(keys.tobytes()).hexdigest()[:16]
med = statistics.median(ms)
print(f"{os.environ.get('GP_ENGINE_LIB', 'default')}: S={S} median {med:.4f} ms min {min(ms):.4f} ms "
      f"-> {S * total / (med * 1e-3):.4e} cand/s; winners sha1 {dig}; first {keys[0].tolist()} "
      f"flags {int(d_flags.sum())}")
