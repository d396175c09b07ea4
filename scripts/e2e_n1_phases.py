"""Where the single-GPU snapshot re-plan's end-to-end time goes (128 C4
snapshots): the public replan.replan_snapshots call vs its pieces (H2D of
the pinned matrices, the device re-plan, the key read-back).  Usage:
python scripts/e2e_n1_phases.py"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import SearchConfig, instances, replan  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import packed_instance  # noqa: E402

spec = instances.config("c4")
model, topo, groups = instances.build(spec)
packed = packed_instance(model, topo, groups, 1.25)
eng = Engine(0).load(packed)
S = 128
bws = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec, j) for j in range(S)])
pin = torch.from_numpy(bws).pin_memory()
bws_p = pin.numpy()
dev = torch.device("cuda", 0)
d_bw = torch.empty_like(pin, device=dev)
d_keys = torch.zeros((S, 2), dtype=torch.int64, device=dev)
d_flags = torch.zeros(S, dtype=torch.int32, device=dev)
h_keys = torch.zeros((S, 2), dtype=torch.int64).pin_memory()
est = torch.cuda.ExternalStream(eng.stream, device=dev)
cfg = SearchConfig(seed=0)
T = {k: [] for k in ("api", "sync_abi", "h2d", "device", "h2d+device+d2h", "api_pageable")}
bws_pageable = np.array(bws_p)
for it in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    replan.replan_snapshots(model, topo, groups, cfg, bws_p, engine=eng)
    t1 = time.perf_counter()
    eng.replan_snapshots(bws_p)
    t2 = time.perf_counter()
    # (copies on torch's stream: pinned blocks must not be tied to the
    # engine's stream, which the engine destroys before torch's allocator)
    cur = torch.cuda.current_stream(dev)
    d_bw.copy_(pin, non_blocking=True)
    cur.synchronize()
    t3 = time.perf_counter()
    eng.replan_snapshots_async(d_bw.data_ptr(), S, d_keys.data_ptr(), d_flags.data_ptr())
    est.synchronize()
    t4 = time.perf_counter()
    d_bw.copy_(pin, non_blocking=True)
    est.wait_stream(cur)
    eng.replan_snapshots_async(d_bw.data_ptr(), S, d_keys.data_ptr(), d_flags.data_ptr())
    cur.wait_stream(est)
    h_keys.copy_(d_keys, non_blocking=True)
    cur.synchronize()
    t5 = time.perf_counter()
    t6 = time.perf_counter()
    replan.replan_snapshots(model, topo, groups, cfg, bws_pageable, engine=eng)
    t7 = time.perf_counter()
    if it >= 5:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t7 - t6)):
            T[k].append(v)
print({k: round(statistics.median(v) * 1e3, 4) for k, v in T.items()})
