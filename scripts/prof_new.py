"""Launch-list workload for the §8(f) kernels: K5 full (adapter + async),
schedule records, K8 validation, K7 grouping, explicit-plan cost."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import grouping as GR, instances, simulate  # noqa: E402
from paper_2505_15536_b200 import schedule as SCH  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402

eng = Engine(0)
rng = np.random.default_rng(5)
n = 10_000
tims = []
for i in range(n):
    S = int(rng.integers(2, 6))
    tims.append(simulate.make_timing(
        fwd=list(rng.uniform(0.2, 2.0, S)), bwd=list(rng.uniform(0.2, 2.0, S)),
        wgt=list(rng.uniform(0.05, 1.0, S)), transfer=list(rng.uniform(0.05, 2.5, S - 1)),
        microbatch=int(rng.choice([2, 4, 8])), micro_count=int(rng.integers(4, 17)),
        sync=list(rng.uniform(0.0, 0.5, S)), opt=list(rng.uniform(0.0, 0.3, S)),
        latency=float(rng.uniform(0.0, 0.2))))
traces = [{f"{b}-{b + 1}": [[float(t), float(m)] for t, m in
                            zip(np.sort(rng.uniform(0, 60, 4)), rng.choice([0.25, 0.5, 1.0], 4))]
           for b in range(4)} for _ in range(64)]
cfg = simulate.SimConfig(iterations=3, async_iterations=True)
out = SCH.generate_schedules(tims, "zb_compact", traces, np.arange(n) % 64, adapter_enabled=True,
                             config=cfg, engine=eng)
msgs = SCH.validate_schedules([s for s, _ in out], tims, engine=eng)
print("schedules", len(out), "with violations", sum(1 for m in msgs if m))
_, t4, _ = instances.load("c4")
ids, pt, bw, pc = GR.topology_arrays(t4)
GR.group_hierarchies(np.repeat(pt[None], 100, axis=0), bw, pc, engine=eng)
from paper_2505_15536_b200 import search_plan, SearchConfig  # noqa: E402
from paper_2505_15536_b200.costmodel import plan_cost  # noqa: E402
m4, t4, g4 = instances.load("c4")
r = search_plan(m4, t4, g4, SearchConfig(seed=0), engine=eng)
print("plan cost", plan_cost(r.plan, t4, m4, g4, engine=eng).plan_cost)
