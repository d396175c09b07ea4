"""1F1B makespans of 2x10^5 memory-feasible random C4 plans (K5,
gp_sim_candidates, iterations=1) and of 10^5 random 1F1B timings
(gp_sim_1f1b) for the engine build in GP_ENGINE_LIB (default: in-tree);
prints the rate and a digest of the makespans."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import instances, simulate  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.enumeration import composition_table, decode_indices  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

m, t, g = instances.load("c4")
eng = Engine(0).load(PackedInstance(m, t, g, 1.25))
total = eng.space_size()
idx = np.random.default_rng(4).integers(0, total, size=3_000_000)
order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
cost, st = eng.eval_batch(order, counts, bm)
feas = np.nonzero(np.isfinite(cost))[0][:200_000]
o, c, b = order[feas], counts[feas], bm[feas]
eng.sim_candidates(o, c, b, 1, 0.0)
reps = []
for _ in range(5):
    t0 = time.perf_counter()
    ms, s = eng.sim_candidates(o, c, b, 1, 0.0)
    reps.append(time.perf_counter() - t0)
el = min(reps)
print(f"{os.environ.get('GP_ENGINE_LIB', 'default')}: sim_candidates {feas.size} plans "
      f"{el * 1e3:.2f} ms -> {feas.size / el:.3e}/s; digest "
      f"{int(np.bitwise_xor.reduce(ms.view(np.uint64))):#x} ok {(s == 0).mean():.3f}")
rng = np.random.default_rng(5)
tims = []
for i in range(100_000):
    S = int(rng.integers(1, 5))
    tims.append(simulate.make_timing(
        fwd=list(rng.uniform(0.2, 2.0, S)), bwd=list(rng.uniform(0.2, 2.0, S)),
        wgt=list(rng.uniform(0.05, 1.0, S)), transfer=list(rng.uniform(0.05, 2.5, S - 1)),
        microbatch=int(rng.choice([1, 2, 4, 8])), micro_count=int(rng.integers(1, 17)),
        latency=float(rng.uniform(0.0, 0.2))))
arr = simulate.pack_timings(tims)
eng.sim_1f1b(arr, len(tims), 1)
reps = []
for _ in range(5):
    t0 = time.perf_counter()
    ms2, s2 = eng.sim_1f1b(arr, len(tims), 1)
    reps.append(time.perf_counter() - t0)
el = min(reps)
print(f"sim_1f1b {len(tims)} timings {el * 1e3:.2f} ms -> {len(tims) / el:.3e}/s; digest "
      f"{int(np.bitwise_xor.reduce(ms2.view(np.uint64))):#x} ok {(s2 == 0).mean():.3f}")
