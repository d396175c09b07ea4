"""Host-call time of the full simulator (adapter + async, ZB_COMPACT, 3
iterations) on 10^5 random timings, three consecutive calls."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import simulate  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402

eng = Engine(0)
rng5 = np.random.default_rng(5)
n5 = 100_000
S5 = rng5.integers(2, 6, n5)
tims = []
for i in range(n5):
    S = int(S5[i])
    tims.append(simulate.make_timing(
        fwd=list(rng5.uniform(0.2, 2.0, S)), bwd=list(rng5.uniform(0.2, 2.0, S)),
        wgt=list(rng5.uniform(0.05, 1.0, S)), transfer=list(rng5.uniform(0.05, 2.5, S - 1)),
        microbatch=int(rng5.choice([2, 4, 8])), micro_count=int(rng5.integers(4, 17)),
        sync=list(rng5.uniform(0.0, 0.5, S)), opt=list(rng5.uniform(0.0, 0.3, S)),
        latency=float(rng5.uniform(0.0, 0.2))))
traces = [{f"{b}-{b + 1}": [[float(t), float(m)] for t, m in
                            zip(np.sort(rng5.uniform(0, 60, 4)), rng5.choice([0.25, 0.5, 1.0], 4))]
           for b in range(4)} for _ in range(64)]
arr5 = simulate.pack_timings(tims)
tr5 = simulate.pack_traces(traces)
ti5 = np.arange(n5) % 64
for ad, asy in ((True, True), (True, False), (False, False)):
    for rep in range(3):
        t0 = time.perf_counter()
        reps5, _, st5 = eng.simulate_report(arr5, n5, 3, 3, tr5, 64, ti5, adapter=ad,
                                            async_iterations=asy)
        el = time.perf_counter() - t0
        print(f"adapter={ad} async={asy} call {rep}: {el * 1e3:.1f} ms ({n5 / el:.3g} sims/s)")
